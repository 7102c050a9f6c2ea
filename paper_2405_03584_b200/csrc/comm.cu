// comm.cu — allgather backends of the row-sharded path (see comm.h).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>

#include "../../include/ipm.h"
#include "comm.h"

bool ipm_group::barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const unsigned long long g = gen;
    if (++count == n) {
        count = 0;
        ++gen;
        cv.notify_all();
        return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g || broken; });
    if (!ok || broken) {
        broken = true;
        cv.notify_all();
        return false;
    }
    return true;
}

namespace ipm {

// ------------------------------------------------------------------------------ NCCL
namespace {
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string &err) {
        if (h) return true;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return false;
        }
        GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        if (!GetUniqueId || !CommInitRank || !AllGather || !CommDestroy || !GetErrorString) {
            err = "libnccl.so.2 lacks a required symbol";
            h = nullptr;
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (c) g_nccl.CommDestroy(c);
    }
    int allgather(const void *send, void *recv, size_t bytes, cudaStream_t st, std::string &err) override {
        ncclResult_t r = g_nccl.AllGather(send, recv, bytes, ncclUint8, c, st);
        if (r != ncclSuccess) {
            err = std::string("ncclAllGather: ") + g_nccl.GetErrorString(r);
            return 1;
        }
        return 0;
    }
};
}  // namespace

int nccl_unique_id(void *out, size_t bytes, std::string &err) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (bytes < sizeof(ncclUniqueId)) {
        err = "unique id buffer smaller than NCCL_UNIQUE_ID_BYTES";
        return 1;
    }
    if (!g_nccl.load(err)) return 1;
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) {
        err = std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r);
        return 1;
    }
    std::memcpy(out, &id, sizeof id);
    return 0;
}

Comm *make_nccl_comm(const void *unique_id, int rank, int nranks, std::string &err) {
    {
        std::lock_guard<std::mutex> lk(g_nccl_mu);
        if (!g_nccl.load(err)) return nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    NcclComm *c = new NcclComm();
    c->rank = rank;
    c->nranks = nranks;
    ncclResult_t r = g_nccl.CommInitRank(&c->c, nranks, id, rank);
    if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r);
        c->c = nullptr;
        delete c;
        return nullptr;
    }
    return c;
}

// ------------------------------------------------------------------------------ host callback
namespace {
struct HostComm : Comm {
    ipm_host_comm hc{};
    int allgather(const void *send, void *recv, size_t bytes, cudaStream_t st, std::string &err) override {
        std::vector<unsigned char> s(bytes), r(bytes * (size_t)nranks);
        cudaError_t e = cudaMemcpyAsync(s.data(), send, bytes, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            err = std::string("host allgather staging: ") + cudaGetErrorString(e);
            return 1;
        }
        if (hc.allgather(s.data(), r.data(), bytes, hc.user) != 0) {
            err = "host allgather callback failed";
            return 1;
        }
        e = cudaMemcpyAsync(recv, r.data(), r.size(), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // r is a stack buffer
        if (e != cudaSuccess) {
            err = std::string("host allgather staging: ") + cudaGetErrorString(e);
            return 1;
        }
        return 0;
    }
};
}  // namespace

Comm *make_host_comm(const void *host_comm, std::string &err) {
    const ipm_host_comm *h = static_cast<const ipm_host_comm *>(host_comm);
    if (!h || !h->allgather || h->nranks < 1 || h->rank < 0 || h->rank >= h->nranks) {
        err = "bad ipm_host_comm";
        return nullptr;
    }
    HostComm *c = new HostComm();
    c->hc = *h;
    c->rank = h->rank;
    c->nranks = h->nranks;
    return c;
}

// ------------------------------------------------------------------------------ local group
namespace {
struct LocalComm : Comm {
    ipm_group *g = nullptr;
    int allgather(const void *send, void *recv, size_t bytes, cudaStream_t st, std::string &err) override {
        int dev = 0;
        cudaGetDevice(&dev);
        if (!g->ready[rank]) {
            cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&g->copied[rank], cudaEventDisableTiming);
        }
        // 1. publish: my block is ready once the work queued so far on my stream is done
        cudaEventRecord(g->ready[rank], st);
        g->send[rank] = send;
        g->dev[rank] = dev;
        if (!g->barrier()) {
            err = "local group barrier failed (a rank left or timed out)";
            return 1;
        }
        // 2. pull every block into my receive buffer, ordered after its producer
        for (int r = 0; r < nranks; ++r) {
            cudaStreamWaitEvent(st, g->ready[r], 0);
            char *dst = static_cast<char *>(recv) + (size_t)r * bytes;
            cudaError_t e = (g->dev[r] == dev)
                                ? cudaMemcpyAsync(dst, g->send[r], bytes, cudaMemcpyDeviceToDevice, st)
                                : cudaMemcpyPeerAsync(dst, dev, g->send[r], g->dev[r], bytes, st);
            if (e != cudaSuccess) {
                err = std::string("local allgather copy: ") + cudaGetErrorString(e);
                return 1;
            }
        }
        cudaEventRecord(g->copied[rank], st);
        if (!g->barrier()) {
            err = "local group barrier failed (a rank left or timed out)";
            return 1;
        }
        // 3. nobody may overwrite its send block before every rank has copied it
        for (int r = 0; r < nranks; ++r)
            if (r != rank) cudaStreamWaitEvent(st, g->copied[r], 0);
        return 0;
    }
};
}  // namespace

Comm *make_local_comm(ipm_group *g, int rank, std::string &err) {
    if (!g || rank < 0 || rank >= g->n) {
        err = "bad local group / rank";
        return nullptr;
    }
    LocalComm *c = new LocalComm();
    c->g = g;
    c->rank = rank;
    c->nranks = g->n;
    return c;
}

}  // namespace ipm
