// comm.h — collectives of the row-sharded path.  The path needs exactly one
// primitive: allgather of equal-size per-rank blocks (the search vector p and the small
// vector of per-rank reduction partials), on the context's stream.
//
// Backends:
//   * NcclComm  — ncclAllGather over NVLink/NVSwitch; libnccl.so.2 is dlopen'd at create so
//                 the library has no link-time NCCL dependency (torch's NCCL is reused when
//                 already loaded).
//   * LocalComm — ranks are contexts inside ONE process (one host thread per rank, any mix of
//                 devices): stream-ordered device copies fenced by CUDA events and a host
//                 barrier.  Used to test the sharded kernels with P virtual ranks on one GPU
//                 and for single-process multi-GPU runs.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

struct ipm_group {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int count = 0;
    unsigned long long gen = 0;
    bool broken = false;
    std::vector<const void *> send;
    std::vector<int> dev;
    std::vector<cudaEvent_t> ready, copied;
    explicit ipm_group(int n_) : n(n_), send(n_, nullptr), dev(n_, 0), ready(n_, nullptr), copied(n_, nullptr) {}
    bool barrier();  // false on timeout / broken group
};

namespace ipm {

struct Comm {
    int rank = 0, nranks = 1;
    virtual ~Comm() {}
    // recv receives nranks * bytes; rank r's block at offset r * bytes.  0 on success.
    virtual int allgather(const void *send, void *recv, size_t bytes, cudaStream_t st, std::string &err) = 0;
};

Comm *make_nccl_comm(const void *unique_id, int rank, int nranks, std::string &err);
// comm_kind 3: the caller's host allgather callback (ipm_host_comm, include/ipm.h) — used only
// to bootstrap the peer-memory data plane and for the create-time certificate exchange
Comm *make_host_comm(const void *host_comm, std::string &err);
Comm *make_local_comm(ipm_group *g, int rank, std::string &err);
int nccl_unique_id(void *out, size_t bytes, std::string &err);

}  // namespace ipm
