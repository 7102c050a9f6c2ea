// ipm_api.cu — host side of libipm.so: the C ABI of include/ipm.h.
//
// Algorithm 1 runs as a host loop over device kernels; ALL vectors
// stay resident on the device (the paper moves residuals, D and the solution across PCIe
// every iteration, P:232-238 — here only ~20 scalars come back per IPM iteration for the
// mu logic of Alg. 1 lines 10-15).  The PCG inner loop (line 2) is a CUDA graph whose
// conditional WHILE node is re-armed by the device, so a whole PCG solve is one launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ipm.h"
#include <unistd.h>

#include "comm.h"
#include "kernels.h"
#include "peer.h"
#include "state.h"

#define IPM_EXPORT extern "C" __attribute__((visibility("default")))

using namespace ipm;

namespace {

thread_local std::string g_create_error;

// IPM_DEBUG=1 in the environment prints host-side progress to stderr (diagnostics only).
bool dbg() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("IPM_DEBUG");
        v = (e && *e && *e != '0') ? 1 : 0;
    }
    return v == 1;
}
#define DBG(...)                                  \
    do {                                          \
        if (dbg()) {                              \
            fprintf(stderr, "[ipm] " __VA_ARGS__); \
            fflush(stderr);                       \
        }                                         \
    } while (0)
// IPM_DEBUG=2: synchronise after each stage and report (localises hangs / faults).
static int dbg_level() {
    const char *e = getenv("IPM_DEBUG");
    return e ? atoi(e) : 0;
}
#define DSYNC(label)                                                                        \
    do {                                                                                    \
        if (dbg_level() >= 2) {                                                             \
            fprintf(stderr, "[ipm] >> %s\n", label);                                        \
            fflush(stderr);                                                                 \
            cudaError_t e2_ = cudaStreamSynchronize(ctx->st);                               \
            fprintf(stderr, "[ipm] << %s: %s\n", label, cudaGetErrorString(e2_));           \
            fflush(stderr);                                                                 \
        }                                                                                   \
    } while (0)

struct Layout {
    size_t total = 0;
    size_t take(size_t bytes) {
        const size_t off = total;
        total += (bytes + 255) & ~size_t(255);
        return off;
    }
};

struct Offsets {
    size_t sc;
    size_t nvec[40];
    size_t mvec[40];
    size_t ypart, part, ATrp, ATcol, ATval, g, l, u, xl, xu, diagH, cnt, bad, gfull, xloc_all;
    size_t kd, ch0, cw, cs, cspart, chpart, symr, symt, symz, zcol, zvec, zall, hashes, peer;
    int n_nvec, n_mvec;
    int nchunk;
};

constexpr int kNVec = 30;   // n-space vectors in Vecs (see assign_vectors)
constexpr int kMVec = 38;   // m-space vectors (24 + 14 segments of the doubly augmented PCG)

// nloc = rows owned by this rank; every n-space vector gets chunk = ceil(n/P) (+2 pad) slots
// so the allgather can send equal blocks and the bulk GEMV may read one padding element.
Offsets plan(int64_t nloc, int64_t ncols, int64_t m, int64_t nnz_loc, int nranks, Layout &L, int64_t ldu = 0,
             int rank = 0, SymPlan *symp = nullptr) {
    Offsets o{};
    SymPlan sp;
    sym_plan_build((int)ncols, nranks, rank, gemv_bulk_grid(), sp);
    if (ldu > 0) {                     // compact Hessian (NEXT-1): h0, w, s = U^T p and partials
        o.ch0 = L.take(sizeof(double) * std::max<int64_t>(nloc, 1));
        o.cw = L.take(sizeof(double) * ldu);
        o.cs = L.take(sizeof(double) * ldu);
        o.cspart = L.take(sizeof(double) * ldu * kCompactGrid);
        o.chpart = L.take(sizeof(double) * kCompactGrid);
    }
    const int64_t chunk = (ncols + nranks - 1) / nranks;
    o.sc = L.take(sizeof(Scalars));
    for (int i = 0; i < kNVec; ++i) o.nvec[i] = L.take(sizeof(double) * (std::max<int64_t>(chunk, 1) + 2));
    for (int i = 0; i < kMVec; ++i) o.mvec[i] = L.take(sizeof(double) * std::max<int64_t>(m, 1));
    o.ypart = L.take(sizeof(double) * std::max<int64_t>(nloc, 1) * std::max(gemv_ncb((int)ncols), sp.ldy));
    o.symr = L.take(sizeof(SymRange) * sp.ranges.size());
    o.symt = L.take(sizeof(SymTile) * std::max<size_t>(1, sp.tiles.size()));
    o.symz = L.take(sizeof(double) * std::max<int64_t>(1, (int64_t)sp.zrows * sp.ldz));
    o.zcol = L.take(sizeof(int) * std::max<size_t>(1, sp.zcol.size()));
    o.zvec = L.take(sizeof(double) * (nranks > 1 ? ncols : 1));
    o.zall = L.take(sizeof(double) * (nranks > 1 ? ncols * nranks : 1));
    o.hashes = L.take(sizeof(unsigned long long) * (size_t)(nranks + 1) * (nranks + 1));
    if (symp) *symp = std::move(sp);
    o.part = L.take(sizeof(double) * kMaxPartials * 8);
    o.ATrp = L.take(sizeof(int64_t) * (nloc + 1));
    o.ATcol = L.take(sizeof(int) * std::max<int64_t>(nnz_loc, 1));
    o.ATval = L.take(sizeof(double) * std::max<int64_t>(nnz_loc, 1));
    o.g = L.take(sizeof(double) * std::max<int64_t>(nloc, 1));
    o.xl = L.take(sizeof(double) * std::max<int64_t>(nloc, 1));
    o.xu = L.take(sizeof(double) * std::max<int64_t>(nloc, 1));
    o.l = L.take(sizeof(double) * std::max<int64_t>(m, 1));
    o.u = L.take(sizeof(double) * std::max<int64_t>(m, 1));
    o.diagH = L.take(sizeof(double) * std::max<int64_t>(nloc, 1));
    o.kd = L.take(ncols <= kWarpMaxN && nranks == 1 ? sizeof(double) * kWarpMaxN * kWarpMaxN : 256);
    o.nchunk = (int)std::max<int64_t>(1, std::min<int64_t>(128, m));
    o.cnt = L.take(sizeof(int) * (size_t)o.nchunk * std::max<int64_t>(nloc, 1));
    o.bad = L.take(sizeof(unsigned long long));
    o.gfull = L.take(sizeof(double) * ((size_t)chunk * nranks + 2));
    o.xloc_all = L.take(sizeof(double) * 8 * (size_t)nranks);
    // peer-memory data plane (peer.h): the region other ranks store into (sharded only)
    o.peer = L.take(nranks > 1 && nranks <= kPeerMax ? peer_layout(ncols, m, nranks).bytes : 256);
    return o;
}

}  // namespace

struct ipm_ctx {
    int device = 0;
    cudaStream_t st = nullptr;   // user stream
    cudaStream_t cap = nullptr;  // private capture stream
    ipm_options opt{};
    int64_t n = 0, m = 0, nnz = 0;
    int row0 = 0, nloc = 0, rank = 0, nranks = 1;
    char *ws = nullptr;
    Prob P{};
    Vecs V{};
    Scalars *sc = nullptr;
    Scalars *hsc = nullptr;  // pinned host copy
    int G = 8;
    int ncb = 1;
    int gemv_grid = 148;
    int64_t nbounds = 0;
    // graph
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaGraphConditionalHandle handle = 0;
    bool graph_ready = false;
    bool fused_p = false;        // PCG iterations use k_pcg_update_fp (p-update fused, cooperative)
    bool sym_sharded = false;    // row-sharded symmetric GEMV: remote column parts exchanged per apply
    int sym_zrows = 0;
    int *sym_zcol = nullptr;
    double *sym_zvec = nullptr, *sym_zall = nullptr;
    // state
    bool have_iterate = false;   // V holds a valid iterate (after a solve or set_iterate)
    bool user_iterate = false;   // set_iterate called: next solve starts from it
    bool warm_pending = false;   // ipm_warm_start called
    bool have_dx = false;        // V.dx holds a previous PCG solution (PCG warm start)
    double mu = 0.0;
    ipm_stats stats{};
    std::vector<ipm_trace_rec> trace;
    std::string err;
    int64_t launches = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    alignas(64) unsigned char tmap_sym[128] = {};   // CUtensorMap for the symmetric GEMV
    ipm::Fork fork{nullptr, nullptr, nullptr};      // SpMV || GEMV branch of a PCG iteration
    // row-sharded mode
    ipm::Comm *comm = nullptr;
    bool sharded = false;
    int64_t chunk = 0;
    // peer-memory data plane (peer.h): device-side exchanges instead of Comm allgathers
    bool peer_on = false;
    bool a_split = false;        // PCG SpMV over this rank's rows of A only (peer plane, opt.a_row_split)
    bool cg = false;             // Chronopoulos-Gear single-reduction PCG (sharded, opt.pcg_single_reduction)
    ipm::PeerArgs peer{};
    std::vector<void *> ipc_opened;
    // one-warp whole-IPM path (tiny.cu): mapped pinned host buffer for its result and trace
    void *tiny_host = nullptr;
    size_t tiny_cap = 0;
};

namespace {

ipm_status fail(ipm_ctx *c, ipm_status s, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    else g_create_error = buf;
    return s;
}

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) return fail(ctx, IPM_ERR_CUDA, "%s: %s (%s:%d)", #call,              \
                                           cudaGetErrorString(e_), __FILE__, __LINE__);            \
    } while (0)

#define CKL()                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = cudaGetLastError();                                                        \
        if (e_ != cudaSuccess) return fail(ctx, IPM_ERR_CUDA, "kernel launch: %s (%s:%d)",         \
                                           cudaGetErrorString(e_), __FILE__, __LINE__);            \
    } while (0)

#define TRY(expr)                          \
    do {                                   \
        ipm_status s_ = (expr);            \
        if (s_ != IPM_OK) return s_;       \
    } while (0)

// Peer-memory data plane setup (peer.h): exchange the peer regions' addresses over the Comm
// (bootstrap only) — raw pointers between ranks of one process (peer access enabled across
// devices), CUDA IPC handles between processes — and point V.gfull at the region's gfull.
// IPM_PEER=0 (experiment switch) keeps the Comm allgather data plane.
using DrvGetAddressRange = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);

ipm_status setup_peer(ipm_ctx *ctx, char *region, char *scratch) {
    const int R = ctx->comm->nranks, me = ctx->comm->rank;
    const char *env = getenv("IPM_PEER");
    if (R < 2 || R > kPeerMax || (env && atoi(env) == 0)) return IPM_OK;
    struct Ex {
        cudaIpcMemHandle_t h;
        int64_t off;
        uint64_t raw;
        int32_t pid, dev;
    };
    Ex mine{};
    mine.raw = reinterpret_cast<uint64_t>(region);
    mine.pid = (int32_t)getpid();
    mine.dev = ctx->device;
    {   // CUDA IPC needs the allocation base (the workspace may be a sub-allocation of torch's pool)
        static DrvGetAddressRange range = nullptr;
        if (!range) {
            cudaDriverEntryPointQueryResult q;
            void *fn = nullptr;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                range = reinterpret_cast<DrvGetAddressRange>(fn);
        }
        CUdeviceptr base = 0;
        size_t sz = 0;
        if (!range || range(&base, &sz, reinterpret_cast<CUdeviceptr>(region)) != CUDA_SUCCESS)
            return fail(ctx, IPM_ERR_CUDA, "cuMemGetAddressRange failed on the workspace");
        mine.off = (int64_t)(reinterpret_cast<CUdeviceptr>(region) - base);
        if (cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void *>(base)) != cudaSuccess) {
            cudaGetLastError();
            std::memset(&mine.h, 0, sizeof mine.h);   // same-process groups do not need it
        }
    }
    Ex *dsend = reinterpret_cast<Ex *>(scratch);
    Ex *drecv = dsend + 1;
    CK(cudaMemcpyAsync(dsend, &mine, sizeof mine, cudaMemcpyHostToDevice, ctx->st));
    std::string e;
    if (ctx->comm->allgather(dsend, drecv, sizeof(Ex), ctx->st, e)) return fail(ctx, IPM_ERR_NCCL, "%s", e.c_str());
    std::vector<Ex> all(R);
    CK(cudaMemcpyAsync(all.data(), drecv, sizeof(Ex) * R, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    PeerArgs pa{};
    if (const char *t = getenv("IPM_PEER_TIMEOUT_S")) pa.timeout_ns = (unsigned long long)(atof(t) * 1e9);
    pa.rank = me;
    pa.P = R;
    pa.chunk = ctx->chunk;
    pa.m = ctx->m;
    pa.L = peer_layout(ctx->n, ctx->m, R);
    for (int r = 0; r < R; ++r) {
        if (r == me) {
            pa.base[r] = region;
        } else if (all[r].pid == mine.pid) {
            if (all[r].dev != ctx->device) {
                const cudaError_t pe = cudaDeviceEnablePeerAccess(all[r].dev, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
                    return fail(ctx, IPM_ERR_CUDA, "peer access %d -> %d: %s", ctx->device, all[r].dev,
                                cudaGetErrorString(pe));
                cudaGetLastError();
            }
            pa.base[r] = reinterpret_cast<char *>(all[r].raw);
        } else {
            void *ptr = nullptr;
            CK(cudaIpcOpenMemHandle(&ptr, all[r].h, cudaIpcMemLazyEnablePeerAccess));
            ctx->ipc_opened.push_back(ptr);
            pa.base[r] = static_cast<char *>(ptr) + all[r].off;
        }
    }
    ctx->peer = pa;
    ctx->peer_on = true;
    ctx->a_split = ctx->opt.a_row_split != 0 && ctx->m > 0;
    const int64_t split = ctx->a_split ? 1 : 0;
    CK(cudaMemcpyAsync(&ctx->sc->spmv_split, &split, sizeof split, cudaMemcpyHostToDevice, ctx->st));
    ctx->V.gfull = reinterpret_cast<double *>(region + pa.L.gfull);
    // everybody's region is zeroed (workspace memset) before anyone may store into it
    CK(cudaStreamSynchronize(ctx->st));
    if (ctx->comm->allgather(dsend, drecv, sizeof(Ex), ctx->st, e)) return fail(ctx, IPM_ERR_NCCL, "%s", e.c_str());
    CK(cudaStreamSynchronize(ctx->st));
    return IPM_OK;
}

ipm_status peer_timeout_error(ipm_ctx *ctx) {
    const unsigned long long *d = ctx->hsc->peer_diag;
    return fail(ctx, IPM_ERR_NCCL,
                "peer exchange timed out on rank %d: exchange %llu (stage %lld) never arrived from rank %llu "
                "(its flag = %llu)",
                ctx->peer.rank, d[0], (long long)d[3] - 1000, d[1], d[2]);
}

ipm_status sync_scalars(ipm_ctx *ctx) {
    CKL();
    CK(cudaMemcpyAsync(ctx->hsc, ctx->sc, sizeof(Scalars), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (ctx->peer_on && ctx->hsc->peer_timeout) return peer_timeout_error(ctx);
    return IPM_OK;
}

void assign_vectors(ipm_ctx *c, const Offsets &o) {
    char *b = c->ws;
    double *nv[kNVec];
    double *mv[kMVec];
    for (int i = 0; i < kNVec; ++i) nv[i] = reinterpret_cast<double *>(b + o.nvec[i]);
    for (int i = 0; i < kMVec; ++i) mv[i] = reinterpret_cast<double *>(b + o.mvec[i]);
    Vecs &V = c->V;
    int k = 0;
    V.x = nv[k++]; V.s_lx = nv[k++]; V.s_ux = nv[k++]; V.lam_lx = nv[k++]; V.lam_ux = nv[k++];
    V.rH = nv[k++]; V.r_lx = nv[k++]; V.r_ux = nv[k++]; V.rc_lx = nv[k++]; V.rc_ux = nv[k++]; V.Hx = nv[k++];
    V.sig_b = nv[k++]; V.Minv = nv[k++]; V.rhs = nv[k++]; V.dx = nv[k++];
    V.ds_lx = nv[k++]; V.ds_ux = nv[k++]; V.dl_lx = nv[k++]; V.dl_ux = nv[k++];
    V.ads_lx = nv[k++]; V.ads_ux = nv[k++]; V.adl_lx = nv[k++]; V.adl_ux = nv[k++];
    V.pr = nv[k++]; V.pz = nv[k++]; V.pp = nv[k++]; V.py = nv[k++]; V.pAt = nv[k++];
    int j = 0;
    V.s_lA = mv[j++]; V.s_uA = mv[j++]; V.lam_lA = mv[j++]; V.lam_uA = mv[j++];
    V.r_lA = mv[j++]; V.r_uA = mv[j++]; V.rc_lA = mv[j++]; V.rc_uA = mv[j++]; V.Ax = mv[j++];
    V.sig_c = mv[j++]; V.r2_l = mv[j++]; V.r2_u = mv[j++]; V.w = mv[j++]; V.Adx = mv[j++];
    V.ds_lA = mv[j++]; V.ds_uA = mv[j++]; V.dl_lA = mv[j++]; V.dl_uA = mv[j++];
    V.ads_lA = mv[j++]; V.ads_uA = mv[j++]; V.adl_lA = mv[j++]; V.adl_uA = mv[j++];
    V.lamd = mv[j++]; V.pt = mv[j++];
    V.ag.xl = mv[j++]; V.ag.xu = mv[j++]; V.ag.rl = mv[j++]; V.ag.ru = mv[j++]; V.ag.zl = mv[j++]; V.ag.zu = mv[j++];
    V.ag.pl = mv[j++]; V.ag.pu = mv[j++]; V.ag.yl = mv[j++]; V.ag.yu = mv[j++]; V.ag.Dl = mv[j++]; V.ag.Du = mv[j++];
    V.ag.Ml = mv[j++]; V.ag.Mu = mv[j++];
    V.ypart = reinterpret_cast<double *>(b + o.ypart);
    for (int i = 0; i < 8; ++i) V.part[i] = reinterpret_cast<double *>(b + o.part) + (size_t)i * kMaxPartials;
    V.gfull = reinterpret_cast<double *>(b + o.gfull);
    V.xloc_all = reinterpret_cast<double *>(b + o.xloc_all);
}

// ------------------------------------------------------------------- sharded collectives
// Full-length copy of an x-space vector: the vector itself on one GPU, else an allgather of
// every rank's chunk into V.gfull (rank r's rows land at [r*chunk, ...), i.e. global order).
ipm_status gather(ipm_ctx *ctx, const double *local, const double **full, cudaStream_t st = nullptr,
                  int check_done = 0) {
    if (!ctx->sharded) {
        *full = local;
        return IPM_OK;
    }
    if (ctx->peer_on) {                // every rank stores its slice into every peer's gfull (peer.h)
        st = st ? st : ctx->st;
        launch_peer_put_vec(ctx->peer, local, ctx->nloc, ctx->peer.L.gfull, ctx->peer.rank * ctx->chunk, 0, ctx->sc,
                            check_done, st);
        launch_peer_wait(ctx->peer, ctx->sc, -1, 0.0, 0.0, 0, check_done, 0, 0, st);
        ctx->launches += 2;
        CKL();
        *full = ctx->V.gfull;          // = the peer region's gfull
        return IPM_OK;
    }
    std::string e;
    if (ctx->comm->allgather(local, ctx->V.gfull, sizeof(double) * ctx->chunk, ctx->st, e))
        return fail(ctx, IPM_ERR_NCCL, "%s", e.c_str());
    *full = ctx->V.gfull;
    return IPM_OK;
}

// Sharded symmetric GEMV: the column parts this rank computed for other ranks' rows (zpart)
// are reduced to a full-length vector, allgathered, and each rank adds the P contributions to
// its rows in rank order into the last ypart slot (shard.cu).  No-op otherwise.
ipm_status sym_exchange(ipm_ctx *ctx, cudaStream_t st = nullptr, int check_done = 0) {
    if (!ctx->sym_sharded) return IPM_OK;
    const Prob &P = ctx->P;
    if (ctx->peer_on) {                // fused zreduce + scatter to the owning ranks, wait, fold
        st = st ? st : ctx->st;
        launch_peer_zput(ctx->peer, ctx->sym_zrows, P.sym_ldz, P.sym_z, ctx->sym_zcol, ctx->sc, check_done, st);
        launch_peer_wait(ctx->peer, ctx->sc, -1, 0.0, 0.0, 0, check_done, 0, 0, st);
        launch_peer_zfold(ctx->peer, P.n, ctx->V.ypart, ctx->ncb, ctx->sc, check_done, st);
        ctx->launches += 3;
        CKL();
        return IPM_OK;
    }
    launch_zreduce(ctx->sym_zrows, P.sym_ldz, P.sym_z, ctx->sym_zcol, ctx->sym_zvec, ctx->st);
    CKL();
    std::string e;
    if (ctx->comm->allgather(ctx->sym_zvec, ctx->sym_zall, sizeof(double) * P.ncols, ctx->st, e))
        return fail(ctx, IPM_ERR_NCCL, "%s", e.c_str());
    launch_zfold(P.n, P.ncols, ctx->comm->nranks, ctx->row0, ctx->sym_zall, ctx->V.ypart, ctx->ncb, ctx->st);
    ctx->launches += 2;
    CKL();
    return IPM_OK;
}

// Combine this stage's per-rank partials (Scalars::loc) across ranks (shard.cu).
ipm_status xcombine(ipm_ctx *ctx, int stage, double p0 = 0.0, double p1 = 0.0, int64_t p2 = 0,
                    cudaStream_t st = nullptr, int check_done = 0, cudaGraphConditionalHandle h = 0, int use_cond = 0) {
    if (!ctx->sharded) return IPM_OK;
    if (ctx->peer_on) {                // this rank's partials into every peer's xall[stage]; wait + combine
        st = st ? st : ctx->st;
        launch_peer_put_loc(ctx->peer, stage, ctx->sc, check_done, st);
        launch_peer_wait(ctx->peer, ctx->sc, stage, p0, p1, p2, check_done, h, use_cond, st);
        ctx->launches += 2;
        CKL();
        return IPM_OK;
    }
    std::string e;
    if (ctx->comm->allgather(ctx->sc->loc, ctx->V.xloc_all, sizeof(double) * 8, ctx->st, e))
        return fail(ctx, IPM_ERR_NCCL, "%s", e.c_str());
    launch_xcombine(ctx->sc, ctx->V.xloc_all, ctx->comm->nranks, stage, p0, p1, p2, ctx->st);
    ctx->launches += 1;
    CKL();
    return IPM_OK;
}

int choose_group(int64_t nnz_loc, int64_t nloc, int ncb) {
    const double avg = nloc > 0 ? (double)nnz_loc / (double)nloc : 0.0;
    const double work = std::max(avg, (double)ncb);
    if (work <= 6) return 4;
    if (work <= 12) return 8;
    if (work <= 24) return 16;
    return 32;
}

double pcg_rtol(const ipm_options &o, double mu) {
    if (o.pcg_schedule == 1) return std::max(1e-10, std::min(1e-2, 0.1 * mu));
    return std::max(o.pcg_rtol_floor, std::min(o.pcg_rtol_max, o.pcg_rtol_mu_factor * mu));
}

// ---------------------------------------------------------------------------- operators
// y = K v with the current sig_b/sig_c (t and ypart are scratch).  mode 1: r = rhs - K v.
// v_local: workspace x-space vector (this rank's rows); v_full: its full-length version or
// nullptr to gather it.  Result rows are local.
ipm_status op_apply(ipm_ctx *ctx, const double *v_local, const double *v_full, double *out, const double *rhs,
                    int mode) {
    const Prob &P = ctx->P;
    const Vecs &V = ctx->V;
    if (!v_full) TRY(gather(ctx, v_local, &v_full));
    // mode 1 on an augmented context: the true residual of eq:2x2_augmented, whose dlam
    // segments are the PCG's own (V.ag.x*); the public operator (mode 0) stays condensed
    const bool aug = P.aug && mode == 1;
    const AugArgs ag = aug_args(P, V);
    if (aug) launch_spmv_aug(P, V, v_full, V.ag.xl, V.ag.xu, ctx->sc, 0, ctx->st);
    else launch_spmv(P, v_full, V.sig_c, V.pt, V.part[3], ctx->sc, 1, 0, ctx->st);
    launch_gemv(P, v_full, nullptr, V.ypart, ctx->ncb, V.part[4], ctx->sc, ctx->gemv_grid, 0, C_GEMV, ctx->st);
    TRY(sym_exchange(ctx));
    launch_apply_reduce(P, ctx->G, ctx->ncb, V.ypart, V.sig_b, v_local, V.pt, out, rhs, V.part[5], ctx->sc, mode,
                        ctx->st, aug ? &ag : nullptr);
    ctx->launches += (P.m > 0 ? 1 : 0) + 2;
    CKL();
    if (mode == 1) TRY(xcombine(ctx, X_RES2));
    return IPM_OK;
}

// One PCG iteration on a row-sharded context (no graph: collectives between the kernels).
// st = nullptr: the context stream (host-driven); otherwise the graph-capture stream, and with
// use_cond the last exchange sets the WHILE condition (peer data plane only: no host calls).
// Peer data plane: the SpMV stage runs on the side branch next to the SYMV (as on one GPU);
// with the A-row split (opt.a_row_split) each rank forms t only for its rows of A and the
// slices are allgathered over peer memory on the side branch's own exchange channel.
ipm_status pcg_iteration_sharded(ipm_ctx *ctx, cudaStream_t st = nullptr, int use_cond = 0) {
    const Prob &P = ctx->P;
    const Vecs &V = ctx->V;
    st = st ? st : ctx->st;
    launch_pcg_p(P, V, ctx->sc, st);
    const double *pf = nullptr;
    TRY(gather(ctx, V.pp, &pf, st, 1));
    const bool par = ctx->peer_on && P.m > 0;
    if (par) {
        cudaStream_t side = ctx->fork.side;
        CK(cudaEventRecord(ctx->fork.ev_fork, st));
        CK(cudaStreamWaitEvent(side, ctx->fork.ev_fork, 0));
        const double *t = V.pt;
        if (ctx->a_split) {
            const PeerArgs &pa = ctx->peer;
            double *tall = reinterpret_cast<double *>(pa.base[pa.rank] + pa.L.tall);
            const int64_t m0 = peer_mrow0(pa, pa.rank), m1 = peer_mrow0(pa, pa.rank + 1);
            launch_spmv_rows(P, pf, V.sig_c, tall, V.part[3], ctx->sc, m0, m1, side, side_block());
            launch_peer_put_vec(pa, tall + m0, m1 - m0, pa.L.tall, m0, 1, ctx->sc, 1, side);
            launch_peer_wait(pa, ctx->sc, -1, 0.0, 0.0, 0, 1, 0, 0, side, 1);
            t = tall;
            ctx->launches += 2;
        } else {
            launch_spmv(P, pf, V.sig_c, V.pt, V.part[3], ctx->sc, 1, 1, side, kMaxGrid, side_block());
        }
        launch_pcg_spmvT(P, V, ctx->G, ctx->sc, t, side);
        CK(cudaEventRecord(ctx->fork.ev_join, side));
        launch_gemv(P, pf, V.pp, V.ypart, ctx->ncb, V.part[4], ctx->sc, ctx->gemv_grid, 1, C_GEMV_PCG, st);
        TRY(sym_exchange(ctx, st, 1));
        CK(cudaStreamWaitEvent(st, ctx->fork.ev_join, 0));
        TRY(xcombine(ctx, X_PCG_ALPHA, 0.0, 0.0, 0, st, 1));
        launch_pcg_update_only(P, V, ctx->G, ctx->ncb, ctx->sc, V.dx, st);
    } else {
        launch_spmv(P, pf, V.sig_c, V.pt, V.part[3], ctx->sc, 1, 1, st, kMaxGrid, side_block());
        launch_gemv(P, pf, V.pp, V.ypart, ctx->ncb, V.part[4], ctx->sc, ctx->gemv_grid, 1, C_GEMV_PCG, st);
        TRY(sym_exchange(ctx, st, 1));
        TRY(xcombine(ctx, X_PCG_ALPHA, 0.0, 0.0, 0, st, 1));
        launch_pcg_update(P, V, ctx->G, ctx->ncb, ctx->sc, V.dx, st);
    }
    TRY(xcombine(ctx, X_PCG_UPDATE, 0.0, 0.0, 0, st, 1, ctx->handle, use_cond));
    ctx->launches += 3 + (P.m > 0 ? 2 : 0);
    CKL();
    return IPM_OK;
}

// Chronopoulos-Gear single-reduction PCG (opt.pcg_single_reduction, sharded): the operator is
// applied to u = M^-1 r; ONE scalar exchange per iteration (X_CG: S_b, S_H, S_c, r^T u, ||r||^2)
// decides the stop and alpha, beta; p and s = K p follow by recurrence in k_cg_update.  The
// standard loop needs two (X_PCG_ALPHA after the operator, X_PCG_UPDATE after the update).
ipm_status pcg_iteration_cg(ipm_ctx *ctx, cudaStream_t st = nullptr, int use_cond = 0) {
    const Prob &P = ctx->P;
    const Vecs &V = ctx->V;
    st = st ? st : ctx->st;
    const double *uf = nullptr;
    TRY(gather(ctx, V.pz, &uf, st, 1));
    const bool par = P.m > 0;
    if (par) {
        cudaStream_t side = ctx->fork.side;
        CK(cudaEventRecord(ctx->fork.ev_fork, st));
        CK(cudaStreamWaitEvent(side, ctx->fork.ev_fork, 0));
        const double *t = V.pt;
        if (ctx->a_split) {
            const PeerArgs &pa = ctx->peer;
            double *tall = reinterpret_cast<double *>(pa.base[pa.rank] + pa.L.tall);
            const int64_t m0 = peer_mrow0(pa, pa.rank), m1 = peer_mrow0(pa, pa.rank + 1);
            launch_spmv_rows(P, uf, V.sig_c, tall, V.part[3], ctx->sc, m0, m1, side, side_block());
            launch_peer_put_vec(pa, tall + m0, m1 - m0, pa.L.tall, m0, 1, ctx->sc, 1, side);
            launch_peer_wait(pa, ctx->sc, -1, 0.0, 0.0, 0, 1, 0, 0, side, 1);
            t = tall;
        } else {
            launch_spmv(P, uf, V.sig_c, V.pt, V.part[3], ctx->sc, 1, 1, side, kMaxGrid, side_block());
        }
        launch_pcg_spmvT(P, V, ctx->G, ctx->sc, t, side);
        CK(cudaEventRecord(ctx->fork.ev_join, side));
    }
    launch_gemv(P, uf, V.pz, V.ypart, ctx->ncb, V.part[4], ctx->sc, ctx->gemv_grid, 1, C_GEMV_PCG, st);
    TRY(sym_exchange(ctx, st, 1));
    if (par) CK(cudaStreamWaitEvent(st, ctx->fork.ev_join, 0));
    TRY(xcombine(ctx, X_CG, 0.0, 0.0, 0, st, 1, ctx->handle, use_cond));
    launch_cg_update(P, V, ctx->ncb, ctx->sc, V.dx, st);
    ctx->launches += 3 + (P.m > 0 ? 2 : 0);
    CKL();
    return IPM_OK;
}

ipm_status build_graph(ipm_ctx *ctx) {
    if (ctx->graph_ready) return IPM_OK;
    CK(cudaGraphCreate(&ctx->graph, 0));
    CK(cudaGraphConditionalHandleCreate(&ctx->handle, ctx->graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = ctx->handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, ctx->graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(ctx->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    // IPM_UNROLL (experiment): k PCG iterations per WHILE trip; an iteration after the stop
    // early-exits in every kernel (sc->done), and the last update sets the condition
    const char *ue = getenv("IPM_UNROLL");
    const int unroll = ue ? std::max(1, std::min(8, atoi(ue))) : 1;
    if (ctx->sharded) {
        // peer data plane: the whole sharded iteration (puts, waits, combines) is device-side
        if (ctx->cg) TRY(pcg_iteration_cg(ctx, ctx->cap, 1));
        else TRY(pcg_iteration_sharded(ctx, ctx->cap, 1));
    } else {
        for (int u = 0; u < unroll; ++u)
            launch_pcg_iteration(ctx->P, ctx->V, ctx->G, ctx->ncb, ctx->gemv_grid, ctx->sc, ctx->V.dx, ctx->handle,
                                 1, ctx->cap, &ctx->fork, ctx->fused_p);
    }
    cudaGraph_t captured = nullptr;
    CK(cudaStreamEndCapture(ctx->cap, &captured));
    CK(cudaGraphInstantiate(&ctx->gexec, ctx->graph, 0));
    ctx->graph_ready = true;
    return IPM_OK;
}

struct PcgOut {
    int64_t iters = 0;
    double relres = 0.0;
    bool stalled = false;
    int restarts = 0;
    bool deferred = false;   // one-warp path launched without a host sync: collect at the next sync
};

// Results of a deferred one-warp PCG solve from the host copy of the scalars (after a sync).
ipm_status pcg_collect(ipm_ctx *ctx, PcgOut &out) {
    if (!out.deferred) return IPM_OK;
    out.deferred = false;
    const Scalars &h = *ctx->hsc;
    out.iters = h.it;
    out.relres = h.rhs2 > 0 ? std::sqrt(h.res2 / h.rhs2) : 0.0;
    out.stalled = h.stalled != 0;
    out.restarts = (int)h.restarts;
    if (h.breakdown)
        return fail(ctx, IPM_ERR_PCG_BREAKDOWN, "PCG breakdown at iteration %lld (p^T K p = %g)", (long long)h.it, h.pKp);
    if (!std::isfinite(h.res2)) return fail(ctx, IPM_ERR_NONFINITE, "non-finite PCG residual");
    return IPM_OK;
}

// Solve K dx = rhs (V.rhs -> V.dx) with the current diagonals; Minv already set.
// fixed > 0 (test hook ipm_pcg_iterate): exactly `fixed` iterations from x0 = 0 — no stopping
// test (tolerance 0), no true-residual confirmation, no restart; same kernels and launch path.
// defer: the one-warp path (n <= kWarpMaxN) returns without a host sync, out.deferred set; the
// caller runs pcg_collect after its next sync_scalars.
ipm_status pcg_solve(ipm_ctx *ctx, double rtol, PcgOut &out, int64_t fixed = 0, bool defer = false) {
    const Prob &P = ctx->P;
    Vecs &V = ctx->V;
    int64_t maxit = ctx->opt.pcg_max_iter > 0 ? ctx->opt.pcg_max_iter : 10 * (int64_t)ctx->n;
    double atol = ctx->opt.pcg_atol;
    if (fixed > 0) {
        maxit = fixed;
        rtol = 0.0;
        atol = 0.0;
    }
    // warm start (option): x0 = the previous direction still held in V.dx
    const int warm = (fixed == 0 && ctx->opt.pcg_warm_start && ctx->have_dx) ? 1 : 0;
    launch_pcg_init(P, V, ctx->sc, V.rhs, V.dx, rtol, atol, maxit, warm, ctx->st);
    DSYNC("pcg_init");
    ctx->launches += 1;
    CKL();
    TRY(xcombine(ctx, X_PCG_INIT, rtol, atol, maxit));
    if (warm) {
        TRY(op_apply(ctx, V.dx, nullptr, V.pr, V.rhs, 1));      // r = rhs - K x0
        launch_pcg_restart(P, V, ctx->sc, ctx->st);              // z, rho, rr, done
        ctx->launches += 1;
        CKL();
        TRY(xcombine(ctx, X_PCG_RESTART));
    }
    ctx->have_dx = true;
    const bool small = !ctx->sharded && !P.aug && !P.hess_compact && P.n <= kSmallN && ctx->opt.use_graph;
    const bool graph = ctx->opt.use_graph && (!ctx->sharded || ctx->peer_on) && !small;
    if (graph) TRY(build_graph(ctx));
    out = PcgOut{};
    if (small && pcg_warp_path(P)) {               // the whole solve, restarts included, in one warp
        ctx->launches += launch_pcg_small(P, V, ctx->sc, V.dx, V.rhs, fixed == 0 ? 1 : 0, ctx->st);
        CKL();
        out.deferred = true;
        if (defer) return IPM_OK;
        TRY(sync_scalars(ctx));
        return pcg_collect(ctx, out);
    }
    int64_t it_prev = 0;
    // kernels per PCG iteration (sharded peer plane: + 2 per exchange, + zfold)
    const int per_it = (ctx->fused_p ? 2 : 3) + (P.m > 0 ? 2 : 0) +
                       (ctx->sharded && ctx->peer_on ? 6 + (ctx->sym_sharded ? 3 : 0) : 0);
    for (int round = 0;; ++round) {
        if (ctx->cg) {                                      // gamma, ||r||^2, S_b of u = M^-1 r
            launch_cg_prime(P, V, ctx->sc, ctx->st);
            ctx->launches += 1;
            CKL();
        }
        if (ctx->fused_p && !small) {
            launch_pcg_p(P, V, ctx->sc, ctx->st);           // p = z after the (re)start; S_b
            ctx->launches += 1;
            CKL();
        }
        if (small) {
            ctx->launches += launch_pcg_small(P, V, ctx->sc, V.dx, V.rhs, 0, ctx->st);
            TRY(sync_scalars(ctx));
        } else if (graph) {
            CK(cudaGraphLaunch(ctx->gexec, ctx->st));
            TRY(sync_scalars(ctx));
            if (ctx->hsc->peer_timeout) return peer_timeout_error(ctx);
        } else if (ctx->sharded) {
            // host-driven batches; every rank sees the same combined `done`, so all ranks run
            // the same number of iterations and collectives
            for (;;) {
                for (int b = 0; b < 16; ++b) TRY(ctx->cg ? pcg_iteration_cg(ctx) : pcg_iteration_sharded(ctx));
                TRY(sync_scalars(ctx));
                if (ctx->hsc->done) break;
            }
        } else {
            // host-driven fallback: batches of 16 iterations with device-side early exit
            for (;;) {
                for (int b = 0; b < 16; ++b)
                    launch_pcg_iteration(P, V, ctx->G, ctx->ncb, ctx->gemv_grid, ctx->sc, V.dx, 0, 0, ctx->st, &ctx->fork,
                                         ctx->fused_p);
                TRY(sync_scalars(ctx));
                DBG("  host batch: it=%lld rr=%.3e done=%lld\n", (long long)ctx->hsc->it, ctx->hsc->rr, (long long)ctx->hsc->done);
                ctx->launches += 16 * per_it;
                if (ctx->hsc->done) break;
            }
        }
        const Scalars &h = *ctx->hsc;
        DBG("pcg round %d: it=%lld rr=%.3e tol2=%.3e done=%lld breakdown=%lld rho=%.3e pKp=%.3e\n", round,
            (long long)h.it, h.rr, h.tol2, (long long)h.done, (long long)h.breakdown, h.rho, h.pKp);
        if (graph) ctx->launches += std::max<int64_t>(1, h.it - it_prev) * per_it;
        it_prev = h.it;
        if (h.breakdown) {
            out.iters = h.it;
            return fail(ctx, IPM_ERR_PCG_BREAKDOWN, "PCG breakdown at iteration %lld (p^T K p = %g)",
                        (long long)h.it, h.pKp);
        }
        if (fixed > 0) {
            out.iters = h.it;
            break;
        }
        // true residual confirmation: r = rhs - K dx
        TRY(op_apply(ctx, V.dx, nullptr, V.pr, V.rhs, 1));
        TRY(sync_scalars(ctx));
        const double res2 = ctx->hsc->res2, tol2 = ctx->hsc->tol2, rhs2 = ctx->hsc->rhs2;
        out.iters = ctx->hsc->it;
        out.relres = rhs2 > 0 ? std::sqrt(res2 / rhs2) : 0.0;
        if (!std::isfinite(res2)) return fail(ctx, IPM_ERR_NONFINITE, "non-finite PCG residual");
        if (res2 <= tol2) break;
        if (ctx->hsc->it >= maxit || round >= 8) {
            out.stalled = true;
            break;
        }
        out.restarts++;
        launch_pcg_restart(P, V, ctx->sc, ctx->st);
        ctx->launches += 1;
        CKL();
        TRY(xcombine(ctx, X_PCG_RESTART));
    }
    return IPM_OK;
}

// Hx (GEMV tiles) + Ax (SpMV), then the residual kernels at the given mu.  reuse: x has not
// moved since the last call (its H x tile partials and A x are still in ypart / Ax) — only the
// residual kernels run (the final report at a new mu).
ipm_status residuals(ipm_ctx *ctx, double mu, bool reuse = false) {
    const Prob &P = ctx->P;
    const Vecs &V = ctx->V;
    if (!reuse) {
        const double *xf = nullptr;
        TRY(gather(ctx, V.x, &xf));
        launch_gemv(P, xf, nullptr, V.ypart, ctx->ncb, V.part[4], ctx->sc, ctx->gemv_grid, 0, C_GEMV, ctx->st);
        TRY(sym_exchange(ctx));
        DSYNC("gemv Hx");
        launch_spmv(P, xf, nullptr, V.Ax, nullptr, ctx->sc, 0, 0, ctx->st);
        DSYNC("spmv Ax");
        ctx->launches += 1 + (P.m > 0 ? 1 : 0);
    }
    launch_residuals(P, V, ctx->G, ctx->sc, mu, ctx->st);
    DSYNC("residual kernels");
    ctx->launches += 1 + (P.m > 0 ? 1 : 0);
    CKL();
    TRY(xcombine(ctx, X_RESID));
    return IPM_OK;
}

double kkt_inf(const Scalars &h) { return std::max(h.rH_max, std::max(h.prim_max, h.comp_max)); }

// One Newton direction (Alg. 1 lines 2-3) into V.dx / V.d* ; step lengths in sc->alpha_*.
ipm_status direction(ipm_ctx *ctx, double mu, int mode, double smu, double tau, int aff, PcgOut &po, float &tpcg) {
    const Prob &P = ctx->P;
    const Vecs &V = ctx->V;
    launch_rhs(P, V, ctx->G, mu, mode, smu, ctx->st);
    ctx->launches += 1 + (P.m > 0 ? 1 : 0);
    CKL();
    CK(cudaEventRecord(ctx->ev[2], ctx->st));
    TRY(pcg_solve(ctx, pcg_rtol(ctx->opt, mu), po, 0, true));
    CK(cudaEventRecord(ctx->ev[3], ctx->st));
    if (!po.deferred) {
        float ms = 0.f;
        CK(cudaEventSynchronize(ctx->ev[3]));
        CK(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
        tpcg += ms;
    }
    const double *dxf = nullptr;
    TRY(gather(ctx, V.dx, &dxf));
    launch_spmv(P, dxf, nullptr, V.Adx, nullptr, ctx->sc, 0, 0, ctx->st);
    launch_recover(P, V, ctx->sc, tau, aff, ctx->st);
    ctx->launches += 1 + 2 * (P.m > 0 ? 1 : 0);
    CKL();
    TRY(xcombine(ctx, X_RECOVER, tau));
    return IPM_OK;
}

ipm_status start_point(ipm_ctx *ctx) {
    const Prob &P = ctx->P;
    const Vecs &V = ctx->V;
    if (ctx->user_iterate) {
        ctx->user_iterate = false;
        return IPM_OK;
    }
    const int warm = ctx->warm_pending ? 1 : 0;
    ctx->warm_pending = false;
    launch_init_x(P, V, warm, ctx->opt.warm_shift, ctx->st);
    DSYNC("init_x");
    const double *xf = nullptr;
    TRY(gather(ctx, V.x, &xf));
    launch_spmv(P, xf, nullptr, V.Ax, nullptr, ctx->sc, 0, 0, ctx->st);
    DSYNC("spmv Ax0");
    launch_init_slacks(P, V, ctx->sc, warm, ctx->opt.warm_shift, ctx->st);
    DSYNC("init_slacks");
    ctx->launches += 2 + 2 * (P.m > 0 ? 1 : 0);
    TRY(xcombine(ctx, X_SUMLS));
    TRY(sync_scalars(ctx));
    if (ctx->nbounds == 0) ctx->mu = ctx->opt.mu_tol;                                   // R13
    else ctx->mu = ctx->opt.mu0_scale * ctx->hsc->sum_ls / (double)ctx->nbounds;      // R5
    return IPM_OK;
}

// n, m <= kWarpMaxN, plain Algorithm 1 (no predictor-corrector, no PCG warm start), condensed
// system, explicit H, one GPU: the whole loop in one warp (tiny.cu).  IPM_TINY=0 disables.
static bool tiny_path(const ipm_ctx *ctx) {
    static int env = -1;
    if (env < 0) {
        const char *e = getenv("IPM_TINY");
        env = e ? atoi(e) : 1;
    }
    const Prob &P = ctx->P;
    return env && !ctx->sharded && !P.aug && !P.hess_compact && tiny_eligible(P.n, P.m) &&
           !ctx->opt.predictor_corrector && !ctx->opt.pcg_warm_start && ctx->opt.use_graph;
}

// Algorithm 1 after the start point, in one launch; stats, trace and status from its result.
ipm_status solve_tiny(ipm_ctx *ctx) {
    const ipm_options &o = ctx->opt;
    const Prob &P = ctx->P;
    Vecs &V = ctx->V;
    ipm_stats &S = ctx->stats;
    const size_t need = sizeof(TinyOut) + sizeof(ipm_trace_rec) * (size_t)std::max(1, o.max_ipm_iter);
    if (ctx->tiny_cap < need) {
        if (ctx->tiny_host) CK(cudaFreeHost(ctx->tiny_host));
        ctx->tiny_host = nullptr;
        ctx->tiny_cap = 0;
        CK(cudaHostAlloc(&ctx->tiny_host, need, cudaHostAllocMapped));
        ctx->tiny_cap = need;
    }
    TinyOut *out = reinterpret_cast<TinyOut *>(ctx->tiny_host);
    ipm_trace_rec *tr = reinterpret_cast<ipm_trace_rec *>(out + 1);
    TinyArgs a{};
    a.n = P.n; a.m = P.m; a.H = P.H; a.ldh = P.ldh; a.Arp = P.Arp; a.Acol = P.Acol; a.Aval = P.Aval;
    a.g = P.g; a.l = P.l; a.u = P.u; a.xl = P.xl; a.xu = P.xu;
    a.x = V.x; a.s_lA = V.s_lA; a.s_uA = V.s_uA; a.lam_lA = V.lam_lA; a.lam_uA = V.lam_uA;
    a.s_lx = V.s_lx; a.s_ux = V.s_ux; a.lam_lx = V.lam_lx; a.lam_ux = V.lam_ux; a.dx = V.dx; a.Hx = V.Hx; a.Ax = V.Ax;
    a.mu0 = ctx->mu; a.mu_tol = o.mu_tol; a.mu_div = o.mu_divisor; a.tau = o.tau;
    a.rtol_floor = o.pcg_rtol_floor; a.rtol_max = o.pcg_rtol_max; a.rtol_fac = o.pcg_rtol_mu_factor; a.atol = o.pcg_atol;
    a.schedule = o.pcg_schedule; a.max_ipm = o.max_ipm_iter; a.trace = o.trace ? 1 : 0; a.pcg_maxit = o.pcg_max_iter;
    a.trace_buf = tr;
    a.out = out;
    a.sc = ctx->sc;
    out->status = -1;
    launch_ipm_tiny(a, ctx->st);
    ctx->launches += 1;
    CKL();
    TRY(sync_scalars(ctx));
    CK(cudaEventRecord(ctx->ev[1], ctx->st));
    CK(cudaEventSynchronize(ctx->ev[1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
    ctx->have_dx = true;
    ctx->mu = out->mu;
    S.ipm_iters = out->ipm_iters;
    S.pcg_iters_total = out->pcg_total;
    S.pcg_iters_max = out->pcg_max;
    S.pcg_stalls = out->stalls;
    S.pcg_restarts = out->restarts;
    S.mu_final = out->mu;
    S.kkt_inf = kkt_inf(*ctx->hsc);
    S.obj = ctx->hsc->obj;
    S.t_solve_ms = ms;
    S.t_pcg_ms = (float)(out->t_pcg_ns * 1e-6);
    if (o.trace)
        for (int i = 0; i < out->ntrace; ++i) ctx->trace.push_back(tr[i]);
    const ipm_status st = (ipm_status)out->status;
    S.status = st;
    if (st == IPM_ERR_PCG_BREAKDOWN)
        return fail(ctx, st, "PCG breakdown at IPM iteration %d (one-warp path)", out->ipm_iters);
    if (st == IPM_ERR_NONFINITE)
        return fail(ctx, st, "non-finite residual or step at IPM iteration %d (one-warp path)", out->ipm_iters);
    return st;
}

ipm_status solve_impl(ipm_ctx *ctx) {
    const ipm_options &o = ctx->opt;
    ctx->trace.clear();
    ipm_stats &S = ctx->stats;
    S = ipm_stats{};
    DSYNC("solve entry");
    CK(cudaMemsetAsync(&ctx->sc->nonfinite, 0, sizeof(int64_t), ctx->st));
    DSYNC("memset");
    CK(cudaEventRecord(ctx->ev[0], ctx->st));
    DSYNC("event");
    TRY(start_point(ctx));
    ctx->have_iterate = true;
    if (tiny_path(ctx)) return solve_tiny(ctx);
    TRY(residuals(ctx, ctx->mu));
    TRY(sync_scalars(ctx));
    // a starting iterate with Inf/NaN entries (ipm_set_iterate) cannot produce a direction
    if (ctx->hsc->nonfinite) return fail(ctx, IPM_ERR_NONFINITE, "non-finite residual at the starting iterate");
    double mu = ctx->mu;
    float tpcg = 0.f;
    ipm_status status = IPM_NOT_CONVERGED;
    const bool pc = o.predictor_corrector && ctx->nbounds > 0;
    int k = 0;
    // a deferred (one-warp) PCG solve is read back at the next sync point
    auto collect = [&](PcgOut &po) -> ipm_status {
        if (!po.deferred) return IPM_OK;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
        tpcg += ms;
        return pcg_collect(ctx, po);
    };
    DBG("solve start: n=%d m=%d mu0=%.3e kkt=%.3e\n", ctx->P.n, ctx->P.m, mu, kkt_inf(*ctx->hsc));
    for (k = 1; k <= o.max_ipm_iter; ++k) {
        launch_sigma(ctx->P, ctx->V, ctx->G, ctx->st);
        ctx->launches += 1 + (ctx->P.m > 0 ? 1 : 0);
        PcgOut po, po2;
        if (!pc) {
            TRY(direction(ctx, mu, 0, 0.0, o.tau, 0, po, tpcg));
        } else {
            // Mehrotra (R18): affine direction, sigma = (mu_aff/mu_cur)^3, corrector
            launch_sum_ls(ctx->P, ctx->V, ctx->sc, ctx->st);
            TRY(xcombine(ctx, X_SUMLS));
            TRY(direction(ctx, mu, 1, 0.0, 1.0, 1, po, tpcg));
            launch_muaff(ctx->P, ctx->V, ctx->sc, ctx->st);
            TRY(xcombine(ctx, X_MUAFF));
            ctx->launches += 2 * (1 + (ctx->P.m > 0 ? 1 : 0));
            TRY(sync_scalars(ctx));
            TRY(collect(po));
            const double nb = (double)ctx->nbounds;
            const double mu_cur = ctx->hsc->sum_ls / nb;
            const double mu_aff = ctx->hsc->muaff / nb;
            const double r = mu_aff / mu_cur;
            const double smu = r * r * r * mu_cur;
            TRY(direction(ctx, mu, 2, smu, o.tau, 0, po2, tpcg));
        }
        launch_update(ctx->P, ctx->V, ctx->sc, ctx->st);
        ctx->launches += 1 + (ctx->P.m > 0 ? 1 : 0);
        if (pc) {
            launch_sum_ls(ctx->P, ctx->V, ctx->sc, ctx->st);
            ctx->launches += 1 + (ctx->P.m > 0 ? 1 : 0);
            TRY(xcombine(ctx, X_SUMLS));
        }
        TRY(residuals(ctx, pc ? 0.0 : mu));
        TRY(sync_scalars(ctx));
        TRY(collect(po));
        TRY(collect(po2));
        const Scalars &h = *ctx->hsc;
        const int64_t its = po.iters + po2.iters;
        S.pcg_iters_total += its;
        S.pcg_iters_max = std::max<int32_t>(S.pcg_iters_max, (int32_t)std::max(po.iters, po2.iters));
        S.pcg_stalls += (po.stalled ? 1 : 0) + (po2.stalled ? 1 : 0);
        S.pcg_restarts += po.restarts + po2.restarts;
        DBG("ipm it %d: mu=%.3e kkt=%.3e (rH %.2e prim %.2e comp %.2e) ax=%.3f al=%.3f pcg=%lld obj=%.10e\n", k, mu,
            kkt_inf(h), h.rH_max, h.prim_max, h.comp_max, h.alpha_x, h.alpha_l, (long long)its, h.obj);
        if (h.nonfinite) {
            status = fail(ctx, IPM_ERR_NONFINITE, "non-finite residual or step at IPM iteration %d", k);
            break;
        }
        double nrm;
        if (pc) {
            mu = h.sum_ls / (double)ctx->nbounds;
            nrm = std::max(h.rH_max, std::max(h.prim_max, h.ls_max));
        } else {
            nrm = kkt_inf(h);
        }
        if (o.trace) {
            ipm_trace_rec r{};
            r.it = k;
            r.pcg_iters = (int32_t)its;
            r.mu = mu;
            r.kkt_inf = nrm;
            r.alpha_x = h.alpha_x;
            r.alpha_lam = h.alpha_l;
            r.pcg_relres = std::max(po.relres, po2.relres);
            r.obj = h.obj;
            ctx->trace.push_back(r);
        }
        if (pc) {
            if (nrm < o.mu_tol) {
                status = IPM_OK;
                break;
            }
            continue;
        }
        if (nrm < mu) {                                  // Alg. 1 lines 10-15
            if (mu <= o.mu_tol) {
                status = IPM_OK;
                break;
            }
            mu = mu / o.mu_divisor;
        }
    }
    ctx->mu = mu;
    // final residuals at the final mu (r_c with the current mu) for reporting; x is unchanged
    // since the last residuals (same H x, A x)
    TRY(residuals(ctx, mu, true));
    TRY(sync_scalars(ctx));
    CK(cudaEventRecord(ctx->ev[1], ctx->st));
    CK(cudaEventSynchronize(ctx->ev[1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]));
    S.status = status;
    S.ipm_iters = std::min(k, o.max_ipm_iter);
    S.mu_final = mu;
    S.kkt_inf = kkt_inf(*ctx->hsc);
    S.obj = ctx->hsc->obj;
    S.t_solve_ms = ms;
    S.t_pcg_ms = tpcg;
    return status;
}

ipm_status validate_host(ipm_ctx *ctx, const ipm_problem *p, std::vector<int64_t> &rp, std::vector<int> &col) {
    const int64_t n = p->n, m = p->m, nnz = p->nnz;
    if (rp.size() != (size_t)(m + 1)) return fail(ctx, IPM_ERR_INVALID, "rowptr size");
    if (rp[0] != 0 || rp[m] != nnz) return fail(ctx, IPM_ERR_INVALID, "A_rowptr[0] must be 0 and A_rowptr[m] == nnz");
    for (int64_t i = 0; i < m; ++i) {
        if (rp[i + 1] < rp[i]) return fail(ctx, IPM_ERR_INVALID, "A_rowptr decreasing at row %lld", (long long)i);
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            if (col[k] < 0 || col[k] >= n)
                return fail(ctx, IPM_ERR_INVALID, "A_col out of range in row %lld", (long long)i);
            if (k > rp[i] && col[k] <= col[k - 1])
                return fail(ctx, IPM_ERR_INVALID, "A_col not strictly increasing (unsorted or duplicate) in row %lld",
                            (long long)i);
        }
    }
    return IPM_OK;
}

ipm_status check_bounds(ipm_ctx *ctx, const std::vector<double> &lo, const std::vector<double> &hi, const char *what) {
    for (size_t i = 0; i < lo.size(); ++i) {
        if (std::isnan(lo[i]) || std::isnan(hi[i])) return fail(ctx, IPM_ERR_INVALID, "%s bound %zu is NaN", what, i);
        if (lo[i] == INFINITY || hi[i] == -INFINITY)
            return fail(ctx, IPM_ERR_INVALID, "%s bound %zu: lower=+inf or upper=-inf", what, i);
        if (std::isfinite(lo[i]) && std::isfinite(hi[i]) && !(lo[i] < hi[i]))
            return fail(ctx, IPM_ERR_INVALID, "%s bounds %zu: need lower < upper (equal bounds are rejected, R10)",
                        what, i);
    }
    return IPM_OK;
}

}  // namespace

// ================================================================================= C ABI
IPM_EXPORT int32_t ipm_abi_version(void) { return IPM_ABI_VERSION; }

IPM_EXPORT void ipm_options_default(ipm_options *o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->size = (int32_t)sizeof(ipm_options);
    o->mu_tol = 1e-8;
    o->mu0_scale = 0.1;
    o->mu_divisor = 10.0;
    o->tau = 0.995;
    o->max_ipm_iter = 100;
    o->pcg_schedule = 0;
    o->pcg_rtol_max = 1e-6;
    o->pcg_rtol_mu_factor = 1e-3;
    o->pcg_rtol_floor = 1e-12;
    o->pcg_atol = 1e-13;
    o->pcg_max_iter = 0;
    o->predictor_corrector = 0;
    o->trace = 0;
    o->use_graph = 1;
    o->warm_shift = 0.1;
    o->a_row_split = 1;
}

static void local_rows(const ipm_problem *p, int64_t &row0, int64_t &nloc) {
    if (p->comm_kind != 0) {
        row0 = p->row_begin;
        nloc = p->row_end - p->row_begin;
    } else {
        row0 = 0;
        nloc = p->n;
    }
}

static int eff_ranks(const ipm_problem *p) { return p->comm_kind != 0 ? std::max(1, p->nranks) : 1; }

// Rows of rank r under the equal-chunk partition (header: chunk = ceil(n / nranks)).
static ipm_status check_partition(const ipm_problem *p) {
    if (p->comm_kind == 0) {
        if (p->nranks > 1)
            return fail(nullptr, IPM_ERR_INVALID, "nranks > 1 needs comm_kind 1 (NCCL), 2 (local group) or 3 (host)");
        return IPM_OK;
    }
    if (p->comm_kind < 1 || p->comm_kind > 3) return fail(nullptr, IPM_ERR_INVALID, "unknown comm_kind");
    if (!p->comm_handle_host) return fail(nullptr, IPM_ERR_INVALID, "comm_handle_host is null");
    const int64_t P = std::max(1, p->nranks);
    if (p->rank < 0 || p->rank >= P) return fail(nullptr, IPM_ERR_INVALID, "rank out of range");
    const int64_t chunk = (p->n + P - 1) / P;
    const int64_t b = std::min<int64_t>(p->n, p->rank * chunk), e = std::min<int64_t>(p->n, (p->rank + 1) * chunk);
    if (p->row_begin != b || p->row_end != e || b >= e)
        return fail(nullptr, IPM_ERR_INVALID,
                    "row block [%lld,%lld) of rank %d must be [%lld,%lld) (chunk = ceil(n/nranks)) and non-empty",
                    (long long)p->row_begin, (long long)p->row_end, p->rank, (long long)b, (long long)e);
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_workspace_size(const ipm_problem *p, const ipm_options *opt, size_t *bytes) {
    (void)opt;
    if (!p || !bytes) return fail(nullptr, IPM_ERR_INVALID, "null argument");
    if (p->n < 1 || p->m < 0 || p->nnz < 0) return fail(nullptr, IPM_ERR_INVALID, "bad dimensions");
    int64_t row0, nloc;
    local_rows(p, row0, nloc);
    if (nloc < 1) return fail(nullptr, IPM_ERR_INVALID, "empty row block");
    Layout L;
    if (p->hess_kind == 1 && (p->ldu < 1 || p->k < 0 || p->k > p->ldu))
        return fail(nullptr, IPM_ERR_INVALID, "compact Hessian needs 0 <= k <= ldu and ldu >= 1");
    // k_compact_us stages w o s (k doubles, k <= ldu) in its 48 KB default dynamic shared memory
    if (p->hess_kind == 1 && p->ldu > kCompactMaxCols)
        return fail(nullptr, IPM_ERR_INVALID, "compact Hessian: ldu = %lld exceeds %d columns", (long long)p->ldu,
                    kCompactMaxCols);
    plan(nloc, p->n, p->m, p->nnz, eff_ranks(p), L, p->hess_kind == 1 ? p->ldu : 0, p->rank);   // local A^T nnz <= nnz
    *bytes = L.total;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_nccl_unique_id(void *out, size_t bytes) {
    if (!out) return fail(nullptr, IPM_ERR_INVALID, "null argument");
    std::string e;
    if (ipm::nccl_unique_id(out, bytes, e)) return fail(nullptr, IPM_ERR_NCCL, "%s", e.c_str());
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_group_create(int32_t nranks, ipm_group **g) {
    if (!g || nranks < 1) return fail(nullptr, IPM_ERR_INVALID, "bad argument");
    *g = new ipm_group(nranks);
    return IPM_OK;
}

IPM_EXPORT void ipm_group_destroy(ipm_group *g) {
    if (!g) return;
    for (auto e : g->ready)
        if (e) cudaEventDestroy(e);
    for (auto e : g->copied)
        if (e) cudaEventDestroy(e);
    delete g;
}

static ipm_status create_impl(ipm_ctx *ctx, const ipm_problem *p, void *workspace, ipm_stream_t stream) {
    // load every kernel now: CUDA's lazy loading must never run while a peer-exchange wait
    // kernel of another rank sharing this device spins (it would wait for that kernel)
    preload_all_kernels();
    cudaGetLastError();
    ctx->st = reinterpret_cast<cudaStream_t>(stream);
    ctx->n = p->n;
    ctx->m = p->m;
    ctx->nnz = p->nnz;
    int64_t row0, nloc;
    local_rows(p, row0, nloc);
    ctx->row0 = (int)row0;
    ctx->nloc = (int)nloc;
    ctx->rank = p->rank;
    ctx->nranks = std::max(1, p->nranks);
    ctx->ws = reinterpret_cast<char *>(workspace);
    ipm_status s = IPM_OK;
        CK(cudaGetDevice(&ctx->device));
        CK(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->fork.side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->fork.ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->fork.ev_join, cudaEventDisableTiming));
        CK(cudaMallocHost(&ctx->hsc, sizeof(Scalars)));
        for (auto &e : ctx->ev) CK(cudaEventCreate(&e));
        // --- host validation of the O(n + m + nnz) data --------------------------------
        std::vector<int64_t> rp(p->m + 1, 0);
        std::vector<int> col(p->nnz);
        std::vector<double> val(p->nnz), l(p->m), u(p->m), xl(p->n), xu(p->n), g(p->n);
        if (p->m > 0) CK(cudaMemcpy(rp.data(), p->A_rowptr, sizeof(int64_t) * (p->m + 1), cudaMemcpyDeviceToHost));
        if (p->nnz > 0) {
            CK(cudaMemcpy(col.data(), p->A_col, sizeof(int) * p->nnz, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(val.data(), p->A_val, sizeof(double) * p->nnz, cudaMemcpyDeviceToHost));
        }
        if (p->m > 0) {
            CK(cudaMemcpy(l.data(), p->l, sizeof(double) * p->m, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(u.data(), p->u, sizeof(double) * p->m, cudaMemcpyDeviceToHost));
        }
        CK(cudaMemcpy(xl.data(), p->xl, sizeof(double) * p->n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(xu.data(), p->xu, sizeof(double) * p->n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(g.data(), p->g, sizeof(double) * p->n, cudaMemcpyDeviceToHost));
        if ((s = validate_host(ctx, p, rp, col)) != IPM_OK) return s;
        for (double v : val)
            if (!std::isfinite(v)) { s = fail(ctx, IPM_ERR_INVALID, "A_val has a non-finite entry"); return s; }
        for (double v : g)
            if (!std::isfinite(v)) { s = fail(ctx, IPM_ERR_INVALID, "g has a non-finite entry"); return s; }
        if ((s = check_bounds(ctx, l, u, "row")) != IPM_OK) return s;
        if ((s = check_bounds(ctx, xl, xu, "variable")) != IPM_OK) return s;
        int64_t nb = 0;
        for (int64_t i = 0; i < p->m; ++i) nb += std::isfinite(l[i]) + std::isfinite(u[i]);
        for (int64_t j = 0; j < p->n; ++j) nb += std::isfinite(xl[j]) + std::isfinite(xu[j]);
        ctx->nbounds = nb;

        // --- device state ------------------------------------------------------------
        Layout L;
        SymPlan symp;
        const Offsets o = plan(nloc, p->n, p->m, p->nnz, eff_ranks(p), L, p->hess_kind == 1 ? p->ldu : 0,
                               eff_ranks(p) > 1 ? p->rank : 0, &symp);
        CK(cudaMemsetAsync(ctx->ws, 0, L.total, ctx->st));
        ctx->sc = reinterpret_cast<Scalars *>(ctx->ws + o.sc);
        assign_vectors(ctx, o);
        if (p->comm_kind != 0) {
            std::string e;
            ctx->comm = (p->comm_kind == 1)   ? ipm::make_nccl_comm(p->comm_handle_host, p->rank,
                                                                        std::max(1, p->nranks), e)
                        : (p->comm_kind == 3) ? ipm::make_host_comm(p->comm_handle_host, e)
                                              : ipm::make_local_comm(const_cast<ipm_group *>(
                                                                         static_cast<const ipm_group *>(
                                                                             p->comm_handle_host)),
                                                                     p->rank, e);
            if (!ctx->comm) return fail(ctx, IPM_ERR_NCCL, "communicator: %s", e.c_str());
            if (ctx->comm->nranks != std::max(1, p->nranks))
                return fail(ctx, IPM_ERR_INVALID, "group size %d != nranks %d", ctx->comm->nranks, p->nranks);
            ctx->sharded = true;
            ctx->chunk = (p->n + ctx->comm->nranks - 1) / ctx->comm->nranks;
            const int64_t one = 1;
            CK(cudaMemcpyAsync(&ctx->sc->sharded, &one, sizeof one, cudaMemcpyHostToDevice, ctx->st));
            if ((s = setup_peer(ctx, ctx->ws + o.peer, ctx->ws + o.part)) != IPM_OK) return s;
            ctx->cg = ctx->opt.pcg_single_reduction != 0 && ctx->opt.pcg_system == 0;
            if (p->comm_kind == 3 && !ctx->peer_on && ctx->comm->nranks > 1)
                return fail(ctx, IPM_ERR_INVALID, "comm_kind 3 needs the peer data plane (2 <= nranks <= %d, "
                            "IPM_PEER not 0)", kPeerMax);
        }
        Prob &P = ctx->P;
        P.n = (int)nloc;
        P.m = (int)p->m;
        P.ncols = (int)p->n;
        P.nnz = p->nnz;
        P.ldh = p->ldh;
        P.H = const_cast<double *>(p->H);
        P.Arp = p->A_rowptr;
        P.Acol = p->A_col;
        P.Aval = p->A_val;
        double *gd = reinterpret_cast<double *>(ctx->ws + o.g);
        double *ld = reinterpret_cast<double *>(ctx->ws + o.l);
        double *ud = reinterpret_cast<double *>(ctx->ws + o.u);
        double *xld = reinterpret_cast<double *>(ctx->ws + o.xl);
        double *xud = reinterpret_cast<double *>(ctx->ws + o.xu);
        CK(cudaMemcpyAsync(gd, p->g + row0, sizeof(double) * nloc, cudaMemcpyDeviceToDevice, ctx->st));
        CK(cudaMemcpyAsync(xld, p->xl + row0, sizeof(double) * nloc, cudaMemcpyDeviceToDevice, ctx->st));
        CK(cudaMemcpyAsync(xud, p->xu + row0, sizeof(double) * nloc, cudaMemcpyDeviceToDevice, ctx->st));
        if (p->m > 0) {
            CK(cudaMemcpyAsync(ld, p->l, sizeof(double) * p->m, cudaMemcpyDeviceToDevice, ctx->st));
            CK(cudaMemcpyAsync(ud, p->u, sizeof(double) * p->m, cudaMemcpyDeviceToDevice, ctx->st));
        }
        P.g = gd;
        P.l = ld;
        P.u = ud;
        P.xl = xld;
        P.xu = xud;
        P.diagH = reinterpret_cast<double *>(ctx->ws + o.diagH);
        P.Kd = reinterpret_cast<double *>(ctx->ws + o.kd);
        int64_t *ATrp = reinterpret_cast<int64_t *>(ctx->ws + o.ATrp);
        int *ATcol = reinterpret_cast<int *>(ctx->ws + o.ATcol);
        double *ATval = reinterpret_cast<double *>(ctx->ws + o.ATval);
        P.ATrp = ATrp;
        P.ATcol = ATcol;
        P.ATval = ATval;
        launch_transpose(P, (int)row0, o.nchunk, reinterpret_cast<int *>(ctx->ws + o.cnt), ATrp, ATcol, ATval, ctx->st);
        unsigned long long *bad = reinterpret_cast<unsigned long long *>(ctx->ws + o.bad);
        if (p->hess_kind == 1) {
            // compact quasi-Newton Hessian (NEXT-1): h0 and w copied, U borrowed, diag cached
            P.hess_compact = 1;
            P.ck = p->k;
            P.ldu = p->ldu;
            P.U = p->U;
            P.h0 = reinterpret_cast<double *>(ctx->ws + o.ch0);
            P.w = reinterpret_cast<double *>(ctx->ws + o.cw);
            P.cs = reinterpret_cast<double *>(ctx->ws + o.cs);
            P.cspart = reinterpret_cast<double *>(ctx->ws + o.cspart);
            P.chpart = reinterpret_cast<double *>(ctx->ws + o.chpart);
            CK(cudaMemcpyAsync(P.h0, p->h0, sizeof(double) * nloc, cudaMemcpyDeviceToDevice, ctx->st));
            if (p->k > 0) CK(cudaMemcpyAsync(P.w, p->w, sizeof(double) * p->k, cudaMemcpyDeviceToDevice, ctx->st));
            launch_compact_diag(P, ctx->st);
            if (p->k > 0) {
                Prob Q = P;                     // non-finite scan over the n x k block of U
                Q.H = p->U;
                Q.ldh = p->ldu;
                Q.ncols = p->k;
                launch_count_nonfinite(Q, bad, ctx->st);
            }
        } else {
            launch_setup_diag(P, (int)row0, ctx->st);
            launch_count_nonfinite(P, bad, ctx->st);
        }
        ctx->launches += 5;
        CKL();
        unsigned long long nbad = 0;
        CK(cudaMemcpyAsync(&nbad, bad, sizeof nbad, cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        if (nbad) { s = fail(ctx, IPM_ERR_INVALID, "H has %llu non-finite entries", nbad); return s; }
        ctx->gemv_grid = gemv_max_grid();
        const int gk = ctx->opt.gemv_kernel;
        const bool bulk_ok = gemv_bulk_ok(P);
        bool sym = false;
        P.row_begin = ctx->row0;
        const bool sym_try = (gk == 0 || gk == 3) && !P.hess_compact && (!ctx->sharded || (ctx->chunk % 2) == 0);
        if (sym_try) {
            // the symmetric GEMV reads only an upper block triangle: require H == H^T bitwise.
            // Unsharded: every entry pair compared.  Sharded: the rank's diagonal block compared
            // entry by entry, the off-diagonal blocks certified by exchanged order-independent
            // hashes (k_sym_hash) — every rank takes the same decision from the same data.
            unsigned long long nasym = bulk_ok ? 0ull : 1ull;
            if (bulk_ok) {
                Prob Q = P;
                Q.H = P.H + (ctx->sharded ? ctx->row0 : 0);      // the local diagonal block
                CK(cudaMemsetAsync(bad, 0, sizeof nasym, ctx->st));
                launch_count_asym(Q, bad, ctx->st);
                CKL();
                CK(cudaMemcpyAsync(&nasym, bad, sizeof nasym, cudaMemcpyDeviceToHost, ctx->st));
                CK(cudaStreamSynchronize(ctx->st));
                ctx->launches += 1;
            }
            sym = (nasym == 0);
            if (ctx->sharded) {
                const int R = ctx->comm->nranks;
                unsigned long long *hs = reinterpret_cast<unsigned long long *>(ctx->ws + o.hashes);
                CK(cudaMemsetAsync(hs, 0, sizeof(unsigned long long) * (R + 1), ctx->st));
                if (bulk_ok) launch_sym_hash(P.n, P.ncols, ctx->row0, (int)ctx->chunk, R, P.H, P.ldh, hs, ctx->st);
                CK(cudaMemcpyAsync(hs + R, &nasym, sizeof nasym, cudaMemcpyHostToDevice, ctx->st));
                std::string e;
                if (ctx->comm->allgather(hs, hs + (R + 1), sizeof(unsigned long long) * (R + 1), ctx->st, e))
                    return fail(ctx, IPM_ERR_NCCL, "%s", e.c_str());
                std::vector<unsigned long long> all((size_t)R * (R + 1));
                CK(cudaMemcpyAsync(all.data(), hs + (R + 1), sizeof(unsigned long long) * all.size(),
                                   cudaMemcpyDeviceToHost, ctx->st));
                CK(cudaStreamSynchronize(ctx->st));
                ctx->launches += 1;
                sym = true;
                for (int a = 0; a < R; ++a) {
                    if (all[(size_t)a * (R + 1) + R] != 0) sym = false;
                    for (int b = 0; b < R; ++b)
                        if (a != b && all[(size_t)a * (R + 1) + b] != all[(size_t)b * (R + 1) + a]) sym = false;
                }
            }
            if (sym) {
                sym = make_sym_tensor_map(P, ctx->tmap_sym);
                P.tmap_sym = ctx->tmap_sym;
            }
        }
        if (gk == 3 && !sym)
            return fail(ctx, IPM_ERR_INVALID,
                        "gemv_kernel=3 needs an exactly symmetric H, even ldh, 16-byte aligned rows (sharded: even chunk)");
        if (gk == 2 && !bulk_ok) return fail(ctx, IPM_ERR_INVALID, "gemv_kernel=2 needs even ldh and 16-byte aligned H");
        P.gemv_sym = sym ? 1 : 0;
        P.sym_keep = 0;
        if (sym) {
            // an upper block triangle of <= 100 MiB is loaded with an evict_last policy so it stays
            // resident across PCG iterations; larger H streams evict_first (measured: no gain from a
            // resident share at C3; C2's 105 MB forced resident: SYMV -2 % but QP +3 %)
            const double tri = 4.0 * (double)p->n * (double)(p->n + kSymB);
            const char *e = getenv("IPM_SYM_KEEP_MB");      // experiment override
            const double mb = e ? atof(e) : (tri <= 100.0 * 1048576.0 ? 1e9 : 0.0);
            const double tiles = mb * 1048576.0 / (8.0 * kSymB * kSymB);
            P.sym_keep = (int)std::min(1e9, tiles / std::max(1, gemv_bulk_grid())) + (mb > 0 ? 1 : 0);
        }
        P.gemv_bulk = (!sym && !P.hess_compact && (gk == 0 || gk == 2) && bulk_ok) ? 1 : 0;
        P.gemv_bulk_grid = gemv_bulk_grid();
        if (sym) {                  // the SYMV work plan (tiles, strip-balanced ranges; kernels.h)
            SymTile *dt = reinterpret_cast<SymTile *>(ctx->ws + o.symt);
            SymRange *dr = reinterpret_cast<SymRange *>(ctx->ws + o.symr);
            int *dz = reinterpret_cast<int *>(ctx->ws + o.zcol);
            CK(cudaMemcpyAsync(dt, symp.tiles.data(), sizeof(SymTile) * symp.tiles.size(), cudaMemcpyHostToDevice,
                               ctx->st));
            CK(cudaMemcpyAsync(dr, symp.ranges.data(), sizeof(SymRange) * symp.ranges.size(),
                               cudaMemcpyHostToDevice, ctx->st));
            if (!symp.zcol.empty())
                CK(cudaMemcpyAsync(dz, symp.zcol.data(), sizeof(int) * symp.zcol.size(), cudaMemcpyHostToDevice,
                                   ctx->st));
            CK(cudaStreamSynchronize(ctx->st));
            P.sym_tiles = dt;
            P.sym_ranges = dr;
            P.sym_z = reinterpret_cast<double *>(ctx->ws + o.symz);
            P.sym_ntma = symp.ntma;
            P.sym_ntiles = (int)symp.tiles.size();
            P.sym_ycarry = symp.nbg;
            P.sym_ldz = symp.ldz;
            P.sym_zcarry = symp.ldz - symp.zcarry_n;
            ctx->sym_zrows = symp.zrows;
            ctx->sym_zcol = dz;
            ctx->sym_zvec = reinterpret_cast<double *>(ctx->ws + o.zvec);
            ctx->sym_zall = reinterpret_cast<double *>(ctx->ws + o.zall);
            ctx->sym_sharded = ctx->sharded;
        }
        ctx->ncb = P.hess_compact ? 1 : (sym ? symp.ldy : gemv_ncb((int)p->n));
        P.ncb = ctx->ncb;
        if (ctx->opt.pcg_system != 0 && ctx->opt.pcg_system != 1) return fail(ctx, IPM_ERR_INVALID, "unknown pcg_system");
        if (ctx->opt.pcg_system == 1 && ctx->sharded)
            return fail(ctx, IPM_ERR_INVALID, "pcg_system = 1 (doubly augmented) is unsharded only");
        P.aug = (ctx->opt.pcg_system == 1 && p->m > 0) ? 1 : 0;
        P.ktimer = ctx->opt.kernel_timer ? 1 : 0;
        ctx->G = choose_group(p->nnz, nloc, ctx->ncb);
        {   // function attributes are per device: set them for this context's device on every create
            CK(configure_linalg_attrs());
            CK(configure_pcg_attrs());
            CK(configure_tiny_attrs());
            const char *ce = getenv("IPM_CARVEOUT");
            if (!(ce && atoi(ce) == 0)) {
                configure_linalg_carveout();
                configure_pcg_carveout();
            }
        }
        {   // fused update + p (cooperative grid barrier): single-GPU condensed PCG
            int coop = 0;
            CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device));
            const char *e = getenv("IPM_FUSED_P");
            ctx->fused_p = coop && !ctx->sharded && !P.aug && !(e && atoi(e) == 0);
        }
        DBG("create: n=%lld m=%lld nnz=%lld gemv=%s ncb=%d G=%d sharded=%d\n", (long long)p->n, (long long)p->m,
            (long long)p->nnz, sym ? "symmetric-bulk" : (P.gemv_bulk ? "bulk" : "ldg"), ctx->ncb, ctx->G,
            (int)ctx->sharded);
    
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_create(ipm_ctx **out, const ipm_problem *p, const ipm_options *opt, void *workspace,
                                 size_t workspace_bytes, ipm_stream_t stream) {
    ipm_ctx *ctx = nullptr;
    if (!out || !p) return fail(nullptr, IPM_ERR_INVALID, "null argument");
    *out = nullptr;
    if (p->n < 1 || p->m < 0 || p->nnz < 0 || p->ldh < p->n)
        return fail(nullptr, IPM_ERR_INVALID, "bad dimensions (n >= 1, m >= 0, nnz >= 0, ldh >= n)");
    if (p->n > INT32_MAX || p->m > INT32_MAX || p->nnz >= INT32_MAX)
        return fail(nullptr, IPM_ERR_INVALID, "dimension exceeds int32 index range");
    if (check_partition(p) != IPM_OK) return IPM_ERR_INVALID;
    if (p->hess_kind != 0 && p->hess_kind != 1) return fail(nullptr, IPM_ERR_INVALID, "unknown hess_kind");
    if (p->hess_kind == 1 && (p->comm_kind != 0 || !p->h0 || !p->U || (p->k > 0 && !p->w)))
        return fail(nullptr, IPM_ERR_INVALID, "compact Hessian: needs h0, U (and w when k > 0); unsharded only");
    if ((p->hess_kind == 0 && !p->H) || !p->g || !p->xl || !p->xu ||
        (p->m > 0 && (!p->l || !p->u || !p->A_rowptr)) || (p->nnz > 0 && (!p->A_col || !p->A_val)))
        return fail(nullptr, IPM_ERR_INVALID, "null data pointer");
    size_t need = 0;
    if (ipm_workspace_size(p, opt, &need) != IPM_OK) return IPM_ERR_INVALID;
    if (!workspace || workspace_bytes < need)
        return fail(nullptr, IPM_ERR_OOM, "workspace too small: %zu < %zu bytes", workspace_bytes, need);
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return fail(nullptr, IPM_ERR_INVALID, "workspace not 256-byte aligned");

    ctx = new ipm_ctx();
    ipm_options_default(&ctx->opt);
    if (opt) {
        if (opt->size != (int32_t)sizeof(ipm_options)) {
            delete ctx;
            return fail(nullptr, IPM_ERR_INVALID, "ipm_options.size mismatch (ABI)");
        }
        ctx->opt = *opt;
    }
    const ipm_status s = create_impl(ctx, p, workspace, stream);
    if (s != IPM_OK) {
        g_create_error = ctx->err;
        ipm_destroy(ctx);
        return s;
    }
    *out = ctx;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_solve(ipm_ctx *ctx) {
    if (!ctx) return fail(nullptr, IPM_ERR_INVALID, "null context");
    ctx->err.clear();
    const ipm_status s = solve_impl(ctx);
    if (s != IPM_OK && s != IPM_NOT_CONVERGED) ctx->stats.status = s;   // early error exits
    return s;
}

IPM_EXPORT ipm_status ipm_get_solution(ipm_ctx *ctx, double *x, double *lam_lA, double *lam_uA, double *lam_lx,
                                       double *lam_ux, double *obj_host) {
    if (!ctx) return fail(nullptr, IPM_ERR_INVALID, "null context");
    if (!ctx->have_iterate) return fail(ctx, IPM_ERR_STATE, "no iterate: call ipm_solve first");
    const size_t nb = sizeof(double) * ctx->nloc, mb = sizeof(double) * ctx->m;
    if (x) CK(cudaMemcpyAsync(x, ctx->V.x, nb, cudaMemcpyDeviceToDevice, ctx->st));
    if (lam_lx) CK(cudaMemcpyAsync(lam_lx, ctx->V.lam_lx, nb, cudaMemcpyDeviceToDevice, ctx->st));
    if (lam_ux) CK(cudaMemcpyAsync(lam_ux, ctx->V.lam_ux, nb, cudaMemcpyDeviceToDevice, ctx->st));
    if (ctx->m > 0) {
        if (lam_lA) CK(cudaMemcpyAsync(lam_lA, ctx->V.lam_lA, mb, cudaMemcpyDeviceToDevice, ctx->st));
        if (lam_uA) CK(cudaMemcpyAsync(lam_uA, ctx->V.lam_uA, mb, cudaMemcpyDeviceToDevice, ctx->st));
    }
    if (obj_host) *obj_host = ctx->stats.obj;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_get_stats(ipm_ctx *ctx, ipm_stats *s) {
    if (!ctx || !s) return fail(ctx, IPM_ERR_INVALID, "null argument");
    *s = ctx->stats;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_get_trace(ipm_ctx *ctx, ipm_trace_rec *recs, int32_t cap, int32_t *count) {
    if (!ctx || !count) return fail(ctx, IPM_ERR_INVALID, "null argument");
    const int32_t nrec = (int32_t)ctx->trace.size();
    *count = nrec;
    if (recs)
        for (int32_t i = 0; i < std::min(cap, nrec); ++i) recs[i] = ctx->trace[i];
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_set_linear_term(ipm_ctx *ctx, const double *g) {
    if (!ctx || !g) return fail(ctx, IPM_ERR_INVALID, "null argument");
    CK(cudaMemcpyAsync(const_cast<double *>(ctx->P.g), g + ctx->row0, sizeof(double) * ctx->nloc,
                       cudaMemcpyDeviceToDevice, ctx->st));
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_set_bounds(ipm_ctx *ctx, const double *l, const double *u, const double *xl,
                                     const double *xu) {
    if (!ctx || !xl || !xu || (ctx->m > 0 && (!l || !u))) return fail(ctx, IPM_ERR_INVALID, "null argument");
    const int64_t m = ctx->m, n = ctx->n;
    std::vector<double> hl(m), hu(m), hxl(n), hxu(n), ol(m), ou(m), oxl(ctx->nloc), oxu(ctx->nloc);
    CK(cudaStreamSynchronize(ctx->st));
    if (m > 0) {
        CK(cudaMemcpy(hl.data(), l, sizeof(double) * m, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hu.data(), u, sizeof(double) * m, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ol.data(), ctx->P.l, sizeof(double) * m, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ou.data(), ctx->P.u, sizeof(double) * m, cudaMemcpyDeviceToHost));
    }
    CK(cudaMemcpy(hxl.data(), xl, sizeof(double) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hxu.data(), xu, sizeof(double) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(oxl.data(), ctx->P.xl, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(oxu.data(), ctx->P.xu, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToHost));
    TRY(check_bounds(ctx, hl, hu, "row"));
    TRY(check_bounds(ctx, hxl, hxu, "variable"));
    // the finite pattern fixes the bound families (masks, #bounds, mu0): it may not change
    for (int64_t i = 0; i < m; ++i)
        if (std::isfinite(hl[i]) != std::isfinite(ol[i]) || std::isfinite(hu[i]) != std::isfinite(ou[i]))
            return fail(ctx, IPM_ERR_INVALID, "row %lld: which bounds are finite may not change", (long long)i);
    for (int64_t j = 0; j < ctx->nloc; ++j)
        if (std::isfinite(hxl[ctx->row0 + j]) != std::isfinite(oxl[j]) ||
            std::isfinite(hxu[ctx->row0 + j]) != std::isfinite(oxu[j]))
            return fail(ctx, IPM_ERR_INVALID, "variable %lld: which bounds are finite may not change",
                        (long long)(ctx->row0 + j));
    if (m > 0) {
        CK(cudaMemcpyAsync(const_cast<double *>(ctx->P.l), l, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->st));
        CK(cudaMemcpyAsync(const_cast<double *>(ctx->P.u), u, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->st));
    }
    CK(cudaMemcpyAsync(const_cast<double *>(ctx->P.xl), xl + ctx->row0, sizeof(double) * ctx->nloc,
                       cudaMemcpyDeviceToDevice, ctx->st));
    CK(cudaMemcpyAsync(const_cast<double *>(ctx->P.xu), xu + ctx->row0, sizeof(double) * ctx->nloc,
                       cudaMemcpyDeviceToDevice, ctx->st));
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_update_hessian_rank2(ipm_ctx *ctx, const double *u, double alpha, const double *v,
                                               double beta) {
    if (!ctx || !u || !v) return fail(ctx, IPM_ERR_INVALID, "null argument");
    Prob &P = ctx->P;
    if (P.hess_compact) {
        // compact form: append (u, v) as columns k, k+1 with weights (alpha, beta)
        if (P.ck + 2 > P.ldu)
            return fail(ctx, IPM_ERR_STATE, "compact Hessian full: k + 2 > ldu (%d + 2 > %lld)", P.ck,
                        (long long)P.ldu);
        launch_compact_append(P, P.U, P.ck, u, v, ctx->st);
        const double wv[2] = {alpha, beta};
        CK(cudaMemcpyAsync(P.w + P.ck, wv, sizeof wv, cudaMemcpyHostToDevice, ctx->st));
        P.ck += 2;
        launch_compact_diag(P, ctx->st);
        CK(cudaStreamSynchronize(ctx->st));   // wv is a host stack buffer
        ctx->launches += 2;
        ctx->graph_ready = false;              // the captured PCG body holds the old k
        if (ctx->gexec) {
            cudaGraphExecDestroy(ctx->gexec);
            ctx->gexec = nullptr;
        }
        if (ctx->graph) {
            cudaGraphDestroy(ctx->graph);
            ctx->graph = nullptr;
        }
        CKL();
        return IPM_OK;
    }
    launch_rank2(P, ctx->row0, u, alpha, v, beta, ctx->st);
    ctx->launches += 1;
    CKL();
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_warm_start(ipm_ctx *ctx) {
    if (!ctx) return fail(nullptr, IPM_ERR_INVALID, "null context");
    if (!ctx->have_iterate) return fail(ctx, IPM_ERR_STATE, "warm start needs a previous solve");
    ctx->warm_pending = true;
    ctx->user_iterate = false;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_set_iterate(ipm_ctx *ctx, const double *x, const double *const s4[4],
                                      const double *const lam4[4], double mu) {
    if (!ctx || !x || !s4 || !lam4) return fail(ctx, IPM_ERR_INVALID, "null argument");
    const Vecs &V = ctx->V;
    double *sd[4] = {V.s_lA, V.s_uA, V.s_lx, V.s_ux};
    double *ld[4] = {V.lam_lA, V.lam_uA, V.lam_lx, V.lam_ux};
    for (int f = 0; f < 4; ++f) {
        const size_t b = sizeof(double) * (f < 2 ? (size_t)ctx->m : (size_t)ctx->nloc);
        if (b == 0) continue;
        const size_t off = (f < 2) ? 0 : (size_t)ctx->row0;
        CK(cudaMemcpyAsync(sd[f], s4[f] + off, b, cudaMemcpyDeviceToDevice, ctx->st));
        CK(cudaMemcpyAsync(ld[f], lam4[f] + off, b, cudaMemcpyDeviceToDevice, ctx->st));
    }
    CK(cudaMemcpyAsync(V.x, x + ctx->row0, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToDevice, ctx->st));
    ctx->mu = mu;
    ctx->user_iterate = true;
    ctx->warm_pending = false;
    ctx->have_iterate = true;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_get_iterate(ipm_ctx *ctx, double *x, double *const s4[4], double *const lam4[4],
                                      double *mu_host) {
    if (!ctx) return fail(nullptr, IPM_ERR_INVALID, "null context");
    if (!ctx->have_iterate) return fail(ctx, IPM_ERR_STATE, "no iterate");
    const Vecs &V = ctx->V;
    const double *sd[4] = {V.s_lA, V.s_uA, V.s_lx, V.s_ux};
    const double *ld[4] = {V.lam_lA, V.lam_uA, V.lam_lx, V.lam_ux};
    for (int f = 0; f < 4; ++f) {
        const size_t b = sizeof(double) * (f < 2 ? (size_t)ctx->m : (size_t)ctx->nloc);
        if (b == 0) continue;
        if (s4 && s4[f]) CK(cudaMemcpyAsync(s4[f], sd[f], b, cudaMemcpyDeviceToDevice, ctx->st));
        if (lam4 && lam4[f]) CK(cudaMemcpyAsync(lam4[f], ld[f], b, cudaMemcpyDeviceToDevice, ctx->st));
    }
    if (x) CK(cudaMemcpyAsync(x, V.x, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToDevice, ctx->st));
    if (mu_host) *mu_host = ctx->mu;
    CK(cudaStreamSynchronize(ctx->st));
    return IPM_OK;
}

static ipm_status load_sigmas(ipm_ctx *ctx, const double *sig_b, const double *sig_c) {
    CK(cudaMemcpyAsync(ctx->V.sig_b, sig_b, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToDevice, ctx->st));
    if (ctx->m > 0) CK(cudaMemcpyAsync(ctx->V.sig_c, sig_c, sizeof(double) * ctx->m, cudaMemcpyDeviceToDevice, ctx->st));
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_op_apply(ipm_ctx *ctx, const double *sig_b, const double *sig_c, const double *v, double *y) {
    if (!ctx || !sig_b || !v || !y || (ctx->m > 0 && !sig_c)) return fail(ctx, IPM_ERR_INVALID, "null argument");
    TRY(load_sigmas(ctx, sig_b, sig_c));
    // operands must live in the workspace (16-B aligned, padded for the bulk GEMV)
    const Vecs &V = ctx->V;
    CK(cudaMemcpyAsync(V.py, v + ctx->row0, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToDevice, ctx->st));
    const double *vf = V.py;
    if (ctx->sharded) {
        CK(cudaMemcpyAsync(V.gfull, v, sizeof(double) * ctx->n, cudaMemcpyDeviceToDevice, ctx->st));
        vf = V.gfull;
    }
    TRY(op_apply(ctx, V.py, vf, y, nullptr, 0));
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_op_diag(ipm_ctx *ctx, const double *sig_b, const double *sig_c, double *d) {
    if (!ctx || !sig_b || !d || (ctx->m > 0 && !sig_c)) return fail(ctx, IPM_ERR_INVALID, "null argument");
    TRY(load_sigmas(ctx, sig_b, sig_c));
    launch_jacobi(ctx->P, ctx->G, ctx->V.sig_b, ctx->V.sig_c, d, 0, ctx->st);
    ctx->launches += 1;
    CKL();
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_pcg(ipm_ctx *ctx, const double *sig_b, const double *sig_c, const double *rhs, double *x,
                              double rtol, int32_t *iters) {
    if (!ctx || !sig_b || !rhs || !x || (ctx->m > 0 && !sig_c)) return fail(ctx, IPM_ERR_INVALID, "null argument");
    if (ctx->P.aug) return fail(ctx, IPM_ERR_STATE, "ipm_pcg solves the condensed system: create with pcg_system = 0");
    TRY(load_sigmas(ctx, sig_b, sig_c));
    launch_jacobi(ctx->P, ctx->G, ctx->V.sig_b, ctx->V.sig_c, ctx->V.Minv, 1, ctx->st);
    CK(cudaMemcpyAsync(ctx->V.rhs, rhs, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToDevice, ctx->st));
    ctx->launches += 1;
    PcgOut po;
    TRY(pcg_solve(ctx, rtol, po));
    CK(cudaMemcpyAsync(x, ctx->V.dx, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToDevice, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (iters) *iters = (int32_t)po.iters;
    if (po.stalled) return fail(ctx, IPM_NOT_CONVERGED, "PCG reached its iteration limit (relres %g)", po.relres);
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_pcg_iterate(ipm_ctx *ctx, const double *sig_b, const double *sig_c, const double *rhs,
                                      int32_t k, double *x, double *r, double *z, double *p, double *scal) {
    if (!ctx || !sig_b || !rhs || k < 1 || (ctx->m > 0 && !sig_c)) return fail(ctx, IPM_ERR_INVALID, "bad argument");
    if (ctx->P.aug) return fail(ctx, IPM_ERR_STATE, "ipm_pcg_iterate runs the condensed system: pcg_system = 0");
    TRY(load_sigmas(ctx, sig_b, sig_c));
    launch_jacobi(ctx->P, ctx->G, ctx->V.sig_b, ctx->V.sig_c, ctx->V.Minv, 1, ctx->st);
    CK(cudaMemcpyAsync(ctx->V.rhs, rhs, sizeof(double) * ctx->nloc, cudaMemcpyDeviceToDevice, ctx->st));
    ctx->launches += 1;
    PcgOut po;
    TRY(pcg_solve(ctx, 0.0, po, k));
    const size_t nb = sizeof(double) * ctx->nloc;
    if (x) CK(cudaMemcpyAsync(x, ctx->V.dx, nb, cudaMemcpyDeviceToDevice, ctx->st));
    if (r) CK(cudaMemcpyAsync(r, ctx->V.pr, nb, cudaMemcpyDeviceToDevice, ctx->st));
    if (z) CK(cudaMemcpyAsync(z, ctx->V.pz, nb, cudaMemcpyDeviceToDevice, ctx->st));
    if (p) CK(cudaMemcpyAsync(p, ctx->V.pp, nb, cudaMemcpyDeviceToDevice, ctx->st));
    TRY(sync_scalars(ctx));
    if (ctx->hsc->it != k) return fail(ctx, IPM_ERR_STATE, "ran %lld PCG iterations, expected %d", (long long)ctx->hsc->it, k);
    if (scal) {
        scal[0] = ctx->hsc->rho;
        scal[1] = ctx->hsc->pKp;
        scal[2] = ctx->hsc->alpha;
        scal[3] = ctx->hsc->rr;
    }
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_profile(ipm_ctx *ctx, int32_t what, int32_t reps, double *ms) {
    if (!ctx || !ms || reps < 1 || what < 0 || what > 2) return fail(ctx, IPM_ERR_INVALID, "bad argument");
    const Prob &P = ctx->P;
    const Vecs &V = ctx->V;
    CK(cudaMemsetAsync(&ctx->sc->done, 0, sizeof(int64_t), ctx->st));
    CK(cudaMemsetAsync(&ctx->sc->it_rs, 0, sizeof(int64_t), ctx->st));
    if (what == 2 && ctx->fused_p) launch_pcg_p(P, V, ctx->sc, ctx->st);
    auto one = [&]() {
        // what 0: the PCG GEMV's full work (tiles + fused p^T H p) without its done/alpha epilogue
        // (sharded: the GEMV reads a full-length vector — the last allgathered one)
        if (what == 0) launch_gemv(P, ctx->sharded ? V.gfull : V.pp, V.pp, V.ypart, ctx->ncb, V.part[4], ctx->sc,
                                   ctx->gemv_grid, 0, C_GEMV_PCG, ctx->st);
        else if (what == 1 && P.aug) launch_spmv_aug(P, V, V.pp, V.ag.pl, V.ag.pu, ctx->sc, 1, ctx->st);
        else if (what == 1) launch_spmv(P, V.pp, V.sig_c, V.pt, V.part[3], ctx->sc, 1, 1, ctx->st);
        else launch_pcg_iteration(P, V, ctx->G, ctx->ncb, ctx->gemv_grid, ctx->sc, V.dx, 0, 0, ctx->st, &ctx->fork,
                                  ctx->fused_p);
    };
    one();  // warm-up
    CK(cudaEventRecord(ctx->ev[2], ctx->st));
    for (int i = 0; i < reps; ++i) {
        if (what == 2) CK(cudaMemsetAsync(&ctx->sc->done, 0, sizeof(int64_t), ctx->st));
        one();
    }
    CK(cudaEventRecord(ctx->ev[3], ctx->st));
    CKL();
    CK(cudaEventSynchronize(ctx->ev[3]));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, ctx->ev[2], ctx->ev[3]));
    *ms = (double)t / reps;
    ctx->launches += (int64_t)(reps + 1) * (what == 2 ? (3 + 2 * (P.m > 0)) : 1);
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_get_info(const ipm_ctx *ctx, ipm_info *info) {
    if (!ctx || !info) return fail(nullptr, IPM_ERR_INVALID, "null argument");
    info->gemv_kernel = ctx->P.gemv_sym ? 3 : (ctx->P.gemv_bulk ? 2 : 1);
    info->ncb = ctx->ncb;
    info->group_lanes = ctx->G;
    info->sharded = ctx->sharded ? 1 : 0;
    info->rank = ctx->comm ? ctx->comm->rank : 0;
    info->nranks = ctx->comm ? ctx->comm->nranks : 1;
    info->row_begin = ctx->row0;
    info->row_end = ctx->row0 + ctx->nloc;
    return IPM_OK;
}

IPM_EXPORT int64_t ipm_kernel_launches(const ipm_ctx *ctx) { return ctx ? ctx->launches : 0; }

IPM_EXPORT ipm_status ipm_sym_plan(int32_t ncols, int32_t nranks, int32_t rank, int32_t grid, int32_t *tiles,
                                   int32_t cap, int32_t *ntiles, int32_t *ranges, int32_t *ldy, int32_t *ldz) {
    if (ncols < 1 || nranks < 1 || rank < 0 || rank >= nranks || grid < 1 || !ntiles)
        return fail(nullptr, IPM_ERR_INVALID, "bad argument");
    SymPlan pl;
    sym_plan_build(ncols, nranks, rank, grid, pl);
    *ntiles = (int32_t)pl.tiles.size();
    if (tiles)
        for (int t = 0; t < std::min<int>(cap, (int)pl.tiles.size()); ++t) {
            const SymTile &T = pl.tiles[t];
            const int32_t v[8] = {T.r0, T.rows, T.c0, T.cols, T.rslot, T.cmode, T.cbase, T.cslot};
            std::memcpy(tiles + 8 * t, v, sizeof v);
        }
    if (ranges)
        for (int b = 0; b < grid; ++b) {
            const SymRange &r = pl.ranges[b];
            const int32_t v[5] = {r.t0, r.s0, r.t1, r.s1, r.carry};
            std::memcpy(ranges + 5 * b, v, sizeof v);
        }
    if (ldy) *ldy = pl.ldy;
    if (ldz) *ldz = pl.ldz;
    return IPM_OK;
}

#ifdef IPM_TIMELINE
// diagnostic builds only: the ring of per-iteration kernel timestamps (64 x 8 u64, ns)
IPM_EXPORT ipm_status ipm_debug_timeline(ipm_ctx *ctx, unsigned long long *host) {
    CK(cudaMemcpyAsync(host, ctx->sc->tl_ring, sizeof(ctx->sc->tl_ring), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    return IPM_OK;
}
#endif

IPM_EXPORT ipm_status ipm_kernel_timer(ipm_ctx *ctx, double *ms_total, int64_t *launches) {
    if (!ctx || !ms_total || !launches) return fail(ctx, IPM_ERR_INVALID, "bad argument");
    unsigned long long v[2] = {0, 0};
    CK(cudaMemcpyAsync(v, &ctx->sc->kt_ns, sizeof v, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    *ms_total = (double)v[0] * 1e-6;
    *launches = (int64_t)v[1];
    return IPM_OK;
}

IPM_EXPORT const char *ipm_last_error(const ipm_ctx *ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

IPM_EXPORT void ipm_destroy(ipm_ctx *ctx) {
    if (!ctx) return;
    if (ctx->st) cudaStreamSynchronize(ctx->st);
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    if (ctx->graph) cudaGraphDestroy(ctx->graph);
    if (ctx->cap) cudaStreamDestroy(ctx->cap);
    if (ctx->fork.side) cudaStreamDestroy(ctx->fork.side);
    if (ctx->fork.ev_fork) cudaEventDestroy(ctx->fork.ev_fork);
    if (ctx->fork.ev_join) cudaEventDestroy(ctx->fork.ev_join);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->hsc) cudaFreeHost(ctx->hsc);
    if (ctx->tiny_host) cudaFreeHost(ctx->tiny_host);
    for (void *p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    delete ctx->comm;
    delete ctx;
}
