// peer.h — device-side exchange over peer memory for the row-sharded path.
//
// Every rank reserves the same "peer region" at the start of its workspace; at create the
// ranks exchange the regions' addresses (raw pointers inside one process, CUDA IPC handles
// across processes — bootstrapped once over the Comm allgather), so each rank can STORE into
// every peer's region over NVLink / NVSwitch.  A collective is then a producer kernel that
// writes its data straight into the receivers' buffers and raises a per-sender sequence flag
// (release, system scope), plus a one-CTA wait kernel on the receiver (acquire) — no host
// round trip, no NCCL call, so the sharded PCG loop is captured in the same CUDA graph with a
// device-side WHILE node as the single-GPU one.
//
// Ordering: every rank executes the same sequence of exchanges (same control flow, decisions
// taken from bitwise-identical combined scalars), numbered by Scalars::peer_seq.  Buffers are
// single-buffered per exchange TYPE: a sender can only overwrite a receiver's buffer of a type
// after passing a later exchange, whose data the receiver only puts after consuming the first.
// Region layout (identical on every rank; offsets in bytes from the region base):
//   gfull  P*chunk + 2 doubles   allgathered x-space vector (p, x, dx, v)
//   zall   P*chunk doubles       column parts of the sharded SYMV for the receiver's rows, per sender
//   xall   kPeerX stages x P x 8 per-stage scalar partials (Scalars::loc) of every sender
//   flags  P uint64              last sequence number each sender completed toward this rank
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "state.h"

namespace ipm {

constexpr int kPeerMax = 8;          // ranks reachable by the peer path (one NVLink domain / node)
constexpr int kPeerX = 12;           // xall stage slots (>= number of XStage values)

struct PeerLayout {
    size_t gfull = 0, zall = 0, xall = 0, flags = 0, bytes = 0;
};
PeerLayout peer_layout(int64_t ncols, int nranks);

// Kernel-side view (by value): base[r] = rank r's region as addressable from this device.
struct PeerArgs {
    char *base[kPeerMax];
    int rank = 0, P = 0;
    int64_t chunk = 0;
    unsigned long long timeout_ns = 30ull * 1000000000ull;   // IPM_PEER_TIMEOUT_S (default 30 s)
    PeerLayout L;
};

// Allgather of an x-space vector: every rank stores its nloc entries into every peer's gfull at
// rank * chunk, then raises its flag; the wait makes the full vector usable in stream order.
void launch_peer_put_vec(const PeerArgs &pa, const double *src, int64_t count, Scalars *sc, int check_done,
                         cudaStream_t st);
// Scalar partials of one XStage: Scalars::loc (8 doubles) into every peer's xall[stage][rank].
void launch_peer_put_loc(const PeerArgs &pa, int stage, Scalars *sc, int check_done, cudaStream_t st);
// Sharded SYMV column parts: zvec entry zcol[q] (the sum of zpart row q) stored straight into
// the owning rank's zall[rank] slot (fused zreduce + scatter); flags to every peer.
void launch_peer_zput(const PeerArgs &pa, int zrows, int ldz, const double *zpart, const int *zcol, Scalars *sc,
                      int check_done, cudaStream_t st);
// One CTA waits until every sender's flag reaches this exchange's sequence number, advances
// Scalars::peer_seq; stage >= 0 also combines xall[stage] (rank order, k_xcombine's epilogue)
// and, with use_cond, sets the WHILE condition from sc->done (X_PCG_UPDATE).
void launch_peer_wait(const PeerArgs &pa, Scalars *sc, int stage, double p0, double p1, int64_t p2, int check_done,
                      cudaGraphConditionalHandle h, int use_cond, cudaStream_t st);
// zfold from the peer zall buffer: ypart slot ldy-1 of row i = sum over senders in rank order.
void launch_peer_zfold(const PeerArgs &pa, int nloc, double *ypart, int ldy, Scalars *sc, int check_done,
                       cudaStream_t st);

}  // namespace ipm
