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
//   tall   m doubles             t = Sigma_c o (A p) when the PCG SpMV's A rows are split
//   flags  kPeerCh x P uint64    per channel: last sequence number each sender completed toward me
// Channels: exchanges issued on different streams (the PCG's SpMV side branch runs next to the
// SYMV) use separate sequence counters and flags (channel 0 = main stream, 1 = side branch).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "state.h"

namespace ipm {

constexpr int kPeerMax = 8;          // ranks reachable by the peer path (one NVLink domain / node)
constexpr int kPeerX = 12;           // xall stage slots (>= number of XStage values)
constexpr int kPeerCh = 2;           // exchange channels (streams)

struct PeerLayout {
    size_t gfull = 0, zall = 0, xall = 0, tall = 0, flags = 0, bytes = 0;
};
PeerLayout peer_layout(int64_t ncols, int64_t m, int nranks);

// Kernel-side view (by value): base[r] = rank r's region as addressable from this device.
struct PeerArgs {
    char *base[kPeerMax];
    int rank = 0, P = 0;
    int64_t chunk = 0;
    int64_t m = 0;              // rows of A; with the split PCG SpMV rank r owns rows [m0(r), m0(r + 1))
    unsigned long long timeout_ns = 30ull * 1000000000ull;   // IPM_PEER_TIMEOUT_S (default 30 s)
    PeerLayout L;
};

// Rows of A owned by rank r for the split PCG SpMV (equal split of m).
inline int64_t peer_mrow0(const PeerArgs &pa, int r) { return pa.m * r / pa.P; }

// Allgather of a vector: every rank stores its `count` entries into every peer's buffer at region
// offset dst_off, element index dst_base (x-space: gfull, rank * chunk; t: tall, m0(rank)), then
// raises its flag on channel ch; the wait makes the full vector usable in stream order.
void launch_peer_put_vec(const PeerArgs &pa, const double *src, int64_t count, size_t dst_off, int64_t dst_base,
                         int ch, Scalars *sc, int check_done, cudaStream_t st);
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
                      cudaGraphConditionalHandle h, int use_cond, cudaStream_t st, int ch = 0);
// zfold from the peer zall buffer: ypart slot ldy-1 of row i = sum over senders in rank order.
void launch_peer_zfold(const PeerArgs &pa, int nloc, double *ypart, int ldy, Scalars *sc, int check_done,
                       cudaStream_t st);

}  // namespace ipm
