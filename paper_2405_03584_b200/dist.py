"""Row-sharded QP solves across ranks.

H is partitioned by contiguous row blocks of equal size chunk = ceil(n / P) (the last rank
may own fewer rows); every x-space vector follows the same partition, A and all m-space
vectors are replicated.  Per PCG iteration the library allgathers the search vector p and
one 8-double vector of reduction partials; all cross-rank sums are taken in rank order, so a
run is bitwise reproducible at a fixed P.

Two ways to form the rank group:
  * ``create_nccl`` — one process per GPU under torchrun: rank 0 asks libipm for an
    ncclUniqueId and broadcasts it over the torch.distributed process group (plumbing only;
    the library talks NCCL itself).
  * ``LocalGroup`` — P contexts in ONE process (threads), e.g. P virtual ranks on one GPU
    for testing, or one process driving several GPUs.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Callable, List, Sequence, Tuple

from . import _lib as L

NCCL_UNIQUE_ID_BYTES = 128


def partition(n: int, nranks: int) -> List[Tuple[int, int]]:
    """Row blocks [b, e) of every rank (the partition ipm_create validates)."""
    if nranks < 1 or n < nranks:
        raise ValueError(f"need 1 <= nranks <= n (n={n}, nranks={nranks})")
    chunk = -(-n // nranks)
    out = [(min(n, r * chunk), min(n, (r + 1) * chunk)) for r in range(nranks)]
    if any(b >= e for b, e in out):
        raise ValueError(f"n={n} cannot be split into {nranks} non-empty blocks of ceil(n/P) rows")
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    L.check(L.ipm_nccl_unique_id(buf, NCCL_UNIQUE_ID_BYTES))
    return buf.raw


def broadcast_unique_id(get_id: Callable[[], bytes], rank: int, broadcast_object_list) -> bytes:
    """Rank 0 creates the id, everyone receives it (torch.distributed.broadcast_object_list
    or any compatible function).  Host-side plumbing; testable with gloo on CPU."""
    obj = [get_id() if rank == 0 else None]
    broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != NCCL_UNIQUE_ID_BYTES:
        raise RuntimeError("bad NCCL unique id received")
    return bytes(uid)


def nccl_shard(rank: int, nranks: int, uid: bytes) -> dict:
    buf = C.create_string_buffer(uid, NCCL_UNIQUE_ID_BYTES)
    return dict(rank=rank, nranks=nranks, comm_kind=1, handle=C.cast(buf, C.c_void_p), _buf=buf)


def host_shard(rank: int, nranks: int, allgather_bytes: Callable[[bytes], List[bytes]]) -> dict:
    """comm_kind 3: the library bootstraps its peer-memory data plane through the caller's host
    allgather (allgather_bytes(my_bytes) -> every rank's bytes in rank order), e.g. over a gloo
    process group — so ranks may be separate processes sharing one GPU (CUDA IPC) or one GPU
    each, without NCCL.  Plumbing only: byte marshalling for ipm_create's bootstrap."""

    def cb(send, recv, nbytes, user):
        try:
            parts = allgather_bytes(C.string_at(send, nbytes))
            if len(parts) != nranks or any(len(p) != nbytes for p in parts):
                return 1
            C.memmove(recv, b"".join(parts), nbytes * nranks)
            return 0
        except Exception:  # noqa: BLE001 — reported to the library as a failed allgather
            return 1

    fn = L.IPM_HOST_ALLGATHER(cb)
    hc = L.ipm_host_comm(rank=rank, nranks=nranks, allgather=fn, user=None)
    return dict(rank=rank, nranks=nranks, comm_kind=3, handle=C.cast(C.pointer(hc), C.c_void_p), _keep=(fn, hc))


def torch_allgather_bytes(group=None) -> Callable[[bytes], List[bytes]]:
    """allgather_bytes over a torch.distributed process group (any backend)."""
    import torch.distributed as dist

    def ag(b: bytes) -> List[bytes]:
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, b, group=group)
        return out
    return ag


def create_nccl(tensors: dict, rank: int, nranks: int, **opts):
    """Collective over the default torch.distributed group: returns this rank's QP.
    tensors: the FULL problem except H, which must be this rank's row block."""
    import torch.distributed as dist
    from .qp import QP
    uid = broadcast_unique_id(nccl_unique_id, rank, dist.broadcast_object_list)
    return QP(shard=nccl_shard(rank, nranks, uid), **tensors, **opts)


class LocalGroup:
    """In-process rank group (comm_kind 2): one context per rank, each driven by its own
    host thread (see ``run``)."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        h = C.c_void_p()
        L.check(L.ipm_group_create(nranks, C.byref(h)))
        self.handle = h

    def shard(self, rank: int) -> dict:
        return dict(rank=rank, nranks=self.nranks, comm_kind=2, handle=self.handle)

    def run(self, fns: Sequence[Callable[[], object]]) -> list:
        """Run fns[r] for every rank concurrently (ctypes drops the GIL inside the library)."""
        out = [None] * len(fns)
        err = [None] * len(fns)

        def body(r):
            try:
                out[r] = fns[r]()
            except BaseException as e:  # noqa: BLE001 — re-raised below
                err[r] = e

        th = [threading.Thread(target=body, args=(r,)) for r in range(len(fns))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in err:
            if e is not None:
                raise e
        return out

    def close(self):
        if self.handle:
            L.ipm_group_destroy(self.handle)
            self.handle = None
