"""Host-side logic of the row-sharded path on CPU: torch.distributed with gloo, world size 2
(127.0.0.1).  Covers the partition every rank derives, the NCCL unique-id broadcast and the
re-assembly of the sharded solution; the device kernels are covered by test_gpu_shard.py."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2405_03584_b200.dist import NCCL_UNIQUE_ID_BYTES, broadcast_unique_id, partition
        n = 1001
        blocks = partition(n, world)
        allb = [None] * world
        dist.all_gather_object(allb, blocks)
        ok_same = all(b == blocks for b in allb)
        b, e = blocks[rank]
        # every rank derives the same partition, blocks tile [0, n) in rank order
        tiles = [x for blk in blocks for x in range(*blk)] == list(range(n))
        fake = lambda: bytes(range(128))
        uid = broadcast_unique_id(fake, rank, dist.broadcast_object_list)
        # re-assemble a "sharded solution": rank r owns x[b:e] (x_j = j / n)
        x_loc = np.arange(b, e) / n
        parts = [None] * world
        dist.all_gather_object(parts, x_loc)
        x = np.concatenate(parts)
        # sharded symmetric GEMV: each rank derives ITS work plan (host-only library hook); the
        # gathered plans use every ordered entry (i, j) of H exactly once across the world
        import ctypes as C
        from paper_2405_03584_b200 import _lib
        nsym = 1000
        nt = C.c_int32()
        _lib.ipm_sym_plan(nsym, world, rank, 148, None, 0, C.byref(nt), None, None, None)
        tl = (C.c_int32 * (8 * nt.value))()
        _lib.ipm_sym_plan(nsym, world, rank, 148, tl, nt.value, C.byref(nt), None, None, None)
        plans = [None] * world
        dist.all_gather_object(plans, (min(rank * -(-nsym // world), nsym), list(tl)))
        used = np.zeros((nsym, nsym), dtype=np.int32)
        for rb, flat in plans:
            for t in range(len(flat) // 8):
                r0, rows, c0, cols, _, cmode, _, _ = flat[8 * t:8 * t + 8]
                used[rb + r0:rb + r0 + rows, c0:c0 + cols] += 1
                if cmode != 0:
                    used[c0:c0 + cols, rb + r0:rb + r0 + rows] += 1
        sym_ok = bool(used.min() == 1 and used.max() == 1)
        q.put((rank, ok_same, tiles, uid == bytes(range(128)) and len(uid) == NCCL_UNIQUE_ID_BYTES,
               bool(np.array_equal(x, np.arange(n) / n)) and sym_ok))
    finally:
        dist.destroy_process_group()


def test_sharding_host_logic_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    for r in res:
        assert r[1] and r[2] and r[3] and r[4], r


def test_nccl_unique_id_available_without_gpu():
    """libipm dlopens libnccl.so.2 for the unique id (host-only call)."""
    from paper_2405_03584_b200 import _lib
    from paper_2405_03584_b200.dist import nccl_unique_id
    try:
        uid = nccl_unique_id()
    except _lib.IpmError as e:
        pytest.skip(f"NCCL not loadable here: {e}")
    assert len(uid) == 128 and any(uid)
