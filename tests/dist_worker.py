"""Worker for the multi-process sharded tests (launched by torch.distributed.run from
tests/test_dist_peer.py and tests/test_dist_nccl.py; not collected by pytest).

  python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 --master-port X \
      tests/dist_worker.py --mode host|nccl --out result.json [--same-gpu]

mode host: bootstrap over a gloo process group (comm_kind 3), data plane over peer memory
(CUDA IPC between the processes).  mode nccl: bootstrap over NCCL (comm_kind 1), same data
plane.  --same-gpu: every rank uses cuda:0 (separate processes sharing one GPU).  Rank 0
writes the gathered solution, statuses and per-rank objectives to --out."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="host", choices=["host", "nccl"])
    ap.add_argument("--out", required=True)
    ap.add_argument("--same-gpu", action="store_true")
    ap.add_argument("--nvars", type=int, default=1000)
    ap.add_argument("--mrows", type=int, default=300)
    ap.add_argument("--seed", type=int, default=44)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", 0 if a.same_gpu else local)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo" if a.mode == "host" else "nccl")
    from gen.planted import planted_qp
    from gen.torch_io import problem_tensors
    from paper_2405_03584_b200 import QP
    from paper_2405_03584_b200.dist import (broadcast_unique_id, host_shard, nccl_shard, nccl_unique_id, partition,
                                            torch_allgather_bytes)
    q = planted_qp(a.nvars, a.mrows, density=0.02, rank=32, seed=a.seed, rows="vmat", var="box")
    b, e = partition(q.n, ws)[rank]
    t = problem_tensors(q, dev)
    t["H"] = t["H"][b:e].contiguous()
    if a.mode == "host":
        shard = host_shard(rank, ws, torch_allgather_bytes())
    else:
        uid = broadcast_unique_id(nccl_unique_id, rank, dist.broadcast_object_list)
        shard = nccl_shard(rank, ws, uid)
    qp = QP(device=dev, shard=shard, **t)
    info = qp.info()
    runs = []
    for _ in range(a.repeat):
        st = qp.solve()
        s = qp.stats()
        x = qp.solution()["x"].cpu().numpy()
        runs.append((st, s["obj"], s["ipm_iters"], s["pcg_iters_total"], x))
    gathered = [None] * ws
    dist.all_gather_object(gathered, [(st, obj, it, pcg, x.tolist()) for st, obj, it, pcg, x in runs])
    if rank == 0:
        res = {"ws": ws, "mode": a.mode, "sharded": info["sharded"], "gemv_kernel": info["gemv_kernel"],
               "runs": []}
        for k in range(a.repeat):
            res["runs"].append({"status": [g[k][0] for g in gathered], "obj": [g[k][1] for g in gathered],
                                "ipm_iters": [g[k][2] for g in gathered], "pcg_iters": [g[k][3] for g in gathered],
                                "x": [v for g in gathered for v in g[k][4]]})
        json.dump(res, open(a.out, "w"))
    qp.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
