"""Multi-GPU path logic on CPU: world_size-2 gloo.  Each rank solves its
cost-ordered shard of the Gram pairs (here with the CPU oracle standing in for
the device solve, which needs a GPU), results are gathered to rank 0 and
assembled with bench.assemble -- the exact code bench.py runs at N > 1."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    from oracle import mgk_oracle as O
    from paper_1910_06310_b200 import synth

    ds = synth.config2(count=9, seed=4)
    order = O.schedule_pairs([g.node_count for g in ds], [2 * g.edge_count for g in ds])
    rows = []
    for pid in range(rank, len(order), world):  # shard: id = rank mod world
        a, b = order[pid]
        r = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0))
        rows.append([a, b, r.value, r.iterations + 0.5 * r.converged])
    gathered = [None] * world
    dist.all_gather_object(gathered, np.array(rows))
    if rank == 0:
        K = bench.assemble(np.concatenate(gathered), len(ds))
        ref, _, _ = O.gram(ds, "delta:0.5", "se:1.0")
        out["ok"] = bool(np.allclose(K, ref, rtol=0, atol=0))
        out["n"] = int(sum(len(g) for g in gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gram_gather_assemble_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["n"] == 9 * 10 // 2
    assert out["ok"]
