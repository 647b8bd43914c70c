"""Multi-GPU path logic on CPU: world_size-2 gloo.  Each rank solves its
cost-ordered shard of the Gram pairs (pair ids congruent to rank mod world, as
mgk_gram_shard_device assigns them; the CPU oracle stands in for the device
solve, which needs a GPU), pads its records, and bench.gather_records -- the
exact gather bench.py runs over NCCL at N > 1 -- brings them to rank 0, where
the host statement of the device assembly kernel builds the mirrored Gram.
The device side (shard records in device tensors + mgk_gram_assemble) is
covered by tests/test_gpu_parity.py::test_gram_shard_device_records_assemble."""
import os
import socket

import numpy as np
import torch
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
    a, b, v, it, cv = [], [], [], [], []
    for pid in range(rank, len(order), world):  # shard: id = rank mod world
        x, y = order[pid]
        r = O.solve_pcg(ds[x], ds[y], ("delta", 0.5), ("se", 1.0))
        a.append(x), b.append(y), v.append(r.value), it.append(r.iterations), cv.append(r.converged)
    n = torch.tensor([len(a)])
    dist.all_reduce(n, op=dist.ReduceOp.MAX)
    cap = int(n.item())
    pad = cap - len(a)
    rec = [torch.tensor(a + [-1] * pad, dtype=torch.int32), torch.tensor(b + [-1] * pad, dtype=torch.int32),
           torch.tensor(v + [0.0] * pad, dtype=torch.float64), torch.tensor(it + [0] * pad, dtype=torch.int32),
           torch.tensor(cv + [False] * pad, dtype=torch.uint8)]
    outs = bench.gather_records(rec, rank, world, dist)
    if rank == 0:
        K, I = bench.assemble_host([t.numpy() for t in outs], len(ds))
        ref, ref_it, _ = O.gram(ds, "delta:0.5", "se:1.0")
        out["ok"] = bool(np.array_equal(K, ref)) and bool(np.array_equal(I, ref_it))
        out["n"] = int((outs[0] >= 0).sum())
    else:
        assert outs is None
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gram_gather_assemble_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["n"] == 9 * 10 // 2
    assert out["ok"]
