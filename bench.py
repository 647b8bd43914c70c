"""Benchmark: all-pairs marginalized-graph-kernel Gram matrices on B200.

Default workload (BASELINE.json configs[1]): QM7-shaped
synthetic molecules, 7165 graphs (n 4..23), Kronecker-delta(0.5) vertex
kernel on the element label, square-exponential(1.0) edge kernel on the bond
length, q = 0.05, tol = 1e-10.  One step = the full N(N+1)/2 = 25,672,195-pair
Gram matrix.  ``--config`` selects the other BASELINE shapes (same JSON line):

    1    16 random labeled graphs, full 16x16 Gram                (configs[0])
    2    QM7-shaped, 7165 graphs, all pairs                       (configs[1], default)
    3    protein-sized, 1000 graphs n 200..600, shuffled + PBR     (configs[2])
    4    large sparse, 4 density buckets x 25 graphs n 2k..5k,
         shuffled + PBR, unlabeled, within-bucket Grams (4 x 325) (configs[3])
    4se  the same with the SE edge kernel (X = 7)
    5    10k mixed-size molecules (n 4..128), all pairs           (configs[4], values)

At N GPUs the pair list of every Gram is sharded (cost-ordered ids round-robin
over ranks) and the compact per-pair results are gathered to rank 0 (the only
collective); total work is fixed, so scaling is "strong".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

``--impl reference`` times the CPU oracle port (oracle/mgk_oracle.py, the
restatement of the reference path; the reference itself is pure Python and
not available on the GPU box) with every host core, on bounded pair samples
of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "graph-pairs/sec and effective GFLOP/s vs FP32 peak at 1/2/4/8 B200 vs CPU ref"


@dataclass
class Config:
    key: str
    text: str
    vspec: str | None
    espec: str | None
    tol: float
    x_flops: int          # 3 unlabeled, 3 + kappa_e.flop_count labeled (product.py:212-220)
    reorder: bool         # PBR (seed 0) before the Gram (shuffled inputs)
    cpu_pairs: int        # default oracle sample for cpu_baseline
    parity_pairs: int
    kernel: str           # dominant solver kernel
    nodewise: bool = False  # stream every pair's nodal-similarity field (mgk_gram_nodewise)


CONFIGS = {
    "1": Config("1", "config1: 16 random labeled graphs (n 18..22), full 16x16 Gram", "delta:0.5", "se:1.0", 1e-10,
                7, False, 136, 136, "k_pcg_warp<SE>"),
    "2": Config("2", "config2: QM7-shaped synthetic molecules, {G} graphs, all-pairs Gram", "delta:0.5", "se:1.0",
                1e-10, 7, False, 300000, 200, "k_pcg_warp<SE>"),
    "3": Config("3", "config3: protein-sized synthetic graphs, {G} graphs n 200..600, shuffled + device PBR, "
                "all-pairs Gram", "delta:0.5", "se:1.0", 1e-10, 7, True, 48, 6, "k_pcg_panel<SE>"),
    "4": Config("4", "config4: large sparse RGGs, 4 density buckets (mean degree 4/8/16/32) x {B} graphs n 2k..5k, "
                "shuffled + device PBR, unlabeled, within-bucket Grams", None, None, 1e-6, 3, True, 4, 5,
                "k_pcg_grid<unlabeled>"),
    "4se": Config("4se", "config4 with the SE(1.0) edge kernel on the scaled edge length: 4 buckets x {B} graphs",
                  None, "se:1.0", 1e-10, 7, True, 0, 2, "k_pcg_grid<SE>"),
    "5": Config("5", "config5: {G} mixed-size synthetic molecules (60% n 4..23, 30% 24..64, 10% 65..128), "
                "all-pairs Gram", "delta:0.5", "se:1.0", 1e-10, 7, False, 20000, 100, "k_pcg_warp + k_pcg_panel"),
    "5nw": Config("5nw", "config5 nodal similarity: {G} mixed-size molecules, every pair's n_a x n_b field streamed "
                  "to the host in 1 GiB chunks", "delta:0.5", "se:1.0", 1e-10, 7, False, 20000, 100,
                  "k_pcg_warp<nodewise> + k_pcg_panel<nodewise>", nodewise=True),
}

NW_CHUNK = 1 << 30


def buckets(cfg: Config, count: int | None):
    """[(name, graphs)] -- one Gram per bucket (config 4: one per density)."""
    from paper_1910_06310_b200 import synth

    if cfg.key == "1":
        return [("all", synth.config1())]
    if cfg.key == "2":
        return [("all", synth.config2(count=count or 7165))]
    if cfg.key == "3":
        return [("all", synth.config3(count=count or 1000))]
    if cfg.key in ("5", "5nw"):
        return [("all", synth.config5(count=count or 10000))]
    per = count or 25
    out = []
    for k, d in enumerate((4, 8, 16, 32)):
        gs = synth.config4(count=per, seed=100 + k, degrees=(d,))
        out.append((f"deg{d}", gs))
    return out


def describe(cfg: Config, bks, pairs):
    graphs = [g for _, b in bks for g in b]
    return {
        "workload": cfg.text.format(G=len(graphs), B=len(bks[0][1])),
        "graphs": len(graphs),
        "pairs": pairs,
        "nodes_mean": float(np.mean([g.node_count for g in graphs])),
        "edges_mean": float(np.mean([g.edge_count for g in graphs])),
        "vertex_kernel": cfg.vspec,
        "edge_kernel": cfg.espec,
        "q": 0.05,
        "tol": cfg.tol,
        "reorder": "pbr seed 0 (device)" if cfg.reorder else "none",
        "cache": "L2 flushed (256 MiB device write) before every timed step; the dataset is smaller than L2, the "
                 "solver state of configs 3-4 is not",
    }


# ---------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------

_POOL = {}


def _oracle_pair(job):
    from oracle import mgk_oracle as O

    b, x, y = job
    ds, vspec, espec, tol = _POOL["ds"][b], _POOL["v"], _POOL["e"], _POOL["tol"]
    if espec is None:
        system = O.FactoredSystem(ds[x], ds[y], vspec)
        r = O.solve_pcg(ds[x], ds[y], vspec, None, tol=tol, system=system)
    else:
        r = O.solve_pcg(ds[x], ds[y], vspec, espec, tol=tol)
    return r.value, r.iterations


def _spec(s):
    from oracle import mgk_oracle as O

    return O.parse_spec(s) if s else None


def sample_pairs(bks, npairs: int, seed: int):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(npairs):
        b = int(rng.integers(0, len(bks)))
        G = len(bks[b][1])
        x, y = sorted(rng.integers(0, G, size=2).tolist())
        out.append((b, x, y))
    return out


def cpu_pairs_per_sec(cfg: Config, bks, npairs: int, seed: int, procs: int):
    """Time the oracle (float64 numpy restatement of solve_pcg) on a random pair sample."""
    import multiprocessing as mp

    _POOL.update(ds=[b for _, b in bks], v=_spec(cfg.vspec), e=_spec(cfg.espec), tol=cfg.tol)
    jobs = sample_pairs(bks, npairs, seed)
    ctx = mp.get_context("fork")
    procs = max(1, min(procs, npairs))
    with ctx.Pool(procs) as pool:
        if npairs >= 4 * procs:
            pool.map(_oracle_pair, jobs[: procs], chunksize=1)  # warm the workers
        t0 = time.perf_counter()
        out = pool.map(_oracle_pair, jobs, chunksize=max(1, npairs // (procs * 8)))
        dt = time.perf_counter() - t0
    return npairs / dt, dt, jobs, out


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def traffic_from_profiles(cfg: Config):
    """dram bytes per launch of the solver kernel from the committed ncu capture of this config, if any."""
    for p in sorted((ROOT / "profiles").glob(f"*ncu_summary_c{cfg.key}.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            return d.get("solver_dram_bytes_per_launch"), p.name
        except Exception:
            continue
    return None, None


def ncu_pipes(cfg: Config):
    """Pipe utilisation of the dominant kernel from the newest committed ncu --set full summary (config 2's
    narrow warp solver), or None."""
    if cfg.key not in ("1", "2"):
        return None
    for p in sorted((ROOT / "profiles").glob("*ncu_full_narrow_c2*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            pipes = {k.split(".")[0]: v for k, v in d.get("pipes", {}).items()}
            out = {"source": p.name, **pipes, "issue_active_pct": d["launches"][0].get("issue_active_pct"),
                   "ipc_active": d["launches"][0].get("ipc_active")}
            # the resource the kernel is bound by: the busiest pipe of the ncu capture (the FP32 fraction
            # above is the reference's flop convention, not what saturates first)
            if pipes:
                k = max(pipes, key=lambda q: pipes[q])
                out["binding"] = {"pipe": k, "pct_of_peak": pipes[k],
                                  "note": "shared-memory data-pipe wavefronts (P gathers, row entries, segment "
                                          "sums)" if "shared" in k else k}
            return out
        except Exception:
            continue
    return None


_PERMS = {}


def reorder_buckets(raw, device: int):
    """Device PBR (seed 0) of every graph of every bucket in ONE launch (two CTAs per graph, so the
    wall time is the slowest graph's, not the sum over buckets), applied on the host (the public API
    path: pbr_reorder_many + apply_permutation)."""
    from paper_1910_06310_b200 import apply_permutation, pbr_reorder_many

    allg = [g for _, ds in raw for g in ds]
    perms = pbr_reorder_many(allg, seed=0, device=device)
    out, k = [], 0
    for name, ds in raw:
        pp = perms[k: k + len(ds)]
        k += len(ds)
        _PERMS[id(ds)] = pp
        out.append((name, [apply_permutation(g, p) for g, p in zip(ds, pp)]))
    return out


def _oracle_pbr(g):
    from oracle import mgk_oracle as O

    return O.pbr_reorder(g, seed=0).tolist()


def pbr_parity(raw, count: int, max_n: int = 600):
    """Device PBR permutations of the `count` smallest graphs (n <= max_n) against the oracle restatement
    (pinned to the reference's forward maps up to n = 600, tests/golden/pbr_large.json), bit for bit."""
    import multiprocessing as mp

    cand = []
    for _, ds in raw:
        perms = _PERMS.get(id(ds))
        if perms is None:
            continue
        cand += [(g.node_count, k, g, perms[k]) for k, g in enumerate(ds) if g.node_count <= max_n]
    cand = sorted(cand, key=lambda c: (c[0], c[1]))[:count]
    if not cand:
        return None
    with mp.get_context("fork").Pool(min(len(cand), os.cpu_count() or 1)) as pool:
        ref = pool.map(_oracle_pbr, [c[2] for c in cand])
    exact = sum(int(c[3].forward.tolist() == r) for c, r in zip(cand, ref))
    return {"graphs": len(cand), "bit_exact": exact, "nodes": [c[0] for c in cand],
            "oracle": "oracle/mgk_oracle.pbr_reorder (pinned to the reference's pbr_reorder, n <= 600)"}


def _oracle_big_pair(job):
    from oracle import mgk_oracle as O

    ga, gb, vspec, espec, tol = job
    system = (O.FactoredSystem(ga, gb, vspec) if espec is None else
              O.ChunkedSystem(ga, gb, vspec, espec, chunk=512))
    r = O.solve_pcg(ga, gb, vspec, espec, tol=tol, system=system)
    return r.value, r.iterations


def parity_jobs(cfg, bks):
    """(bucket, x, y) pairs checked against the oracle: uniform samples, except config 4se, whose
    full-size SE systems only fit the chunked matrix-free oracle on the smallest graphs -- the smallest
    graph of the sparsest bucket against itself and against the second smallest."""
    if cfg.key != "4se":
        return sample_pairs(bks, cfg.parity_pairs, 1)
    ds = bks[0][1]
    order = sorted(range(len(ds)), key=lambda k: (2 * ds[k].edge_count, k))
    a, b = order[0], order[1]
    return [(0, a, a), (0, min(a, b), max(a, b))]


_T0 = time.perf_counter()


def log(msg: str):
    """Phase progress on stderr (the JSON line stays alone on stdout)."""
    print(f"[bench +{time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1910_06310_b200 import native
    from paper_1910_06310_b200.gram import compute_gram, stream_nodewise

    cfg = CONFIGS[args.config]
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    raw = buckets(cfg, args.count)
    log(f"config {cfg.key}: {sum(len(b) for _, b in raw)} graphs synthesised")
    t_pre = time.perf_counter()
    bks = reorder_buckets(raw, local_rank) if cfg.reorder else list(raw)
    reorder_s = time.perf_counter() - t_pre
    if cfg.reorder:
        log(f"device PBR + apply: {reorder_s:.1f} s")
    ctxs = []
    for _, ds in bks:
        ctx = native.Context(local_rank)
        ctx.upload(native.PackedDataset(ds))
        ctx.set_kernels(cfg.vspec, cfg.espec)
        ctxs.append(ctx)
    npairs = sum(len(ds) * (len(ds) + 1) // 2 for _, ds in bks)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()

    gram_out = {}

    bucket_ms = [[] for _ in bks]

    def step():
        """One Gram per bucket (N=1: device-resident result; N>1: shard + gather to rank 0)."""
        ms_tot, nl_tot, g_tot = 0.0, 0, 0.0
        for bi, (ctx, (_, ds)) in enumerate(zip(ctxs, bks)):
            ms_before = ms_tot
            if cfg.nodewise:
                ctx.gram_nodewise(rank, world, cfg.tol, _discard, NW_CHUNK)
                ms, launches = ctx.last_timing()
                ms_tot += ms
                nl_tot += launches
                bucket_ms[bi].append(ms)
                continue
            if world == 1:
                ctx.gram(cfg.tol, fetch=False)
                ms, launches = ctx.last_timing()
                ms_tot += ms
                nl_tot += launches
                bucket_ms[bi].append(ms)
                continue
            # shard records straight into device tensors (mgk_gram_shard_device), NCCL gather of the
            # padded records to rank 0, device-side assembly of the mirrored matrix (mgk_gram_assemble)
            n = ctx.gram_shard_device(rank, world, cfg.tol)
            nmax = torch.tensor([n], device=dev)
            dist.all_reduce(nmax, op=dist.ReduceOp.MAX)
            cap = int(nmax.item())
            rec = [torch.full((cap,), -1, dtype=torch.int32, device=dev), torch.full((cap,), -1, dtype=torch.int32,
                   device=dev), torch.empty(cap, dtype=torch.float64, device=dev),
                   torch.empty(cap, dtype=torch.int32, device=dev), torch.zeros(cap, dtype=torch.uint8, device=dev)]
            ctx.gram_shard_device(rank, world, cfg.tol, out=rec)
            ms, launches = ctx.last_timing()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            outs = gather_records(rec, rank, world, dist)
            if rank == 0:
                G = len(ds)
                if gram_out.get(G) is None:
                    gram_out[G] = (torch.empty((G, G), dtype=torch.float64, device=dev),
                                   torch.empty((G, G), dtype=torch.int32, device=dev),
                                   torch.empty((G, G), dtype=torch.uint8, device=dev))
                native.gram_assemble(local_rank, outs, G, *gram_out[G])
            t1.record()
            torch.cuda.synchronize(dev)
            ms_tot += ms
            nl_tot += launches + (1 if rank == 0 else 0)
            g_tot += t0.elapsed_time(t1)
            bucket_ms[bi].append(ms)
        return ms_tot, nl_tot, g_tot

    for w in range(args.warmup):
        flush.zero_()
        barrier()
        step()
        log(f"warmup {w + 1}/{args.warmup} done")
    solve_ms, gather_ms, launches = [], [], 0
    barrier()
    with ClockSampler(local_rank) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            ms, nl, gms = step()
            barrier()
            solve_ms.append(ms)
            gather_ms.append(gms)
            launches += nl
            log(f"timed step: solve {ms:.1f} ms, gather {gms:.1f} ms")
    per_step = np.array(solve_ms) + np.array(gather_ms)
    t_local = torch.tensor([float(np.mean(per_step)), float(np.mean(solve_ms))], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_step, ms_solve = float(t_local[0]), float(t_local[1])
    value = npairs / (ms_step * 1e-3)

    result = None
    if rank == 0:
        # ---- parity sample + algorithmic flops from the iteration counts (outside the timed region)
        from oracle import mgk_oracle as O

        flops = exps = dense = 0.0
        Ks = []
        fp32_peak, ex2_peak = ctxs[0].peaks(local_rank)
        per_bucket = []
        for bi, (ctx, (bname, ds)) in enumerate(zip(ctxs, bks)):
            K, it, cv = ctx.gram(cfg.tol)
            Ks.append((K, it))
            G = len(ds)
            n = np.array([g.node_count for g in ds], dtype=np.float64)
            S = 2.0 * np.array([g.edge_count for g in ds], dtype=np.float64)
            iu, ju = np.triu_indices(G)
            iters = it[iu, ju].astype(np.float64)
            f_b = float(np.sum(iters * (cfg.x_flops * S[iu] * S[ju] + 15.0 * n[iu] * n[ju])))
            flops += f_b
            T = np.array([octile_count(g) for g in ds], dtype=np.float64)
            d_b = float(np.sum(iters * cfg.x_flops * 4096.0 * T[iu] * T[ju]))
            dense += d_b
            exps += float(np.sum(iters * S[iu] * S[ju])) if cfg.espec == "se:1.0" else 0.0
            if len(bks) > 1:  # per-density-bucket evidence (BASELINE configs[3])
                ms_b = float(np.mean(bucket_ms[bi]))
                per_bucket.append({
                    "bucket": bname, "graphs": G, "pairs": G * (G + 1) // 2, "ms": ms_b,
                    "pairs_per_s": G * (G + 1) / 2 / (ms_b * 1e-3),
                    "mean_tile_nnz": float(S.sum() / T.sum()) if T.sum() else 0.0,
                    "mean_iterations": float(iters.mean()),
                    "eff_tflops": f_b / (ms_b * 1e-3) / 1e12,
                    "fp32_frac": f_b / (ms_b * 1e-3) / 1e12 / fp32_peak,
                    "dense_tile_tflops": d_b / (ms_b * 1e-3) / 1e12,
                })
            del iu, ju
        worst, it_dev, checked = 0.0, 0, 0
        if cfg.parity_pairs:
            import multiprocessing as mp

            vs, es = _spec(cfg.vspec), _spec(cfg.espec)
            jobs = parity_jobs(cfg, bks)
            big = cfg.key in ("4", "4se")
            args_ = [(bks[b][1][x], bks[b][1][y], vs, es, cfg.tol) for b, x, y in jobs]
            if big:
                with mp.get_context("fork").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
                    refs = pool.map(_oracle_big_pair, args_)
            else:
                refs = [(o.value, o.iterations) for o in
                        (O.solve_pcg(ga, gb, v, e, tol=t) for ga, gb, v, e, t in args_)]
            for (b, x, y), (ov, oit) in zip(jobs, refs):
                K, it = Ks[b]
                worst = max(worst, abs(K[x, y] - ov) / abs(ov))
                it_dev = max(it_dev, abs(int(it[x, y]) - oit))
                checked += 1
        pbr = pbr_parity(raw, 5) if cfg.reorder else None
        del Ks
        log(f"parity sample done ({checked} pairs)")
        achieved = flops / world / (ms_solve * 1e-3) / 1e12
        traffic, traffic_src = traffic_from_profiles(cfg)

        # ---- end to end through the public API with host buffers (rank 0)
        e2e_ms = []
        nrep = max(1, min(args.steps, 3))
        # short configs get one untimed warm-up call of the public API path (its first call creates the
        # process-wide context); the long ones (minutes per call) are timed from their first call
        plan = ([False] if cfg.key in ("1", "2", "5") else []) + [True] * nrep
        h0 = d0 = None
        for timed in plan:
            if timed and h0 is None:
                h0, d0 = ctxs[0].transfer_bytes()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            srcs = reorder_buckets(raw, local_rank) if cfg.reorder else raw
            for (_, ds), (_, src) in zip(raw, srcs):
                if cfg.nodewise:
                    got = stream_nodewise(src, _checksum, cfg.vspec, cfg.espec, _solver_cfg(cfg), NW_CHUNK,
                                          device=local_rank)
                    assert got[0] == len(ds) * (len(ds) + 1) // 2
                    continue
                res = compute_gram(src, cfg.vspec, cfg.espec, cfg=_solver_cfg(cfg), device=local_rank)
                assert res.matrix.shape == (len(ds), len(ds))
            torch.cuda.synchronize(dev)
            if timed:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h1, d1 = ctxs[0].transfer_bytes()
        e2e_val = npairs / (float(np.mean(e2e_ms)) * 1e-3)
        log(f"e2e done: {np.mean(e2e_ms):.1f} ms")

        # ---- CPU oracle baseline on this host
        cores = os.cpu_count() or 1
        cpu = None
        ncpu = args.cpu_pairs if args.cpu_pairs is not None else cfg.cpu_pairs
        if ncpu:
            cpu_rate, cpu_dt, _, _ = cpu_pairs_per_sec(cfg, bks, ncpu, 7, cores)
            log(f"cpu baseline done: {cpu_rate:.1f} pairs/s")
            cpu = {
                "value": cpu_rate,
                "unit": "pairs/s",
                "cores": min(cores, ncpu),
                "kind": "port",
                "sample": f"{ncpu} uniformly sampled pairs of this workload, oracle/mgk_oracle.solve_pcg (float64 "
                          f"numpy{', factored unlabeled system' if cfg.espec is None else ''}), multiprocessing "
                          f"pool of {min(cores, ncpu)} processes, {cpu_dt:.1f} s",
            }

        result = {
            "metric": METRIC,
            "value": value,
            "unit": "pairs/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded generators, paper_1910_06310_b200/synth.py)",
            "config": describe(cfg, bks, npairs),
            "effective_gflops": flops / (ms_step * 1e-3) / 1e9,
            "roofline": {
                "bound": "fp32",
                "achieved": achieved,
                "peak": fp32_peak,
                "unit": "TFLOP/s",
                "frac": achieved / fp32_peak,
                "traffic": traffic,
                "peak_source": "FFMA microbenchmark measured live in this run (mgk_bench_peaks); "
                               "MEASURED_PEAKS.json has no FP32 CUDA-core figure",
                "flops_per_launch": flops / world,
                "flops_convention": f"sum over pairs of I*(X*S_a*S_b + 15*n_a*n_b), X={cfg.x_flops} (SURVEY §8d)",
                "ex2_convention": "one edge-kernel evaluation per directed contribution (the reference's "
                                  "formulation); the solvers evaluate one per undirected lane-graph edge, half of it",
                "ncu_pipes": ncu_pipes(cfg),
                "ex2_per_launch": exps / world,
                "ex2_achieved_tops": exps / world / (ms_solve * 1e-3) / 1e12,
                "ex2_peak_tops": ex2_peak,
                "ex2_frac": exps / world / (ms_solve * 1e-3) / 1e12 / ex2_peak,
                "kernel": cfg.kernel,
                "traffic_source": traffic_src,
                "dense_tile_equivalent": {
                    "flops_per_launch": dense / world,
                    "tflops": dense / world / (ms_solve * 1e-3) / 1e12,
                    "convention": "SURVEY §8d F_dense = I*X*4096*T_a*T_b (the reference's dense-stream counter, "
                                  "product.py:249-253): the work a dense 8x8 tile-pair kernel would issue; the "
                                  "solvers here skip the zeros, so this exceeds the FP32 peak",
                },
            },
            "cpu_baseline": cpu,
            "e2e": {
                "value": e2e_val,
                "unit": "pairs/s",
                "h2d_bytes_per_step": (h1 - h0) // nrep,
                "d2h_bytes_per_step": (d1 - d0) // nrep,
                "ms_per_step": float(np.mean(e2e_ms)),
                "api": ("paper_1910_06310_b200.stream_nodewise (validate, pack, C-ABI upload, device octiles, "
                        "chunked solve, D2H of every pair's field into pinned buffers, host checksum of each chunk)"
                        if cfg.nodewise else
                        "paper_1910_06310_b200.compute_gram (validate, pack, C-ABI upload, device octiles, solve, "
                        "D2H of the N x N matrix, iterations and flags)")
                       + (" after pbr_reorder_many + apply_permutation" if cfg.reorder else ""),
            },
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "parity": {"sample_pairs": checked, "max_rel_err": worst, "max_iter_diff": it_dev,
                       "bar": "1e-5 relative, +-1 iteration", "pbr_permutations": pbr},
            "solve_ms_per_step": ms_solve,
        }
        if per_bucket:
            result["buckets"] = per_bucket
        if cfg.reorder:
            result["preprocess_s"] = {"device_pbr_and_apply": reorder_s}
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return result


def octile_count(g) -> int:
    """Non-empty 8x8 tiles of the symmetric adjacency (build_tiles, tiles.py:85-127)."""
    ei, ej = np.asarray(g.edges_i, np.int64), np.asarray(g.edges_j, np.int64)
    if len(ei) == 0:
        return 0
    k = (max(g.node_count, 1) + 7) // 8
    keys = np.concatenate([(ei // 8) * k + ej // 8, (ej // 8) * k + ei // 8])
    return int(len(np.unique(keys)))


def _discard(*_chunk):
    """Device-timed nodewise leg: the fields reach pinned host memory and are dropped."""


_NW_SUM = [0.0]


def _checksum(a, b, v, it, cv, off, field):
    """End-to-end nodewise leg: touch every streamed field (a float64 sum over the chunk)."""
    _NW_SUM[0] += float(np.sum(field, dtype=np.float64))


def _solver_cfg(cfg: Config):
    from paper_1910_06310_b200 import SolverConfig

    return SolverConfig(tolerance=cfg.tol)


def gather_records(rec, rank: int, world: int, dist):
    """Gather every rank's padded shard records (pair_a, pair_b, value, iterations, converged; equal
    lengths, graph id -1 = padding) to rank 0: one collective per field (NCCL on device tensors in the
    bench, gloo on CPU tensors in tests/test_dist_gloo.py).  Returns the concatenated fields on rank 0,
    None elsewhere."""
    import torch

    outs = []
    for t in rec:
        o = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
        dist.gather(t, o, dst=0)
        outs.append(torch.cat(o) if rank == 0 else None)
    return outs if rank == 0 else None


def assemble_host(recs, G: int):
    """Host statement of mgk_gram_assemble (gram_post.cu) for the CPU multi-rank test: mirrored writes,
    NaN where not converged, padding skipped."""
    a, b, v, it, cv = [np.asarray(t) for t in recs]
    keep = a >= 0
    a, b, v, it, cv = a[keep].astype(np.int64), b[keep].astype(np.int64), v[keep], it[keep], cv[keep].astype(bool)
    K = np.zeros((G, G))
    I = np.zeros((G, G), dtype=np.int32)
    vv = np.where(cv, v, np.nan)
    K[a, b] = K[b, a] = vv
    I[a, b] = I[b, a] = it
    return K, I


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle port on all host cores
# ---------------------------------------------------------------------------


def run_reference(args, rank, world):
    if rank != 0:
        return None
    cfg = CONFIGS[args.config]
    bks = buckets(cfg, args.count)
    npairs = sum(len(ds) * (len(ds) + 1) // 2 for _, ds in bks)
    if not cfg.cpu_pairs:
        return {"impl": "reference", "unavailable": f"config {cfg.key}: the labeled product systems are too large "
                "for the float64 oracle (S_a*S_b up to 1e10 nonzeros)"}
    cores = os.cpu_count() or 1
    per_step = args.ref_pairs if args.ref_pairs is not None else max(cfg.cpu_pairs // 3, cores)
    for w in range(args.warmup):
        cpu_pairs_per_sec(cfg, bks, max(cores, per_step // 8), 100 + w, cores)
    rates, times = [], []
    for k in range(args.steps):
        r, dt, _, _ = cpu_pairs_per_sec(cfg, bks, per_step, 1000 + k, cores)
        rates.append(r)
        times.append(dt)
    value = per_step * len(times) / sum(times)
    sample = (f"{per_step} uniformly sampled pairs of this workload per step, oracle/mgk_oracle.solve_pcg (float64 "
              f"numpy restatement of the reference solve_pcg), {min(cores, per_step)} processes")
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "pairs/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generators)",
        "config": describe(cfg, bks, npairs),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": min(cores, per_step), "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="2")
    ap.add_argument("--count", type=int, default=None, help="graphs (per bucket for config 4)")
    ap.add_argument("--cpu-pairs", type=int, default=None)
    ap.add_argument("--ref-pairs", type=int, default=None)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local_rank)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
