"""CPU checks of bench.py's workload table and the oracle legs it times
(no GPU: the device arm is exercised by the gpu suite and the bench runs)."""
import numpy as np

import bench
from oracle import mgk_oracle as O


def test_configs_cover_baseline_shapes():
    # BASELINE.json configs[0..4] -> bench --config 1..5 (4 and 4se share the config-4 graphs)
    assert {"1", "2", "3", "4", "4se", "5"} <= set(bench.CONFIGS)
    for key, cfg in bench.CONFIGS.items():
        assert cfg.x_flops == (3 if cfg.espec is None else 7), key


def test_config1_buckets_and_cpu_leg():
    cfg = bench.CONFIGS["1"]
    bks = bench.buckets(cfg, None)
    assert len(bks) == 1 and len(bks[0][1]) == 16
    rate, dt, jobs, out = bench.cpu_pairs_per_sec(cfg, bks, 6, 0, 2)
    assert rate > 0 and len(out) == 6
    for (b, x, y), (val, it) in zip(jobs, out):
        ref = O.solve_pcg(bks[b][1][x], bks[b][1][y], ("delta", 0.5), ("se", 1.0))
        assert val == ref.value and it == ref.iterations


def test_factored_system_matches_coo_plan():
    from paper_1910_06310_b200 import LabeledGraph, synth

    rng = np.random.default_rng(3)
    g1, g2 = synth.rgg(rng, 60, 6), synth.rgg(rng, 45, 8)
    # labeled graphs with kappa_e = None (ones) and the same graphs unlabeled: one system
    for ga, gb in ((g1, g2), tuple(LabeledGraph.from_arrays(g.node_count, g.edges_i, g.edges_j, g.weights)
                                   for g in (g1, g2))):
        coo = O.ProductSystem(ga, gb)
        fac = O.FactoredSystem(ga, gb)
        p = rng.random(coo.size)
        assert np.allclose(coo.apply(p), fac.apply(p), rtol=1e-12, atol=1e-12)
        a = O.solve_pcg(ga, gb, tol=1e-8)
        b = O.solve_pcg(ga, gb, tol=1e-8, system=fac)
        assert a.iterations == b.iterations and abs(a.value - b.value) <= 1e-12 * abs(a.value)


def test_octile_count_matches_oracle():
    from paper_1910_06310_b200 import synth

    for g in synth.config2(count=40) + synth.config3(count=2, n_lo=200, n_hi=220):
        assert bench.octile_count(g) == O.build_octiles(g).count
