"""Cost model and counters of the product matvec, mirroring ``mgksolver.costs``
(costs.py:27-128) and the counter side of ``ProductOperator`` (product.py:
38-66, 212-272, 423-436).

The counters are a *convention* -- the abstract traffic / flop totals of the
reference's tile-pair plan -- not a measurement of the device kernels (those
are reported by bench.py against the FP32 / MUFU roofline).  ``kernel()``
fills ``KernelResult.counters`` from the device octiles: libmgk builds a
per-graph histogram of nonzeros per octile (``k_tile_hist``) and sums the
plan's per-tile-pair increments over the density classes
(``mgk_counters``), so no tile pair is enumerated on the host.
``predict_costs`` is the reference's closed form for dense inputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

PRIMITIVES = ("naive", "shared-tiling", "register-blocking", "tiling-blocking")


@dataclass
class CostModel:
    """Bytes per edge label ``E``, bytes per float ``F``, flops per fused contribution ``X``,
    tile size ``t`` and chunk length ``r`` (costs.py:27-43)."""

    E: int = 0
    F: int = 4
    X: int = 3
    t: int = 8
    r: int = 8

    def __post_init__(self):
        if self.E < 0 or self.F <= 0 or self.X <= 0:
            raise ValueError("require E >= 0, F > 0, X > 0")
        if self.t <= 0 or self.r <= 0 or self.t % self.r:
            raise ValueError("chunk length r must divide tile size t")


@dataclass
class CounterReport:
    """Totals of the off-diagonal product (costs.py:46-71)."""

    flops: float = 0.0
    t1_load: float = 0.0
    t1_store: float = 0.0
    t2_load: float = 0.0
    t2_store: float = 0.0
    tile_pairs: int = 0
    ai1: Optional[float] = field(default=None)
    ai2: Optional[float] = field(default=None)

    def finalize(self) -> "CounterReport":
        tier1 = self.t1_load + self.t1_store
        tier2 = self.t2_load + self.t2_store
        self.ai1 = self.flops / tier1 if tier1 > 0 else None
        self.ai2 = self.flops / tier2 if tier2 > 0 else None
        return self

    def reset(self) -> None:
        self.flops = self.t1_load = self.t1_store = self.t2_load = self.t2_store = 0.0
        self.tile_pairs = 0
        self.ai1 = self.ai2 = None


@dataclass
class SelectionThresholds:
    """Tile micro-kernel crossovers (product.py:38-53): sparse x sparse iff min(nnz) <= sparse_min_max and
    max(nnz) <= sparse_max_max; dense x dense iff min(nnz) >= dense_min; dense x sparse otherwise."""

    sparse_min_max: int
    sparse_max_max: int
    dense_min: int

    @staticmethod
    def for_mode(mode: str) -> "SelectionThresholds":
        return SelectionThresholds(10, 16, 32) if mode == "unlabeled" else SelectionThresholds(16, 24, 32)


def select_tile_kernel(nnz_a: int, nnz_b: int, mode: str, thresholds: SelectionThresholds | None = None) -> str:
    """product.py:56-66.  Value-transparent on the device (every solver skips the zeros itself); kept for
    the counters and for callers that inspect the reference's plan."""
    th = thresholds or SelectionThresholds.for_mode(mode)
    lo, hi = sorted((nnz_a, nnz_b))
    if lo <= th.sparse_min_max and hi <= th.sparse_max_max:
        return "sparse-sparse"
    return "dense-dense" if lo >= th.dense_min else "dense-sparse"


def _tile_pairs_dense(n: int, m: int, t: int) -> int:
    a, b = -(-n // t), -(-m // t)
    return a * a * b * b


def predict_costs(model: CostModel, n: int, m: int, primitive: str) -> CounterReport:
    """Closed-form per-iteration totals of the four strategies for a dense n x m pair (costs.py:74-128)."""
    E, F, X, t, r = model.E, model.F, model.X, model.t, model.r
    n2m2 = float(n) * n * m * m
    out_store = float(n) * m * F
    if primitive == "naive":
        return CounterReport(flops=2 * n2m2, t1_load=n2m2 * F, t1_store=out_store, t2_load=0.0, t2_store=0.0,
                             tile_pairs=0, ai1=2 / F, ai2=None)
    if primitive not in PRIMITIVES:
        raise ValueError(f"unknown primitive {primitive!r}; expected one of {PRIMITIVES}")
    tiles = _tile_pairs_dense(n, m, t)
    block = (t / r) * E + ((r + t) / r) * F  # bytes of one streamed operand tile + RHS block, per t^2
    ai1_shared = t**2 * X / ((t / r) * E + (1 + t / r) * F)
    if primitive == "shared-tiling":
        return CounterReport(flops=n2m2 * X, t1_load=n2m2 * block / t**2, t1_store=out_store,
                             t2_load=n2m2 * (((r + 1) / r) * E + ((2 * r + 1) / r) * F),
                             t2_store=n2m2 * block / t**2, tile_pairs=tiles, ai1=ai1_shared,
                             ai2=X / ((1 + 1 / r) * E + (2 + 1 / r) * F))
    if primitive == "register-blocking":
        return CounterReport(flops=n2m2 * X, t1_load=n2m2 * block / t**2, t1_store=out_store, t2_load=n2m2 * F,
                             t2_store=n2m2 * F / t**2, tile_pairs=tiles, ai1=ai1_shared,
                             ai2=X / ((1 + 1 / t**2) * F))
    return CounterReport(flops=n2m2 * X, t1_load=n2m2 * (E + 2 * F) / t**2, t1_store=out_store,
                         t2_load=n2m2 * ((r + t) / (r * t)) * (E + F), t2_store=n2m2 * (E + F) / t**2,
                         tile_pairs=tiles, ai1=t**2 * X / (E + 2 * F),
                         ai2=X / ((1 / r + 1 / t) * E + (1 / r + 1 / t) * F))


def default_model(g_a, g_b, mode: str, edge_kernel) -> CostModel:
    """The operator's default model (product.py:212-220): E = 4 bytes per label component in labeled
    mode, F = 4, X = 3 unlabeled / 3 + edge_kernel.flop_count labeled."""
    comps = 0
    if mode == "labeled":
        lab = g_a.edge_labels if g_a.edge_labels is not None else g_b.edge_labels
        comps = 1 if lab.ndim == 1 else lab.shape[1]
        x = 3 + (edge_kernel.flop_count if edge_kernel is not None else 0)
    else:
        x = 3
    return CostModel(E=4 * comps, F=4, X=x)
