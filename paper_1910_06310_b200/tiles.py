"""Octile storage views, mirroring ``mgksolver.tiles`` (tiles.py:19-185).

``build_tiles`` runs the device octile builder (csrc/tiles.cu) and copies the
result back as the reference's ``Tile``/``TiledMatrix`` objects (row, col,
64-bit bitmap, compact values in bit order); it exists for inspection and
bit-exact parity -- the solver reads the octiles straight from HBM.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import native
from .graphs import LabeledGraph

TILE_SIZE = 8
_FULL = (1 << 64) - 1


@dataclass
class Tile:
    tile_row: int
    tile_col: int
    bitmap: int
    weights: np.ndarray
    labels: Optional[np.ndarray] = None
    local_rows: np.ndarray = field(init=False)
    local_cols: np.ndarray = field(init=False)

    def __post_init__(self):
        if not (0 < self.bitmap <= _FULL):
            raise ValueError("tile bitmap must be a nonzero 64-bit mask")
        bits = np.array([b for b in range(64) if self.bitmap >> b & 1], dtype=np.int64)
        if len(self.weights) != len(bits):
            raise ValueError("weight count does not match bitmap population")
        self.local_rows = bits // TILE_SIZE
        self.local_cols = bits % TILE_SIZE

    @property
    def nnz(self) -> int:
        return bin(self.bitmap).count("1")


@dataclass
class TiledMatrix:
    node_count: int
    tile_size: int
    tiles: list

    @property
    def tile_count(self) -> int:
        return len(self.tiles)

    @property
    def padded_size(self) -> int:
        return -(-self.node_count // self.tile_size) * self.tile_size

    def offdiag_tile_count(self) -> int:
        return sum(1 for t in self.tiles if t.tile_row != t.tile_col)


def build_tiles(g: LabeledGraph, device: int = 0) -> TiledMatrix:
    """Device octiles of one graph (tiles.py:85-127) as the reference's host objects.

    Rows, columns and bitmaps come from the device builder; each tile's payload
    follows its bitmap in ascending bit order, as the reference stores it, with
    the graph's float64 weights and its edge labels (the device streams float32
    copies; the host view keeps the caller's values)."""
    from .solver import _ctx_lock, context

    ctx = context(device)
    with _ctx_lock:
        ctx.upload(native.PackedDataset([g], with_labels=False))
        ctx.set_kernels(None, None)
        rc, bm, _ = ctx.tiles(0)
    n = g.node_count
    ei, ej = np.asarray(g.edges_i, dtype=np.int64), np.asarray(g.edges_j, dtype=np.int64)
    # edge index of every (row, col) entry of the symmetric matrix, both directions
    key = np.concatenate([ei * n + ej, ej * n + ei])
    eid = np.concatenate([np.arange(len(ei)), np.arange(len(ei))])
    order = np.argsort(key, kind="stable")
    key, eid = key[order], eid[order]
    w64 = np.asarray(g.weights, dtype=np.float64)
    labels = None if g.edge_labels is None else np.asarray(g.edge_labels)
    tiles = []
    for (r, c), b in zip(rc.tolist(), bm.tolist()):
        b = int(b)
        bits = np.array([k for k in range(64) if b >> k & 1], dtype=np.int64)
        rows, cols = r * TILE_SIZE + bits // TILE_SIZE, c * TILE_SIZE + bits % TILE_SIZE
        e = eid[np.searchsorted(key, rows * n + cols)]
        tiles.append(Tile(int(r), int(c), b, w64[e], None if labels is None else labels[e]))
    return TiledMatrix(n, TILE_SIZE, tiles)


def dump_tiles(m: TiledMatrix) -> str:
    """tiles.py:181-185: ``r c 0x<16 hex> nnz`` per tile."""
    return "\n".join(f"{t.tile_row} {t.tile_col} 0x{t.bitmap:016x} {t.nnz}" for t in m.tiles)


def expand_tile(tile: Tile):
    """tiles.py:130-146 (host view helper)."""
    w = np.zeros((TILE_SIZE, TILE_SIZE))
    w[tile.local_rows, tile.local_cols] = tile.weights
    lab = None
    if tile.labels is not None:
        lab = np.full((TILE_SIZE, TILE_SIZE), -1, dtype=np.int64) if tile.labels.dtype.kind in "iu" else \
            np.zeros((TILE_SIZE, TILE_SIZE) + tile.labels.shape[1:])
        lab[tile.local_rows, tile.local_cols] = tile.labels
    return w, lab


@dataclass
class TileHistogram:
    buckets: np.ndarray
    total: int
    mean_density: float


def tile_histogram(m: TiledMatrix) -> TileHistogram:
    """tiles.py:172-178."""
    b = np.zeros(65, dtype=np.int64)
    for t in m.tiles:
        b[t.nnz] += 1
    dens = float(np.mean([t.nnz for t in m.tiles]) / 64.0) if m.tiles else 0.0
    return TileHistogram(b, int(b.sum()), dens)
