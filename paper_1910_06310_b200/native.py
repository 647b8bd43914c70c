"""ctypes binding of libmgk.so (the C-ABI in include/mgk.h).

The product path has no CPU fallback: if the shared object is missing, or no
CUDA device is visible, every compute call raises ``NativeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("MGK_LIB", HERE / "libmgk.so"))

MGK_E_INVALID, MGK_E_SHAPE, MGK_E_CUDA, MGK_E_UNSUPPORTED, MGK_E_STATE = -1, -2, -3, -4, -5
LABEL_NONE, LABEL_CAT, LABEL_VEC = 0, 1, 2

# name -> (restype, argtypes); the authoritative list of exported symbols
_P = C.c_void_p
SIGNATURES = {
    "mgk_version": (C.c_char_p, []),
    "mgk_last_error": (C.c_char_p, []),
    "mgk_ctx_create": (C.c_int, [C.POINTER(_P), C.c_int]),
    "mgk_ctx_destroy": (C.c_int, [_P]),
    "mgk_upload": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, C.c_int, C.c_int, _P, C.c_int, C.c_int, _P]),
    "mgk_set_kernels": (C.c_int, [_P, C.c_char_p, C.c_char_p]),
    "mgk_set_vertex_floor": (C.c_int, [_P, C.c_double]),
    "mgk_reorder": (C.c_int, [_P, C.c_int, C.c_uint64, C.c_int, _P]),
    "mgk_tiles": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, _P]),
    "mgk_degrees": (C.c_int, [_P, C.c_int32, _P]),
    "mgk_gram": (C.c_int, [_P, C.c_double, C.c_int64, _P, _P, _P]),
    "mgk_gram_normalized": (C.c_int, [_P, C.c_double, C.c_int64, _P, _P, _P]),
    "mgk_gram_shard": (C.c_int, [_P, C.c_int, C.c_int, C.c_double, C.c_int64, _P, _P, _P, _P, _P, _P]),
    "mgk_pairs": (C.c_int, [_P, C.c_int64, _P, _P, C.c_double, C.c_int64, _P, _P, _P, _P, _P]),
    "mgk_kernel": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_double, C.c_int64, _P, _P, _P, _P, _P]),
    "mgk_gram_nodewise": (C.c_int, [_P, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_int64, _P, _P, _P, _P]),
    "mgk_last_timing": (C.c_int, [_P, _P, _P]),
    "mgk_spatial_edges": (C.c_int, [C.c_int, C.c_int32, _P, C.c_int, _P, C.c_double, _P, _P, _P, _P, _P]),
    "mgk_bench_peaks": (C.c_int, [C.c_int, _P, _P]),
    "mgk_transfer_bytes": (C.c_int, [_P, _P]),
    "mgk_counters": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int64, _P, _P, C.c_int, _P]),
    "mgk_gram_shard_device": (C.c_int, [_P, C.c_int, C.c_int, C.c_double, C.c_int64, _P, _P, _P, _P, _P, _P]),
    "mgk_gram_assemble": (C.c_int, [C.c_int, C.c_int64, _P, _P, _P, _P, _P, C.c_int64, _P, _P, _P]),
    "mgk_gram_multi": (C.c_int, [_P, C.c_int, C.c_double, C.c_int64, _P, _P, _P]),
    "mgk_gram_iterations64": (C.c_int, [_P, _P]),
}


# mgk_nodewise_sink (include/mgk.h)
NODEWISE_SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                            C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_uint8),
                            C.POINTER(C.c_int64), C.POINTER(C.c_float))


class NativeError(RuntimeError):
    """libmgk failed (missing library, no device, CUDA error)."""


_lib = None
_lock = threading.Lock()


def load(path: Path | None = None):
    """Load libmgk.so and bind every symbol of SIGNATURES (fails loudly)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path or LIB_PATH)
        if not p.exists():
            raise NativeError(f"libmgk.so not found at {p}; build it with `python -m paper_1910_06310_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def check(rc: int):
    if rc == 0:
        return
    msg = load().mgk_last_error().decode(errors="replace")
    from .basekernels import KernelShapeError

    if rc == MGK_E_INVALID:
        raise ValueError(msg)
    if rc == MGK_E_SHAPE:
        raise KernelShapeError(msg)
    if rc == MGK_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(msg)


class Context:
    """Owns one mgk_ctx (one CUDA device)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = C.c_void_p()
        check(self.lib.mgk_ctx_create(C.byref(h), int(device)))
        self.h = h
        self.G = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.mgk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, packed: "PackedDataset"):
        pk = packed
        check(self.lib.mgk_upload(
            self.h, pk.G, _ptr(pk.node_off), _ptr(pk.edge_off), _ptr(pk.ei), _ptr(pk.ej), _ptr(pk.w), _ptr(pk.p),
            _ptr(pk.q), pk.nl_kind, pk.nl_dim, _ptr(pk.node_labels), pk.el_kind, pk.el_dim, _ptr(pk.edge_labels)))
        self.G = pk.G
        self.packed = pk

    def set_kernels(self, vspec: str | None, espec: str | None):
        check(self.lib.mgk_set_kernels(self.h, (vspec or "").encode(), (espec or "").encode()))

    def set_vertex_floor(self, v_min: float):
        check(self.lib.mgk_set_vertex_floor(self.h, float(v_min)))

    REORDER = {"none": 0, "pbr": 1, "rcm": 2, "morton": 3}

    def reorder(self, method: str, seed: int, apply: bool) -> np.ndarray:
        """mgk_reorder: forward maps (old -> new, local per graph) of every graph, [sum n]."""
        out = np.empty(int(self.packed.node_off[-1]), dtype=np.int64)
        check(self.lib.mgk_reorder(self.h, self.REORDER[method], C.c_uint64(seed & ((1 << 64) - 1)), int(apply),
                                   _ptr(out)))
        return out

    def reorder_pbr(self, seed: int, apply: bool) -> np.ndarray:
        return self.reorder("pbr", seed, apply)

    def tiles(self, g: int):
        nt, nz = C.c_int32(), C.c_int32()
        check(self.lib.mgk_tiles(self.h, int(g), C.byref(nt), C.byref(nz), None, None, None))
        rc = np.empty(2 * nt.value, dtype=np.int32)
        bm = np.empty(nt.value, dtype=np.uint64)
        w = np.empty(nz.value, dtype=np.float32)
        check(self.lib.mgk_tiles(self.h, int(g), C.byref(nt), C.byref(nz), _ptr(rc), _ptr(bm), _ptr(w)))
        return rc.reshape(-1, 2), bm, w

    def degrees(self, g: int, n: int) -> np.ndarray:
        d = np.empty(n, dtype=np.float64)
        check(self.lib.mgk_degrees(self.h, int(g), _ptr(d)))
        return d

    def gram(self, tol: float, max_iter: int = 0, fetch: bool = True):
        G = self.G
        if not fetch:
            check(self.lib.mgk_gram(self.h, float(tol), int(max_iter), None, None, None))
            return None
        K = np.empty((G, G), dtype=np.float64)
        cv = np.empty((G, G), dtype=np.uint8)
        check(self.lib.mgk_gram(self.h, float(tol), int(max_iter), _ptr(K), None, _ptr(cv)))
        it = np.empty((G, G), dtype=np.int64)  # int32 over PCIe, widened by libmgk's host copy threads
        check(self.lib.mgk_gram_iterations64(self.h, _ptr(it)))
        return K, it, cv.view(bool)

    def gram_normalized(self, tol: float, max_iter: int = 0):
        """Gram matrix normalised on the device (normalize_gram, gram.py:98-107)."""
        G = self.G
        K = np.empty((G, G), dtype=np.float64)
        cv = np.empty((G, G), dtype=np.uint8)
        check(self.lib.mgk_gram_normalized(self.h, float(tol), int(max_iter), _ptr(K), None, _ptr(cv)))
        it = np.empty((G, G), dtype=np.int64)
        check(self.lib.mgk_gram_iterations64(self.h, _ptr(it)))
        return K, it, cv.view(bool)

    def gram_shard(self, rank: int, world: int, tol: float, max_iter: int = 0):
        """This rank's share of the Gram pairs: (a, b, value, iterations, converged)."""
        n = C.c_int64()
        check(self.lib.mgk_gram_shard(self.h, rank, world, float(tol), int(max_iter), C.byref(n),
                                      None, None, None, None, None))
        k = n.value
        pa, pb = np.empty(k, np.int32), np.empty(k, np.int32)
        v, it, cv = np.empty(k, np.float64), np.empty(k, np.int32), np.empty(k, np.uint8)
        check(self.lib.mgk_gram_shard(self.h, rank, world, float(tol), int(max_iter), C.byref(n), _ptr(pa),
                                      _ptr(pb), _ptr(v), _ptr(it), _ptr(cv)))
        return pa, pb, v, it, cv

    def gram_nodewise(self, rank: int, world: int, tol: float, consumer, chunk_bytes: int = 1 << 30,
                      max_iter: int = 0):
        """Stream this rank's Gram pairs with their nodewise fields to ``consumer(a, b, value, iterations,
        converged, offsets, field)`` (numpy views valid during the call).  Returns (pairs, floats)."""
        err = []

        def cb(_user, k, pa, pb, val, it, cv, off, nw):
            try:
                a = np.ctypeslib.as_array(pa, (k,))
                b = np.ctypeslib.as_array(pb, (k,))
                v = np.ctypeslib.as_array(val, (k,))
                i = np.ctypeslib.as_array(it, (k,))
                c = np.ctypeslib.as_array(cv, (k,)).astype(bool)
                o = np.ctypeslib.as_array(off, (k + 1,))
                f = np.ctypeslib.as_array(nw, (int(o[-1]),)) if o[-1] > 0 else np.zeros(0, np.float32)
                consumer(a, b, v, i, c, o, f)
                return 0
            except BaseException as e:  # surfaced after the C call returns
                err.append(e)
                return 1

        fn = NODEWISE_SINK(cb)
        n, f = C.c_int64(), C.c_int64()
        rc = self.lib.mgk_gram_nodewise(self.h, int(rank), int(world), float(tol), int(max_iter), int(chunk_bytes),
                                        C.cast(fn, C.c_void_p), None, C.byref(n), C.byref(f))
        if err:
            raise err[0]
        check(rc)
        return n.value, f.value

    def pairs(self, a, b, tol: float, max_iter: int = 0, nodewise: bool = False, sizes=None):
        a = np.ascontiguousarray(a, dtype=np.int32)
        b = np.ascontiguousarray(b, dtype=np.int32)
        k = len(a)
        val = np.empty(k, dtype=np.float64)
        it = np.empty(k, dtype=np.int32)
        res = np.empty(k, dtype=np.float64)
        cv = np.empty(k, dtype=np.uint8)
        nw = None
        if nodewise:
            n = np.asarray(sizes, dtype=np.int64)
            nw = np.empty(int(np.sum(n[a] * n[b])), dtype=np.float64)
        check(self.lib.mgk_pairs(self.h, k, _ptr(a), _ptr(b), float(tol), int(max_iter), _ptr(val), _ptr(it),
                                 _ptr(res), _ptr(cv), _ptr(nw)))
        return val, it, res, cv.astype(bool), nw

    def gram_shard_device(self, rank: int, world: int, tol: float, max_iter: int = 0, out=None) -> int:
        """mgk_gram_shard_device: out = (pair_a, pair_b, value, iters, conv) device tensors (torch) on this
        context's device, or None to count the shard's pairs."""
        n = C.c_int64()
        ptrs = [C.c_void_p(t.data_ptr()) for t in out] if out is not None else [None] * 5
        check(self.lib.mgk_gram_shard_device(self.h, int(rank), int(world), float(tol), int(max_iter), C.byref(n),
                                             *ptrs))
        return n.value

    def counters(self, a: int, b: int, applies: int, model, thresholds, force_dense: bool) -> np.ndarray:
        """mgk_counters: {flops, t1_load, t1_store, t2_load, t2_store, tile_pairs} after `applies` applies."""
        m = np.array([model.E, model.F, model.X, model.r], dtype=np.float64)
        th = np.array([thresholds.sparse_min_max, thresholds.sparse_max_max, thresholds.dense_min], dtype=np.int32)
        out = np.empty(6, dtype=np.float64)
        check(self.lib.mgk_counters(self.h, int(a), int(b), int(applies), _ptr(m), _ptr(th), int(bool(force_dense)),
                                    _ptr(out)))
        return out

    def peaks(self, device: int = 0):
        f, e = C.c_double(), C.c_double()
        check(self.lib.mgk_bench_peaks(int(device), C.byref(f), C.byref(e)))
        return f.value, e.value

    def transfer_bytes(self):
        h, d = C.c_int64(), C.c_int64()
        check(self.lib.mgk_transfer_bytes(C.byref(h), C.byref(d)))
        return h.value, d.value

    def last_timing(self):
        ms, n = C.c_double(), C.c_int32()
        check(self.lib.mgk_last_timing(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value


def spatial_edges(clouds, cutoff: float, device: int = 0):
    """mgk_spatial_edges for a list of (n, dim) float64 point arrays -> per-cloud (ei, ej, w, d)."""
    lib = load()
    pts = [np.ascontiguousarray(np.asarray(p, dtype=np.float64)) for p in clouds]
    dims = {p.shape[1] for p in pts if p.ndim == 2}
    if any(p.ndim != 2 for p in pts) or len(dims) > 1:
        raise ValueError("points must be (n, 2) or (n, 3) arrays of one dimension")
    dim = dims.pop() if dims else 3
    node_off = np.concatenate([[0], np.cumsum([len(p) for p in pts])]).astype(np.int64)
    flat = np.ascontiguousarray(np.concatenate(pts).reshape(-1)) if pts else np.zeros(0)
    eoff = np.empty(len(pts) + 1, dtype=np.int64)
    check(lib.mgk_spatial_edges(int(device), len(pts), _ptr(node_off), dim, _ptr(flat), float(cutoff), _ptr(eoff),
                                None, None, None, None))
    ne = int(eoff[-1])
    ei, ej = np.empty(ne, np.int32), np.empty(ne, np.int32)
    w, d = np.empty(ne, np.float64), np.empty(ne, np.float64)
    check(lib.mgk_spatial_edges(int(device), len(pts), _ptr(node_off), dim, _ptr(flat), float(cutoff), _ptr(eoff),
                                _ptr(ei), _ptr(ej), _ptr(w), _ptr(d)))
    return [(ei[eoff[k]:eoff[k + 1]], ej[eoff[k]:eoff[k + 1]], w[eoff[k]:eoff[k + 1]], d[eoff[k]:eoff[k + 1]])
            for k in range(len(pts))]


class PackedDataset:
    """Graphs packed into the flat arrays mgk_upload takes (the device layout's host image)."""

    def __init__(self, graphs, with_labels: bool = True):
        from .basekernels import KernelShapeError

        graphs = list(graphs)
        if not graphs:
            raise ValueError("dataset must hold at least one graph")
        self.G = len(graphs)
        n = np.array([g.node_count for g in graphs], dtype=np.int64)
        e = np.array([len(g.weights) for g in graphs], dtype=np.int64)
        self.sizes = n
        self.nnz = 2 * e
        self.node_off = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
        self.edge_off = np.concatenate([[0], np.cumsum(e)]).astype(np.int64)
        cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0), dtype=dt)  # noqa: E731
        self.ei = cat([np.asarray(g.edges_i) for g in graphs], np.int32)
        self.ej = cat([np.asarray(g.edges_j) for g in graphs], np.int32)
        self.w = cat([np.asarray(g.weights, float) for g in graphs], np.float64)
        self.p = cat([np.asarray(g.start_prob, float) for g in graphs], np.float64)
        self.q = cat([np.asarray(g.stop_prob, float) for g in graphs], np.float64)
        self.nl_kind, self.nl_dim, self.node_labels = LABEL_NONE, 0, None
        self.el_kind, self.el_dim, self.edge_labels = LABEL_NONE, 0, None
        if with_labels:
            self.nl_kind, self.nl_dim, self.node_labels = self._labels([g.node_labels for g in graphs], "node", n,
                                                                       KernelShapeError, None)
            self.el_kind, self.el_dim, self.edge_labels = self._labels([g.edge_labels for g in graphs], "edge", e,
                                                                       KernelShapeError, e)

    @staticmethod
    def _labels(labs, what, counts, err, edge_counts):
        # presence must be uniform (product.py:158-159, 170-171); edgeless graphs carry no evidence
        present = [lab is not None for lab in labs]
        relevant = [p for p, c in zip(present, counts) if (edge_counts is None or c > 0)]
        if not any(present):
            return LABEL_NONE, 0, None
        if any(relevant) and not all(relevant):
            raise err(f"{what} label presence must be uniform across a pair")
        kinds = {("c" if np.asarray(lab).dtype.kind in "iu" else "v") for lab in labs if lab is not None}
        if len(kinds) > 1:
            raise err(f"{what} label kinds differ across the dataset")
        if kinds == {"c"}:
            data = [np.asarray(lab, np.int64).reshape(-1) if lab is not None else np.zeros(c, np.int64)
                    for lab, c in zip(labs, counts)]
            return LABEL_CAT, 1, np.ascontiguousarray(np.concatenate(data), dtype=np.int64)
        dims = {np.asarray(lab).reshape(len(lab), -1).shape[1] for lab in labs if lab is not None and len(lab)}
        if len(dims) > 1:
            raise err(f"label dimensions differ: {sorted(dims)}")
        d = dims.pop() if dims else 1
        data = [np.asarray(lab, np.float64).reshape(-1, d) if lab is not None else np.zeros((c, d))
                for lab, c in zip(labs, counts)]
        return LABEL_VEC, d, np.ascontiguousarray(np.concatenate(data).reshape(-1), dtype=np.float64)


def gram_multi(ctxs: list, tol: float, max_iter: int = 0):
    """mgk_gram_multi: one host process, one context per device; returns (K, iterations, converged)."""
    lib = load()
    G = ctxs[0].G
    K = np.empty((G, G), dtype=np.float64)
    it = np.empty((G, G), dtype=np.int32)
    cv = np.empty((G, G), dtype=np.uint8)
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    check(lib.mgk_gram_multi(arr, len(ctxs), float(tol), int(max_iter), _ptr(K), _ptr(it), _ptr(cv)))
    return K, it, cv.astype(bool)


def gram_assemble(device: int, records, G: int, K=None, iters=None, conv=None):
    """mgk_gram_assemble on device tensors: records = (pair_a, pair_b, value, iters, conv)."""
    lib = load()
    pa, pb, v, it, cv = records
    p = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
    check(lib.mgk_gram_assemble(int(device), int(pa.numel()), p(pa), p(pb), p(v), p(it), p(cv), int(G), p(K),
                                p(iters), p(conv)))
