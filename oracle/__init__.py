"""ctypes binding of the CPU oracle (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs, nothing else.  The product
package ``paper_2402_06859_b200`` never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
LIB_OMP_PATH = os.path.join(_HERE, "liboracle_omp.so")  # same source, -fopenmp
CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    newest = max(os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h")))
    for path, extra in ((LIB_PATH, []), (LIB_OMP_PATH, ["-fopenmp"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < newest:
            subprocess.check_call(["gcc", *CFLAGS, *extra, src, "-o", path, "-lm"])
    return LIB_PATH


class _Cfg(C.Structure):
    _fields_ = [("num_tables", C.c_int32), ("table_rows", C.POINTER(C.c_int64)),
                ("dim", C.c_int32), ("num_features", C.c_int32),
                ("feature_table", C.POINTER(C.c_int32)), ("pooling", C.c_int32)]


_libs = {}
_parallel = False


def set_parallel(on: bool, threads: int = 0) -> int:
    """Route every oracle call to the OpenMP build (on) or the sequential one (off).  Both
    give bit-identical results; returns the thread count now in use."""
    global _parallel
    _parallel = bool(on)
    L = lib()
    if on and threads > 0:
        L.ora_set_threads(int(threads))
    return int(L.ora_threads())


def lib():
    path = LIB_OMP_PATH if _parallel else LIB_PATH
    if path not in _libs:
        build()
        L = C.CDLL(path)
        P = C.c_void_p
        i32, i64, f32, f64 = C.c_int32, C.c_int64, C.c_float, C.c_double
        sig = {
            "ora_forward": (i64, [P, P, P, P, i32, P]),
            "ora_dedup": (i64, [P, P, P, i32, P, P, P, P]),
            "ora_segment_reduce": (None, [P, P, i32, i64, P, P, P, P]),
            "ora_sq_norm": (f64, [P, i64, i32, f64]),
            "ora_clip_factor": (f32, [f64, f32, P]),
            "ora_clip": (None, [P, i64, f32, P]),
            "ora_adagrad_rowwise": (None, [P, P, P, i64, P, i32, f32, f32]),
            "ora_adagrad_elementwise": (None, [P, P, P, i64, P, i32, f32, f32]),
            "ora_quantize_row": (i32, [P, i32, P, P, P]),
            "ora_quantize_mm8": (i64, [P, i64, i32, P, P, P]),
            "ora_forward_q8": (i64, [P, P, P, P, P, P, i32, P]),
            "ora_train_step": (i32, [P, P, P, i32, P, P, i32, P, f32, f32, f32, f64, P, P, P, P]),
            "ora_murmur3_x64_128": (None, [P, i64, C.c_uint32, P]),
            "ora_hash_ids": (None, [P, P, i64, P]),
            "ora_qr_expand": (None, [P, P, i64, i64, i32, i64, i32, P, P]),
            "ora_quantize_row_minmax": (i32, [P, i32, P, P, P]),
            "ora_quantize_minmax": (i64, [P, i64, i32, P, P, P]),
            "ora_forward_q8_minmax": (i64, [P, P, P, P, P, P, i32, P]),
            "ora_cold_weight_init": (None, [P, P, i64, f32, P]),
            "ora_fim_penalty": (f64, [P, i64, P, P, P, P, f32, f32]),
            "ora_fim_penalty_grad": (None, [P, P, i64, i32, P, P, P, P, f32, f32, P]),
            "ora_train_step_fim": (i32, [P, P, P, i32, P, P, i32, P, f32, f32, f32, f64, P, P, P, P, f32, f32, P, P]),
            "ora_threads": (i32, []),
            "ora_set_threads": (None, [i32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _libs[path] = L
    return _libs[path]


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Problem:
    """Static description of the tables/features (mirrors ``ora_cfg``)."""

    def __init__(self, table_rows, dim, feature_table, pooling=0):
        self.table_rows = np.ascontiguousarray(table_rows, dtype=np.int64)
        self.feature_table = np.ascontiguousarray(feature_table, dtype=np.int32)
        self.dim = int(dim)
        self.pooling = int(pooling)
        self._c = _Cfg(len(self.table_rows), self.table_rows.ctypes.data_as(C.POINTER(C.c_int64)),
                       self.dim, len(self.feature_table),
                       self.feature_table.ctypes.data_as(C.POINTER(C.c_int32)), self.pooling)

    @property
    def F(self):
        return len(self.feature_table)

    @property
    def total_rows(self):
        return int(self.table_rows.sum())

    @property
    def ref(self):
        return C.byref(self._c)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def forward(pb: Problem, W, ids, offsets, B):
    W, ids, offsets = _f32(W), _i32(ids), _i32(offsets)
    out = np.zeros((B, pb.F, pb.dim), dtype=np.float32)
    bad = lib().ora_forward(pb.ref, _p(W), _p(ids), _p(offsets), B, _p(out))
    return out, int(bad)


def dedup(pb: Problem, ids, offsets, B):
    ids, offsets = _i32(ids), _i32(offsets)
    nnz = int(offsets[-1])
    keys = np.zeros(max(nnz, 1), dtype=np.int64)
    segs = np.zeros(max(nnz, 1) + 1, dtype=np.int64)
    bags = np.zeros(max(nnz, 1), dtype=np.int64)
    nv = C.c_int64(0)
    U = lib().ora_dedup(pb.ref, _p(ids), _p(offsets), B, _p(keys), _p(segs), _p(bags), C.byref(nv))
    return keys[:U].copy(), segs[:U + 1].copy(), bags[:nv.value].copy()


def segment_reduce(pb: Problem, offsets, B, segs, bags, grad):
    offsets, grad = _i32(offsets), _f32(grad)
    segs = np.ascontiguousarray(segs, dtype=np.int64)
    bags = np.ascontiguousarray(bags, dtype=np.int64)
    U = len(segs) - 1
    G = np.zeros((max(U, 0), pb.dim), dtype=np.float32)
    lib().ora_segment_reduce(pb.ref, _p(offsets), B, U, _p(segs), _p(bags), _p(grad), _p(G))
    return G


def sq_norm(G, extra=0.0):
    G = _f32(G)
    U = G.shape[0] if G.ndim == 2 else 0
    D = G.shape[1] if G.ndim == 2 else 1
    return float(lib().ora_sq_norm(_p(G), U, D, float(extra)))


def clip_factor(S, max_norm=1.0):
    nf = C.c_int(0)
    c = lib().ora_clip_factor(float(S), float(max_norm), C.byref(nf))
    return np.float32(c), bool(nf.value)


def clip(G, c):
    G = _f32(G)
    g = np.empty_like(G)
    lib().ora_clip(_p(G), G.size, float(c), _p(g))
    return g


def adagrad(W, A, keys, g, lr, eps, mode="rowwise"):
    """In place on W, A (float32 C-contiguous numpy arrays)."""
    assert W.dtype == np.float32 and W.flags.c_contiguous
    assert A.dtype == np.float32 and A.flags.c_contiguous
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    g = _f32(g)
    D = W.shape[1]
    fn = lib().ora_adagrad_rowwise if mode == "rowwise" else lib().ora_adagrad_elementwise
    fn(_p(W), _p(A), _p(keys), len(keys), _p(g), D, float(lr), float(eps))


def quantize(X):
    X = _f32(X)
    rows, D = X.shape
    codes = np.zeros((rows, D), dtype=np.int8)
    mid = np.zeros(rows, dtype=np.float32)
    sc = np.zeros(rows, dtype=np.float32)
    bad = lib().ora_quantize_mm8(_p(X), rows, D, _p(codes), _p(mid), _p(sc))
    return codes, mid, sc, int(bad)


def forward_q8(pb: Problem, codes, middle, scale, ids, offsets, B):
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    middle, scale = _f32(middle), _f32(scale)
    ids, offsets = _i32(ids), _i32(offsets)
    out = np.zeros((B, pb.F, pb.dim), dtype=np.float32)
    bad = lib().ora_forward_q8(pb.ref, _p(codes), _p(middle), _p(scale), _p(ids), _p(offsets), B, _p(out))
    return out, int(bad)


def train_step(pb: Problem, W, A, ids, offsets, B, grad, lr, eps, max_norm,
               mode="rowwise", extra_sq_norm=0.0, want_out=True):
    """In place on W, A.  Returns dict(out, S, c, U, nonfinite)."""
    assert W.dtype == np.float32 and W.flags.c_contiguous
    assert A.dtype == np.float32 and A.flags.c_contiguous
    ids, offsets, grad = _i32(ids), _i32(offsets), _f32(grad)
    out = np.zeros((B, pb.F, pb.dim), dtype=np.float32) if want_out else None
    S = C.c_double(0)
    c = C.c_float(0)
    U = C.c_int64(0)
    nf = lib().ora_train_step(pb.ref, _p(W), _p(A), 0 if mode == "rowwise" else 1, _p(ids), _p(offsets),
                              B, _p(grad), float(lr), float(eps), float(max_norm), float(extra_sq_norm),
                              _p(out), C.byref(S), C.byref(c), C.byref(U))
    return dict(out=out, S=S.value, c=np.float32(c.value), U=U.value, nonfinite=bool(nf))


# ---- NEXT-1: unlimited-dictionary ids (oracle.h: ora_murmur3_x64_128, ora_qr_expand) ----

def murmur3_x64_128(key: bytes, seed: int = 0):
    """(h1, h2) of MurmurHash3 x64-128."""
    buf = np.frombuffer(bytes(key), dtype=np.uint8).copy() if len(key) else np.zeros(1, np.uint8)
    out = np.zeros(2, dtype=np.uint64)
    lib().ora_murmur3_x64_128(_p(buf), len(key), seed, _p(out))
    return int(out[0]), int(out[1])


def pack_strings(strings):
    """UTF-8 bytes of the strings concatenated + int64 offsets [n+1]."""
    enc = [s.encode("utf-8") if isinstance(s, str) else bytes(s) for s in strings]
    off = np.zeros(len(enc) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(e) for e in enc])
    data = np.frombuffer(b"".join(enc), dtype=np.uint8).copy() if off[-1] else np.zeros(1, np.uint8)
    return data, off


def hash_ids(strings):
    """int64 ids (as uint64) of id strings: h1 of MurmurHash3 x64-128, seed 0."""
    data, off = pack_strings(strings)
    h = np.zeros(max(len(strings), 1), dtype=np.uint64)
    lib().ora_hash_ids(_p(data), _p(off), len(strings), _p(h))
    return h[:len(strings)]


def qr_expand(h, offsets, R: int, Q: int, dual: bool):
    """QR expansion of hashed ids into rows of the concatenated QR table (oracle.h)."""
    h = np.ascontiguousarray(h, dtype=np.uint64)
    offsets = _i32(offsets)
    k = 4 if dual else 2
    ids = np.zeros(max(k * len(h), 1), dtype=np.int32)
    off = np.zeros(len(offsets), dtype=np.int32)
    lib().ora_qr_expand(_p(h), _p(offsets), len(offsets) - 1, len(h), R, Q, 1 if dual else 0, _p(ids), _p(off))
    return ids[:k * len(h)], off


def qr_rows(R: int, Q: int, dual: bool) -> int:
    return (2 if dual else 1) * (Q + R)


# ---- NEXT-4: min-max row-wise 8-bit quantization (oracle.h) ---------------------------

def quantize_minmax(X):
    """(codes uint8 [rows][dim], min [rows], scale [rows], #non-finite rows)."""
    X = _f32(X)
    rows, dim = X.shape
    codes = np.zeros((rows, dim), dtype=np.uint8)
    mn = np.zeros(rows, dtype=np.float32)
    sc = np.zeros(rows, dtype=np.float32)
    bad = lib().ora_quantize_minmax(_p(X), rows, dim, _p(codes), _p(mn), _p(sc))
    return codes, mn, sc, int(bad)


def forward_q8_minmax(pb: Problem, codes, mn, scale, ids, offsets, B):
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    mn, scale, ids, offsets = _f32(mn), _f32(scale), _i32(ids), _i32(offsets)
    out = np.zeros((B, pb.F, pb.dim), dtype=np.float32)
    inv = lib().ora_forward_q8_minmax(pb.ref, _p(codes), _p(mn), _p(scale), _p(ids), _p(offsets), B, _p(out))
    return out, int(inv)


# ---- NEXT-3: incremental training (oracle.h) ------------------------------------------

def cold_weight_init(w0, w1, alpha):
    w0, w1 = _f32(w0), _f32(w1)
    out = np.zeros_like(w0)
    lib().ora_cold_weight_init(_p(w0), _p(w1), w0.size, float(alpha), _p(out))
    return out


def _opt(a):
    return None if a is None else _f32(a)


def fim_penalty(W, w0, H0, w1, H1, lam, alpha):
    W = _f32(W)
    return float(lib().ora_fim_penalty(_p(W), W.size, _p(_opt(w0)), _p(_opt(H0)), _p(_opt(w1)),
                                       _p(_opt(H1)), float(lam), float(alpha)))


def fim_penalty_grad(W, keys, G, w0, H0, w1, H1, lam, alpha):
    """G (float32 [U][dim]) + the penalty gradient of rows `keys` (returns a new array)."""
    W, G = _f32(W), _f32(G).copy()
    keys = np.ascontiguousarray(keys, dtype=np.int64)
    lib().ora_fim_penalty_grad(_p(W), _p(keys), len(keys), G.shape[1], _p(_opt(w0)), _p(_opt(H0)),
                               _p(_opt(w1)), _p(_opt(H1)), float(lam), float(alpha), _p(G))
    return G


def train_step_fim(pb: Problem, W, A, ids, offsets, B, grad, lr, eps, max_norm, w0, H0, w1, H1,
                   lam, alpha, mode="rowwise", extra_sq_norm=0.0):
    """In place on W, A.  Returns dict(S, c, nonfinite)."""
    assert W.dtype == np.float32 and W.flags.c_contiguous and A.dtype == np.float32
    ids, offsets, grad = _i32(ids), _i32(offsets), _f32(grad)
    anchors = [_opt(x) for x in (w0, H0, w1, H1)]
    S = C.c_double(0)
    c = C.c_float(0)
    nf = lib().ora_train_step_fim(pb.ref, _p(W), _p(A), 0 if mode == "rowwise" else 1, _p(ids), _p(offsets), B,
                                  _p(grad), float(lr), float(eps), float(max_norm), float(extra_sq_norm),
                                  *[_p(a) for a in anchors], float(lam), float(alpha), C.byref(S), C.byref(c))
    return dict(S=S.value, c=np.float32(c.value), nonfinite=bool(nf))
