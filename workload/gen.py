"""Seeded synthetic inputs for the LiRank sparse-embedding hot path.

This module is the ONLY code shared by the CUDA path's tests/bench and the
CPU oracle (``oracle/``).  It holds none of the method's arithmetic: no
pooling, no dedup, no clipping, no AdaGrad, no quantization.  It only draws
numbers.

Two kinds of draws:

* **Counter-based values** (table rows, upstream gradients).  SplitMix64
  (Steele, Lea & Flood 2014) outputs ``mix(state0 + n * GAMMA)`` for
  n = 1, 2, ...; we address them directly by counter so any row can be drawn
  on its own.  The CUDA generator in ``workload/csrc/gen.cu`` implements the
  same function bit for bit (pinned by ``tests/test_workload.py`` on CPU and
  ``tests/test_gpu_parity.py::test_gpu_generator_matches_numpy`` on GPU).
  A value is an Irwin-Hall(4) sum of 22-bit uniform integers, centred and
  scaled by a power of two, so it is exact in fp32 and roughly normal
  (embeddings "typically follow a normal distribution").

* **Ids and bag lengths** come from numpy's PCG64 (seeded) on the host, once;
  the same int32 arrays feed both the GPU and the oracle.
  Ids are bounded Zipf(alpha) ranks (Hörmann & Derflinger rejection-
  inversion), mapped to rows by the bijection
  ``row = ((rank-1) * 2654435761 + 977 * t) mod rows_t`` which scatters hot
  rows across the table (and across row-wise shards).
"""
from __future__ import annotations

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GAMMA = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
M22 = np.uint64((1 << 22) - 1)

GRAD_STREAM_BASE = 1 << 32  # stream ids >= this are upstream-gradient streams


def mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser (uint64 in, uint64 out, wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * C1
        z = (z ^ (z >> np.uint64(27))) * C2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> np.uint64:
    """Key of stream ``stream``: the (stream+1)-th SplitMix64 output from state ``seed``."""
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + np.uint64(stream + 1) * GAMMA
    return np.uint64(mix64(np.array([s], dtype=np.uint64))[0])


def ih4_values(key: np.uint64, elem: np.ndarray, shift: int) -> np.ndarray:
    """Irwin-Hall(4) value for each element counter ``elem`` (uint64 array).

    h1 = mix(key + (2e+1)*GAMMA), h2 = mix(key + (2e+2)*GAMMA);
    s = (h1 & M22) + (h1>>22 & M22) + (h2 & M22) + (h2>>22 & M22) - 2^23;
    value = s * 2^-shift  (exact in fp32: |s| <= 2^23).
    """
    e = np.asarray(elem, dtype=np.uint64)
    with np.errstate(over="ignore"):
        two_e = e * np.uint64(2)
        h1 = mix64(key + (two_e + np.uint64(1)) * GAMMA)
        h2 = mix64(key + (two_e + np.uint64(2)) * GAMMA)
    s = ((h1 & M22) + ((h1 >> np.uint64(22)) & M22)
         + (h2 & M22) + ((h2 >> np.uint64(22)) & M22)).astype(np.int64) - (1 << 23)
    return np.ldexp(s.astype(np.float64), -shift).astype(np.float32)


TABLE_SHIFT = 26  # table values: sigma = 2^22/sqrt(3) * 2^-26 ~= 0.036


def table_rows(seed: int, table: int, rows: np.ndarray, dim: int,
               shift: int = TABLE_SHIFT) -> np.ndarray:
    """Initial values of rows ``rows`` (int array) of table ``table``: fp32 [len(rows), dim].

    Element counter e = row * dim + d, stream = table.
    """
    rows = np.asarray(rows, dtype=np.uint64).reshape(-1, 1)
    key = stream_key(seed, table)
    out = np.empty((rows.shape[0], dim), dtype=np.float32)
    step = max(1, (1 << 22) // max(dim, 1))  # bound temporaries to ~4M elements
    cols = np.arange(dim, dtype=np.uint64).reshape(1, -1)
    for i in range(0, rows.shape[0], step):
        e = rows[i:i + step] * np.uint64(dim) + cols
        out[i:i + step] = ih4_values(key, e, shift)
    return out


def grad_values(seed: int, step: int, batch: int, num_features: int, dim: int,
                shift: int, sample0: int = 0) -> np.ndarray:
    """Upstream gradient dL/d(pooled) for samples [sample0, sample0+batch): fp32 [batch, F, dim].

    Element counter e = ((sample0+b) * F + f) * dim + d, stream = 2^32 + step.
    ``sample0`` lets each data-parallel rank draw its slice of the global batch.
    """
    b = np.arange(sample0, sample0 + batch, dtype=np.uint64).reshape(-1, 1, 1)
    f = np.arange(num_features, dtype=np.uint64).reshape(1, -1, 1)
    d = np.arange(dim, dtype=np.uint64).reshape(1, 1, -1)
    e = (b * np.uint64(num_features) + f) * np.uint64(dim) + d
    return ih4_values(stream_key(seed, GRAD_STREAM_BASE + step), e, shift)


# ----------------------------------------------------------------------------
# Ids: bounded Zipf by rejection-inversion (Hörmann & Derflinger 1996).
# ----------------------------------------------------------------------------

def _zipf_rejection_inversion(rng: np.random.Generator, n: int, s: float, size: int) -> np.ndarray:
    """Ranks in {1..n} with P(k) ∝ k^-s.  Vectorised; redraws rejected samples."""
    if size == 0:
        return np.zeros(0, dtype=np.int64)
    if s == 0.0 or n == 1:
        return rng.integers(1, n + 1, size=size, dtype=np.int64)
    one_m_s = 1.0 - s

    def helper1(x):  # log1p(x)/x, ->1 at 0
        out = np.ones_like(x)
        nz = np.abs(x) > 1e-8
        out[nz] = np.log1p(x[nz]) / x[nz]
        out[~nz] = 1.0 - x[~nz] * (0.5 - x[~nz] * (1.0 / 3.0 - 0.25 * x[~nz]))
        return out

    def helper2(x):  # expm1(x)/x, ->1 at 0
        out = np.ones_like(x)
        nz = np.abs(x) > 1e-8
        out[nz] = np.expm1(x[nz]) / x[nz]
        out[~nz] = 1.0 + x[~nz] * 0.5 * (1.0 + x[~nz] * (1.0 / 3.0) * (1.0 + 0.25 * x[~nz]))
        return out

    def h(x):
        return np.exp(-s * np.log(x))

    def h_integral(x):
        lx = np.log(x)
        return helper2(one_m_s * lx) * lx

    def h_integral_inv(x):
        t = np.maximum(x * one_m_s, -1.0)
        return np.exp(helper1(t) * x)

    a = lambda v: np.array([v], dtype=np.float64)
    hx1 = h_integral(a(1.5))[0] - 1.0
    hn = h_integral(a(n + 0.5))[0]
    sd = 2.0 - h_integral_inv(h_integral(a(2.5)) - h(a(2.0)))[0]

    out = np.empty(size, dtype=np.int64)
    todo = np.arange(size)
    while todo.size:
        u = hn + rng.random(todo.size) * (hx1 - hn)
        x = h_integral_inv(u)
        k = np.clip(np.floor(x + 0.5), 1, n)
        ok = (k - x <= sd) | (u >= h_integral(k + 0.5) - h(k))
        out[todo[ok]] = k[ok].astype(np.int64)
        todo = todo[~ok]
    return out


ROW_MULT = 2654435761  # prime > any table size used here, so the map is a bijection


def zipf_rows(rng: np.random.Generator, rows: int, alpha: float, table: int, size: int) -> np.ndarray:
    """Row ids (int64) of one table: Zipf(alpha) ranks scattered by a bijection."""
    assert rows < ROW_MULT
    ranks = _zipf_rejection_inversion(rng, rows, alpha, size)
    return ((ranks - 1) * ROW_MULT + 977 * table) % rows


def bag_lengths(rng: np.random.Generator, kind, batch: int) -> np.ndarray:
    """Bag lengths for one feature.  kind: ('onehot',) | ('multi', m) -> U{1..2m-1} | ('range', lo, hi)."""
    if kind[0] == "onehot":
        return np.ones(batch, dtype=np.int64)
    if kind[0] == "multi":
        m = kind[1]
        return rng.integers(1, 2 * m, size=batch, dtype=np.int64)
    if kind[0] == "range":
        return rng.integers(kind[1], kind[2] + 1, size=batch, dtype=np.int64)
    raise ValueError(kind)


def make_batch(table_rows_list, features, batch: int, seed: int, step: int,
               alpha: float = 1.05):
    """One batch of multi-hot bags, feature-major.

    features: list of (table_index, kind).
    Returns (ids int32 [nnz], offsets int32 [F*batch+1]); bag (f, b) is
    ids[offsets[f*batch+b] : offsets[f*batch+b+1]].
    """
    rng = np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, step, 0x2402]))
    lens = []
    for (t, kind) in features:
        lens.append(bag_lengths(rng, kind, batch))
    lens = np.concatenate(lens) if lens else np.zeros(0, dtype=np.int64)
    offsets = np.zeros(len(features) * batch + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    nnz = int(offsets[-1])
    assert nnz < 2**31
    ids = np.empty(nnz, dtype=np.int64)
    for f, (t, kind) in enumerate(features):
        a, b = offsets[f * batch], offsets[(f + 1) * batch]
        ids[a:b] = zipf_rows(rng, table_rows_list[t], alpha, t, int(b - a))
    return ids.astype(np.int32), offsets.astype(np.int32)


def grad_shift_for(nnz: int, dim: int, target_norm: float = 4.0) -> int:
    """Power-of-two scale for upstream grads so the pre-clip global norm is ~target_norm.

    ||G||^2 ~= nnz * dim * sigma^2 (independent terms); sigma = 2^22/sqrt(3) * 2^-shift.
    """
    sigma = target_norm / np.sqrt(max(nnz, 1) * dim)
    return int(round(np.log2((2.0 ** 22) / np.sqrt(3.0) / sigma)))
