"""Shared test utilities: build a GPU embedding for a workload config, initialise it from the
seeded generator, and build the matching oracle problem (dense for small configs, or
'compact' -- only the touched rows -- for full-size configs)."""
from __future__ import annotations

import numpy as np

import oracle as O
from workload import gen


def make_emb(cfg, *, max_nnz, max_batch, **kw):
    import torch
    from paper_2402_06859_b200 import ShardedEmbedding
    emb = ShardedEmbedding(cfg.table_rows, cfg.dim, cfg.feature_table, max_nnz=max_nnz,
                           max_batch=max_batch, device=torch.device("cuda:0"), **kw)
    return emb


def init_tables_gpu(emb, cfg, seed=None):
    """Fill every local table from the generator on the GPU (workload/libwlgen.so)."""
    from workload import gpu
    seed = cfg.seed if seed is None else seed
    for t in range(cfg.num_tables):
        v = emb.table_view(t)
        if v.shape[0]:
            gpu.fill_table(v, v.shape[0], cfg.dim, emb.pitch, seed, t, row0=int(emb.row_lo[t]),
                           stream=emb.stream)


def init_tables_host(emb, cfg, seed=None):
    """Fill every local table from the numpy generator (small configs)."""
    import torch
    seed = cfg.seed if seed is None else seed
    for t in range(cfg.num_tables):
        v = emb.table_view(t)
        n = v.shape[0]
        if n:
            rows = np.arange(int(emb.row_lo[t]), int(emb.row_lo[t]) + n)
            vals = gen.table_rows(seed, t, rows, cfg.dim)
            full = np.zeros((n, emb.pitch), dtype=np.float32)
            full[:, :cfg.dim] = vals
            v.copy_(torch.from_numpy(full))


def dense_tables(cfg, seed=None):
    seed = cfg.seed if seed is None else seed
    return np.concatenate([gen.table_rows(seed, t, np.arange(r), cfg.dim)
                           for t, r in enumerate(cfg.table_rows)]).astype(np.float32)


def problem(cfg, pooling=0):
    return O.Problem(cfg.table_rows, cfg.dim, cfg.feature_table, pooling)


class Compact:
    """Oracle problem restricted to the rows a batch touches.

    All features read one compact table whose row k is global key keys[k]; ids are
    remapped to k (invalid ids to -1).  The map is monotone, so dedup order is preserved.
    """

    def __init__(self, cfg, ids, offsets, B, seed=None, pooling=0):
        seed = cfg.seed if seed is None else seed
        base = np.concatenate([[0], np.cumsum(cfg.table_rows)]).astype(np.int64)
        F = cfg.num_features
        bag_of = np.repeat(np.arange(F * B), np.diff(offsets.astype(np.int64)))
        t = np.asarray(cfg.feature_table, dtype=np.int64)[bag_of // B]
        ids64 = ids.astype(np.int64)
        rows = np.asarray(cfg.table_rows, dtype=np.int64)[t]
        valid = (ids64 >= 0) & (ids64 < rows)
        gkey = np.where(valid, base[t] + ids64, -1)
        self.keys = np.unique(gkey[valid])
        self.cids = np.where(valid, np.searchsorted(self.keys, np.where(valid, gkey, 0)), -1).astype(np.int32)
        tk = np.searchsorted(base, self.keys, side="right") - 1
        self.table_of_key = tk
        self.row_of_key = self.keys - base[tk]
        W = np.zeros((len(self.keys), cfg.dim), dtype=np.float32)
        for tt in np.unique(tk):
            m = tk == tt
            W[m] = gen.table_rows(seed, int(tt), self.row_of_key[m], cfg.dim)
        self.W = W
        self.pb = O.Problem([max(len(self.keys), 1)], cfg.dim, [0] * F, pooling)
        self.offsets = offsets
        self.B = B


def sample_bags(cfg, ids, offsets, B, samples):
    """Sub-batch made of the given sample indices (all features), feature-major."""
    F = cfg.num_features
    off = offsets.astype(np.int64)
    new_ids, lens = [], []
    for f in range(F):
        for b in samples:
            bag = f * B + b
            new_ids.append(ids[off[bag]:off[bag + 1]])
            lens.append(off[bag + 1] - off[bag])
    o = np.zeros(len(lens) + 1, dtype=np.int64)
    o[1:] = np.cumsum(lens)
    return np.concatenate(new_ids).astype(np.int32) if new_ids else np.zeros(0, np.int32), o.astype(np.int32)


def cond_close(gpu, ora, mag, rel=1e-5):
    """Condition-aware pooled-output gate: |gpu-ora| <= rel*sum|terms|."""
    return np.abs(gpu.astype(np.float64) - ora.astype(np.float64)) <= rel * mag + 1e-30


def w_close(gpu, ora, w_old, step, rel=1e-6):
    tol = rel * np.maximum(np.maximum(np.abs(ora), np.abs(w_old)), np.abs(step)) + 1e-12
    return np.abs(gpu.astype(np.float64) - ora.astype(np.float64)) <= tol


# Global squared norm S (a7) against the oracle.  G is each segment's fp64 sum rounded to
# fp32; a segment split across segment-reduce chunks is summed in another fp64 order, so a G
# element may round to the neighbouring fp32 value (SURVEY.md §8(c) comparison classes:
# "an occasional 1-ulp difference"; reading 13).  A 1-ulp change of every element
# moves S = sum G^2 by at most 2 * 2^-24 relative: the bound below.  Unsplit segments (and
# fp64 sums that stay exact) agree bit for bit.
S_REL = 2.0 ** -22


def S_close(gpu, ora):
    return abs(gpu - ora) <= S_REL * abs(ora)
