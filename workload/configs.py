"""Workload configurations (BASELINE.json "configs").

Shapes only: table sizes, feature->table map, bag-length laws, batch.  The
synthetic recipe (Zipf ids, Irwin-Hall values) lives in ``workload/gen.py``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np


@dataclass
class Config:
    name: str
    table_rows: List[int]
    dim: int
    features: List[Tuple[int, tuple]]  # (table, bag-length kind)
    batch: int                         # global batch
    alpha: float = 1.05
    seed: int = 240206859
    note: str = ""

    @property
    def num_tables(self) -> int:
        return len(self.table_rows)

    @property
    def num_features(self) -> int:
        return len(self.features)

    @property
    def feature_table(self) -> List[int]:
        return [t for (t, _) in self.features]

    @property
    def total_rows(self) -> int:
        return int(sum(self.table_rows))

    def mean_bag(self) -> float:
        m = 0.0
        for (_, k) in self.features:
            if k[0] == "onehot":
                m += 1
            elif k[0] == "multi":
                m += k[1]
            else:
                m += (k[1] + k[2]) / 2
        return m

    def expected_nnz(self) -> int:
        return int(round(self.batch * self.mean_bag()))

    def with_(self, **kw) -> "Config":
        d = dict(self.__dict__)
        d.update(kw)
        return Config(**d)


def _ads_rows(n=200, lo=3500, hi=3_500_000, total=100_000_000):
    r = (hi / lo) ** (1.0 / (n - 1))
    g = lo * r ** np.arange(n)
    g = g * (total / g.sum())
    return [int(round(x)) for x in g]


def tiny() -> Config:
    """4 tables x 10k rows x dim 32, batch 256, <=10 ids/bag (empty bags included)."""
    return Config("tiny", [10_000] * 4, 32,
                  [(t, ("range", 0, 10)) for t in range(4)], 256,
                  note="BASELINE.json configs[0]")


def jobs() -> Config:
    """50 tables x 1M x 64, batch 16k: 20 one-hot, 20 multi(10), 10 multi(30) (1:1)."""
    feats = ([(t, ("onehot",)) for t in range(20)]
             + [(t, ("multi", 10)) for t in range(20, 40)]
             + [(t, ("multi", 30)) for t in range(40, 50)])
    return Config("jobs", [1_000_000] * 50, 64, feats, 16_384, note="BASELINE.json configs[1]")


def jobs_shared() -> Config:
    """Jobs variant: 40 features through 5 shared tables."""
    feats = []
    for f in range(40):
        t = f % 5
        kind = ("onehot",) if f < 16 else (("multi", 10) if f < 32 else ("multi", 30))
        feats.append((t, kind))
    return Config("jobs_shared", [1_000_000] * 5, 64, feats, 16_384, note="PAPER.md:457 sharing")


def ads() -> Config:
    """200 tables, ~100M rows total (log-spaced 3.5k..3.5M) x 64, batch 64k; 120 one-hot + 80 multi(8)."""
    feats = [(t, ("multi", 8) if t % 5 in (1, 3) else ("onehot",)) for t in range(200)]
    return Config("ads", _ads_rows(), 64, feats, 65_536, note="BASELINE.json configs[2]")


FEED_FEATURES = [
    (0, ("multi", 32)),  # viewer historical actor ids  -> member/actor table
    (0, ("onehot",)),    # actor id                      -> member/actor table
    (0, ("multi", 32)),  # actor historical actor ids    -> member/actor table
    (1, ("multi", 16)),  # viewer hashtag ids            -> hashtag table
    (1, ("multi", 16)),  # actor hashtag ids             -> hashtag table
    (1, ("multi", 4)),   # post hashtag ids              -> hashtag table
]


def feed1() -> Config:
    """1-GPU Feed shard: member/actor 120M + hashtag 5M rows x 64, batch 128k (the >=60% HBM gate config)."""
    return Config("feed1", [120_000_000, 5_000_000], 64, list(FEED_FEATURES), 131_072,
                  note="SURVEY.md §8(d) Feed-1; 1/8 of BASELINE.json configs[3] tables, full batch")


def feed8() -> Config:
    """Feed: member 960M + hashtag 40M = 1B rows x 64, batch 128k (row-wise over 8 GPUs)."""
    return Config("feed8", [960_000_000, 40_000_000], 64, list(FEED_FEATURES), 131_072,
                  note="BASELINE.json configs[3]")


def feedq8() -> Config:
    """Feed inference: 1B rows quantized (72 GB), q8 pooled lookup batch 256k."""
    return Config("feedq8", [960_000_000, 40_000_000], 64, list(FEED_FEATURES), 262_144,
                  note="BASELINE.json configs[4]")


def bag_mean(kind) -> float:
    if kind[0] == "onehot":
        return 1.0
    if kind[0] == "multi":
        return float(kind[1])
    return (kind[1] + kind[2]) / 2.0


def table_cost(cfg: Config, batch: int = None) -> List[float]:
    """Table-wise planning weight: per table, the algorithmic bytes one step
    moves for it, sum over the features reading it of B * L_f * (4 + 4 D) (ids + row gathers)
    + B * 4 D (the pooled row).  Passed as emb_config.table_cost so the LPT placement balances
    lookup traffic, not rows."""
    B = cfg.batch if batch is None else batch
    row = 4 * cfg.dim
    cost = [0.0] * cfg.num_tables
    for (t, kind) in cfg.features:
        cost[t] += B * bag_mean(kind) * (4 + row) + B * row
    return cost


CONFIGS = {c.__name__: c for c in (tiny, jobs, jobs_shared, ads, feed1, feed8, feedq8)}


def get(name: str) -> Config:
    return CONFIGS[name]()
