#!/usr/bin/env python
"""Minimal driver for ncu: set up a workload, run `--warmup` untimed steps and `--steps`
steps of the bench's hot-path step (a2, a5-a8 + requant, a10), nothing else."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2402_06859_b200 import ShardedEmbedding  # noqa: E402
from workload import configs, gen  # noqa: E402
from workload import gpu as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="feed1")
ap.add_argument("--alpha", type=float, default=None)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--quantize", action="store_true", help="also run one full-table quantize")
a = ap.parse_args()
cfg = configs.get(a.config)
if a.alpha is not None:
    cfg = cfg.with_(alpha=a.alpha)
dev = torch.device("cuda:0")
B, D, F = cfg.batch, cfg.dim, cfg.num_features
ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0, alpha=cfg.alpha)
emb = ShardedEmbedding(cfg.table_rows, D, cfg.feature_table, max_nnz=len(ids), max_batch=B, q8=True,
                       requant=True, device=dev)
for t in range(cfg.num_tables):
    v = emb.table_view(t)
    G.fill_table(v, v.shape[0], D, emb.pitch, cfg.seed, t)
emb.quantize()
g = torch.empty((B, F, D), device=dev)
G.fill_grad(g, B, F, D, cfg.seed, 0, gen.grad_shift_for(len(ids), D))
ids_d, off_d = torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev)
out = torch.empty((B, F, D), device=dev)
for _ in range(a.warmup + a.steps):
    emb.forward(ids_d, off_d, B, out=out)
    emb.backward_adagrad(g, 0.05)
    emb.forward_q8(ids_d, off_d, B, out=out)
if a.quantize:
    emb.quantize()
assert emb.sync() == 0
torch.cuda.synchronize()
print("ok", len(ids), emb.last_stats())
