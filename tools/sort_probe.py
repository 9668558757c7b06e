#!/usr/bin/env python
"""a5 alone: forward -> backward steps (no q8 lookup beside the dedup), per-phase CUDA-event
times from the library's profiler; prints the sort / rle ms and their own-bytes fraction."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_06859_b200 import ShardedEmbedding  # noqa: E402
from workload import configs, gen  # noqa: E402
from workload import gpu as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="feed1")
ap.add_argument("--alpha", type=float, default=None)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
cfg = configs.get(a.config)
if a.alpha is not None:
    cfg = cfg.with_(alpha=a.alpha)
dev = torch.device("cuda:0")
B, D, F = cfg.batch, cfg.dim, cfg.num_features
ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0, alpha=cfg.alpha)
emb = ShardedEmbedding(cfg.table_rows, D, cfg.feature_table, max_nnz=len(ids), max_batch=B, device=dev)
for t in range(cfg.num_tables):
    v = emb.table_view(t)
    G.fill_table(v, v.shape[0], D, emb.pitch, cfg.seed, t)
g = torch.empty((B, F, D), device=dev)
G.fill_grad(g, B, F, D, cfg.seed, 0, gen.grad_shift_for(len(ids), D))
ids_d, off_d = torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev)
out = torch.empty((B, F, D), device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    emb.forward(ids_d, off_d, B, out=out)
    emb.backward_adagrad(g, 0.05)
torch.cuda.synchronize()
emb.profile(True)
emb.profile_read(reset=True)
for _ in range(a.steps):
    G.flush_l2(flush)
    emb.forward(ids_d, off_d, B, out=out)
    emb.backward_adagrad(g, 0.05)
ph = emb.profile_read()
assert emb.sync() == 0
n = len(ids)
U = emb.last_stats()[2]
kbits = int(emb.local_rows).bit_length()
dbits = 9 if (24 < kbits <= 27 or 16 < kbits <= 18) else 8
passes = -(-kbits // dbits)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
sort_ms = ph["sort"][0] / ph["sort"][1]
rle_ms = ph["rle"][0] / ph["rle"][1]
sb, rb = n * (8 + 16 * passes), n * 8 + U * 8
print(json.dumps({"config": cfg.name, "alpha": cfg.alpha, "nnz": n, "U": U, "passes": passes,
                  "variant": os.environ.get("LIRANK_OS_VARIANT", "0"),
                  "sort_ms": sort_ms, "rle_ms": rle_ms,
                  "sort_own_frac": sb / (sort_ms / 1e3) / 1e9 / peak,
                  "a5_own_frac": (sb + rb) / ((sort_ms + rle_ms) / 1e3) / 1e9 / peak,
                  "segreduce_ms": ph["segreduce"][0] / ph["segreduce"][1],
                  "update_ms": ph["update"][0] / ph["update"][1]}))
