#!/usr/bin/env python
"""Writes a config's batch-0 ids as global row indices (uint32) for tools/q8_layout_probe.cu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workload import configs, gen  # noqa: E402

cfg = configs.get(sys.argv[1])
ids, off = gen.make_batch(cfg.table_rows, cfg.features, cfg.batch, cfg.seed, 0, alpha=cfg.alpha)
row_lo = np.concatenate([[0], np.cumsum(cfg.table_rows)[:-1]]).astype(np.int64)
feat_table = np.array([t for (t, _) in cfg.features])
f_of = np.repeat(np.arange(len(cfg.features)), np.diff(off[::cfg.batch]))
g = (ids.astype(np.int64) + row_lo[feat_table[f_of]]).astype(np.uint32)
g.tofile(sys.argv[2])
print(sys.argv[1], len(g), int(sum(cfg.table_rows)))
