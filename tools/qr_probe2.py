"""Run bench.qr_section alone on Feed-1 batch 0 (debug helper)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from workload import configs, gen  # noqa: E402

cfg = configs.get("feed1")
ids, off = gen.make_batch(cfg.table_rows, cfg.features, cfg.batch, cfg.seed, 0, alpha=cfg.alpha)
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(json.dumps(bench.qr_section(cfg, ids, off, cfg.batch, dev, stream, flush, 6529.7)))
