"""Bisect emb_hash_ids failures on the bench's Feed-1 strings (debug helper)."""
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")
if len(sys.argv) > 1:
    import torch
    import bench
    from paper_2402_06859_b200 import qr
    from workload import configs, gen
    cfg = configs.get("feed1")
    B = cfg.batch
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0, alpha=cfg.alpha)
    f = int(sys.argv[1]); k = int(sys.argv[2])
    a, b = off[f * B], off[(f + 1) * B]
    d, o = bench.id_strings(ids[a:b][:k], [b"member:", b"hashtag:"][cfg.feature_table[f]])
    dev = torch.device("cuda:0")
    h = qr.hash_ids(torch.from_numpy(d).to(dev), torch.from_numpy(o).to(dev))
    torch.cuda.synchronize()
    print("ok", f, k, len(d), o[-1], flush=True)
else:
    for f in range(6):
        for k in [100, 100000, 10**9]:
            r = subprocess.run([sys.executable, __file__, str(f), str(k)], capture_output=True, text=True,
                               env={"CUDA_LAUNCH_BLOCKING": "1", **__import__("os").environ})
            print(f, k, r.returncode, (r.stdout.strip().splitlines() or [""])[-1], (r.stderr.strip().splitlines() or [""])[-1][:120])
