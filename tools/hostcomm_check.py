#!/usr/bin/env python
"""The sharded path across real process boundaries on one GPU, launched by torchrun:

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/hostcomm_check.py

Every rank uses cuda:0 and the host transport (EMB_F_HOSTCOMM over gloo, CUDA IPC peer
mappings); row- and table-wise, fused and collective exchange, two steps each against the
oracle on the global batch (tests/test_hostcomm_gpu.py's check).  Exit code 0 iff all pass."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch.distributed as dist  # noqa: E402

from test_hostcomm_gpu import run_check  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
res = {}
for sharding in ("row", "table"):
    for p2p in (True, False):
        res[f"{sharding}-{'p2p' if p2p else 'collective'}"] = run_check(rank, world, sharding, p2p)
good = all(all(v.values()) for v in res.values())
print(json.dumps({"rank": rank, "world": world, "ok": good, "checks": res}), flush=True)
dist.destroy_process_group()
sys.exit(0 if good else 1)
