"""bench.py's N-GPU plan (host logic, CPU): the default N > 1 run is BASELINE.json's
strong-scaling configuration -- Feed: global batch 128k row-wise, the 1B-row tables at N = 8
(125M rows and 16k samples per GPU); Ads: 200 tables / 100M rows table-wise at global batch
64k -- and --weak keeps the per-GPU batch."""
import importlib.util
import os

import pytest

from workload import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_feed_strong_scaling_reaches_baseline_feed_config_at_8():
    b = bench()
    cfg, B, sharding, scaling = b.scale_plan(configs.feed1(), 8)
    assert cfg.table_rows == configs.feed8().table_rows  # 960M + 40M = 1B rows (BASELINE configs[3])
    assert sum(cfg.table_rows) // 8 == 125_000_000       # per GPU: the 1-GPU Feed shard
    assert cfg.batch == 131_072 and B == 16_384           # global 128k, 16k per GPU
    assert sharding == "row" and scaling == "strong"


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_ads_strong_scaling_keeps_tables_and_global_batch(N):
    b = bench()
    cfg, B, sharding, scaling = b.scale_plan(configs.ads(), N)
    assert cfg.table_rows == configs.ads().table_rows and sum(cfg.table_rows) == pytest.approx(1e8, rel=1e-3)
    assert B * N == 65_536 and sharding == "table" and scaling == "strong"


def test_weak_keeps_per_gpu_batch():
    b = bench()
    cfg, B, sharding, scaling = b.scale_plan(configs.feed1(), 4, weak=True)
    assert B == 131_072 and cfg.batch == 4 * 131_072 and scaling == "weak"
    assert sum(cfg.table_rows) == 4 * 125_000_000


def test_spot_check_accepts_oracle_readings_and_rejects_a_perturbed_row():
    """bench.py's in-run parity spot check (its oracle side): readings equal to the oracle's own
    step pass; one perturbed row fails."""
    import numpy as np
    import oracle as O
    from workload import gen
    b = bench()
    cfg = configs.tiny()
    W, B = 2, cfg.batch // 2
    per = [gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed + 7919 * r, 0, alpha=cfg.alpha) for r in range(W)]
    ids_g, off_g = b.global_batch(per, cfg.num_features, B)
    gshift = gen.grad_shift_for(len(ids_g), cfg.dim)
    smp = b.OracleSample(cfg, ids_g, off_g, W * B, None, "rowwise", gshift=gshift)
    r = O.train_step(smp.pb, smp.W, smp.A, smp.cids, smp.soff, smp.Bs, smp.grad, b.LR, 1e-7, 1.0)
    keys = smp.keys[::7]
    t = np.searchsorted(smp.base, keys, side="right") - 1
    rows = {}
    for tt in np.unique(t):
        k = np.searchsorted(smp.keys, keys[t == tt])
        rows[int(tt)] = (keys[t == tt] - smp.base[tt], (smp.W[k].copy(), smp.A[k].copy()))
    rd = {"samples": 16, "pooled": r["out"][:16].copy(), "rows": rows}
    res = b.spot_check(cfg, rd, W, B, gshift, "rowwise")
    assert res["ok"] and res["rows_checked"] == len(keys) and res["pooled_bit_exact_frac"] == 1.0
    t0 = next(iter(rows))
    rows[t0][1][0][0, 3] += 1e-3
    assert not b.spot_check(cfg, rd, W, B, gshift, "rowwise")["ok"]
