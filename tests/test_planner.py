"""Table-wise placement ("greedy LPT over tables by cost B*L_t*260 B +
B*256 B"; "Each embedding table is placed on a GPU").  Host-only: emb_plan +
emb_local_layout, no device."""
import ctypes as C

import numpy as np
import pytest

from paper_2402_06859_b200 import _lib as L
from workload import configs


def owners(cfg, W, cost=None):
    lib = L.load()
    rows = np.asarray(cfg.table_rows, dtype=np.int64)
    ft = np.asarray(cfg.feature_table, dtype=np.int32)
    keep = [rows, ft]
    own = np.full(cfg.num_tables, -1)
    for r in range(W):
        c = L.EmbConfig(abi_version=L.EMB_ABI_VERSION, num_tables=cfg.num_tables,
                        table_rows=rows.ctypes.data_as(C.POINTER(C.c_int64)), dim=cfg.dim,
                        num_features=cfg.num_features, feature_table=ft.ctypes.data_as(C.POINTER(C.c_int32)),
                        pooling=0, adagrad_mode=0, init_accumulator=0.1, eps=1e-7, max_norm=1.0,
                        max_nnz=1 << 20, max_batch=1024, sharding=L.EMB_SHARD_TABLE, rank=r, world_size=W,
                        flags=0)
        if cost is not None:
            ca = np.asarray(cost, dtype=np.float64)
            keep.append(ca)
            c.table_cost = ca.ctypes.data_as(C.POINTER(C.c_double))
        base = np.zeros(cfg.num_tables, dtype=np.int64)
        assert lib.emb_local_layout(C.byref(c), base.ctypes.data_as(C.c_void_p), None, None) == 0
        assert (own[base >= 0] == -1).all()  # every table on exactly one rank
        own[base >= 0] = r
    assert (own >= 0).all()
    return own


def expected_ids(cfg):
    ids = np.zeros(cfg.num_tables)
    for (t, kind) in cfg.features:
        ids[t] += cfg.batch * configs.bag_mean(kind)
    return ids


@pytest.mark.parametrize("W", [2, 4, 8])
def test_ads_traffic_plan_balances_lookups(W):
    cfg = configs.ads()
    own = owners(cfg, W, configs.table_cost(cfg))
    ids = expected_ids(cfg)
    per = np.array([ids[own == r].sum() for r in range(W)])
    assert np.abs(per - per.mean()).max() <= 0.10 * per.mean(), per
    # the rows-only plan is what the cost plan fixes: at W=8 it leaves ids far less even
    if W == 8:
        per_rows = np.array([ids[owners(cfg, W) == r].sum() for r in range(W)])
        assert np.abs(per_rows - per_rows.mean()).max() > np.abs(per - per.mean()).max()


def test_lpt_cost_matches_reference_greedy():
    """The planner is the textbook LPT: sort by cost descending (stable), each table to the
    least-loaded rank, ties to the lower rank -- re-derived here in Python."""
    cfg = configs.ads()
    cost = configs.table_cost(cfg)
    W = 8
    order = sorted(range(cfg.num_tables), key=lambda t: -cost[t])
    load = [0.0] * W
    ref = np.zeros(cfg.num_tables, dtype=int)
    for t in order:
        r = min(range(W), key=lambda q: (load[q], q))
        ref[t] = r
        load[r] += cost[t]
    assert (owners(cfg, W, cost) == ref).all()


def test_negative_cost_rejected():
    cfg = configs.ads()
    cost = configs.table_cost(cfg)
    cost[3] = -1.0
    with pytest.raises(AssertionError):
        owners(cfg, 2, cost)
