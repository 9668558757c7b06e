"""C-ABI library: loads, exports every symbol include/lirank_emb.h declares, host-only
planning logic (CPU, no compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2402_06859_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lirank_emb.h")).read()
    return sorted(set(re.findall(r"EMB_API\s+[\w\s\*]+?\b(emb_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = L.load()
    names = declared_symbols()
    assert len(names) >= 17
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(L.SIGNATURES)  # the binding covers exactly the header


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {L.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_status_strings():
    lib = L.load()
    assert lib.emb_abi_version() == L.EMB_ABI_VERSION
    for code in range(8):
        assert lib.emb_status_string(code)


def make_cfg(rows, dim, ft, **kw):
    rows_a = np.asarray(rows, dtype=np.int64)
    ft_a = np.asarray(ft, dtype=np.int32)
    owner = kw.pop("table_owner", None)
    cfg = L.EmbConfig(abi_version=L.EMB_ABI_VERSION, num_tables=len(rows), table_rows=rows_a.ctypes.data_as(C.POINTER(C.c_int64)),
                      dim=dim, num_features=len(ft), feature_table=ft_a.ctypes.data_as(C.POINTER(C.c_int32)),
                      pooling=0, adagrad_mode=0, init_accumulator=0.1, eps=1e-7, max_norm=1.0,
                      max_nnz=1000, max_batch=64, sharding=0, table_owner=None, rank=0, world_size=1,
                      nccl_unique_id=None, stream=None, flags=0)
    keep = [rows_a, ft_a]
    if owner is not None:
        ow = np.asarray(owner, dtype=np.int32)
        keep.append(ow)
        cfg.table_owner = ow.ctypes.data_as(C.POINTER(C.c_int32))
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg, keep


def plan(cfg):
    s = L.EmbSizes()
    code = L.load().emb_plan(C.byref(cfg), C.byref(s))
    return code, s


def test_plan_sizes():
    cfg, keep = make_cfg([100, 50], 30, [0, 1, 0], flags=L.EMB_F_Q8)
    code, s = plan(cfg)
    assert code == 0
    assert s.row_pitch == 32 and s.q8_pitch == 64 and s.local_rows == 150  # 30 codes+2 pad+8 meta, to 32 B
    assert s.weights_bytes == 150 * 32 * 4 and s.accum_bytes == 150 * 4
    assert s.q8_codes_bytes == 150 * 64 and s.q8_meta_bytes == 0
    assert s.workspace_bytes > 0 and s.workspace_bytes % 256 == 0
    cfg.adagrad_mode = 1
    assert plan(cfg)[1].accum_bytes == 150 * 32 * 4


@pytest.mark.parametrize("field,value", [("dim", 0), ("dim", 1025), ("num_tables", 0), ("abi_version", 99),
                                         ("max_nnz", 1 << 30), ("pooling", 3), ("adagrad_mode", 7),
                                         ("max_norm", 0.0), ("world_size", 0), ("flags", L.EMB_F_REQUANT)])
def test_plan_rejects(field, value):
    cfg, keep = make_cfg([100], 8, [0])
    setattr(cfg, field, value)
    assert plan(cfg)[0] == L.EMB_EINVAL


def test_plan_rejects_bad_feature_table():
    cfg, keep = make_cfg([100], 8, [1])
    assert plan(cfg)[0] == L.EMB_EINVAL
    cfg, keep = make_cfg([2**31], 8, [0])
    assert plan(cfg)[0] == L.EMB_EINVAL


def layout(cfg, T):
    lb, lo, hi = (np.zeros(T, dtype=np.int64) for _ in range(3))
    code = L.load().emb_local_layout(C.byref(cfg), lb.ctypes.data_as(C.c_void_p), lo.ctypes.data_as(C.c_void_p),
                                     hi.ctypes.data_as(C.c_void_p))
    assert code == 0
    return lb, lo, hi


@pytest.mark.parametrize("W", [2, 3, 8])
@pytest.mark.parametrize("mode", [L.EMB_SHARD_TABLE, L.EMB_SHARD_ROW])
def test_sharded_layout_covers_every_row_once(W, mode):
    rows = [1000, 7, 3500, 64, 999_983]
    cover = [np.zeros(r, dtype=np.int32) for r in rows]
    total_local = 0
    for r in range(W):
        cfg, keep = make_cfg(rows, 16, [0, 1, 2, 3, 4, 0], sharding=mode, rank=r, world_size=W)
        code, s = plan(cfg)
        assert code == 0
        lb, lo, hi = layout(cfg, len(rows))
        seen = 0
        for t in range(len(rows)):
            if lb[t] >= 0:
                assert lb[t] == seen  # local tables packed in table order
                cover[t][lo[t]:hi[t]] += 1
                seen += hi[t] - lo[t]
        assert seen == s.local_rows
        total_local += seen
    assert total_local == sum(rows)
    for c in cover:
        assert (c == 1).all()


def test_table_plan_explicit_owner_and_lpt():
    rows = [10, 1000, 100, 500]
    cfg, keep = make_cfg(rows, 8, [0, 1, 2, 3], sharding=L.EMB_SHARD_TABLE, rank=0, world_size=2,
                         table_owner=[1, 1, 0, 0])
    lb, lo, hi = layout(cfg, 4)
    assert (lb >= 0).tolist() == [False, False, True, True]
    # greedy LPT: 1000 -> r0, 500 -> r1, 100 -> r1, 10 -> r1
    cfg, keep = make_cfg(rows, 8, [0, 1, 2, 3], sharding=L.EMB_SHARD_TABLE, rank=0, world_size=2)
    lb, lo, hi = layout(cfg, 4)
    assert (lb >= 0).tolist() == [False, True, False, False]


def test_qr_rows_host_only():
    """emb_qr_rows is host arithmetic (no device needed): (dual ? 2 : 1) * (Q + R)."""
    from paper_2402_06859_b200 import _lib as L
    lib = L.load()
    assert lib.emb_qr_rows(1000, 4294968, 1) == 2 * (4294968 + 1000)
    assert lib.emb_qr_rows(7, 11, 0) == 18
    assert lib.emb_qr_rows(0, 11, 0) < 0 and lib.emb_qr_rows(7, 0, 1) < 0


def test_plan_serving_handle_has_no_fp32_tables():
    """EMB_F_Q8_ONLY (serving): no fp32 weights / accumulators and no training workspace."""
    from paper_2402_06859_b200 import _lib as L
    lib = L.load()
    rows = np.array([1_000_000, 5000], dtype=np.int64)
    ft = np.array([0, 1, 0], dtype=np.int32)

    def plan(flags):
        cfg = L.EmbConfig(abi_version=L.EMB_ABI_VERSION, num_tables=2, table_rows=rows.ctypes.data_as(C.POINTER(C.c_int64)), dim=64,
                          num_features=3, feature_table=ft.ctypes.data_as(C.POINTER(C.c_int32)), pooling=0,
                          adagrad_mode=0, init_accumulator=0.1, eps=1e-7, max_norm=1.0, max_nnz=200_000,
                          max_batch=4096, sharding=0, table_owner=None, rank=0, world_size=1,
                          nccl_unique_id=None, stream=None, flags=flags, max_recv_nnz=0)
        s = L.EmbSizes()
        return lib.emb_plan(C.byref(cfg), C.byref(s)), s
    st, train = plan(L.EMB_F_Q8)
    st2, serve = plan(L.EMB_F_Q8 | L.EMB_F_Q8_ONLY)
    assert st == 0 and st2 == 0
    assert serve.weights_bytes == 0 and serve.accum_bytes == 0
    assert serve.q8_codes_bytes == train.q8_codes_bytes == 1_005_000 * 96
    assert serve.workspace_bytes < train.workspace_bytes / 4
    assert plan(L.EMB_F_Q8_ONLY)[0] == L.EMB_EINVAL  # needs EMB_F_Q8
    assert plan(L.EMB_F_Q8 | L.EMB_F_Q8_ONLY | L.EMB_F_REQUANT)[0] == L.EMB_EINVAL
