"""ctypes binding of liblirank_emb.so (include/lirank_emb.h).  Argument marshalling only.

There is no fallback: if the sm_100a library is missing or no CUDA device is present,
every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblirank_emb.so")

EMB_ABI_VERSION = 2
EMB_POOL_SUM, EMB_POOL_MEAN = 0, 1
EMB_ADAGRAD_ROWWISE, EMB_ADAGRAD_ELEMENTWISE = 0, 1
EMB_SHARD_NONE, EMB_SHARD_TABLE, EMB_SHARD_ROW = 0, 1, 2
EMB_F_Q8, EMB_F_REQUANT, EMB_F_LOOPBACK, EMB_F_EXCHANGE, EMB_F_Q8_MINMAX, EMB_F_Q8_ONLY, EMB_F_P2P, \
    EMB_F_HOSTCOMM = 1, 2, 4, 8, 16, 32, 64, 128
PHASES = ["fwd", "sort", "rle", "segreduce", "norm", "update", "fwd_q8", "quantize", "copy", "exchange"]

STATUS = {0: "EMB_OK", 1: "EMB_EINVAL", 2: "EMB_ENOMEM", 3: "EMB_ECUDA", 4: "EMB_ENCCL",
          5: "EMB_EIDRANGE", 6: "EMB_ENONFINITE", 7: "EMB_ESTATE"}
EMB_OK, EMB_EINVAL, EMB_ENOMEM, EMB_ECUDA, EMB_ENCCL, EMB_EIDRANGE, EMB_ENONFINITE, EMB_ESTATE = range(8)


class EmbError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)}")


class EmbConfig(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32),
        ("num_tables", C.c_int32),
        ("table_rows", C.POINTER(C.c_int64)),
        ("dim", C.c_int32),
        ("num_features", C.c_int32),
        ("feature_table", C.POINTER(C.c_int32)),
        ("pooling", C.c_int32),
        ("adagrad_mode", C.c_int32),
        ("init_accumulator", C.c_float),
        ("eps", C.c_float),
        ("max_norm", C.c_float),
        ("max_nnz", C.c_int64),
        ("max_batch", C.c_int32),
        ("sharding", C.c_int32),
        ("table_owner", C.POINTER(C.c_int32)),
        ("rank", C.c_int32),
        ("world_size", C.c_int32),
        ("nccl_unique_id", C.c_void_p),
        ("stream", C.c_void_p),
        ("flags", C.c_uint32),
        ("max_recv_nnz", C.c_int64),
        ("table_cost", C.POINTER(C.c_double)),
    ]


# int32 (*allgather)(void* ctx, const void* send, void* recv, int64 bytes)
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)


class EmbHostComm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", HOST_ALLGATHER)]


class EmbSizes(C.Structure):
    _fields_ = [
        ("weights_bytes", C.c_int64),
        ("accum_bytes", C.c_int64),
        ("q8_codes_bytes", C.c_int64),
        ("q8_meta_bytes", C.c_int64),
        ("workspace_bytes", C.c_int64),
        ("local_rows", C.c_int64),
        ("row_pitch", C.c_int32),
        ("q8_pitch", C.c_int32),
    ]


class EmbBuffers(C.Structure):
    _fields_ = [("weights", C.c_void_p), ("accum", C.c_void_p), ("q8_codes", C.c_void_p),
                ("q8_meta", C.c_void_p), ("workspace", C.c_void_p)]


# name -> (restype, argtypes); the exported symbol set of include/lirank_emb.h
P = C.c_void_p
SIGNATURES = {
    "emb_abi_version": (C.c_int32, []),
    "emb_status_string": (C.c_char_p, [C.c_int]),
    "emb_plan": (C.c_int, [P, P]),
    "emb_local_layout": (C.c_int, [P, P, P, P]),
    "emb_create": (C.c_int, [P, P, P]),
    "emb_forward": (C.c_int, [P, P, P, C.c_int32, C.c_int64, P]),
    "emb_backward_adagrad": (C.c_int, [P, P, C.c_float, C.c_double, P]),
    "emb_quantize_mm8": (C.c_int, [P]),
    "emb_forward_q8": (C.c_int, [P, P, P, C.c_int32, C.c_int64, P]),
    "emb_sync": (C.c_int, [P]),
    "emb_read_rows": (C.c_int, [P, C.c_int32, P, C.c_int64, P, P]),
    "emb_write_rows": (C.c_int, [P, C.c_int32, P, C.c_int64, P, P]),
    "emb_read_q8": (C.c_int, [P, C.c_int32, P, C.c_int64, P, P, P]),
    "emb_last_dedup": (C.c_int, [P, P, P, C.c_int64, P, C.c_int64, P, P]),
    "emb_last_stats": (C.c_int, [P, P, P, P]),
    "emb_kernel_launches": (C.c_int64, [P]),
    "emb_nccl_unique_id": (C.c_int, [P]),
    "emb_loopback_hub_create": (C.c_int, [C.c_int32, P]),
    "emb_loopback_hub_destroy": (C.c_int, [P]),
    "emb_profile": (C.c_int, [P, C.c_int32]),
    "emb_profile_read": (C.c_int, [P, P, P, C.c_int32]),
    "emb_destroy": (C.c_int, [P]),
    "emb_backward_adagrad_dev": (C.c_int, [P, P, C.c_float, P, P, P]),
    "emb_allreduce_f32": (C.c_int, [P, P, C.c_int64]),
    "emb_set_incremental": (C.c_int, [P, P, P, P, P, C.c_float, C.c_float]),
    "emb_quantize_block": (C.c_int, [P, C.c_int32, C.c_int64, C.c_int64, P, C.c_int64]),
    "emb_cold_weight_init": (C.c_int, [P, P, P, C.c_float]),
    "emb_hash_ids": (C.c_int, [P, P, C.c_int64, P, P]),
    "emb_qr_expand": (C.c_int, [P, P, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int32, P, P, P]),
    "emb_qr_rows": (C.c_int64, [C.c_int32, C.c_int64, C.c_int32]),
}

_lib = None


def load(build_if_missing: bool = True):
    """Load the sm_100a library (building it in-tree with nvcc if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from . import build as _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2402_06859_b200.build`")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.emb_abi_version() != EMB_ABI_VERSION:
        raise ImportError("liblirank_emb.so ABI version mismatch")
    _lib = lib
    return lib


def check(code, where):
    if code != EMB_OK:
        raise EmbError(code, where)
