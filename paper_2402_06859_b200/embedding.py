"""Thin Python front end of the C ABI: torch tensors supply device memory and streams.

Every step of the hot path runs in liblirank_emb.so; this module only allocates the
buffers emb_plan() asks for, passes pointers, and converts statuses to exceptions.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; every rank passes it to the constructor)."""
    lib = L.load()
    buf = C.create_string_buffer(128)
    L.check(lib.emb_nccl_unique_id(buf), "emb_nccl_unique_id")
    return buf.raw


class HostComm:
    """Test transport (EMB_F_HOSTCOMM): one rank per process -- e.g. several processes on one
    GPU -- with the library's collectives moved through host memory by a torch.distributed
    all-gather over `group` (gloo).  Keep this object alive as long as the handle."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)

        def _allgather(ctx, send, recv, nbytes):
            try:
                n = int(nbytes)
                src = torch.zeros(n, dtype=torch.uint8)
                if n:
                    C.memmove(src.data_ptr(), send, n)
                outs = [torch.empty(n, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(outs, src, group=self.group)
                if n:
                    for r, o in enumerate(outs):
                        C.memmove(recv + r * n, o.data_ptr(), n)
                return 0
            except Exception:  # pragma: no cover - reported to the library as a failure
                return 1

        self._cb = L.HOST_ALLGATHER(_allgather)
        self.struct = L.EmbHostComm(None, self._cb)
        self.ptr = C.cast(C.pointer(self.struct), C.c_void_p)


class LoopbackHub:
    """Test transport: W ranks as W threads of one process on one device (EMB_F_LOOPBACK)."""

    def __init__(self, world: int):
        self.lib = L.load()
        self.ptr = C.c_void_p()
        L.check(self.lib.emb_loopback_hub_create(int(world), C.byref(self.ptr)), "emb_loopback_hub_create")
        self.world = world

    def close(self):
        if self.ptr.value:
            self.lib.emb_loopback_hub_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _arr(a, ctype):
    a = np.ascontiguousarray(a)
    return a, a.ctypes.data_as(C.POINTER(ctype))


class ShardedEmbedding:
    """Embedding tables of the LiRank sparse path on one GPU (one shard when world_size > 1).

    Tables: ``table_rows[t]`` rows of width ``dim``; feature f reads table
    ``feature_table[f]``.  Inputs per call: feature-major ids [nnz] and offsets [F*B+1]
    (int32, CUDA or CPU-pinned tensors); output [B, F, dim] fp32.
    """

    def __init__(self, table_rows: Sequence[int], dim: int, feature_table: Sequence[int], *,
                 max_nnz: int, max_batch: int, pooling: str = "sum",
                 adagrad: str = "rowwise", init_accumulator: float = 0.1, eps: float = 1e-7,
                 max_norm: float = 1.0, q8: bool = False, requant: bool = False,
                 device: Optional[torch.device] = None, stream: Optional[torch.cuda.Stream] = None,
                 rank: int = 0, world_size: int = 1, sharding: str = "none",
                 table_owner: Optional[Sequence[int]] = None, nccl_unique_id: Optional[bytes] = None,
                 loopback_hub: Optional["LoopbackHub"] = None, force_exchange: bool = False,
                 max_recv_nnz: int = 0, q8_mode: str = "middle_max", q8_only: bool = False,
                 p2p: bool = False, guard_bytes: int = 0, table_cost: Optional[Sequence[float]] = None,
                 host_comm: Optional["HostComm"] = None):
        self.lib = L.load()
        assert q8_mode in ("middle_max", "min_max")
        self.q8_mode = q8_mode
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.dim = int(dim)
        self.num_features = len(feature_table)
        self.table_rows = [int(r) for r in table_rows]
        self._rows, rows_p = _arr(np.asarray(table_rows, dtype=np.int64), C.c_int64)
        self._ft, ft_p = _arr(np.asarray(feature_table, dtype=np.int32), C.c_int32)
        owner_p = None
        if table_owner is not None:
            self._owner, owner_p = _arr(np.asarray(table_owner, dtype=np.int32), C.c_int32)
        self._uid = None
        uid_ptr = None
        if nccl_unique_id is not None:
            self._uid = C.create_string_buffer(bytes(nccl_unique_id), len(nccl_unique_id))
            uid_ptr = C.cast(self._uid, C.c_void_p)
        self._hub = loopback_hub
        if loopback_hub is not None:
            uid_ptr = loopback_hub.ptr
        self._host_comm = host_comm
        if host_comm is not None:
            uid_ptr = host_comm.ptr
        cost_p = None
        if table_cost is not None:
            self._cost, cost_p = _arr(np.asarray(table_cost, dtype=np.float64), C.c_double)
        self.cfg = L.EmbConfig(
            abi_version=L.EMB_ABI_VERSION, num_tables=len(self.table_rows), table_rows=rows_p,
            dim=self.dim, num_features=self.num_features, feature_table=ft_p,
            pooling={"sum": L.EMB_POOL_SUM, "mean": L.EMB_POOL_MEAN}[pooling],
            adagrad_mode={"rowwise": L.EMB_ADAGRAD_ROWWISE, "elementwise": L.EMB_ADAGRAD_ELEMENTWISE}[adagrad],
            init_accumulator=init_accumulator, eps=eps, max_norm=max_norm,
            max_nnz=int(max_nnz), max_batch=int(max_batch),
            sharding={"none": L.EMB_SHARD_NONE, "table": L.EMB_SHARD_TABLE, "row": L.EMB_SHARD_ROW}[sharding],
            table_owner=owner_p, rank=rank, world_size=world_size,
            nccl_unique_id=uid_ptr,
            stream=C.c_void_p(self.stream.cuda_stream),
            flags=(L.EMB_F_Q8 if (q8 or requant or q8_only) else 0) | (L.EMB_F_REQUANT if requant else 0)
            | (L.EMB_F_Q8_ONLY if q8_only else 0)
            | (L.EMB_F_LOOPBACK if loopback_hub is not None else 0)
            | (L.EMB_F_EXCHANGE if force_exchange else 0)
            | (L.EMB_F_P2P if p2p else 0)
            | (L.EMB_F_Q8_MINMAX if q8_mode == "min_max" else 0)
            | (L.EMB_F_HOSTCOMM if host_comm is not None else 0),
            max_recv_nnz=int(max_recv_nnz), table_cost=cost_p)
        self.sizes = L.EmbSizes()
        L.check(self.lib.emb_plan(C.byref(self.cfg), C.byref(self.sizes)), "emb_plan")
        s = self.sizes
        nT = len(self.table_rows)
        self.local_base = np.zeros(nT, dtype=np.int64)
        self.row_lo = np.zeros(nT, dtype=np.int64)
        self.row_hi = np.zeros(nT, dtype=np.int64)
        L.check(self.lib.emb_local_layout(C.byref(self.cfg), self.local_base.ctypes.data_as(C.c_void_p),
                                          self.row_lo.ctypes.data_as(C.c_void_p),
                                          self.row_hi.ctypes.data_as(C.c_void_p)), "emb_local_layout")
        dev = self.device

        # guard_bytes > 0 (tests): every buffer gets a 0xA5-filled tail the library must never
        # touch (a write past a planned size shows up in guards_intact())
        self._guards = []

        def alloc(nbytes, dtype=torch.uint8):
            n = max(int(nbytes), 16)
            t = torch.empty(n + int(guard_bytes), dtype=torch.uint8, device=dev)
            if guard_bytes:
                t[n:].fill_(0xA5)
                self._guards.append((t, n))
            return t

        self.q8_only = bool(q8_only)  # serving handle: no fp32 tables (EMB_F_Q8_ONLY)
        self.weights_buf = alloc(s.weights_bytes) if s.weights_bytes else None
        self.accum_buf = alloc(s.accum_bytes) if s.accum_bytes else None
        self.workspace = alloc(s.workspace_bytes)
        self.codes_buf = alloc(s.q8_codes_bytes) if s.q8_codes_bytes else None
        self.meta_buf = alloc(s.q8_meta_bytes) if s.q8_meta_bytes else None
        self.local_rows = int(s.local_rows)
        self.pitch = int(s.row_pitch)
        self.q8_pitch = int(s.q8_pitch)
        bufs = L.EmbBuffers(_ptr(self.weights_buf), _ptr(self.accum_buf), _ptr(self.codes_buf),
                            _ptr(self.meta_buf), _ptr(self.workspace))
        self.h = C.c_void_p()
        L.check(self.lib.emb_create(C.byref(self.cfg), C.byref(bufs), C.byref(self.h)), "emb_create")

    def guards_intact(self) -> bool:
        torch.cuda.synchronize(self.device)
        return all(bool((t[n:] == 0xA5).all()) for t, n in self._guards)

    # ---- views -------------------------------------------------------------------------
    @property
    def weights(self) -> torch.Tensor:
        """fp32 [local_rows, row_pitch] view of the stored tables (device)."""
        n = self.local_rows * self.pitch
        return self.weights_buf[: 4 * n].view(torch.float32).view(self.local_rows, self.pitch)

    def quantize_block(self, table: int, row0: int, rows: torch.Tensor) -> None:
        """Quantize fp32 rows [row0, row0 + n) of `table` (device tensor [n, ld], ld % 4 == 0,
        ld >= dim) into the q8 store -- how a serving (q8_only) handle is filled."""
        assert rows.is_cuda and rows.dtype == torch.float32 and rows.dim() == 2 and rows.stride(1) == 1
        L.check(self.lib.emb_quantize_block(self.h, int(table), int(row0), int(rows.shape[0]), _ptr(rows),
                                            int(rows.stride(0))), "emb_quantize_block")

    def table_view(self, t: int) -> torch.Tensor:
        b = int(self.local_base[t])
        if b < 0:
            return self.weights[:0]
        return self.weights[b: b + int(self.row_hi[t] - self.row_lo[t])]

    # ---- hot path ----------------------------------------------------------------------
    def forward(self, ids: torch.Tensor, offsets: torch.Tensor, batch: int,
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty((batch, self.num_features, self.dim), dtype=torch.float32,
                              device=ids.device if ids.is_cuda else "cpu", pin_memory=not ids.is_cuda)
        _check_io(ids, offsets, out)
        L.check(self.lib.emb_forward(self.h, _ptr(ids), _ptr(offsets), int(batch), int(ids.numel()),
                                     _ptr(out)), "emb_forward")
        return out

    def set_incremental(self, w0: Optional[torch.Tensor], H0: Optional[torch.Tensor],
                        w1: Optional[torch.Tensor], H1: Optional[torch.Tensor], lambda_f: float,
                        alpha: float) -> None:
        """NEXT-3: diagonal-FIM penalty toward the cold-start (w0, H0) and prior (w1, H1) models
        on every later backward (tensors in the weights' layout: [local_rows, pitch] fp32, kept
        alive by this object)."""
        for t in (w0, H0, w1, H1):
            assert t is None or (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                                 and t.numel() == self.local_rows * self.pitch)
        self._fim_refs = (w0, H0, w1, H1)
        L.check(self.lib.emb_set_incremental(self.h, _ptr(w0), _ptr(H0), _ptr(w1), _ptr(H1), float(lambda_f),
                                             float(alpha)), "emb_set_incremental")

    def cold_weight_init(self, w0: torch.Tensor, w1: torch.Tensor, alpha: float) -> None:
        """NEXT-3: W = alpha w0 + (1 - alpha) w1, tensors in the weights' layout."""
        for t in (w0, w1):
            assert t.is_cuda and t.dtype == torch.float32 and t.numel() == self.local_rows * self.pitch
        L.check(self.lib.emb_cold_weight_init(self.h, _ptr(w0), _ptr(w1), float(alpha)), "emb_cold_weight_init")

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over the ranks of a device fp32 tensor, on the library's stream and
        transport (the data-parallel dense side of NEXT-2)."""
        assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
        L.check(self.lib.emb_allreduce_f32(self.h, _ptr(t), int(t.numel())), "emb_allreduce_f32")
        return t

    def backward_adagrad_dev(self, grad: torch.Tensor, lr: float,
                             extra_sq_norm: Optional[torch.Tensor] = None,
                             clip_out: Optional[torch.Tensor] = None,
                             sq_norm_out: Optional[torch.Tensor] = None) -> None:
        """a5-a8 with the dense side's squared norm read on the device (fp64 scalar tensor) and
        the clip factor / S written to device tensors: no host synchronisation (NEXT-2)."""
        assert grad.dtype == torch.float32 and grad.is_contiguous()
        for t, dt in ((extra_sq_norm, torch.float64), (clip_out, torch.float32), (sq_norm_out, torch.float64)):
            assert t is None or (t.is_cuda and t.dtype == dt and t.numel() == 1)
        L.check(self.lib.emb_backward_adagrad_dev(self.h, _ptr(grad), float(lr), _ptr(extra_sq_norm),
                                                  _ptr(clip_out), _ptr(sq_norm_out)), "emb_backward_adagrad_dev")

    def backward_adagrad(self, grad: torch.Tensor, lr: float, extra_sq_norm: float = 0.0,
                         want_norm: bool = False):
        assert grad.dtype == torch.float32 and grad.is_contiguous()
        if want_norm:
            S = C.c_double(0)
            L.check(self.lib.emb_backward_adagrad(self.h, _ptr(grad), float(lr), float(extra_sq_norm),
                                                  C.byref(S)), "emb_backward_adagrad")
            return S.value
        L.check(self.lib.emb_backward_adagrad(self.h, _ptr(grad), float(lr), float(extra_sq_norm), None),
                "emb_backward_adagrad")
        return None

    def quantize(self):
        L.check(self.lib.emb_quantize_mm8(self.h), "emb_quantize_mm8")

    def forward_q8(self, ids: Optional[torch.Tensor], offsets: Optional[torch.Tensor], batch: int,
                   out: Optional[torch.Tensor] = None, nnz: Optional[int] = None) -> torch.Tensor:
        """a10.  ids = offsets = None: the batch of the last forward() (its staged copy when it
        came from host memory; pass nnz = its id count)."""
        if ids is None and offsets is None:
            assert out is not None and nnz is not None
            assert out.dtype == torch.float32 and out.is_contiguous()
            L.check(self.lib.emb_forward_q8(self.h, None, None, int(batch), int(nnz), _ptr(out)), "emb_forward_q8")
            return out
        if out is None:
            out = torch.empty((batch, self.num_features, self.dim), dtype=torch.float32,
                              device=ids.device if ids.is_cuda else "cpu", pin_memory=not ids.is_cuda)
        _check_io(ids, offsets, out)
        L.check(self.lib.emb_forward_q8(self.h, _ptr(ids), _ptr(offsets), int(batch), int(ids.numel()),
                                        _ptr(out)), "emb_forward_q8")
        return out

    def sync(self, raise_on_error: bool = False) -> int:
        code = self.lib.emb_sync(self.h)
        if raise_on_error:
            L.check(code, "emb_sync")
        return code

    # ---- introspection -----------------------------------------------------------------
    def read_rows(self, table: int, rows, with_acc: bool = True):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        w = np.zeros((len(rows), self.dim), dtype=np.float32)
        acc = None
        if with_acc:
            acc = np.zeros((len(rows),) if self.cfg.adagrad_mode == L.EMB_ADAGRAD_ROWWISE
                           else (len(rows), self.dim), dtype=np.float32)
        L.check(self.lib.emb_read_rows(self.h, int(table), rows.ctypes.data_as(C.c_void_p), len(rows),
                                       w.ctypes.data_as(C.c_void_p),
                                       acc.ctypes.data_as(C.c_void_p) if acc is not None else None),
                "emb_read_rows")
        return (w, acc) if with_acc else w

    def write_rows(self, table: int, rows, w=None, acc=None):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        wp = None if w is None else np.ascontiguousarray(w, dtype=np.float32)
        ap = None if acc is None else np.ascontiguousarray(acc, dtype=np.float32)
        L.check(self.lib.emb_write_rows(self.h, int(table), rows.ctypes.data_as(C.c_void_p), len(rows),
                                        None if wp is None else wp.ctypes.data_as(C.c_void_p),
                                        None if ap is None else ap.ctypes.data_as(C.c_void_p)),
                "emb_write_rows")

    def read_q8(self, table: int, rows):
        """(codes, base, scale): int8 codes + middle (middle-max) or uint8 codes + min (min-max)."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        codes = np.zeros((len(rows), self.dim), dtype=np.uint8 if self.q8_mode == "min_max" else np.int8)
        mid = np.zeros(len(rows), dtype=np.float32)
        sc = np.zeros(len(rows), dtype=np.float32)
        L.check(self.lib.emb_read_q8(self.h, int(table), rows.ctypes.data_as(C.c_void_p), len(rows),
                                     codes.ctypes.data_as(C.c_void_p), mid.ctypes.data_as(C.c_void_p),
                                     sc.ctypes.data_as(C.c_void_p)), "emb_read_q8")
        return codes, mid, sc

    def last_dedup(self, with_bags: bool = True):
        U = C.c_int64(0)
        nv = C.c_int64(0)
        L.check(self.lib.emb_last_dedup(self.h, None, None, 0, None, 0, C.byref(U), C.byref(nv)),
                "emb_last_dedup")
        uniq = np.zeros(max(U.value, 1), dtype=np.int32)
        seg = np.zeros(U.value + 1, dtype=np.int32)
        bags = np.zeros(max(nv.value, 1), dtype=np.int32) if with_bags else None
        L.check(self.lib.emb_last_dedup(self.h, uniq.ctypes.data_as(C.c_void_p), seg.ctypes.data_as(C.c_void_p),
                                        len(uniq), None if bags is None else bags.ctypes.data_as(C.c_void_p),
                                        0 if bags is None else len(bags), C.byref(U), C.byref(nv)),
                "emb_last_dedup")
        return uniq[:U.value], seg, (bags[:nv.value] if bags is not None else None)

    def last_stats(self):
        S = C.c_double(0)
        c = C.c_float(0)
        U = C.c_int64(0)
        L.check(self.lib.emb_last_stats(self.h, C.byref(S), C.byref(c), C.byref(U)), "emb_last_stats")
        return S.value, np.float32(c.value), U.value

    @property
    def launches(self) -> int:
        return int(self.lib.emb_kernel_launches(self.h))

    def profile(self, enable: bool = True):
        L.check(self.lib.emb_profile(self.h, 1 if enable else 0), "emb_profile")

    def profile_read(self, reset: bool = False):
        """{phase: (total ms, instances)} accumulated from the library's CUDA events."""
        ms = np.zeros(len(L.PHASES), dtype=np.float64)
        n = np.zeros(len(L.PHASES), dtype=np.int64)
        L.check(self.lib.emb_profile_read(self.h, ms.ctypes.data_as(C.c_void_p), n.ctypes.data_as(C.c_void_p),
                                          1 if reset else 0), "emb_profile_read")
        return {p: (float(ms[i]), int(n[i])) for i, p in enumerate(L.PHASES)}

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            # the library's kernels may still use the buffers this object owns (torch tensors
            # whose memory the caching allocator would hand out again): drain the stream first
            try:
                self.stream.synchronize()
            except Exception:
                pass
            self.lib.emb_destroy(self.h)  # also drains the library's side stream
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_io(ids, offsets, out):
    assert ids.dtype == torch.int32 and offsets.dtype == torch.int32 and out.dtype == torch.float32
    assert ids.is_contiguous() and offsets.is_contiguous() and out.is_contiguous()
