#!/usr/bin/env python
"""Benchmark of the LiRank sparse-embedding hot path on B200 (BASELINE.json metric:
"pooled lookups/s and train samples/s at 1/2/4/8 B200; % HBM roofline").

One step = the whole hot path over one batch: a2 fp32 pooled lookup
-> a5 dedup -> a6 segment-reduce -> a7 global norm/clip -> a8 clip+row-wise AdaGrad with
a9 re-quantization of every updated row fused in -> a10 q8 pooled lookup of the same
batch from the refreshed int8 store.  The full-table a9 pass is timed separately
(`quantize_full`).  Workload at N=1: Feed-1 (the north_star's
"1-GPU Feed-shaped config"), synthetic Zipf(1.05) ids, seeded tables.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config feed1] [--impl reference]

Under torchrun (N>1) every rank runs; timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from workload import configs, gen  # noqa: E402

METRIC = "pooled lookups/s and train samples/s at 1/2/4/8 B200; % HBM roofline"
LR = 0.05


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="feed1")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--batches", type=int, default=3, help="distinct resident batches, rotated")
    ap.add_argument("--adagrad", default="rowwise", choices=["rowwise", "elementwise"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-qr", action="store_true", help="skip the NEXT-1 QR/Murmur section")
    ap.add_argument("--no-model", action="store_true", help="skip the NEXT-2 end-to-end model section")
    ap.add_argument("--dense-features", type=int, default=256, help="NEXT-2 dense feature count")
    ap.add_argument("--exchange", action="store_true",
                    help="N=1: run the sharded exchange path on a 1-rank NCCL communicator (its overhead)")
    ap.add_argument("--sharding", default=None, choices=["row", "table"],
                    help="sharding for N>1 / --exchange (default: row for the Feed tables, table otherwise)")
    ap.add_argument("--weak", action="store_true",
                    help="N>1: weak scaling (batch per GPU fixed, Feed tables x N) instead of the default "
                         "strong scaling of BASELINE's global batch")
    ap.add_argument("--exchange-mode", default="p2p", choices=["p2p", "nccl"],
                    help="sharded: p2p = fused exchange over NVLink peer memory (EMB_F_P2P; falls back to "
                         "nccl on every rank if any rank cannot map its peers), nccl = collectives")
    ap.add_argument("--no-fim", action="store_true", help="skip the NEXT-3 incremental-training section")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay section")
    ap.add_argument("--no-lib", action="store_true", help="skip the library (torch embedding_bag) baseline")
    ap.add_argument("--serve", action="store_true",
                    help="serving bench: q8-only handle, a10 lookups only (default for --config feedq8)")
    ap.add_argument("--q8-mode", default="middle_max", choices=["middle_max", "min_max"],
                    help="q8 store: the paper's middle-max (default) or NEXT-4's min-max")
    ap.add_argument("--cpu-samples", type=int, default=8192,
                    help="samples of the single-core oracle timing (the all-core one runs the full batch)")
    ap.add_argument("--no-spot", action="store_true", help="skip the in-run oracle spot check")
    ap.add_argument("--no-a5", action="store_true", help="skip the a5-alone timing (launch lists: every step the same)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="N>1: NCCL (one GPU per rank), or the library's host transport over a gloo group "
                         "(EMB_F_HOSTCOMM: a functional check of the N-rank bench with every rank on the "
                         "same GPU; times are not NVLink numbers)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# algorithmic bytes per unit
# ---------------------------------------------------------------------------

def alg_bytes(phase, cfg, nnz, U, B, pitch, mode="rowwise"):
    D = cfg.dim
    F = cfg.num_features
    row = 4 * pitch
    if phase == "fwd":       # per id: 4 B id + one fp32 row; per bag: 4 B offset + 4D B output
        return nnz * (4 + row) + B * F * (4 + 4 * D)
    if phase == "fwd_q8":    # per id: 4 B id + D B codes + 8 B (middle, scale); per bag as fwd
        return nnz * (4 + D + 8) + B * F * (4 + 4 * D)
    if phase == "segreduce":  # per id: 4 B key + 4 B bag + one grad row; per unique: G row write
        return nnz * (8 + 4 * D) + U * row
    if phase == "update":    # per unique: G read + w read/write + A (+ key); + requant 72 B out
        acc = 8 if mode == "rowwise" else 2 * row
        return U * (row + 2 * row + acc + 4 + (D + 8))
    return None


def impl_bytes(phase, nnz, U, passes):
    """a5 is implementation overhead, not algorithmic bytes: its own traffic
    is one histogram read of the 8-B {key, grad row} pairs + 16 B per pair per onesweep pass
    (read + write); the run-length encode reads the keys (8 B/pair incl. the neighbour's, L1-
    served) and writes unique + segment offsets (8 B/unique)."""
    if phase == "sort":
        return nnz * (8 + 16 * passes)
    if phase == "rle":
        return nnz * 8 + U * 8
    return None


def compulsory_bytes(phase, cfg, nnz, U, B, pitch, mode="rowwise"):
    """Each row touched ONCE (SURVEY.md §8(d) "compulsory"): the U unique rows of the batch
    instead of one row per occurrence; the bag's gradient row once instead of once per id."""
    D, F = cfg.dim, cfg.num_features
    row = 4 * pitch
    if phase == "fwd":
        return nnz * 4 + U * row + B * F * (4 + 4 * D)
    if phase == "fwd_q8":
        return nnz * 4 + U * (D + 8) + B * F * (4 + 4 * D)
    if phase == "segreduce":
        return nnz * 8 + B * F * 4 * D + U * row
    return None


# ---------------------------------------------------------------------------
# clocks during the timed region (pynvml)
# ---------------------------------------------------------------------------

REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
           0x2: "applications_clocks_setting", 0x10: "sync_boost"}


class ClockSampler(threading.Thread):
    def __init__(self, index):
        super().__init__(daemon=True)
        self.index = index
        self.samples = []
        self.reasons = 0
        self.stop_ev = threading.Event()
        self.max_mhz = None
        self.ok = False
        self.ready = threading.Event()

    def run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            first = True
            while not self.stop_ev.is_set() or first:
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                try:
                    self.reasons |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    self.reasons |= pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                if first:
                    first = False
                    self.ready.set()
                time.sleep(0.005)
        except Exception as e:  # no NVML: report that
            self.err = repr(e)
        self.ready.set()

    def begin(self):
        """Start sampling and return once NVML is up (so the timed region is covered)."""
        self.start()
        self.ready.wait(timeout=30)
        self.samples.clear()
        self.reasons = 0
        return self

    def result(self):
        self.stop_ev.set()
        self.join(timeout=2)
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(n for b, n in REASONS.items() if self.reasons & b and b != 0x1),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU oracle on a bounded sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------

class OracleSample:
    """The oracle's whole step (a2, a5-a8, a9 on the touched rows, a10) on the first
    `samples` samples of batch 0 (all of them: samples=None), over the compact table of the
    rows they touch (the Feed tables' 32 GB do not fit host RAM; the touched rows do)."""

    def __init__(self, cfg, ids, off, B, samples, mode, gshift=None, sample0=0):
        import oracle as O
        self.O = O
        F = cfg.num_features
        Bs = B if samples is None else min(samples, B)
        off64 = off.astype(np.int64)
        sub_ids, lens = [], []
        for f in range(F):
            a, b = off64[f * B], off64[f * B + Bs]
            sub_ids.append(ids[a:b])
            lens.append(np.diff(off64[f * B:f * B + Bs + 1]))
        sids = np.concatenate(sub_ids)
        soff = np.zeros(F * Bs + 1, dtype=np.int64)
        soff[1:] = np.cumsum(np.concatenate(lens))
        base = np.concatenate([[0], np.cumsum(cfg.table_rows)]).astype(np.int64)
        bag_of = np.repeat(np.arange(F * Bs), np.diff(soff))
        t = np.asarray(cfg.feature_table, dtype=np.int64)[bag_of // Bs]
        gkey = base[t] + sids.astype(np.int64)
        keys = np.unique(gkey)
        self.keys = keys
        self.base = base
        self.cids = np.searchsorted(keys, gkey).astype(np.int32)
        tk = np.searchsorted(base, keys, side="right") - 1
        W = np.zeros((len(keys), cfg.dim), dtype=np.float32)
        for tt in np.unique(tk):
            m = tk == tt
            W[m] = gen.table_rows(cfg.seed, int(tt), keys[m] - base[tt], cfg.dim)
        self.W0 = W
        self.soff = soff.astype(np.int32)
        self.Bs = Bs
        self.nnz = len(sids)
        self.pb = O.Problem([len(keys)], cfg.dim, [0] * F)
        gshift = gen.grad_shift_for(len(ids), cfg.dim) if gshift is None else gshift
        self.grad = gen.grad_values(cfg.seed, 0, Bs, F, cfg.dim, gshift, sample0=sample0)
        self.mode = mode
        self.reset()

    def reset(self):
        self.W = self.W0.copy()
        shape = (len(self.W),) if self.mode == "rowwise" else self.W.shape
        self.A = np.full(shape, 0.1, dtype=np.float32)

    def step(self):
        O = self.O
        r = O.train_step(self.pb, self.W, self.A, self.cids, self.soff, self.Bs, self.grad, LR, 1e-7, 1.0,
                         mode=self.mode)
        codes, mid, sc, _ = O.quantize(self.W)  # a9 of the touched rows (every row here is touched)
        O.forward_q8(self.pb, codes, mid, sc, self.cids, self.soff, self.Bs)
        return r

    def time(self, steps, warmup=0):
        for _ in range(warmup):
            self.step()
        t0 = time.perf_counter()
        for _ in range(steps):
            self.step()
        return (time.perf_counter() - t0) / max(steps, 1)


def host_info():
    """CPU model, logical cores and RAM of this host (for the oracle timings)."""
    model, ram = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except Exception:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "ram_gib": ram}


def cpu_baseline(cfg, ids, off, B, samples, mode, budget_s=15.0):
    """The oracle as it stands, on this host: the OpenMP build (liboracle_omp.so, bit-identical
    to the sequential one) on ALL cores over the FULL batch 0, and the sequential build on one
    core over its first `samples` samples."""
    import oracle as O
    cores = O.set_parallel(True, threads=os.cpu_count() or 1)
    try:
        full = OracleSample(cfg, ids, off, B, None, mode)
        t1 = full.time(1)
        reps = max(1, min(5, int(budget_s / max(t1, 1e-3))))
        t = full.time(reps)
    finally:
        O.set_parallel(False)
    one = OracleSample(cfg, ids, off, B, samples, mode)
    t1s = one.time(1)
    reps1 = max(1, int(0.5 * budget_s / max(t1s, 1e-3)))
    ts = one.time(reps1)
    res = {"value": full.Bs / t, "unit": "samples/s", "cores": cores, "kind": "oracle",
           "sample": f"the full batch 0 ({full.Bs} samples, {full.nnz} ids), whole step (a2, a5-a8, a9 on the "
                     f"touched rows, a10) over the {len(full.W)} touched rows (compact table), OpenMP C oracle "
                     f"on {cores} threads, {reps + 1} reps",
           "single_core": {"value": one.Bs / ts, "unit": "samples/s", "cores": 1,
                           "sample": f"{one.Bs} of {B} samples of batch 0 ({one.nnz} ids), sequential C oracle, "
                                     f"{reps1 + 1} reps"}}
    res.update(host_info())
    return res


# ---------------------------------------------------------------------------
# reference arm: the oracle, as it stands, on the host cores
# ---------------------------------------------------------------------------

def run_reference(args, cfg, rank, world, serve=False):
    if rank != 0:
        return
    B = cfg.batch
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed, 0, alpha=cfg.alpha)
    if serve:  # the serving arm's metric: the oracle's a10 on the full batch, all host cores
        r = serving_cpu_baseline(cfg, ids, off, B, args.cpu_samples, args.q8_mode,
                                 budget_s=max(1.0, 0.5 * args.steps))
        value = r["value"]
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * B / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8 codes, f32 accumulate",
            "data": "synthetic",
            "config": {"workload": cfg.name, "global_batch": B, "alpha": cfg.alpha, "parallelism": "cpu-oracle"},
            "cpu_baseline": r,
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    import oracle as O
    cores = O.set_parallel(True, threads=os.cpu_count() or 1)
    smp = OracleSample(cfg, ids, off, B, None, args.adagrad)
    t = smp.time(args.steps, args.warmup)
    O.set_parallel(False)
    value = smp.Bs / t
    cb = {"value": value, "unit": "samples/s", "cores": cores, "kind": "oracle",
          "sample": f"the full batch 0 ({smp.Bs} samples, {smp.nnz} ids) per step, whole step (a2, a5-a8, a9 "
                    f"on the touched rows, a10) over the {len(smp.W)} touched rows, OpenMP C oracle on "
                    f"{cores} threads"}
    cb.update(host_info())
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "global_batch": B, "alpha": cfg.alpha, "parallelism": "cpu-oracle"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# NEXT-1 section: unlimited-dictionary ids (hash -> QR expand -> train step on QR tables)
# ---------------------------------------------------------------------------

def id_strings(ids, prefix: bytes):
    """UTF-8 bytes of prefix + decimal(id) for every id (vectorised) + int64 offsets."""
    ids = np.asarray(ids, dtype=np.int64)
    n = len(ids)
    nd = 1 + sum((ids >= 10 ** k).astype(np.int64) for k in range(1, 10))
    maxd = int(nd.max()) if n else 1
    digits = np.zeros((n, maxd), dtype=np.uint8)
    x = ids.copy()
    for j in range(maxd - 1, -1, -1):
        digits[:, j] = 48 + x % 10
        x //= 10
    pre = np.frombuffer(prefix, dtype=np.uint8)
    mat = np.concatenate([np.broadcast_to(pre, (n, len(pre))), digits], axis=1)
    keep = np.concatenate([np.ones((n, len(pre)), bool), np.arange(maxd)[None, :] >= (maxd - nd)[:, None]], axis=1)
    lens = len(pre) + nd
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    return mat[keep], off


def qr_section(cfg, ids, off, B, dev, stream, flush, hbm_peak, reps=5):
    """Feed-1 ids as strings ("member:<id>", "hashtag:<id>") -> emb_hash_ids -> emb_qr_expand
    (dual, R = 1000, Q = ceil(2^32 / R): P:335's 1000x example) -> a2 + a5-a8 on the QR tables.
    CUDA events on the library stream, L2 flushed before each repetition."""
    import torch

    from paper_2402_06859_b200 import ShardedEmbedding, qr
    from workload import gpu as G
    R = 1000
    Q = -(-(1 << 32) // R)
    F, D = cfg.num_features, cfg.dim
    prefixes = [b"member:", b"hashtag:"] + [b"t%d:" % t for t in range(2, cfg.num_tables)]
    datas, offs, base = [], [np.zeros(1, np.int64)], 0
    for f in range(F):
        a, b = off[f * B], off[(f + 1) * B]
        d, o = id_strings(ids[a:b], prefixes[cfg.feature_table[f]])
        datas.append(d)
        offs.append(o[1:] + base)
        base += int(o[-1])
    data = torch.from_numpy(np.concatenate(datas)).to(dev)
    soff = torch.from_numpy(np.concatenate(offs)).to(dev)
    offd = torch.from_numpy(off).to(dev)
    nnz = len(ids)
    h = torch.empty(nnz, dtype=torch.int64, device=dev)
    ids_x = torch.empty(4 * nnz, dtype=torch.int32, device=dev)
    off_x = torch.empty(F * B + 1, dtype=torch.int32, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]

    def timed(fn):
        # a ~0.5 ms device spin before the start event keeps the GPU busy while the host
        # enqueues the calls, so host launch overhead is not inside the events
        ts = []
        for _ in range(reps):
            G.flush_l2(flush, stream=stream)
            with torch.cuda.stream(stream):
                torch.cuda._sleep(1_000_000)
                ev[0][0].record(stream)
                fn()
                ev[0][1].record(stream)
            stream.synchronize()
            ts.append(ev[0][0].elapsed_time(ev[0][1]))
        return float(np.median(ts))

    with torch.cuda.stream(stream):
        hash_ms = timed(lambda: qr.hash_ids(data, soff, out=h))
        exp_ms = timed(lambda: qr.qr_expand(h, offd, R, Q, True, ids_out=ids_x, offsets_out=off_x))
    rows = [qr.qr_rows(R, Q, True)] * cfg.num_tables
    emb = ShardedEmbedding(rows, D, cfg.feature_table, max_nnz=4 * nnz, max_batch=B, device=dev, stream=stream)
    with torch.cuda.stream(stream):
        for t in range(cfg.num_tables):
            v = emb.table_view(t)
            G.fill_table(v, v.shape[0], D, emb.pitch, cfg.seed, t, stream=stream)
        gd = torch.empty((B, F, D), device=dev)
        G.fill_grad(gd, B, F, D, cfg.seed, 0, gen.grad_shift_for(4 * nnz, D), stream=stream)
        out = torch.empty((B, F, D), device=dev)
    for _ in range(3):
        emb.forward(ids_x, off_x, B, out=out)
        emb.backward_adagrad(gd, LR)
    stream.synchronize()
    emb.profile(True)
    emb.profile_read(reset=True)
    step_ms = timed(lambda: (emb.forward(ids_x, off_x, B, out=out), emb.backward_adagrad(gd, LR)))
    ph = emb.profile_read()
    emb.profile(False)
    assert emb.sync() == 0
    fwd_ms = ph["fwd"][0] / max(ph["fwd"][1], 1)
    _, _, U = emb.last_stats()
    sbytes = int(soff[-1].item())
    hash_b = sbytes + 8 * (nnz + 1) + 8 * nnz
    exp_b = 8 * nnz + 16 * nnz + 8 * (F * B + 1)
    res = {
        "what": "Feed-1 batch 0 ids as strings -> emb_hash_ids (MurmurHash3 x64-128) -> emb_qr_expand "
                "(dual, R=1000, Q=ceil(2^32/R)) -> a2 + a5-a8 on the two QR tables (4 rows per id)",
        "strings": nnz, "string_bytes": sbytes, "qr_rows_per_table": rows[0], "unique_rows": U,
        "hash_ms": hash_ms, "hash_strings_per_s": nnz / (hash_ms / 1e3),
        "hash_gbs": hash_b / (hash_ms / 1e3) / 1e9, "hash_frac_of_hbm": hash_b / (hash_ms / 1e3) / 1e9 / hbm_peak,
        "expand_ms": exp_ms, "expand_ids_per_s": nnz / (exp_ms / 1e3),
        "expand_gbs": exp_b / (exp_ms / 1e3) / 1e9, "expand_frac_of_hbm": exp_b / (exp_ms / 1e3) / 1e9 / hbm_peak,
        "train_step_ms": step_ms, "train_samples_per_s": B / (step_ms / 1e3), "fwd_ms": fwd_ms,
        "qr_lookups_per_s": 4 * nnz / (fwd_ms / 1e3),
    }
    del emb
    return res


# ---------------------------------------------------------------------------
# NEXT-2 section: the end-to-end Feed train step (embedding + MLP tower, one global clip)
# ---------------------------------------------------------------------------

def graph_section(emb, cfg, dev_in, B, out, out_q8, stream, flush, steps=10, small_batch=4096):
    """The W = 1 step captured once per resident batch as a CUDA graph and replayed (the step has
    no host synchronisation and its look-back epochs live in device memory), at the full batch
    (L2 flushed between replays, as the main line) and at a small batch where host launch cost
    matters (no flush: latency)."""
    import torch
    from workload import gpu as G

    def step(ids_d, off_d, g, b, o, oq):
        emb.forward(ids_d, off_d, b, out=o)
        emb.forward_q8(None, None, b, out=oq, nnz=ids_d.numel())  # the same batch, as the main step
        emb.backward_adagrad(g, LR)

    def timed(fn, n, flush_between):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        torch.cuda.synchronize()
        for k in range(n):
            if flush_between:
                G.flush_l2(flush, stream=stream)
            with torch.cuda.stream(stream):
                evs[k][0].record(stream)
                fn(k)
                evs[k][1].record(stream)
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b_) for a, b_ in evs]))

    res = {"what": "whole W=1 step (a2, a10, a5-a8 + requant) as one CUDA graph per batch, replayed"}
    graphs = []
    for (ids_d, off_d, g) in dev_in:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            step(ids_d, off_d, g, B, out, out_q8)
        graphs.append(gr)
    res["full_ms_per_step_graph"] = timed(lambda k: graphs[k % len(graphs)].replay(), steps, True)
    # small batch: latency, host launch cost visible
    ids, off = gen.make_batch(cfg.table_rows, cfg.features, small_batch, cfg.seed + 1, 0, alpha=cfg.alpha)
    F, D = cfg.num_features, cfg.dim
    ids_d, off_d = torch.from_numpy(ids).cuda(), torch.from_numpy(off).cuda()
    gs = torch.empty((small_batch, F, D), device=out.device)
    G.fill_grad(gs, small_batch, F, D, cfg.seed, 1, gen.grad_shift_for(len(ids), D), stream=stream)
    o_s, oq_s = torch.empty_like(gs), torch.empty_like(gs)
    for _ in range(3):
        with torch.cuda.stream(stream):
            step(ids_d, off_d, gs, small_batch, o_s, oq_s)
    res["small_batch"] = small_batch
    res["small_ms_per_step_eager"] = timed(lambda k: step(ids_d, off_d, gs, small_batch, o_s, oq_s), 3 * steps, False)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        step(ids_d, off_d, gs, small_batch, o_s, oq_s)
    res["small_ms_per_step_graph"] = timed(lambda k: gr.replay(), 3 * steps, False)
    assert emb.sync() == 0
    return res


def library_section(emb, cfg, dev_in, B, stream, flush, steps=10):
    """Library baseline beside a2 on the same tables and batches: torch.nn.functional.embedding_bag
    (PyTorch's CUDA kernel, mode='sum') over the stored tables with the same global row keys and
    offsets (feature-major bags; its output is [F*B, D] instead of [B, F, D])."""
    import torch
    import torch.nn.functional as Fn
    from workload import gpu as G
    D, F = cfg.dim, cfg.num_features
    W = emb.weights[:, :D] if emb.pitch != D else emb.weights
    inputs = []
    for (ids_d, off_d, _) in dev_in:
        base = torch.tensor([int(emb.local_base[cfg.feature_table[f]]) for f in range(F)], dtype=torch.int64,
                            device=ids_d.device)
        counts = (off_d[1:] - off_d[:-1]).view(F, B).sum(1)
        keys = (ids_d.to(torch.int64) + torch.repeat_interleave(base, counts.to(torch.int64))).contiguous()
        inputs.append((keys, off_d[:-1].to(torch.int64).contiguous()))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for keys, offs in inputs:  # warm-up: first-call allocations and module loading
            Fn.embedding_bag(keys, W, offs, mode="sum")
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for k in range(steps):
            keys, offs = inputs[k % len(inputs)]
            G.flush_l2(flush, stream=stream)
            evs[k][0].record(stream)
            out = Fn.embedding_bag(keys, W, offs, mode="sum")
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b_) for a, b_ in evs]))
    return {"what": "torch.nn.functional.embedding_bag(mode='sum') on the same tables / bags (a2's work)",
            "torch_embedding_bag_ms": ms, "rows_out": int(out.shape[0])}


def model_section(emb, batches, dev_in, B, dense_dim, stream, flush, steps=10, warmup=3):
    """FeedModel (paper_2402_06859_b200/feed_model.py) on the bench's Feed-1 tables: pooled
    embeddings ++ dense features -> 4 x 100 MLP, BCE loss, AdaGrad on sparse + dense
    under one global clip.  Steps issued back to back; CUDA events on the library
    stream; L2 not flushed between steps (whole-model throughput)."""
    import torch

    from paper_2402_06859_b200.feed_model import FeedModel
    torch.backends.cuda.matmul.allow_tf32 = False
    model = FeedModel(emb, dense_dim, lr=LR, seed=1)
    g = torch.Generator(device=emb.device).manual_seed(5)
    with torch.cuda.stream(stream):
        xs = [torch.randn(B, dense_dim, device=emb.device, generator=g) for _ in dev_in]
        ys = [(torch.rand(B, device=emb.device, generator=g) > 0.5).float() for _ in dev_in]
    for k in range(warmup):
        ids_d, off_d, _ = dev_in[k % len(dev_in)]
        model.train_step(ids_d, off_d, B, xs[k % len(xs)], ys[k % len(ys)])
    stream.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        torch.cuda._sleep(1_000_000)
        t0.record(stream)
    for k in range(steps):
        ids_d, off_d, _ = dev_in[k % len(dev_in)]
        loss = model.train_step(ids_d, off_d, B, xs[k % len(xs)], ys[k % len(ys)])
    with torch.cuda.stream(stream):
        t1.record(stream)
    stream.synchronize()
    ms = t0.elapsed_time(t1) / steps
    assert emb.sync() == 0
    tower = sum(p.numel() for p in model.params)
    return {"what": "Feed-1 tables + %d dense features -> MLP 4 x 100 -> BCE; AdaGrad sparse + dense, "
                    "one global clip (emb_backward_adagrad_dev, no host sync)" % dense_dim,
            "ms_per_step": ms, "train_samples_per_s": B / (ms / 1e3), "tower_params": tower,
            "loss_last": float(loss), "clip_last": float(model.c), "steps": steps, "warmup": warmup,
            "tf32": False}


# ---------------------------------------------------------------------------
# NEXT-3 section: incremental training (FIM penalty on touched rows, cold-weight init)
# ---------------------------------------------------------------------------

def fim_section(emb, dev_in, B, stream, flush, hbm_peak, steps=10, warmup=3):
    """Eq. (2) (alpha = 0: the prior-model anchor w1 = w_{t-1} with its FIM diagonal H1) on
    the Feed-1 tables -- the anchors of Eq. (3)'s cold-start term would need 2 more copies of
    the 32 GB table -- and the cold-weight init as a full-table streaming pass."""
    import torch

    from workload import gpu as G
    n = emb.local_rows * emb.pitch
    with torch.cuda.stream(stream):
        base = emb.weights_buf[: 4 * n].view(torch.float32).view(emb.local_rows, emb.pitch)
        w1 = base.clone()
        H1 = torch.rand_like(w1)
    stream.synchronize()

    def run(k0):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(warmup):
            ids_d, off_d, gd = dev_in[k % len(dev_in)]
            emb.forward(ids_d, off_d, B)
            emb.backward_adagrad(gd, LR)
        stream.synchronize()
        emb.profile(True)
        emb.profile_read(reset=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(1_000_000)
            t0.record(stream)
        for k in range(steps):
            ids_d, off_d, gd = dev_in[k % len(dev_in)]
            emb.forward(ids_d, off_d, B)
            emb.backward_adagrad(gd, LR)
        with torch.cuda.stream(stream):
            t1.record(stream)
        stream.synchronize()
        ph = emb.profile_read()
        emb.profile(False)
        assert emb.sync() == 0
        return t0.elapsed_time(t1) / steps, ph["norm"][0] / max(ph["norm"][1], 1)

    plain_ms, plain_norm = run(0)
    emb.set_incremental(None, None, w1, H1, 1e-3, 0.0)
    fim_ms, fim_norm = run(1)
    emb.set_incremental(None, None, None, None, 0.0, 0.0)
    _, _, U = emb.last_stats()
    ts = []
    for _ in range(3):
        G.flush_l2(flush, stream=stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            emb.cold_weight_init(w1, H1, 0.5)
            e1.record(stream)
        stream.synchronize()
        ts.append(e0.elapsed_time(e1))
    ci_ms = float(np.median(ts))
    ci_b = 3 * 4 * n
    pen_b = U * 4 * (3 * emb.pitch) + U * 4 * (2 * emb.pitch)  # G r/w, W, w1, H1 per touched row
    del w1, H1
    torch.cuda.empty_cache()
    return {"what": "Feed-1 fwd + bwd with the Eq. (2) penalty (w1 = prior model, H1 = its FIM diagonal, "
                    "lambda 1e-3) on the touched rows; cold-weight init over the 125M-row table",
            "step_ms_plain": plain_ms, "step_ms_fim": fim_ms, "unique_rows": U,
            "penalty_ms": fim_norm - plain_norm, "penalty_alg_bytes": pen_b,
            "penalty_gbs": pen_b / max(fim_norm - plain_norm, 1e-9) * 1e3 / 1e9,
            "cold_init_ms": ci_ms, "cold_init_gbs": ci_b / (ci_ms / 1e3) / 1e9,
            "cold_init_frac_of_hbm": ci_b / (ci_ms / 1e3) / 1e9 / hbm_peak}


# ---------------------------------------------------------------------------
# serving arm: the Feed-shaped inference config (q8 store only, a10 lookups)
# ---------------------------------------------------------------------------

def serving_cpu_baseline(cfg, ids, off, B, samples, q8_mode, budget_s=10.0):
    """The oracle's a10 (as it stands) on ALL host cores (the OpenMP build, bit-identical to
    the sequential one) over the full batch 0, on the compact q8 table of the rows it touches
    (quantized by the oracle, untimed)."""
    import time as _t
    import oracle as O
    cores = O.set_parallel(True, threads=os.cpu_count() or 1)
    try:
        smp = OracleSample(cfg, ids, off, B, None, "rowwise")
        if q8_mode == "min_max":
            codes, base_, sc, _ = O.quantize_minmax(smp.W0)
            fn = O.forward_q8_minmax
        else:
            codes, base_, sc, _ = O.quantize(smp.W0)
            fn = O.forward_q8
        t0 = _t.perf_counter()
        fn(smp.pb, codes, base_, sc, smp.cids, smp.soff, smp.Bs)
        t1 = _t.perf_counter() - t0
        reps = max(1, min(20, int(budget_s / max(t1, 1e-3))))
        t0 = _t.perf_counter()
        for _ in range(reps):
            fn(smp.pb, codes, base_, sc, smp.cids, smp.soff, smp.Bs)
        t = (_t.perf_counter() - t0) / reps
    finally:
        O.set_parallel(False)
    res = {"value": smp.Bs / t, "unit": "samples/s", "cores": cores, "kind": "oracle",
           "sample": f"the full batch 0 ({smp.Bs} samples, {smp.nnz} ids), a10 over the {len(smp.W0)} touched rows "
                     f"quantized by the oracle (untimed), OpenMP C oracle on {cores} threads, {reps + 1} reps"}
    res.update(host_info())
    return res


def run_serving(args, cfg, rank, world, local_rank):
    """BASELINE.json's Feed-shaped inference config: the 1B-row Feed tables middle-max 8-bit
    quantized (96 GB: one q8-only replica per GPU), q8 pooled lookups of B = 262144
    samples per step.  N GPUs = N independent replicas, each with its own batch ("replicas
    only": the serving path has no exchange)."""
    import torch
    import torch.distributed as dist

    from paper_2402_06859_b200 import ShardedEmbedding
    from workload import gpu as G

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    B, D, F = cfg.batch, cfg.dim, cfg.num_features
    batches = [gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed + 7919 * rank, k, alpha=cfg.alpha)
               for k in range(args.batches)]
    max_nnz = max(len(i) for i, _ in batches)
    emb = ShardedEmbedding(cfg.table_rows, D, cfg.feature_table, max_nnz=max_nnz, max_batch=B, q8_only=True,
                           q8_mode=args.q8_mode, device=dev, stream=stream)
    chunk = 1 << 25  # 32M rows (8 GB fp32) per generated block
    with torch.cuda.stream(stream):
        scratch = torch.empty(min(chunk, max(cfg.table_rows)) * D, device=dev)
        for t, rows in enumerate(cfg.table_rows):
            r = 0
            while r < rows:
                n = min(chunk, rows - r)
                blk = scratch[: n * D].view(n, D)
                G.fill_table(blk, n, D, D, cfg.seed, t, row0=r, stream=stream)
                emb.quantize_block(t, r, blk)
                r += n
        del scratch
        dev_in = [(torch.from_numpy(i).to(dev), torch.from_numpy(o).to(dev)) for i, o in batches]
        out = torch.empty((B, F, D), device=dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream.synchronize()
    torch.cuda.empty_cache()
    assert emb.sync() == 0

    def barrier():
        if world > 1:
            dist.barrier()

    for k in range(args.warmup):
        ids_d, off_d = dev_in[k % len(dev_in)]
        emb.forward_q8(ids_d, off_d, B, out=out)
    stream.synchronize()
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = ClockSampler(dev.index).begin()
    barrier()
    torch.cuda.synchronize(dev)
    launches0 = emb.launches
    emb.profile(True)
    emb.profile_read(reset=True)
    for k in range(K):
        G.flush_l2(flush, stream=stream)
        ids_d, off_d = dev_in[(args.warmup + k) % len(dev_in)]
        with torch.cuda.stream(stream):
            evs[k][0].record(stream)
        emb.forward_q8(ids_d, off_d, B, out=out)
        with torch.cuda.stream(stream):
            evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.result()
    launches = emb.launches - launches0
    ph = emb.profile_read()
    emb.profile(False)
    assert emb.sync() == 0
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    nnz_avg = float(np.mean([len(i) for i, _ in batches]))
    # e2e: ids/offsets H2D (pinned) and the pooled result D2H, every step, through the API
    e2e = None
    if not args.no_e2e:
        host_in = [(torch.from_numpy(i).pin_memory(), torch.from_numpy(o).pin_memory()) for i, o in batches]
        out_h = torch.empty((B, F, D), dtype=torch.float32).pin_memory()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            t0.record(stream)
        for k in range(K):
            ids_h, off_h = host_in[k % len(host_in)]
            emb.forward_q8(ids_h, off_h, B, out=out_h)
        with torch.cuda.stream(stream):
            t1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        assert emb.sync() == 0
        e_ms = t0.elapsed_time(t1) / K
        if world > 1:
            t = torch.tensor([e_ms], device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": world * B / (e_ms / 1e3), "unit": "samples/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(nnz_avg * 4 + (F * B + 1) * 4), "d2h_bytes_per_step": B * F * D * 4,
               "path": "emb_forward_q8 with pinned host ids/offsets/out (staging copies inside the call)"}
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    q_ms = ph["fwd_q8"][0] / max(ph["fwd_q8"][1], 1)
    ab = alg_bytes("fwd_q8", cfg, nnz_avg, 0, B, emb.pitch)
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get("serve_fwd_q8", {}).get(
            "dram_bytes_per_launch")
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": world * B / (ms / 1e3), "unit": "samples/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 codes, f32 accumulate", "data": "synthetic (seeded Zipf ids, Irwin-Hall tables)",
        "config": {"workload": cfg.name, "tables": cfg.table_rows, "dim": D, "features": F, "global_batch": world * B,
                   "batch_per_gpu": B, "nnz_per_step": nnz_avg, "alpha": cfg.alpha, "q8": args.q8_mode,
                   "q8_store_bytes": int(emb.local_rows * emb.q8_pitch),
                   "parallelism": "single" if world == 1 else f"replicas x{world} (one q8 replica per GPU)",
                   "step": "a10 q8 pooled lookup (serving handle, EMB_F_Q8_ONLY)",
                   "l2": "flushed between timed steps (256 MiB write, untimed)", "batches_rotated": len(batches)},
        "q8_lookups_per_s": world * nnz_avg / (ms / 1e3),
        "roofline": {"bound": "hbm", "kernel": "fwd_q8", "achieved": ab / (q_ms / 1e3) / 1e9, "peak": hbm_peak,
                     "unit": "GB/s", "frac": ab / (q_ms / 1e3) / 1e9 / hbm_peak, "traffic": traffic,
                     "alg_bytes_per_launch": ab,
                     "timing": "CUDA events on the library stream around the kernel phase, mean over timed steps"},
        "clocks": clk, "gpu_launches": launches, "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = serving_cpu_baseline(cfg, batches[0][0], batches[0][1], B, args.cpu_samples,
                                                        args.q8_mode)
        except Exception as e:  # report, never hide
            line["cpu_baseline"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)

# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def global_batch(per_rank, F, B):
    """Concatenate per-rank feature-major batches into the global batch (sample r*B + b)."""
    ids_g, lens = [], []
    for f in range(F):
        for (ids, off) in per_rank:
            o = off.astype(np.int64)
            ids_g.append(ids[o[f * B]:o[(f + 1) * B]])
            lens.append(np.diff(o[f * B:(f + 1) * B + 1]))
    off_g = np.zeros(F * B * len(per_rank) + 1, dtype=np.int64)
    off_g[1:] = np.cumsum(np.concatenate(lens))
    return np.concatenate(ids_g).astype(np.int32), off_g.astype(np.int32)


def spot_readings(emb, cfg, ids, off, B, out, samples=64, max_rows=2048):
    """Right after the first step (rank 0): its pooled outputs of its first samples and a
    sample of the rows of its batch that it stores, as updated by that step."""
    F = cfg.num_features
    S = min(samples, B)
    pooled = out[:S].cpu().numpy().copy()
    bag_of = np.repeat(np.arange(F * B), np.diff(off.astype(np.int64)))
    t = np.asarray(cfg.feature_table, dtype=np.int64)[bag_of // B]
    pairs = np.unique(t * (1 << 32) + ids.astype(np.int64))
    tt, rr = pairs >> 32, pairs & 0xffffffff
    lo, hi, lb = emb.row_lo[tt], emb.row_hi[tt], emb.local_base[tt]
    mine = (lb >= 0) & (rr >= lo) & (rr < hi)
    tt, rr = tt[mine], rr[mine]
    if len(tt) > max_rows:
        pick = np.linspace(0, len(tt) - 1, max_rows).astype(np.int64)
        tt, rr = tt[pick], rr[pick]
    rows = {}
    for t_ in np.unique(tt):
        r_ = rr[tt == t_]
        rows[int(t_)] = (r_, emb.read_rows(int(t_), r_, with_acc=True))
    return {"samples": S, "pooled": pooled, "rows": rows}


def spot_check(cfg, rd, world, B, gshift, mode, rank_batches=None):
    """The oracle on the GLOBAL batch 0 (every rank's batch, regenerated from the seeds),
    over the compact table of its touched rows, OpenMP build: rank 0's pooled outputs within
    the pooled gate, its sampled rows and accumulators within the update gates."""
    import oracle as O
    F, D = cfg.num_features, cfg.dim
    t0 = time.perf_counter()
    if rank_batches is None:
        rank_batches = [gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed + 7919 * r, 0, alpha=cfg.alpha)
                        for r in range(world)]
    ids_g, off_g = global_batch(rank_batches, F, B)
    threads = O.set_parallel(True, threads=os.cpu_count() or 1)
    try:
        smp = OracleSample(cfg, ids_g, off_g, world * B, None, mode, gshift=gshift)
        W0 = smp.W.copy()
        A0 = smp.A.copy()
        r = O.train_step(smp.pb, smp.W, smp.A, smp.cids, smp.soff, smp.Bs, smp.grad, LR, 1e-7, 1.0, mode=mode)
        mag, _ = O.forward(smp.pb, np.abs(W0), smp.cids, smp.soff, smp.Bs)
    finally:
        O.set_parallel(False)
    S = rd["samples"]
    ref = r["out"][:S]
    pooled_ok = np.abs(rd["pooled"].astype(np.float64) - ref) <= 1e-5 * mag[:S] + 1e-30
    n_rows, rows_ok, acc_ok, exact = 0, 0, 0, 0
    for t_, (rr, (w, a)) in rd["rows"].items():
        k = np.searchsorted(smp.keys, smp.base[t_] + rr)
        assert (smp.keys[k] == smp.base[t_] + rr).all()
        wo, w0 = smp.W[k], W0[k]
        step = np.abs(wo - w0)
        tol = 1e-6 * np.maximum(np.maximum(np.abs(wo), np.abs(w0)), step) + 1e-12
        rows_ok += int((np.abs(w.astype(np.float64) - wo) <= tol).all(axis=1).sum())
        exact += int((w == wo).all(axis=1).sum())
        ao = smp.A[k]
        acc_ok += int((np.abs(a - ao) <= 1e-6 * np.abs(ao)).reshape(len(k), -1).all(axis=1).sum())
        n_rows += len(k)
    return {"what": "oracle (OpenMP C, bit-identical to the sequential build) on the global batch 0 "
                    f"({smp.Bs} samples, {smp.nnz} ids, {len(smp.keys)} touched rows): rank 0's pooled outputs of "
                    f"its first {S} samples and {n_rows} sampled rows it stores, after the first step",
            "pooled_within_gate": bool(pooled_ok.all()), "pooled_bit_exact_frac": float((rd["pooled"] == ref).mean()),
            "rows_checked": n_rows, "rows_within_gate": rows_ok, "acc_within_gate": acc_ok,
            "rows_bit_exact": exact, "ok": bool(pooled_ok.all()) and rows_ok == n_rows and acc_ok == n_rows,
            "oracle_threads": threads, "seconds": time.perf_counter() - t0}


def run_ours(args, cfg, rank, world, local_rank, B=None, sharding="row", scaling="strong"):
    import torch
    import torch.distributed as dist

    from paper_2402_06859_b200 import ShardedEmbedding
    from workload import gpu as G

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())  # (host transport: ranks may share a GPU)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    B = cfg.batch if B is None else B  # this rank's batch (strong scaling: global / N)
    cdev = torch.device("cpu") if args.transport == "host" else dev  # tensors of torch.distributed calls
    D, F = cfg.dim, cfg.num_features

    # inputs: nb distinct batches, resident in HBM (and pinned on the host for e2e)
    batches = []
    for k in range(args.batches):
        ids, off = gen.make_batch(cfg.table_rows, cfg.features, B, cfg.seed + 7919 * rank, k, alpha=cfg.alpha)
        batches.append((ids, off))
    max_nnz = max(len(i) for i, _ in batches)
    shard_kw = {}
    if world > 1 or args.exchange:
        # sharded over NCCL (or the exchange path on 1 rank); rank 0 makes the unique id, a broadcast distributes it
        from paper_2402_06859_b200 import nccl_unique_id

        def new_uid():  # one NCCL unique id per communicator
            uid = torch.zeros(128, dtype=torch.uint8, device=cdev)
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
            if world > 1:
                dist.broadcast(uid, 0)
            return uid.cpu().numpy().tobytes()

        # receive capacity: a 1-rank exchange receives exactly its own ids; with N ranks an owner
        # receives about the average share (table-wise placement by traffic; row-wise the owner of
        # the Zipf-hottest rows ~1/3 more): 2x (the sharded a5/a6 grids are sized for it)
        shard_kw = dict(rank=rank, world_size=world, sharding=sharding,
                        max_recv_nnz=(2 if world > 1 else 1) * max_nnz, force_exchange=args.exchange)
        if args.transport == "host" and world > 1:
            from paper_2402_06859_b200 import HostComm
            shard_kw["host_comm"] = HostComm()
        else:
            shard_kw["nccl_unique_id"] = new_uid()
        if sharding == "table":  # LPT placement by lookup traffic
            shard_kw["table_cost"] = configs.table_cost(cfg, batch=world * B)
    xmode = None
    if shard_kw:
        xmode = args.exchange_mode
        shard_kw["p2p"] = xmode == "p2p"

    def make_emb():
        e = ShardedEmbedding(cfg.table_rows, D, cfg.feature_table, max_nnz=max_nnz, max_batch=B,
                             adagrad=args.adagrad, q8=True, requant=True, device=dev, stream=stream,
                             q8_mode=args.q8_mode, **shard_kw)
        with torch.cuda.stream(stream):
            for t in range(cfg.num_tables):
                v = e.table_view(t)
                G.fill_table(v, v.shape[0], D, e.pitch, cfg.seed, t, row0=int(e.row_lo[t]), stream=stream)
            e.quantize()
        return e

    emb = make_emb()
    with torch.cuda.stream(stream):
        # one grad scale for every rank: from the GLOBAL batch's expected ids (pre-clip |g| ~ 4)
        gshift = gen.grad_shift_for(int(round(cfg.mean_bag() * B * world)), D)
        dev_in = []
        for k, (ids, off) in enumerate(batches):
            gd = torch.empty((B, F, D), device=dev)
            G.fill_grad(gd, B, F, D, cfg.seed, k, gshift, sample0=rank * B, stream=stream)
            dev_in.append((torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev), gd))
        out = torch.empty((B, F, D), device=dev)
        out_q8 = torch.empty((B, F, D), device=dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream.synchronize()
    assert emb.sync() == 0

    def step(k):
        ids_d, off_d, gd = dev_in[k % len(dev_in)]
        emb.forward(ids_d, off_d, B, out=out)          # a2 (+ a5 dedup starts on the side stream)
        # a10 from the q8 store on the same batch (overlaps a5; sharded: its ids exchange is reused)
        emb.forward_q8(None, None, B, out=out_q8, nnz=ids_d.numel())
        emb.backward_adagrad(gd, LR)                   # a6-a8 (+ a9 requant of touched rows)

    def barrier():
        if world > 1:
            dist.barrier()

    first_done = False
    if xmode == "p2p":
        # the first sharded forward maps the peers (collective: every rank gets the same verdict)
        try:
            step(0)
            first_done = True
        except RuntimeError as e:
            if "EMB_ENCCL" not in str(e) and "ENCCL" not in str(e):
                raise
            xmode = f"nccl (p2p unavailable: {e})"
            emb.close()
            shard_kw["p2p"] = False
            if "nccl_unique_id" in shard_kw:
                shard_kw["nccl_unique_id"] = new_uid()
            emb = make_emb()
    if not first_done:
        step(0)
    # the first (warm-up) step is the in-run parity spot check's: rank 0 reads its pooled
    # outputs and a sample of its updated rows now; the oracle runs after the timed region
    stream.synchronize()
    barrier()
    readings = None
    if rank == 0 and not args.no_spot:
        readings = spot_readings(emb, cfg, batches[0][0], batches[0][1], B, out)
    barrier()
    for k in range(1, args.warmup):
        step(k)
    stream.synchronize()
    st = emb.sync()
    assert st == 0, f"status {st} after warm-up"

    # ---- timed region: device-resident inputs --------------------------------------
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = ClockSampler(dev.index).begin()
    barrier()
    torch.cuda.synchronize(dev)
    launches0 = emb.launches
    emb.profile(True)
    emb.profile_read(reset=True)
    for k in range(K):
        G.flush_l2(flush, stream=stream)
        with torch.cuda.stream(stream):
            evs[k][0].record(stream)
        emb.profile(True)
        step(args.warmup + k)
        emb.profile(False)
        with torch.cuda.stream(stream):
            evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.result()
    launches = emb.launches - launches0
    phases = emb.profile_read()
    st = emb.sync()
    assert st == 0, f"status {st} in timed region"
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms))
    per_rank = None
    if world > 1:
        # every rank's mean step and phase times (row-wise: the owner of the Zipf-hottest rows
        # does more a5-a8 work); the line's time is the max over ranks
        ph_ms = [phases[p][0] / max(phases[p][1], 1) for p in ("fwd", "sort", "segreduce", "update", "exchange")
                 if p in phases]
        mine = torch.tensor([ms] + ph_ms, device=cdev, dtype=torch.float64)
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = [[round(float(x), 4) for x in r.tolist()] for r in allr]
        ms = max(r[0] for r in per_rank)
    S, c, U = emb.last_stats()

    # ---- e2e: the user's pipeline through the C ABI's host-pointer path -----------------
    # Every step's batch (ids, offsets) starts in pinned HOST memory and is handed to the
    # library as host pointers: emb_forward stages it into one of its two staging slots on
    # its copy stream (inside the timed region; the transfer overlaps the previous step's
    # kernels), emb_forward_q8(NULL, NULL) looks up the same staged batch from the q8 store,
    # and emb_backward_adagrad_dev writes the step's result S (global squared grad norm) to
    # the device, copied to pinned host memory at the end of the step; the host reads step
    # k-1's S before it issues step k+1 (a training loop one step deep).  The upstream
    # gradient dL/d(pooled) is a device tensor: in a training step the dense tower's backward
    # produces it on the GPU (the `model` object runs that tower for real), not host input.
    e2e = None
    if not args.no_e2e:
        host_in = [(torch.from_numpy(ids).pin_memory(), torch.from_numpy(off).pin_memory()) for ids, off in batches]
        S_dev = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(2)]
        S_host = [torch.zeros(1, dtype=torch.float64).pin_memory() for _ in range(2)]
        evS = [torch.cuda.Event() for _ in range(2)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        S_seen = []
        barrier()
        torch.cuda.synchronize(dev)
        G.flush_l2(flush, stream=stream)
        with torch.cuda.stream(stream):
            t0.record(stream)
        for k in range(K):
            slot = k % 2
            ids_h, off_h = host_in[k % len(host_in)]
            g_d = dev_in[k % len(dev_in)][2]
            emb.forward(ids_h, off_h, B, out=out)                             # H2D staged by the library
            emb.forward_q8(None, None, B, out=out_q8, nnz=ids_h.numel())     # the same staged batch
            emb.backward_adagrad_dev(g_d, LR, sq_norm_out=S_dev[slot])       # S on the device
            with torch.cuda.stream(stream):
                S_host[slot].copy_(S_dev[slot], non_blocking=True)           # D2H of the step's result
                evS[slot].record(stream)
            if k >= 1:
                evS[1 - slot].synchronize()
                S_seen.append(float(S_host[1 - slot]))
        with torch.cuda.stream(stream):
            t1.record(stream)
        torch.cuda.synchronize(dev)
        S_seen.append(float(S_host[(K - 1) % 2]))
        barrier()
        assert emb.sync() == 0 and len(S_seen) == K and min(S_seen) > 0.0
        e_ms = t0.elapsed_time(t1) / K
        if world > 1:
            t = torch.tensor([e_ms], device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        nnz_avg = float(np.mean([len(i) for i, _ in batches]))
        h2d_b = int(nnz_avg * 4 + (F * B + 1) * 4)
        e2e = {"value": world * B / (e_ms / 1e3), "unit": "samples/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": 8,
               "path": "pinned host ids/offsets passed to emb_forward as HOST pointers (staged H2D by the "
                       "library on its copy stream, double-buffered) -> emb_forward_q8(NULL, NULL) on the "
                       "staged batch -> emb_backward_adagrad_dev (device grad = the tower's output) -> S D2H "
                       "every step; the host reads step k-1's S before issuing step k+1"}

    # ---- a5 alone: forward -> backward with nothing beside the dedup -------------------
    # (in the step above the dedup shares the GPU with the a10 lookup on the main stream, so
    # its phase time there is not its own)
    a5_alone = None
    if world == 1 and not args.no_a5:
        emb.profile(True)
        emb.profile_read(reset=True)
        for k in range(5):
            ids_d, off_d, gd = dev_in[k % len(dev_in)]
            G.flush_l2(flush, stream=stream)
            emb.forward(ids_d, off_d, B, out=out)
            emb.backward_adagrad(gd, LR)
        ph5 = emb.profile_read()
        emb.profile(False)
        assert emb.sync() == 0
        a5_alone = {"sort_ms": ph5["sort"][0] / max(ph5["sort"][1], 1), "rle_ms": ph5["rle"][0] / max(ph5["rle"][1], 1)}

    # ---- full-table quantize (a9), timed alone ----------------------------------------
    emb.profile(True)
    emb.profile_read(reset=True)
    for _ in range(3):
        G.flush_l2(flush, stream=stream)
        emb.quantize()
    q = emb.profile_read()["quantize"]
    emb.profile(False)
    q_ms = q[0] / max(q[1], 1)
    q_bytes = emb.local_rows * (4 * emb.pitch + D + 8)

    # ---- roofline ----------------------------------------------------------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if "hbm_gbs" in peaks else "fallback 6650 GB/s (B200_PROFILING.md)"
    nnz_avg = float(np.mean([len(i) for i, _ in batches]))
    per_phase = {}
    kbits = int(emb.local_rows).bit_length()  # keys in [0, local_rows] (sentinel = local_rows)
    dbits = 9 if (24 < kbits <= 27 or 16 < kbits <= 18) else 8
    passes = -(-kbits // dbits)
    for p, (tot, n) in phases.items():
        if n == 0:
            continue
        per = tot / n
        ab = alg_bytes(p, cfg, nnz_avg, U, B, emb.pitch, args.adagrad)
        ent = {"ms": per, "instances": n}
        if ab:
            ent["alg_bytes"] = ab
            ent["gbs"] = ab / (per / 1e3) / 1e9
            ent["frac_of_hbm"] = ent["gbs"] / hbm_peak
            cb = compulsory_bytes(p, cfg, nnz_avg, U, B, emb.pitch, args.adagrad)
            if cb:  # every touched row (and every bag's gradient row) moved once
                ent["compulsory_bytes"] = cb
                ent["compulsory_frac_of_hbm"] = cb / (per / 1e3) / 1e9 / hbm_peak
            if p in ("fwd", "fwd_q8") and cfg.alpha > 0:
                ent["frac_note"] = ("per-occurrence bytes at Zipf alpha > 0: L1/L2 serve the repeated hot rows, "
                                    "so this fraction is reuse-inflated; the HBM-bound figure is the alpha = 0 "
                                    "run (--alpha 0) or compulsory_frac_of_hbm")
        ib = impl_bytes(p, nnz_avg, U, passes)
        if ib:  # a5: its own (implementation) bytes, SURVEY.md §8(d)
            ent["own_bytes"] = ib
            ent["own_gbs"] = ib / (per / 1e3) / 1e9
            ent["own_frac_of_hbm"] = ent["own_gbs"] / hbm_peak
            if p == "sort":
                ent["passes"] = passes
        per_phase[p] = ent
    if "sort" in per_phase and "rle" in per_phase:
        a5_b = per_phase["sort"]["own_bytes"] + per_phase["rle"]["own_bytes"]
        a5_ms = per_phase["sort"]["ms"] + per_phase["rle"]["ms"]
        ent = {"ms_in_step": a5_ms, "own_bytes": a5_b, "passes": passes,
               "note": "radix sort + run-length encode, on the library's side stream; in the step it shares "
                       "the GPU with the a10 lookup, so its own rate is measured alone (fwd -> bwd, 5 steps)"}
        if a5_alone:
            ms5 = a5_alone["sort_ms"] + a5_alone["rle_ms"]
            ent.update({"ms": ms5, "sort_ms": a5_alone["sort_ms"], "rle_ms": a5_alone["rle_ms"],
                        "own_gbs": a5_b / (ms5 / 1e3) / 1e9, "own_frac_of_hbm": a5_b / (ms5 / 1e3) / 1e9 / hbm_peak,
                        "sort_own_frac_of_hbm": per_phase["sort"]["own_bytes"] / (a5_alone["sort_ms"] / 1e3) / 1e9 / hbm_peak})
        per_phase["a5_dedup"] = ent
    single = [p for p in ("fwd", "fwd_q8", "update", "segreduce") if p in per_phase]
    dom = max(single, key=lambda p: per_phase[p]["ms"])
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(dom, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roof = {"bound": "hbm", "kernel": dom, "achieved": per_phase[dom]["gbs"], "peak": hbm_peak, "unit": "GB/s",
            "frac": per_phase[dom]["gbs"] / hbm_peak, "traffic": traffic,
            "alg_bytes_per_launch": per_phase[dom]["alg_bytes"], "peak_source": peak_src,
            "timing": "CUDA events on the library stream around the kernel phase, mean over timed steps"}
    if traffic:
        # physical DRAM throughput of the same phase (ncu bytes / live time): below the
        # algorithmic figure when L2 serves repeated rows (Zipf-hot rows, a bag's gradient
        # row gathered once per id in the bag)
        roof["dram_achieved"] = traffic / (per_phase[dom]["ms"] / 1e3) / 1e9
        roof["dram_frac"] = roof["dram_achieved"] / hbm_peak

    spot = None
    if readings is not None:
        try:
            spot = spot_check(cfg, readings, world, B, gshift, args.adagrad,
                              rank_batches=[batches[0]] if world == 1 else None)
        except Exception as e:  # report, never hide
            spot = {"error": repr(e), "ok": False}
    value = world * B / (ms / 1e3)
    fwd_ms = per_phase["fwd"]["ms"]
    bwd_ms = sum(per_phase[p]["ms"] for p in ("sort", "rle", "segreduce", "norm", "update") if p in per_phase)
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded Zipf ids, Irwin-Hall tables/grads)",
        "config": {"workload": cfg.name, "baseline_config": cfg.note, "tables": cfg.table_rows, "dim": D, "features": F,
                   "global_batch": world * B, "batch_per_gpu": B, "nnz_per_step_per_gpu": nnz_avg, "alpha": cfg.alpha,
                   "unique_rows": U, "adagrad": args.adagrad, "q8": args.q8_mode,
                   "parallelism": ("single" if not args.exchange else f"{sharding}-sharded exchange path on a 1-rank NCCL communicator")
                   if world == 1 else f"{sharding}-sharded x{world}" + (" (LPT placement by lookup traffic)" if sharding == "table" else ""),
                   "exchange": None if xmode is None else (
                       "p2p: ids stored by one kernel at their compacted place in the owners' receive buffers "
                       "after a device-side count all-gather (no host sync); pooled rows stored by the owners' "
                       "pooling kernels into the destination's buffer over NVLink peer memory (row-wise: "
                       "per-owner slots summed in rank order); grad rows pushed to the owners by one kernel; "
                       + ("NCCL 4-byte all-gather barriers" if args.transport == "nccl" else
                          "host-transport barriers (stream drain + gloo all-gather; ranks share one GPU)")
                       if xmode == "p2p" else
                       f"{xmode}: ids all-to-all of capacity-padded slots (no host sync); " +
                       ("reduce-scatter pooled, all-gather grads" if sharding == "row"
                        else "all-to-all pooled / grad blocks + permute")),
                   "transport": None if world == 1 and not args.exchange else args.transport,
                   "step": "a2 fwd -> a10 q8 fwd (overlapping a5 dedup on a side stream) -> a6-a8 bwd (a9 requant of touched rows fused)",
                   "l2": "flushed between timed steps (256 MiB write, untimed)",
                   "batches_rotated": len(batches)},
        "lookups_per_s": world * nnz_avg / (fwd_ms / 1e3),
        "q8_lookups_per_s": world * nnz_avg / (per_phase["fwd_q8"]["ms"] / 1e3) if "fwd_q8" in per_phase else None,
        "train_samples_per_s": world * B / ((fwd_ms + bwd_ms) / 1e3),
        "phases": per_phase,
        "quantize_full": {"ms": q_ms, "rows": emb.local_rows, "alg_bytes": q_bytes,
                          "gbs": q_bytes / (q_ms / 1e3) / 1e9, "frac_of_hbm": q_bytes / (q_ms / 1e3) / 1e9 / hbm_peak},
        "roofline": roof,
        "clocks": clk,
        "gpu_launches": launches,
        "e2e": e2e,
        "clip": {"sq_norm": S, "c": float(c)},
        "spot_check": spot,
        "per_rank_ms": None if per_rank is None else {
            "columns": ["step"] + [p for p in ("fwd", "sort", "segreduce", "update", "exchange") if p in phases],
            "ranks": per_rank},
    }
    if world == 1 and not args.no_lib:
        try:
            line["library"] = library_section(emb, cfg, dev_in, B, stream, flush)
            line["library"]["ours_a2_ms"] = per_phase["fwd"]["ms"]
        except Exception as e:  # report, never hide
            line["library"] = {"error": repr(e)}
    if world == 1 and not args.no_graph:  # (the exchange path is host-sync free too: graphed at N=1)
        try:
            line["graph"] = graph_section(emb, cfg, dev_in, B, out, out_q8, stream, flush)
        except Exception as e:  # report, never hide
            line["graph"] = {"error": repr(e)}
    if world == 1 and not args.no_model:
        try:
            line["model"] = model_section(emb, batches, dev_in, B, args.dense_features, stream, flush)
        except Exception as e:  # report, never hide
            line["model"] = {"error": repr(e)}
    if world == 1 and not args.no_fim:
        try:
            line["fim"] = fim_section(emb, dev_in, B, stream, flush, hbm_peak)
        except Exception as e:  # report, never hide
            line["fim"] = {"error": repr(e)}
    if world == 1 and not args.no_qr:
        try:
            line["qr"] = qr_section(cfg, batches[0][0], batches[0][1], B, dev, stream, flush, hbm_peak)
        except Exception as e:  # report, never hide
            line["qr"] = {"error": repr(e)}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, batches[0][0], batches[0][1], B, args.cpu_samples,
                                                args.adagrad)
        except Exception as e:  # report, never hide
            line["cpu_baseline"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)


def scale_plan(cfg, world, sharding=None, weak=False, serve=False):
    """(config, this rank's batch, sharding, scaling) of an N-GPU run.

    Strong scaling (default): BASELINE's GLOBAL batch (Feed 128k, Ads 64k, Jobs 16k) split
    over the N GPUs.  The Feed tables grow with N from the 1-GPU shard (125M rows per GPU): at
    N = 8 they are BASELINE.json's Feed config, "~1B total rows x dim 64 fp32 row-wise sharded
    over 8xB200"; Ads / Jobs keep their tables (table-wise, LPT by lookup traffic).  Weak:
    every GPU keeps the 1-GPU batch.  Serving (q8 replicas) keeps its per-replica batch."""
    sharding = sharding or ("row" if cfg.name.startswith("feed") else "table")
    scaling = "weak" if weak else "strong"
    if world <= 1 or serve:
        return cfg, cfg.batch, sharding, scaling
    if cfg.name == "feed1":
        cfg = cfg.with_(name=f"feed-x{world}", table_rows=[r * world for r in cfg.table_rows],
                        note=f"feed1 tables x {world}" + (" = BASELINE.json configs[3] (1B rows)" if world == 8 else ""))
    if weak:
        cfg = cfg.with_(name=f"{cfg.name}-weak", batch=cfg.batch * world)
    assert cfg.batch % world == 0
    return cfg, cfg.batch // world, sharding, scaling


def main():
    args = parse()
    cfg = configs.get(args.config)
    if args.alpha is not None:
        cfg = cfg.with_(alpha=args.alpha)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    serve = args.serve or cfg.name.startswith("feedq8")
    cfg, B_local, sharding, scaling = scale_plan(cfg, world, args.sharding, args.weak, serve)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world, serve=serve)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.transport == "host":
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if serve:
            run_serving(args, cfg, rank, world, local_rank)
        else:
            run_ours(args, cfg, rank, world, local_rank, B=B_local, sharding=sharding, scaling=scaling)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
