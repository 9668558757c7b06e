"""Multi-process (gloo, world size 2-3) tests of the sharded path's host logic on CPU (-m "not gpu").

1. The C planner (emb_plan / emb_local_layout, host-only) gives every rank a consistent
   plan: the union of the ranks' stored rows covers every row exactly once.
2. The forward exchange protocol the CUDA path implements (exchange.cu: a1 per-destination
   [features][B] lengths + keys in (feature, sample, id) order, owner pooling per source,
   a3 return of [B][Fo][D] blocks summed/placed in rank order) executed with gloo
   all-to-all-v and the CPU oracle as the owner's local compute, against the unsharded
   oracle on each rank's batch.  (a4 and the rank-ordered norm are covered on the GPU by
   tests/test_sharded_gpu.py through the loopback transport.)
3. The fused-exchange (EMB_F_P2P) addressing: the owner's peer stores of pooled rows
   (final [B][F] column table-wise; per-owner slots summed in rank order row-wise) and the
   grad-row pushes to the owners, simulated as (row index, row) messages: every destination
   row is written exactly once and the result equals the unsharded oracle.
4. The sync-free a1 (device-side count all-gather, then fused key push at the lower ranks'
   prefix, or capacity-padded slots + compaction): both land the keys exactly where the
   variable-size all-to-all puts them (sources in rank order), and a capacity overflow is
   decided identically on every rank from the gathered count matrix (world sizes 2 and 3).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def layout_of(rows, ft, D, rank, world, sharding):
    from paper_2402_06859_b200 import _lib as L
    lib = L.load()
    ra = np.asarray(rows, dtype=np.int64)
    fa = np.asarray(ft, dtype=np.int32)
    cfg = L.EmbConfig(abi_version=L.EMB_ABI_VERSION, num_tables=len(rows), table_rows=ra.ctypes.data_as(C.POINTER(C.c_int64)),
                      dim=D, num_features=len(ft), feature_table=fa.ctypes.data_as(C.POINTER(C.c_int32)),
                      pooling=0, adagrad_mode=0, init_accumulator=0.1, eps=1e-7, max_norm=1.0, max_nnz=10000,
                      max_batch=256, sharding={"table": 1, "row": 2}[sharding], table_owner=None, rank=rank,
                      world_size=world, nccl_unique_id=None, stream=None, flags=0, max_recv_nnz=0)
    T = len(rows)
    lb, lo, hi = (np.zeros(T, dtype=np.int64) for _ in range(3))
    s = L.EmbSizes()
    assert lib.emb_plan(C.byref(cfg), C.byref(s)) == 0
    assert lib.emb_local_layout(C.byref(cfg), lb.ctypes.data_as(C.c_void_p), lo.ctypes.data_as(C.c_void_p),
                                hi.ctypes.data_as(C.c_void_p)) == 0
    return lb, lo, hi, int(s.local_rows)


def _plan_worker(rank, world, port, sharding, q):
    try:
        _init(rank, world, port)
        rows = [1000, 7, 3500, 64, 99_983]
        lb, lo, hi, lr = layout_of(rows, [0, 1, 2, 3, 4, 2], 16, rank, world, sharding)
        mine = torch.tensor(np.stack([lb, lo, hi]), dtype=torch.int64)
        allp = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allp, mine)
        if rank == 0:
            cover = [np.zeros(r, dtype=np.int32) for r in rows]
            for m in allp:
                m = m.numpy()
                for t in range(len(rows)):
                    if m[0, t] >= 0:
                        cover[t][m[1, t]:m[2, t]] += 1
            q.put(all((c == 1).all() for c in cover))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(repr(e))


@pytest.mark.parametrize("sharding", ["table", "row"])
def test_plan_consistent_across_gloo_ranks(sharding):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_plan_worker, args=(r, 2, port, sharding, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
    assert res is True, res


# ---------------------------------------------------------------------------------------
# protocol simulation
# ---------------------------------------------------------------------------------------

def _protocol_worker(rank, world, port, sharding, q, mode="collective"):
    try:
        _init(rank, world, port)
        import oracle as O
        from workload import configs, gen
        rows = [900, 300, 50]
        ft = [0, 1, 2, 0]
        D, B = 8, 32
        cfg = configs.Config("p", rows, D, [(t, ("range", 0, 7)) for t in ft], B, seed=2)
        F = len(ft)
        lay = [layout_of(rows, ft, D, r, world, sharding) for r in range(world)]
        base = np.concatenate([[0], np.cumsum(rows)])
        per_rank = [gen.make_batch(rows, cfg.features, B, cfg.seed + r, 0) for r in range(world)]
        ids, off = per_rank[rank]

        def owner(t, i):
            for o in range(world):
                lb, lo, hi, _ = lay[o]
                if lb[t] >= 0 and lo[t] <= i < hi[t]:
                    return o
            raise AssertionError

        feats_of = [[f for f in range(F) if lay[o][0][ft[f]] >= 0] for o in range(world)]
        # a1: per destination: lengths [Fo][B] and global row keys in (feature, sample, bag) order
        lens = [np.zeros((len(feats_of[o]), B), dtype=np.int64) for o in range(world)]
        keys = [[] for _ in range(world)]
        for o in range(world):
            for j, f in enumerate(feats_of[o]):
                t = ft[f]
                for b in range(B):
                    for i in ids[off[f * B + b]:off[f * B + b + 1]]:
                        if owner(t, i) == o:
                            lens[o][j, b] += 1
                            keys[o].append(base[t] + i)
        def a2a(chunks, dtype):  # all-to-all-v: counts first, then the payload
            send = [np.asarray(c, dtype=dtype).ravel() for c in chunks]
            ssz = torch.tensor([len(s) for s in send], dtype=torch.int64)
            rsz = torch.zeros(world, dtype=torch.int64)
            dist.all_to_all_single(rsz, ssz)
            flat = torch.from_numpy(np.concatenate(send)) if sum(ssz.tolist()) else torch.zeros(0, dtype=torch.from_numpy(send[0]).dtype)
            recv = torch.zeros(int(rsz.sum()), dtype=flat.dtype)
            dist.all_to_all_single(recv, flat, rsz.tolist(), ssz.tolist())
            return [x.numpy() for x in torch.split(recv, rsz.tolist())]
        r_lens = a2a(lens, np.int64)
        r_keys = a2a(keys, np.int64)
        # owner: pool every source's bags with the oracle over the global table
        Wfull = np.concatenate([gen.table_rows(cfg.seed, t, np.arange(r), D) for t, r in enumerate(rows)])
        pb1 = O.Problem([len(Wfull)], D, [0])
        Fr = len(feats_of[rank])
        pooled = []
        for s_ in range(world):
            L_ = r_lens[s_].reshape(Fr, B)
            o_ = np.zeros(Fr * B + 1, dtype=np.int64)
            o_[1:] = np.cumsum(L_.ravel())
            out_s = np.zeros((B, Fr, D), dtype=np.float32)
            for j in range(Fr):
                sub_off = (o_[j * B:(j + 1) * B + 1] - o_[j * B]).astype(np.int32)
                sub_ids = r_keys[s_][o_[j * B]:o_[(j + 1) * B]].astype(np.int32)
                ob, _ = O.forward(pb1, Wfull, sub_ids, sub_off, B)
                out_s[:, j] = ob[:, 0]
            pooled.append(out_s)
        ok = True
        if mode == "collective":
            # a3: return: each source sums (row-wise) / places (table-wise) owner blocks in rank order
            back = a2a([p.ravel() for p in pooled], np.float32)
            out = np.zeros((B, F, D), dtype=np.float32)
            for o in range(world):
                blk = back[o].reshape(B, len(feats_of[o]), D)
                for j, f in enumerate(feats_of[o]):
                    out[:, f] = out[:, f] + blk[:, j]
        else:
            # a3 fused (EMB_F_P2P, exchange.cu peer_out / forward.cu dst_row): the owner stores
            # the pooled row of (source s, owner-local feature j, sample b) at row
            # (slot * B + b) * F + fcol[j] of rank s's buffer -- table-wise slot 0 and fcol[j]
            # = the global feature (final [B][F] place), row-wise slot = owner rank into a
            # [W][B][F] slot array summed in rank order.  Peer stores are simulated by
            # shipping (row index, row) pairs.
            row_wise = sharding == "row"
            slot = rank if row_wise else 0
            fcol = feats_of[rank]
            idx_to, rows_to = [], []
            for s_ in range(world):
                # row-wise: a bag with no id on this owner is not stored (skip_empty)
                L_ = r_lens[s_].reshape(Fr, B)
                keep = [(b, j) for b in range(B) for j in range(Fr) if not row_wise or L_[j, b] > 0]
                idx_to.append(np.array([(slot * B + b) * F + fcol[j] for b, j in keep], dtype=np.int64))
                rows_to.append(np.array([pooled[s_][b, j] for b, j in keep], dtype=np.float32).reshape(-1))
            r_idx = a2a(idx_to, np.int64)
            r_rows = a2a(rows_to, np.float32)
            nslots = world if row_wise else 1
            buf = np.full((nslots * B * F, D), np.nan, dtype=np.float32)
            hits = np.zeros(nslots * B * F, dtype=np.int64)
            for o in range(world):
                buf[r_idx[o]] = r_rows[o].reshape(-1, D)
                np.add.at(hits, r_idx[o], 1)
            if row_wise:
                # slot o row (b, f) is written iff this rank sent ids of bag (f, b) to owner o
                # (its a1 lengths), exactly once; the sum skips the others (k_sum_slots)
                sent = np.stack([lens[o].T for o in range(world)])  # [W][B][F]
                ok &= bool((hits == (sent > 0).ravel()).all())
                sl = buf.reshape(world, B, F, D)
                out = np.zeros((B, F, D), dtype=np.float32)
                for b_ in range(B):
                    for f in range(F):
                        first = True
                        for o in range(world):
                            if sent[o, b_, f] == 0:
                                continue
                            out[b_, f] = sl[o, b_, f] if first else out[b_, f] + sl[o, b_, f]
                            first = False
            else:
                ok &= bool((hits == 1).all())  # every destination row written exactly once
                out = buf.reshape(B, F, D)
            # a4 fused (k_push_grad): grad row (b, f) of this rank goes to every owner o with
            # jmap[o][f] = j >= 0, at row (rank * B + b) * Fo[o] + j of o's pooled buffer
            grad = gen.grad_values(cfg.seed, 0, world * B, F, D, 0)[rank * B:(rank + 1) * B]
            jmap = [{f: j for j, f in enumerate(feats_of[o])} for o in range(world)]
            idx_to, rows_to = [], []
            for o in range(world):
                pairs = [((rank * B + b) * len(feats_of[o]) + jmap[o][f], grad[b, f]) for b in range(B)
                         for f in range(F) if f in jmap[o]]
                idx_to.append(np.array([i for i, _ in pairs], dtype=np.int64))
                rows_to.append(np.array([g for _, g in pairs], dtype=np.float32).reshape(-1))
            r_idx = a2a(idx_to, np.int64)
            r_rows = a2a(rows_to, np.float32)
            gbuf = np.full((world * B * Fr, D), np.nan, dtype=np.float32)
            ghits = np.zeros(world * B * Fr, dtype=np.int64)
            for s_ in range(world):
                gbuf[r_idx[s_]] = r_rows[s_].reshape(-1, D)
                np.add.at(ghits, r_idx[s_], 1)
            ok &= bool((ghits == 1).all())
            # the owner's recorded occurrences point at grad row (src * B + b) * Fr + j: it must
            # hold source src's gradient of (b, feats_of[rank][j])
            gsrc = [gen.grad_values(cfg.seed, 0, world * B, F, D, 0)[s_ * B:(s_ + 1) * B] for s_ in range(world)]
            g3 = gbuf.reshape(world, B, Fr, D)
            for s_ in range(world):
                for j, f in enumerate(feats_of[rank]):
                    ok &= bool((g3[s_, :, j] == gsrc[s_][:, f]).all())
        # reference: unsharded oracle on this rank's batch
        pb = O.Problem(rows, D, ft)
        ref, _ = O.forward(pb, Wfull, ids, off, B)
        mag, _ = O.forward(pb, np.abs(Wfull), ids, off, B)
        ok &= bool((np.abs(out - ref) <= 1e-5 * mag + 1e-30).all())
        if sharding == "table":
            ok &= bool((out == ref).all())
        oks = [torch.zeros(1) for _ in range(world)]
        dist.all_gather(oks, torch.tensor([1.0 if ok else 0.0]))
        if rank == 0:
            q.put(all(x.item() == 1.0 for x in oks))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(traceback.format_exc())


@pytest.mark.parametrize("mode", ["collective", "p2p"])
@pytest.mark.parametrize("sharding", ["table", "row"])
def test_exchange_protocol_gloo_matches_unsharded_oracle(sharding, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_protocol_worker, args=(r, 2, port, sharding, q, mode)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
    assert res is True, res


# ---------------------------------------------------------------------------------------
# sync-free a1 (exchange.cu k_push_ids / k_compact_ids / k_recv_guard): the count matrix is
# all-gathered (device-side in the library); keys land compacted in SOURCE order -- fused: each
# source stores at base = sum of lower ranks' counts for that owner; collective: capacity-padded
# [W][pair_cap] slots then compaction -- and an overflow is decided identically on every rank.
# ---------------------------------------------------------------------------------------

def _a1_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        rng = np.random.default_rng(100 + rank)
        # this rank's keys per owner (variable counts, one owner much hotter)
        counts = [int(rng.integers(0, 50)) + (120 if o == 1 else 0) for o in range(world)]
        keys = [rng.integers(0, 1 << 20, counts[o]).astype(np.int64) + (o << 24) for o in range(world)]
        cnt = torch.tensor(counts, dtype=torch.int64)
        allc = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, cnt)
        M = torch.stack(allc).numpy()  # M[s][o] = keys rank s sends owner o
        # reference: the variable-size all-to-all, sources concatenated in rank order
        sz = torch.tensor(counts, dtype=torch.int64)
        rsz = torch.zeros(world, dtype=torch.int64)
        dist.all_to_all_single(rsz, sz)
        flat = torch.from_numpy(np.concatenate(keys))
        recv = torch.zeros(int(rsz.sum()), dtype=torch.int64)
        dist.all_to_all_single(recv, flat, rsz.tolist(), sz.tolist())
        ref = recv.numpy()
        ok = bool((rsz.numpy() == M[:, rank]).all())
        # fused: source s writes its keys for owner o at base_o = sum_{s' < s} M[s'][o]
        tot_me = int(M[:, rank].sum())
        buf = np.full(tot_me, -1, dtype=np.int64)
        msgs = []
        for o in range(world):
            base = int(M[:rank, o].sum())
            msgs.append(np.concatenate([[base], keys[o]]).astype(np.int64))
        lens_ = torch.tensor([len(m) for m in msgs], dtype=torch.int64)
        rl = torch.zeros(world, dtype=torch.int64)
        dist.all_to_all_single(rl, lens_)
        rbuf = torch.zeros(int(rl.sum()), dtype=torch.int64)
        dist.all_to_all_single(rbuf, torch.from_numpy(np.concatenate(msgs)), rl.tolist(), lens_.tolist())
        for m in torch.split(rbuf, rl.tolist()):
            m = m.numpy()
            buf[m[0]:m[0] + len(m) - 1] = m[1:]
        ok &= bool((buf == ref).all())
        # collective: [W][pair_cap] padded slots, then compaction in source order
        pair_cap = 200
        send = np.full((world, pair_cap), -7, dtype=np.int64)
        for o in range(world):
            send[o, :counts[o]] = keys[o]
        pad = torch.zeros(world * pair_cap, dtype=torch.int64)
        dist.all_to_all_single(pad, torch.from_numpy(send.ravel()))
        pad = pad.numpy().reshape(world, pair_cap)
        comp = np.concatenate([pad[s, :M[s, rank]] for s in range(world)])
        ok &= bool((comp == ref).all())
        # overflow: owner 1 is over a capacity below its total -> every rank discards
        for cap, pcap in ((int(M[:, 1].sum()) - 1, 0), (10 ** 9, int(M.max()) - 1), (10 ** 9, 0)):
            over = bool((M.sum(0) > cap).any() or (pcap and (M > pcap).any()))
            flags = [torch.zeros(1) for _ in range(world)]
            dist.all_gather(flags, torch.tensor([1.0 if over else 0.0]))
            ok &= len({f.item() for f in flags}) == 1  # the same verdict everywhere
            ok &= over == (cap < 10 ** 9 or pcap > 0)
        oks = [torch.zeros(1) for _ in range(world)]
        dist.all_gather(oks, torch.tensor([1.0 if ok else 0.0]))
        if rank == 0:
            q.put(all(x.item() == 1.0 for x in oks))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put(traceback.format_exc())


@pytest.mark.parametrize("world", [2, 3])
def test_syncfree_a1_compaction_and_overflow_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_a1_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
    assert res is True, res
