"""NEXT-1 GPU parity: MurmurHash3 id hashing and QR expansion on sm_100a (csrc/qr.cu, through
the C ABI) vs the CPU oracle, bit-exact; and a QR-feature training step (hash -> expand ->
a2 -> a5-a8) vs the oracle on the same strings."""
import numpy as np
import pytest

import oracle as O
from helpers import cond_close, dense_tables, init_tables_host, w_close
from workload import configs, gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def random_strings(rng, n, maxlen=70):
    out = []
    for i in range(n):
        k = i % 4
        if k == 0:
            out.append(f"member:{int(rng.integers(0, 10**9))}")
        elif k == 1:
            out.append(bytes(rng.integers(0, 256, size=int(rng.integers(0, maxlen)), dtype=np.uint8).tolist()))
        elif k == 2:
            out.append("hashtag:#" + "é" * int(rng.integers(0, 20)))
        else:
            out.append("")
    return out


def test_hash_ids_bit_exact(gpu):
    from paper_2402_06859_b200 import qr
    rng = np.random.default_rng(11)
    strings = random_strings(rng, 20_000)
    data, off = qr.pack_strings(strings, gpu)
    h = qr.hash_ids(data, off)
    torch.cuda.synchronize()
    ref = O.hash_ids(strings)
    assert (h.cpu().numpy().view(np.uint64) == ref).all()
    # every length 0..255 (all tails, multi-block), against the oracle's digests
    key = bytes(range(256))
    strings = [key[:i] for i in range(256)]
    data, off = qr.pack_strings(strings, gpu)
    h = qr.hash_ids(data, off).cpu().numpy().view(np.uint64)
    assert [int(x) for x in h] == [O.murmur3_x64_128(s, 0)[0] for s in strings]


@pytest.mark.parametrize("n", [1, 31, 33, 1000, 32 * 4737 + 17])
def test_hash_ids_ragged_counts(gpu, n):
    """String counts that leave the last warp partly empty (regression: dead lanes must not
    read outside the warp's staged bytes)."""
    from paper_2402_06859_b200 import qr
    rng = np.random.default_rng(n)
    strings = [f"member:{int(x)}" for x in rng.integers(0, 10**6, size=n)]
    data, off = qr.pack_strings(strings, gpu)
    h = qr.hash_ids(data, off).cpu().numpy().view(np.uint64)
    k = min(n, 3000)
    assert (h[-k:] == O.hash_ids(strings[-k:])).all()


@pytest.mark.parametrize("dual", [False, True])
@pytest.mark.parametrize("R,Q", [(1000, -(-(1 << 32) // 1000)), (97, 1000), (1, 7), ((1 << 31) - 5, 3)])
def test_qr_expand_bit_exact(gpu, dual, R, Q):
    from paper_2402_06859_b200 import qr
    rng = np.random.default_rng(R % 1000 + Q % 1000)
    if 2 * (Q + R) >= (1 << 31) and dual:
        pytest.skip("rows do not fit int32")
    nb = 777
    lens = rng.integers(0, 9, size=nb)
    lens[::50] = 0
    off = np.zeros(nb + 1, dtype=np.int32)
    off[1:] = np.cumsum(lens)
    nnz = int(off[-1])
    h = rng.integers(0, 2**63, size=nnz, dtype=np.int64).view(np.uint64)
    h[:5] = [0, 2**64 - 1, 2**32 - 1, 2**32, 4_000_001]
    ids_ref, off_ref = O.qr_expand(h, off, R, Q, dual)
    hd = torch.from_numpy(h.view(np.int64)).to(gpu)
    od = torch.from_numpy(off).to(gpu)
    ids, offs = qr.qr_expand(hd, od, R, Q, dual)
    assert (ids.cpu().numpy() == ids_ref).all() and (offs.cpu().numpy() == off_ref).all()
    # misaligned output (scalar-store path)
    k = 4 if dual else 2
    buf = torch.zeros(k * nnz + 1, dtype=torch.int32, device=gpu)
    ids2, _ = qr.qr_expand(hd, od, R, Q, dual, ids_out=buf[1:])
    assert (ids2.cpu().numpy() == ids_ref).all()
    assert qr.qr_rows(R, Q, dual) == O.qr_rows(R, Q, dual)


def test_qr_expand_rejects_oversized_tables(gpu):
    from paper_2402_06859_b200 import EmbError, qr
    h = torch.zeros(4, dtype=torch.int64, device=gpu)
    o = torch.tensor([0, 4], dtype=torch.int32, device=gpu)
    with pytest.raises(EmbError):
        qr.qr_expand(h, o, 1000, 1 << 30, True)
    with pytest.raises(EmbError):
        qr.qr_expand(h, o, 0, 10, False)


def test_qr_feature_train_step_matches_oracle(gpu):
    """Strings -> MurmurHash3 -> QR rows of two dual QR tables -> a2 SUM pooling (the paper's
    sum aggregation) -> a5-a8, GPU vs oracle on the same strings."""
    from paper_2402_06859_b200 import ShardedEmbedding, qr
    rng = np.random.default_rng(5)
    D, B = 32, 96
    qr_cfg = [(97, 1000), (13, 500)]  # (R, Q) of table 0 (member) and 1 (hashtag); dual
    rows = [O.qr_rows(R, Q, True) for R, Q in qr_cfg]
    ft = [0, 0, 1]  # viewer actors, actor, hashtags
    F = len(ft)
    cfg = configs.Config("qr", rows, D, [(t, ("range", 0, 6)) for t in ft], B, seed=9)
    strings, lens = [], []
    for f in range(F):
        for b in range(B):
            L = int(rng.integers(0, 7))
            lens.append(L)
            pool = 300 if ft[f] == 0 else 40  # repeats -> duplicate QR rows
            strings += [(f"member:{int(rng.integers(0, pool))}" if ft[f] == 0 else f"hashtag:{int(rng.integers(0, pool))}")
                        for _ in range(L)]
    off = np.zeros(F * B + 1, dtype=np.int32)
    off[1:] = np.cumsum(lens)
    # oracle: hash, expand per table, train step on the expanded bags
    h_ref = O.hash_ids(strings)
    ids_x = np.zeros(4 * len(strings), dtype=np.int32)
    off_x = np.zeros_like(off)
    for f0, f1, t in [(0, 2, 0), (2, 3, 1)]:
        a, b = off[f0 * B], off[f1 * B]
        sub_off = off[f0 * B:f1 * B + 1]
        i_, o_ = O.qr_expand(h_ref[a:b], sub_off, *qr_cfg[t], True)
        ids_x[4 * a:4 * b] = i_
        off_x[f0 * B:f1 * B + 1] = o_
    pb = O.Problem(rows, D, ft)
    W0 = dense_tables(cfg)
    W = W0.copy()
    A = np.full(sum(rows), 0.1, dtype=np.float32)
    grad = gen.grad_values(cfg.seed, 0, B, F, D, gen.grad_shift_for(len(ids_x), D))
    r = O.train_step(pb, W, A, ids_x, off_x, B, grad, 0.05, 1e-7, 1.0)
    # GPU: the same strings through the library
    emb = ShardedEmbedding(rows, D, ft, max_nnz=len(ids_x), max_batch=B, device=gpu)
    init_tables_host(emb, cfg)
    data, soff = qr.pack_strings(strings, gpu)
    h = qr.hash_ids(data, soff)
    od = torch.from_numpy(off).to(gpu)
    ids_d = torch.empty(4 * len(strings), dtype=torch.int32, device=gpu)
    off_d = torch.empty(F * B + 1, dtype=torch.int32, device=gpu)
    for f0, f1, t in [(0, 2, 0), (2, 3, 1)]:
        a, b = int(off[f0 * B]), int(off[f1 * B])
        qr.qr_expand(h[a:b], od[f0 * B:f1 * B + 1], *qr_cfg[t], True, ids_out=ids_d[4 * a:4 * b],
                     offsets_out=off_d[f0 * B:f1 * B + 1])
    assert (ids_d.cpu().numpy() == ids_x).all() and (off_d.cpu().numpy() == off_x).all()
    out = emb.forward(ids_d, off_d, B)
    emb.backward_adagrad(torch.from_numpy(grad).to(gpu), 0.05)
    assert emb.sync() == 0
    mag, _ = O.forward(pb, np.abs(W0), ids_x, off_x, B)
    assert cond_close(out.cpu().numpy(), r["out"], mag).all()
    keys, _, _ = O.dedup(pb, ids_x, off_x, B)
    Wg = np.concatenate([emb.read_rows(t, np.arange(rows[t]))[0] for t in range(2)])
    step = np.abs(Wg - W0) + np.abs(W - W0)
    assert w_close(Wg[keys], W[keys], W0[keys], step[keys]).all()
    untouched = np.setdiff1d(np.arange(sum(rows)), keys)
    assert (Wg[untouched] == W0[untouched]).all()
