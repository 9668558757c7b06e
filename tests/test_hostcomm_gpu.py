"""The sharded path across REAL process boundaries on one GPU (PAPER.md:576 exchange):
two processes (torch.multiprocessing, gloo on 127.0.0.1), one rank each, both on cuda:0,
talking through the host transport (EMB_F_HOSTCOMM: every collective drains the stream and
moves its bytes through host memory with a gloo all-gather; no kernel ever waits on another
rank's kernel -- two processes time-sliced on one GPU cannot guarantee co-scheduling).

What this exercises that the in-process loopback cannot: the CUDA IPC mapping of another
process's workspace allocation (cuMemGetAddressRange base + cudaIpcGetMemHandle +
cudaIpcOpenMemHandle), the fused exchange's peer stores into that mapping (a1 key push, a3
pooled rows, a4 grad rows) followed by a system-scope fence and a barrier, and the rank-
ordered global norm -- against the unsharded oracle on the global batch."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_check(rank, world, sharding, p2p):
    """One rank of the check (the process group is up): two steps of forward -> q8 forward ->
    backward through the host transport on cuda:0, against the oracle on the global batch.
    Returns {check: bool}.  Also run by tools/hostcomm_check.py under torchrun."""
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    import oracle as O
    from helpers import S_close, cond_close, dense_tables, init_tables_host, w_close
    from paper_2402_06859_b200 import HostComm, ShardedEmbedding
    from workload import configs, gen
    from test_sharded_gpu import global_batch
    dev = torch.device("cuda:0")
    rows = [3000, 1200, 500, 77, 2000]
    ft = [0, 1, 2, 3, 4, 0, 1]
    cfg = configs.Config("proc", rows, 32, [(t, ("range", 0, 12)) for t in ft], 64, seed=53)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    steps = 2
    per = [[gen.make_batch(rows, cfg.features, B, cfg.seed + 10 * k + r, 0) for r in range(world)]
           for k in range(steps)]
    nnz_max = max(len(i) for bk in per for i, _ in bk)
    gshift = gen.grad_shift_for(world * nnz_max, D)
    grads = [gen.grad_values(cfg.seed, k, world * B, F, D, gshift) for k in range(steps)]
    hc = HostComm()
    e = ShardedEmbedding(rows, D, ft, max_nnz=nnz_max, max_batch=B, max_recv_nnz=world * nnz_max, device=dev,
                         stream=torch.cuda.Stream(), rank=rank, world_size=world, sharding=sharding,
                         host_comm=hc, p2p=p2p, q8=True, requant=True)
    init_tables_host(e, cfg)
    e.quantize()
    torch.cuda.synchronize()
    outs, q8s = [], []
    with torch.cuda.stream(e.stream):
        for k in range(steps):
            ids, off = per[k][rank]
            ids_d, off_d = torch.from_numpy(ids).to(dev), torch.from_numpy(off).to(dev)
            outs.append(e.forward(ids_d, off_d, B).clone())
            q8s.append(e.forward_q8(ids_d, off_d, B).clone())
            e.backward_adagrad(torch.from_numpy(grads[k][rank * B:(rank + 1) * B].copy()).to(dev), 0.05)
    st = e.sync()
    ok = {"status": st == 0}
    # the oracle, step by step on the global batch (every rank computes it)
    pb = O.Problem(rows, D, ft)
    W0 = dense_tables(cfg)
    Wo = W0.copy()
    A = np.full(cfg.total_rows, 0.1, dtype=np.float32)
    fwd_ok, q8_ok = True, True
    for k in range(steps):
        ids_g, off_g = global_batch(per[k], F, B)
        mag, _ = O.forward(pb, np.abs(Wo), ids_g, off_g, world * B)
        Wq = Wo.copy()
        r_or = O.train_step(pb, Wo, A, ids_g, off_g, world * B, grads[k], 0.05, 1e-7, 1.0)
        sl = slice(rank * B, (rank + 1) * B)
        got = outs[k].cpu().numpy()
        fwd_ok &= bool(cond_close(got, r_or["out"][sl], mag[sl]).all())
        if sharding == "table":
            fwd_ok &= bool((got == r_or["out"][sl]).all())
        if k > 0:  # (later steps read rows re-quantized from GPU-updated rows: 1-ulp codes)
            continue
        codes, mid, sc, _ = O.quantize(Wq)
        ref_q8, _ = O.forward_q8(pb, codes, mid, sc, ids_g, off_g, world * B)
        deq = np.abs(mid.astype(np.float64))[:, None] + np.abs(codes.astype(np.float64) * sc[:, None])
        magq, _ = O.forward(pb, deq.astype(np.float32), ids_g, off_g, world * B)
        q8_ok &= bool(cond_close(q8s[k].cpu().numpy(), ref_q8[sl], magq[sl]).all())
    ok["forward"] = fwd_ok
    ok["q8"] = q8_ok
    S_mine = e.last_stats()[0]
    Ss = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(Ss, torch.tensor([S_mine], dtype=torch.float64))
    ok["norm_same_on_ranks"] = all(float(x) == S_mine for x in Ss)
    ok["norm"] = S_close(S_mine, r_or["S"])
    base = np.concatenate([[0], np.cumsum(rows)])
    rows_ok = True
    for t, R in enumerate(rows):
        lo, hi = int(e.row_lo[t]), int(e.row_hi[t])
        if e.local_base[t] < 0 or hi <= lo:
            continue
        w, a = e.read_rows(t, np.arange(lo, hi))
        s = slice(base[t] + lo, base[t] + hi)
        rows_ok &= bool((np.abs(a - A[s]) <= 1e-6 * A[s]).all())
        rows_ok &= bool(w_close(w, Wo[s], W0[s], np.abs(Wo[s] - W0[s]) + 1e-3).all())
    ok["rows"] = rows_ok
    dist.barrier()  # every rank is done with the peers' mappings
    e.close()
    dist.barrier()
    return ok


def _worker(rank, world, port, sharding, p2p, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put((rank, run_check(rank, world, sharding, p2p)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("p2p", [True, False])
@pytest.mark.parametrize("sharding", ["row", "table"])
def test_two_processes_one_gpu_match_oracle(gpu, sharding, p2p):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, sharding, p2p, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
    for r in range(2):
        assert isinstance(res[r], dict), res[r]
        assert all(res[r].values()), (r, res[r])
