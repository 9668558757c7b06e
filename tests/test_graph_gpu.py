"""CUDA-graph capture of a whole W = 1 training step (a2 forward -> a10 q8 forward -> a5-a8
backward with the fused a9 re-quantization) through the C ABI.

A W = 1 step has no host synchronisation (U, the clip factor and every count stay on the
device) and the look-back epochs of the radix sort / run-length encode live in device memory
(advanced by a kernel in stream order, not baked into launch parameters), so a step captured
once can be replayed: graph replays must reproduce eager execution bit for bit, also when the
same graph is replayed again (fresh epochs per replay) and with the a5 dedup forked onto the
library's side stream inside the capture."""
import numpy as np
import pytest

from helpers import init_tables_host
from workload import configs, gen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_graph_replay_matches_eager(gpu):
    from paper_2402_06859_b200 import ShardedEmbedding
    rows = [200_000, 30_000, 5000]
    ft = [0, 1, 0, 2, 1]
    cfg = configs.Config("graph", rows, 64, [(t, ("range", 0, 40)) for t in ft], 2048, seed=17)
    B, F, D = cfg.batch, cfg.num_features, cfg.dim
    nb = 3
    batches = [gen.make_batch(rows, cfg.features, B, cfg.seed, k, alpha=1.05) for k in range(nb)]
    nnz_max = max(len(i) for i, _ in batches)
    gshift = gen.grad_shift_for(nnz_max, D)
    dev_in = [(torch.from_numpy(i).cuda(), torch.from_numpy(o).cuda(),
               torch.from_numpy(gen.grad_values(cfg.seed, k, B, F, D, gshift)).cuda())
              for k, (i, o) in enumerate(batches)]
    embs, outs = [], []
    for _ in range(2):
        s = torch.cuda.Stream()
        e = ShardedEmbedding(rows, D, ft, max_nnz=nnz_max, max_batch=B, q8=True, requant=True,
                             device=gpu, stream=s)
        init_tables_host(e, cfg)
        e.quantize()
        embs.append(e)
        outs.append([(torch.empty((B, F, D), device=gpu), torch.empty((B, F, D), device=gpu))
                     for _ in range(nb)])
    torch.cuda.synchronize()

    def step(e, k, out):
        ids_d, off_d, g = dev_in[k]
        e.forward(ids_d, off_d, B, out=out[0])
        e.forward_q8(ids_d, off_d, B, out=out[1])
        e.backward_adagrad(g, 0.05)

    eager, graphed = embs
    # one eager warm-up step on both (first-use attributes, lazy module loading)
    for e, o in zip(embs, outs):
        with torch.cuda.stream(e.stream):
            step(e, 0, o[0])
    torch.cuda.synchronize()
    # eager: batches 1, 2, 0, 1
    order = [1, 2, 0, 1]
    ref = []
    with torch.cuda.stream(eager.stream):
        for k in order:
            step(eager, k, outs[0][k])
            eager.stream.synchronize()
            ref.append((outs[0][k][0].clone(), outs[0][k][1].clone()))
    assert eager.sync() == 0
    # graphed: one graph per batch, captured on the library stream, replayed in the same order
    graphs = {}
    for k in (1, 2, 0):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=graphed.stream):
            step(graphed, k, outs[1][k])
        graphs[k] = g
    torch.cuda.synchronize()
    got = []
    for k in order:  # graph 1 is replayed twice
        with torch.cuda.stream(graphed.stream):
            graphs[k].replay()
        graphed.stream.synchronize()
        got.append((outs[1][k][0].clone(), outs[1][k][1].clone()))
    assert graphed.sync() == 0
    for (a, aq), (b, bq) in zip(ref, got):
        assert torch.equal(a, b) and torch.equal(aq, bq)
    assert torch.equal(eager.weights, graphed.weights)
    assert torch.equal(eager.accum_buf, graphed.accum_buf)
    assert torch.equal(eager.codes_buf, graphed.codes_buf)
    for e in embs:
        e.close()
