"""NEXT-2 oracle -- TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench cpu legs).

The end-to-end Feed train step (pooled sparse embeddings concatenated with
dense features into an MLP of "4 connected layers, each with output dimension of 100";
PAPER.md:17: AdaGrad with the global gradient clipped to unit norm) in plain PyTorch CPU
float64 for the dense tower, and the C oracle (oracle.c) for everything sparse:

  pooled  = ora_forward (fp32, bag order)                                  a2
  loss    = mean BCE-with-logits(MLP([pooled | dense]), labels)
  grads   = autograd (float64)                                             dL/dpooled, dL/dW_l
  S       = sum_rows G^2 (ora_train_step, fp64) + sum_l |dL/dW_l|^2        P:17, reading 11
  c       = clip factor (ora_clip_factor);  sparse rows: ora_train_step    a5-a8
  dense   : g <- c g;  A <- A + g^2;  w <- w - lr g / (sqrt(A) + eps)      reading 9 (float64)

The upstream gradient handed to the sparse oracle is the float64 dL/dpooled rounded to fp32
(the library receives fp32).  Pinned in tests/test_feed_oracle.py.
"""
import numpy as np

from . import forward, train_step


def tower_forward(x, params):
    """params = [W1, b1, ..., W5, b5] (torch float64, Linear layout [out, in])."""
    import torch
    h = x
    for i in range(0, len(params) - 2, 2):
        h = torch.relu(h @ params[i].T + params[i + 1])
    return (h @ params[-2].T + params[-1]).squeeze(1)


def feed_train_step(pb, W, A, ids, offsets, B, dense_x, labels, params, accs, lr, eps, max_norm,
                    mode="rowwise"):
    """In place on W, A (numpy fp32).  params/accs: lists of numpy float64 arrays, updated in
    place.  Returns dict(loss, S, c, dense_sq, grad_pooled)."""
    import torch
    out, _ = forward(pb, W, ids, offsets, B)
    p = torch.tensor(out, dtype=torch.float64, requires_grad=True)
    x = torch.cat([p.reshape(B, -1), torch.tensor(np.asarray(dense_x), dtype=torch.float64)], dim=1)
    ws = [torch.tensor(q, dtype=torch.float64, requires_grad=True) for q in params]
    logits = tower_forward(x, ws)
    y = torch.tensor(np.asarray(labels), dtype=torch.float64)
    loss = torch.nn.functional.binary_cross_entropy_with_logits(logits, y)
    grads = torch.autograd.grad(loss, [p] + ws)
    g_dense = [g.detach().numpy() for g in grads[1:]]
    dense_sq = float(sum(np.sum(g * g) for g in g_dense))
    gp = grads[0].detach().numpy().astype(np.float32)
    r = train_step(pb, W, A, ids, offsets, B, gp, lr, eps, max_norm, mode=mode, extra_sq_norm=dense_sq,
                   want_out=False)
    c = float(r["c"]) if not r["nonfinite"] else 0.0
    for w, a, g in zip(params, accs, g_dense):
        gc = g * c
        a += gc * gc
        w -= lr * gc / (np.sqrt(a) + eps)
    return {"loss": float(loss.item()), "S": r["S"], "c": r["c"], "dense_sq": dense_sq, "grad_pooled": gp}
