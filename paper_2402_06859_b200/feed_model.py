"""NEXT-2: the end-to-end Feed train step -- pooled sparse embeddings (the sm_100a library)
concatenated with dense features and passed through the paper's MLP, "4 connected layers,
each with output dimension of 100", trained with AdaGrad under ONE global
gradient norm clipped to unit norm over sparse + dense gradients.

The dense tower is plain PyTorch (cuBLAS GEMMs in fp32, TF32 off: a library GEMM, not the
hot path this package implements).  Everything sparse runs in ``liblirank_emb.so``.  The
step has no host synchronisation: the dense squared norm is handed to the library on the
device (``emb_backward_adagrad_dev``), the library returns the clip factor on the device,
and the dense AdaGrad update reads it there.  The a5 dedup the forward launched on the
library's side stream overlaps the tower's forward and backward.

Data parallel (world_size > 1, "Other layers ... processed in a data parallel
way"): every rank holds the same tower and its local batch; the loss each rank
differentiates is its local mean / W, so the sum over ranks is the global-batch mean loss.
The dense gradients are summed over ranks (emb_allreduce_f32, on the library stream and
transport) BEFORE their squared norm is formed, so every rank folds the same dense term into
the one global norm and applies the same dense update.
"""
from typing import List, Optional

import torch

from .embedding import ShardedEmbedding


class FeedTower(torch.nn.Module):
    """x = [pooled (B x F*D) | dense (B x Dd)] -> 4 x (Linear(100) + ReLU) -> Linear(1)."""

    def __init__(self, in_dim: int, width: int = 100, depth: int = 4):
        super().__init__()
        layers: List[torch.nn.Module] = []
        d = in_dim
        for _ in range(depth):
            layers += [torch.nn.Linear(d, width), torch.nn.ReLU()]
            d = width
        layers.append(torch.nn.Linear(d, 1))
        self.net = torch.nn.Sequential(*layers)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return self.net(x).squeeze(1)


class FeedModel:
    """ShardedEmbedding + FeedTower with one clipped AdaGrad step over both.

    Dense AdaGrad matches the sparse one's element-wise form (SURVEY §8(c) reading 9):
    A' = A + g^2, w' = w - lr * g / (sqrt(A') + eps), A0 = init_accumulator, g = c * grad."""

    def __init__(self, emb: ShardedEmbedding, dense_dim: int, lr: float = 0.05,
                 init_accumulator: float = 0.1, eps: float = 1e-7, seed: int = 0):
        self.emb = emb
        self.F, self.D, self.Dd = emb.num_features, emb.dim, dense_dim
        dev = emb.device
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.tower = FeedTower(self.F * self.D + dense_dim)
        for p in self.tower.parameters():  # seeded init (independent of torch's global RNG)
            with torch.no_grad():
                p.copy_((torch.rand(p.shape, generator=g) - 0.5) * (2.0 / max(p.shape[-1], 1) ** 0.5))
        self.tower.to(dev)
        self.params = list(self.tower.parameters())
        self.acc = [torch.full_like(p, init_accumulator) for p in self.params]
        self.lr, self.eps = float(lr), float(eps)
        self.c = torch.zeros(1, dtype=torch.float32, device=dev)
        self.S = torch.zeros(1, dtype=torch.float64, device=dev)
        self.dense_sq = torch.zeros(1, dtype=torch.float64, device=dev)
        self.world = int(emb.cfg.world_size)
        self._pooled: Optional[torch.Tensor] = None

    def train_step(self, ids: torch.Tensor, offsets: torch.Tensor, batch: int, dense_x: torch.Tensor,
                   labels: torch.Tensor) -> torch.Tensor:
        """One step; returns the (device) mean BCE loss.  All work is enqueued on emb.stream."""
        emb = self.emb
        with torch.cuda.stream(emb.stream):
            if self._pooled is None or self._pooled.shape[0] != batch:
                self._pooled = torch.empty((batch, self.F, self.D), device=emb.device)
            pooled = emb.forward(ids, offsets, batch, out=self._pooled)           # a2 (+a5 on side stream)
            p = pooled.detach().requires_grad_(True)
            x = torch.cat([p.view(batch, self.F * self.D), dense_x], dim=1)
            logits = self.tower(x)
            loss = torch.nn.functional.binary_cross_entropy_with_logits(logits, labels)
            # local mean / W: summed over the ranks this is the global-batch mean loss
            grads = torch.autograd.grad(loss / self.world if self.world > 1 else loss, [p] + self.params)
            g_pooled, g_dense = grads[0].contiguous(), list(grads[1:])
            flat = torch.cat([g.reshape(-1) for g in g_dense])
            if self.world > 1:  # data-parallel dense side: one all-reduce of all tower grads
                emb.allreduce_(flat)
                g_dense = [f.view_as(g) for f, g in zip(torch.split(flat, [g.numel() for g in g_dense]), g_dense)]
            fd = flat.double()
            torch.sum(fd * fd, dim=0, keepdim=True, out=self.dense_sq)
            emb.backward_adagrad_dev(g_pooled, self.lr, extra_sq_norm=self.dense_sq, clip_out=self.c,
                                     sq_norm_out=self.S)                       # a6-a8, global clip
            # c = -1: the global norm was not finite (possibly because a dense gradient is
            # inf/NaN) -- the sparse update was skipped, so skip the dense one too: the
            # scaled gradient is masked to 0 (not multiplied by 0, which keeps a NaN)
            ok = self.c >= 0
            c = self.c.reshape(())
            with torch.no_grad():  # multi-tensor (foreach) AdaGrad: a few launches for all layers
                gc = [torch.where(ok, g * c, torch.zeros((), device=g.device)) for g in g_dense]
                torch._foreach_addcmul_(self.acc, gc, gc)
                den = torch._foreach_sqrt(self.acc)
                torch._foreach_add_(den, self.eps)
                torch._foreach_mul_(gc, self.lr)
                torch._foreach_div_(gc, den)
                torch._foreach_sub_(self.params, gc)
        return loss.detach()
