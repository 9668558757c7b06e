"""B200-native LiRank (arXiv 2402.06859) sparse-embedding hot path.

The product is the sm_100a C-ABI library ``liblirank_emb.so`` (include/lirank_emb.h);
this package is its thin binding.  It never imports ``oracle/`` and has no CPU
fallback: without the library or a CUDA device, compute calls raise.
"""
from ._lib import EmbError, load  # noqa: F401
from .embedding import HostComm, LoopbackHub, ShardedEmbedding, nccl_unique_id  # noqa: F401
from . import qr  # noqa: F401

__all__ = ["ShardedEmbedding", "LoopbackHub", "HostComm", "nccl_unique_id", "EmbError", "load", "qr"]
