"""NEXT-1 binding: unlimited-dictionary ids -- argument marshalling only.

``hash_ids`` (MurmurHash3 x64-128, seed 0, h1 of each id string) and ``qr_expand`` (the
int64 split into B / C, quotient/remainder rows of one concatenated QR table) run in
``liblirank_emb.so`` (``csrc/qr.cu``); see include/lirank_emb.h for the layout.  The
expanded ids/offsets feed ``ShardedEmbedding.forward`` / ``backward_adagrad`` unchanged
(SUM pooling over the expanded rows is the paper's sum aggregation)."""
from typing import Optional, Sequence, Tuple

import torch

from . import _lib as L


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def pack_strings(strings: Sequence[str], device) -> Tuple[torch.Tensor, torch.Tensor]:
    """UTF-8 bytes of the strings, concatenated, + int64 offsets [n+1], on `device`."""
    enc = [s.encode("utf-8") if isinstance(s, str) else bytes(s) for s in strings]
    off = torch.zeros(len(enc) + 1, dtype=torch.int64)
    if enc:
        off[1:] = torch.cumsum(torch.tensor([len(e) for e in enc], dtype=torch.int64), 0)
    data = torch.frombuffer(bytearray(b"".join(enc)) or bytearray(1), dtype=torch.uint8)
    return data.to(device), off.to(device)


def hash_ids(data: torch.Tensor, str_offsets: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """int64 ids (uint64 bits in an int64 tensor) of the strings data[off[i]:off[i+1]]."""
    assert data.dtype == torch.uint8 and str_offsets.dtype == torch.int64
    n = str_offsets.numel() - 1
    if out is None:
        out = torch.empty(max(n, 0), dtype=torch.int64, device=str_offsets.device)
    L.check(L.load().emb_hash_ids(_ptr(data), _ptr(str_offsets), n, _ptr(out), _stream(str_offsets.device)),
            "emb_hash_ids")
    return out


def qr_rows(R: int, Q: int, dual: bool) -> int:
    return int(L.load().emb_qr_rows(int(R), int(Q), 1 if dual else 0))


def qr_expand(hashes: torch.Tensor, offsets: torch.Tensor, R: int, Q: int, dual: bool,
              ids_out: Optional[torch.Tensor] = None,
              offsets_out: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Rows of the concatenated QR table for every hashed id (k = 2 or 4 per id) and the
    bag offsets scaled by k."""
    assert hashes.dtype == torch.int64 and offsets.dtype == torch.int32
    k = 4 if dual else 2
    nnz, nbags = hashes.numel(), offsets.numel() - 1
    dev = offsets.device
    if ids_out is None:
        ids_out = torch.empty(k * nnz, dtype=torch.int32, device=dev)
    if offsets_out is None:
        offsets_out = torch.empty(nbags + 1, dtype=torch.int32, device=dev)
    L.check(L.load().emb_qr_expand(_ptr(hashes), _ptr(offsets), nbags, nnz, int(R), int(Q), 1 if dual else 0,
                                   _ptr(ids_out), _ptr(offsets_out), _stream(dev)), "emb_qr_expand")
    return ids_out, offsets_out
