"""fp64 block-sparse attention on the GPU with torch (TEST INFRASTRUCTURE):
the reference's sparse_attention (ref executor.py:104-158) restated as one
softmax over each query block's selected keys, for checking full outputs at
benchmark scale where the CPU oracle is too slow.  It is itself checked
against the oracle (oracle/blocksift_port.py sparse_attention) on sampled
query blocks by the tests that use it."""

from __future__ import annotations

import math

import numpy as np
import torch


def block_sparse_fp64(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, grid: np.ndarray, blk: int = 128,
                      qblocks=None) -> torch.Tensor:
    """q, k, v [S, d] CUDA (any float dtype, upcast to fp64); grid [nb, nb]
    bool.  Returns fp64 [S, d] (rows of query blocks not in `qblocks` NaN)."""
    S, d = q.shape
    qd, kd, vd = q.double(), k.double(), v.double()
    nb = grid.shape[0]
    out = torch.full((S, d), float("nan"), dtype=torch.float64, device=q.device)
    scale = 1.0 / math.sqrt(d)
    ar = np.arange(blk)
    for qb in (range(nb) if qblocks is None else qblocks):
        a, b = qb * blk, min(S, (qb + 1) * blk)
        kbs = np.flatnonzero(grid[qb])
        keys = (kbs[:, None] * blk + ar[None, :]).ravel()
        keys = torch.from_numpy(keys[keys < S]).to(q.device)
        s = (qd[a:b] * scale) @ kd[keys].T
        rows = torch.arange(a, b, device=q.device)
        s = s.masked_fill(keys[None, :] > rows[:, None], float("-inf"))
        out[a:b] = torch.softmax(s, dim=1) @ vd[keys]
    return out
