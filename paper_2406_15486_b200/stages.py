"""The three hot-path stages behind the reference's stage functions.

    sample_scores + block_reduce   (sampler.py:135-191)   -> sa_stage1
    find_k / arg_topk / select     (filtering.py:30-62)   -> sa_select
    merge_index / select_and_merge (filtering.py:198-256) -> sa_merge
    sparse_attention               (executor.py:104-158)  -> sa_sparse_forward
    flop_accounting                (executor.py:51-73)    -> integer math on the CSR

Every call is stream-ordered on the current torch stream of the tensors'
device; nothing here synchronises except the explicit host views
(`.chunks`, FlopReport fields, find_k's return value).

Selection guard.  bf16 tensor-core stage-1 scores carry ~1e-7 relative
error against the reference's fp64; whenever a (head, chunk)'s alpha cut or
top-k boundary sits closer than GUARD_EPS * total to a decision, that pair is
re-scored by the exact fp64 stage 1 and re-selected, so the selected index
sets match the reference bit-for-bit (policy "auto").  "always" runs the
exact stage 1 for every pair; "never" skips the guard.
"""

from __future__ import annotations

import ctypes

import contextlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import ChunkPlan, SparseConfig, n_blocks
from .errors import InputError
from .heads import AttentionHead, HeadBatch, HeadSet, check_status, dcall
from .masks import BlockMask, SelectedIndices, _tri

__all__ = [
    "GUARD_EPS", "SampledScores", "ChunkScores", "ReducedScores", "FlopReport", "sample_scores",
    "block_reduce", "find_k", "arg_topk", "select", "merge_index", "select_and_merge",
    "sparse_attention", "flop_accounting", "as_batch", "sampled_retained",
]

# ~7x the worst prefix-sum error of the tensor-core scores measured at 96K-128K
# (tools/guard_diag.py, profiles/r2/guard_*.txt: max |cum_tc - cum_exact| / total
# = 5.5e-8 at C3, 1.0e-7 at C4 with 10 % sampling)
GUARD_EPS = 4e-7
# The tensor-core error grows with sum_i |q_i k_i|, bounded per (head, chunk)
# by B = max ||q_r|| * max ||k_j|| / sqrt(d) (sa_stage1's logit bound).
# Measured (C3, C4 at 10 % sampling, and large-logit / heavy-sink heads up to
# B = 930): prefix-sum error / total <= 4.75e-10 * B.  GUARD_EPS applies up to
# B = GUARD_LOGIT_REF (the synthetic benchmark heads reach 305); above it the
# margin grows in proportion, keeping it >= 2.6x the worst measured error at
# every B.
GUARD_LOGIT_REF = 320.0
# Band refinement: the refined scores of tied blocks carry the relative error of
# stage 1's tensor-core row normalisers (tools/rownorm_diag.py: <= 5.2e-6 at C3 /
# C4 10 %, profiles/r2/rownorm_*.txt), scaled like GUARD_EPS with the logit
# bound; the cut between two refined scores is trusted when they differ by more
# than BAND_EPS * (s_a + s_b) (~6x the worst measured error), else the pair is
# re-scored in full.
BAND_EPS = 3e-5

_WS_CACHE: dict = {}


_WS_PRIVATE: dict = {}


def _ws_key(b: HeadBatch, blk: int, cn: int, stream: bool = True):
    # per stream: calls on different streams may run concurrently
    geom = (b.q.device, b.S, b.Hq, b.Hkv, b.d, blk, cn, b.dtype_code)
    return geom + (b.stream,) if stream else geom


def _workspace(b: HeadBatch, blk: int, cn: int) -> torch.Tensor:
    ws = _WS_PRIVATE.get(_ws_key(b, blk, cn, stream=False))
    if ws is not None:
        return ws
    key = _ws_key(b, blk, cn)
    ws = _WS_CACHE.get(key)
    if ws is None:
        nbytes = int(_lib.load().sa_workspace_bytes(b.S, b.Hq, b.Hkv, b.d, blk, cn, b.dtype_code))
        if len(_WS_CACHE) > 16:
            _WS_CACHE.clear()
        ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=b.q.device)
        _WS_CACHE[key] = ws
    return ws


@contextlib.contextmanager
def private_workspace(b: HeadBatch, blk: int, cn: int):
    """Within the block, stage calls on this geometry (on any stream) use a
    fresh workspace that is NOT shared with later calls (CUDA-graph capture:
    the graph keeps the pointer, so it must own the buffer).  Yields it."""
    geom = _ws_key(b, blk, cn, stream=False)
    nbytes = int(_lib.load().sa_workspace_bytes(b.S, b.Hq, b.Hkv, b.d, blk, cn, b.dtype_code))
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=b.q.device)
    saved = _WS_PRIVATE.get(geom)
    _WS_PRIVATE[geom] = ws
    try:
        yield ws
    finally:
        if saved is None:
            _WS_PRIVATE.pop(geom, None)
        else:
            _WS_PRIVATE[geom] = saved


def as_batch(heads, dtype=None) -> HeadBatch:
    """Accept a HeadBatch, a (q, k, v) tuple of tensors, or reference-style
    AttentionHead / HeadSet objects."""
    if isinstance(heads, HeadBatch):
        return heads
    if isinstance(heads, tuple) and len(heads) == 3:
        return HeadBatch.from_tensors(*heads)
    if isinstance(heads, (AttentionHead, HeadSet, list)):
        return HeadBatch.from_heads(heads, dtype=dtype or torch.bfloat16)
    raise InputError(f"unsupported head container {type(heads)!r}")


# ---------------------------------------------------------------- stage 1
@dataclass
class SampledScores:
    """Stage-1 handle.  The reference materialises [rows x S] probability
    rows here (sampler.py:135-149); the fused kernel never does, so this only
    binds the heads to the plan and block_reduce does the work."""

    batch: HeadBatch
    plan: ChunkPlan

    @property
    def S(self) -> int:
        return self.plan.S


def sample_scores(heads, plan: ChunkPlan) -> SampledScores:
    b = as_batch(heads)
    if plan.S != b.S:
        raise InputError(f"plan built for S={plan.S}, head has S={b.S}")
    return SampledScores(b, plan)


@dataclass(frozen=True)
class ChunkScores:
    col_scores: np.ndarray
    slash_scores: np.ndarray
    total_mass: float


@dataclass
class ReducedScores:
    """col / slash [H, cn, nb] fp64 on the device (sampler.py:152-165)."""

    S: int
    blk: int
    plan: ChunkPlan
    batch: HeadBatch
    col: torch.Tensor
    slash: torch.Tensor
    mode: str
    logit_bound: torch.Tensor | None = None  # [H, cn] fp64 (tensor mode): the guard's error scale
    row_stats: torch.Tensor | None = None    # [H*cn*blk*2] fp64 (tensor mode): sampled rows' (log2 max, sum)

    @property
    def chunks(self) -> tuple:
        """Reference-shaped per-chunk scores of head 0 (single-head use)."""
        return self.head_chunks(0)

    def head_chunks(self, h: int) -> tuple:
        col = self.col[h].cpu().numpy()
        slash = self.slash[h].cpu().numpy()
        return tuple(ChunkScores(col[c], slash[c], float(col[c].sum())) for c in range(col.shape[0]))


def _stage1(b: HeadBatch, plan: ChunkPlan, col, slash, mode: int, only=None, bound=None) -> None:
    ws = _workspace(b, plan.blk, plan.chunk_n)
    dcall(b.q.device, "sa_stage1", b.q.data_ptr(), b.k.data_ptr(), b.dtype_code, b.S, b.Hq, b.Hkv, b.d, plan.blk,
          b.group, b.q_head0, plan.chunk_n, plan.itv, col.data_ptr(), slash.data_ptr(),
          None if bound is None else bound.data_ptr(), mode, None if only is None else only.data_ptr(),
          ws.data_ptr(), ws.numel(), b.stream)


def block_reduce(samples: SampledScores, blk: int, mode: str | None = None) -> ReducedScores:
    """Fused sampled attention + column/slash block reduction.

    mode "tensor" (default for bf16): tcgen05 scores; "exact" (default for
    fp32, and available for bf16): fp64 SIMT scores."""
    b, plan = samples.batch, samples.plan
    if blk != plan.blk:
        raise InputError(f"blk={blk} differs from the plan's blk={plan.blk}")
    if mode is None:
        mode = "tensor" if b.dtype_code == _lib.SA_BF16 else "exact"
    if mode not in ("tensor", "exact"):
        raise InputError(f"unknown stage-1 mode {mode!r}")
    nb = n_blocks(b.S, blk)
    col = torch.empty((b.Hq, plan.chunk_n, nb), dtype=torch.float64, device=b.q.device)
    slash = torch.empty_like(col)
    bound = torch.empty((b.Hq, plan.chunk_n), dtype=torch.float64, device=b.q.device) if mode == "tensor" else None
    _stage1(b, plan, col, slash, _lib.SA_STAGE1_TENSOR if mode == "tensor" else _lib.SA_STAGE1_EXACT, bound=bound)
    row_stats = None
    if mode == "tensor":  # the guard's band refinement needs them after later stage-1 calls reuse the workspace
        off = int(_lib.load().sa_workspace_offset(b.S, b.Hq, b.Hkv, b.d, blk, plan.chunk_n, b.dtype_code,
                                                   _lib.SA_WS_ROW_STATS))
        rows = b.Hq * plan.chunk_n * blk
        row_stats = _workspace(b, blk, plan.chunk_n)[off: off + rows * 16].view(torch.float64).clone()
    return ReducedScores(b.S, blk, plan, b, col, slash, mode, bound, row_stats)


# ---------------------------------------------------------------- stage 2
def _vector_select(scores, alpha, k=None):
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1 or s.size == 0:
        raise InputError(f"scores must be a nonempty 1-D sequence, got shape {s.shape}")
    dev = torch.device("cuda")
    t = torch.from_numpy(s.copy()).to(dev).view(1, 1, -1)
    k_out = torch.empty((1, 1, 2), dtype=torch.int32, device=dev)
    idx = torch.empty((1, 1, 2, s.size), dtype=torch.int32, device=dev)
    k_in = None
    if k is not None:
        k_in = torch.tensor([[[k, k]]], dtype=torch.int32, device=dev)
    dcall(dev, "sa_select", t.data_ptr(), t.data_ptr(), 1, 1, s.size, alpha, alpha, 0.0, None, 1.0, None, None,
              None if k_in is None else k_in.data_ptr(), k_out.data_ptr(), idx.data_ptr(), None, 0.0,
              torch.cuda.current_stream(dev).cuda_stream)
    kk = int(k_out[0, 0, 0].item())
    return kk, tuple(int(x) for x in idx[0, 0, 0, :kk].cpu().numpy())


def find_k(scores, alpha: float) -> int:
    """Minimal quota (filtering.py:30-48), computed by the stage-2 kernel:
    descending sort, sequential fp64 cumsum, first cum >= alpha * cum[-1]."""
    if not 0.0 <= alpha <= 1.0:
        raise InputError(f"alpha must be in [0, 1], got {alpha}")
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim == 1 and (s < 0).any():
        raise InputError("scores must be nonnegative")
    return _vector_select(s, alpha)[0]


def arg_topk(scores, k: int) -> tuple:
    """k largest, ties toward the lower index, ascending (filtering.py:51-62).
    The kernel sorts by the nonnegative-score bit pattern, so scores must be
    >= 0 (all stage-1 scores are)."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1:
        raise InputError(f"scores must be 1-D, got shape {s.shape}")
    if not 0 <= k <= s.size:
        raise InputError(f"k={k} out of range for {s.size} scores")
    if k == 0:
        return ()
    if (s < 0).any():
        raise InputError("device arg_topk needs nonnegative scores")
    return _vector_select(s, 0.0, k=k)[1]


@dataclass
class Selection:
    k_sel: torch.Tensor     # int32 [H, cn, 2]
    idx_sel: torch.Tensor   # int32 [H, cn, 2, nb]
    flags: torch.Tensor | None = None  # int32 [H*cn]: pairs the guard re-scored in full (fp64)
    guard: str = "auto"
    band_pairs: torch.Tensor | None = None  # int32 [H*cn]: pairs whose tie band was refined

    def n_rescored(self) -> int:
        return 0 if self.flags is None else int(self.flags.sum().item())

    def n_band_refined(self) -> int:
        """Pairs settled by the band refinement alone (not re-scored in full)."""
        if self.band_pairs is None:
            return 0
        return int(((self.band_pairs != 0) & (self.flags == 0)).sum().item())


def select(reduced: ReducedScores, cfg: SparseConfig, guard: str = "auto",
           guard_eps: float = GUARD_EPS) -> Selection:
    """find_k + arg_topk for every (head, chunk, direction), with the
    selection guard described in the module docstring."""
    if guard not in ("auto", "always", "never"):
        raise InputError(f"unknown guard policy {guard!r}")
    b, plan = reduced.batch, reduced.plan
    H, cn, nb = b.Hq, plan.chunk_n, n_blocks(b.S, plan.blk)
    dev = b.q.device
    st = b.stream
    if guard == "always" and reduced.mode == "tensor":
        _stage1(b, plan, reduced.col, reduced.slash, _lib.SA_STAGE1_EXACT)
        reduced.mode = "exact"
    k_sel = torch.empty((H, cn, 2), dtype=torch.int32, device=dev)
    idx_sel = torch.empty((H, cn, 2, nb), dtype=torch.int32, device=dev)
    use_guard = guard == "auto" and reduced.mode == "tensor"
    flags = torch.zeros(H * cn, dtype=torch.int32, device=dev) if use_guard else None
    bound = reduced.logit_bound if use_guard else None
    band = band_pairs = None
    if use_guard:
        band = torch.empty(_lib.load().sa_band_table_len(H, cn), dtype=torch.int32, device=dev)
        band_pairs = torch.empty(H * cn, dtype=torch.int32, device=dev)
    col, slash = reduced.col.data_ptr(), reduced.slash.data_ptr()
    dcall(dev, "sa_select", col, slash, H, cn, nb, cfg.alpha_c, cfg.alpha_s, guard_eps if use_guard else 0.0,
          None if bound is None else bound.data_ptr(), GUARD_LOGIT_REF, None if flags is None else flags.data_ptr(),
          None, None, k_sel.data_ptr(), idx_sel.data_ptr(), None if band is None else band.data_ptr(), 0.0, st)
    if use_guard:
        # boundary ties alone: exact scores of the blocks within 2E of the cut,
        # then a re-select that certifies the refined cut (else the pair joins
        # the full re-score)
        ws = _workspace(b, plan.blk, plan.chunk_n)
        dcall(dev, "sa_refine_bands", b.q.data_ptr(), b.k.data_ptr(), b.dtype_code, b.S, b.Hq, b.Hkv, b.d, plan.blk,
              b.group, b.q_head0, plan.chunk_n, plan.itv, band.data_ptr(), flags.data_ptr(), band_pairs.data_ptr(),
              reduced.row_stats.data_ptr(), col, slash, ws.data_ptr(), ws.numel(), st)
        dcall(dev, "sa_select", col, slash, H, cn, nb, cfg.alpha_c, cfg.alpha_s, guard_eps, bound.data_ptr(),
              GUARD_LOGIT_REF, flags.data_ptr(), band_pairs.data_ptr(), None, k_sel.data_ptr(), idx_sel.data_ptr(),
              band.data_ptr(), BAND_EPS, st)
        dcall(dev, "sa_certify_band_ties", b.dtype_code, b.S, b.Hq, b.Hkv, b.d, plan.blk, plan.chunk_n, plan.itv,
              band.data_ptr(), flags.data_ptr(), reduced.row_stats.data_ptr(), col, slash, bound.data_ptr(),
              GUARD_LOGIT_REF, BAND_EPS, ws.data_ptr(), ws.numel(), st)
        # everything else the guard flagged: the exact (fp64) stage 1 of the pair, then a fresh selection
        _stage1(b, plan, reduced.col, reduced.slash, _lib.SA_STAGE1_EXACT, only=flags)
        dcall(dev, "sa_select", col, slash, H, cn, nb, cfg.alpha_c, cfg.alpha_s, 0.0, None, 1.0, None,
              flags.data_ptr(), None, k_sel.data_ptr(), idx_sel.data_ptr(), None, 0.0, st)
    return Selection(k_sel, idx_sel, flags, guard, band_pairs)


def _selection_from_indices(selected, n_chunks: int, nb: int, device) -> Selection:
    """Host SelectedIndices (one head) or a list of them (one per head) -> device arrays."""
    heads = selected if isinstance(selected, (list, tuple)) and selected and isinstance(selected[0], SelectedIndices) \
        else [selected]
    H = len(heads)
    k = np.zeros((H, n_chunks, 2), dtype=np.int32)
    ix = np.zeros((H, n_chunks, 2, nb), dtype=np.int32)
    for h, sel in enumerate(heads):
        if len(sel.chunks) != n_chunks:
            raise InputError(f"{len(sel.chunks)} selections for {n_chunks} chunks")
        for c, ch in enumerate(sel.chunks):
            for dir_, picks in enumerate((ch.i_c, ch.i_s)):
                p = np.asarray(picks, dtype=np.int64)
                if p.size and (p.min() < 0 or p.max() >= nb):
                    raise InputError("picked block index out of range")
                k[h, c, dir_] = p.size
                ix[h, c, dir_, : p.size] = p
    return Selection(torch.from_numpy(k).to(device), torch.from_numpy(ix).to(device), None, "never")


def merge_index(selected, plan: ChunkPlan, blk: int, S: int, sink_blocks: int = 0,
                local_blocks: int = 1, device=None) -> BlockMask:
    """Extend picks over their query regions, union, force the diagonal
    (filtering.py:198-230).  `selected` is a device Selection, a
    SelectedIndices (one head) or a list of them (one per head)."""
    nb = n_blocks(S, blk)
    if plan.S != S or plan.blk != blk:
        raise InputError("plan does not match (S, blk)")
    if not isinstance(selected, Selection):
        selected = _selection_from_indices(selected, plan.chunk_n, nb, torch.device(device or "cuda"))
    H = int(selected.k_sel.shape[0])
    if int(selected.k_sel.shape[1]) != plan.chunk_n:
        raise InputError(f"{int(selected.k_sel.shape[1])} selections for {plan.chunk_n} chunks")
    dev = selected.k_sel.device
    kv_cnt = torch.empty((H, nb), dtype=torch.int32, device=dev)
    kv_idx = torch.empty((H, _tri(nb)), dtype=torch.int32, device=dev)
    ab = torch.empty(H, dtype=torch.int64, device=dev)
    ae = torch.empty(H, dtype=torch.int64, device=dev)
    dcall(dev, "sa_merge", selected.k_sel.data_ptr(), selected.idx_sel.data_ptr(), H, plan.chunk_n, nb, S,
              blk, plan.itv, sink_blocks, local_blocks, kv_cnt.data_ptr(), kv_idx.data_ptr(), ab.data_ptr(),
              ae.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    mask = BlockMask(blk, S, kv_cnt, kv_idx, selected.k_sel, selected.idx_sel, ab, ae)
    mask.selection = selected
    return mask


def select_and_merge(reduced: ReducedScores, plan: ChunkPlan, cfg: SparseConfig, guard: str = "auto",
                     sink_blocks: int = 0, local_blocks: int = 1) -> BlockMask:
    """filtering.py:233-256 for every head of the batch."""
    if plan.chunk_n != reduced.plan.chunk_n:
        raise InputError("reduced scores and plan disagree on chunk count")
    sel = select(reduced, cfg, guard=guard)
    return merge_index(sel, plan, reduced.blk, reduced.S, sink_blocks, local_blocks)


def sampled_retained(reduced: ReducedScores, mask: BlockMask, rescored: torch.Tensor | None = None) -> torch.Tensor:
    """Per head, the probability mass every sampled row keeps inside the mask
    (ref pipeline.py:37-58 `_retained_by_block` over the sampled rows, whose
    min / mean are cra_sampled), from stage 1's own partials
    (sa_sampled_retained) -- no recomputation of the sampled rows.  Must follow
    the stage-1 / select calls of `reduced` on the same stream (it reads their
    workspace).  `rescored`: the guard flags of the select call.  Returns fp64
    [H, sampled rows] in plan order."""
    b, plan = reduced.batch, reduced.plan
    ws = _workspace(b, plan.blk, plan.chunk_n)
    out = torch.empty((b.Hq, plan.chunk_n, plan.blk), dtype=torch.float64, device=b.q.device)
    mode = _lib.SA_STAGE1_TENSOR if reduced.mode == "tensor" else _lib.SA_STAGE1_EXACT
    dcall(b.q.device, "sa_sampled_retained", b.dtype_code, b.S, b.Hq, b.Hkv, b.d, plan.blk, plan.chunk_n, plan.itv,
          mode, None if rescored is None else rescored.data_ptr(), mask.kv_cnt.data_ptr(), mask.kv_idx.data_ptr(),
          ws.data_ptr(), ws.numel(), out.data_ptr(), b.stream)
    n = [c.sample_end - c.sample_start for c in plan.chunks]
    if all(x == plan.blk for x in n):
        return out.view(b.Hq, -1)
    return torch.cat([out[:, c, :x] for c, x in enumerate(n)], dim=1)


# ---------------------------------------------------------------- stage 3
@dataclass
class FlopReport:
    """executor.py:31-48: block counts and GEMM FLOP estimates (4*d*m*n per
    active block pair, trailing partial blocks pro-rated), summed over the
    batch's heads; per-head arrays in `per_head_*`."""

    active_blocks: int
    causal_blocks: int
    block_density: float
    estimated_flops_sparse: int
    estimated_flops_dense: int
    wall_time_sparse: float = 0.0
    wall_time_dense: float = 0.0
    per_head_active: np.ndarray = field(default=None, repr=False)
    per_head_flops_sparse: np.ndarray = field(default=None, repr=False)

    @property
    def flop_ratio(self) -> float:
        return self.estimated_flops_sparse / self.estimated_flops_dense


def flop_accounting(mask: BlockMask, S: int, d: int) -> FlopReport:
    nb, blk = mask.n_qblocks, mask.blk
    if n_blocks(S, blk) != nb:
        raise InputError(f"mask has {nb} blocks of {blk}, cannot cover S={S}")
    sizes = np.minimum(blk, S - np.arange(nb, dtype=np.int64) * blk)
    cnt = mask.kv_cnt.cpu().numpy().astype(np.int64)  # [H, nb]
    # every listed kb < nb-1 is a full block; kb = nb-1 only appears (as the diagonal) in row nb-1
    area = (cnt * blk) * sizes[None, :]
    area[:, nb - 1] -= sizes[nb - 1] * (blk - sizes[nb - 1])
    per_head_sparse = 4 * d * area.sum(axis=1)
    dense_one = 4 * d * int(sum(int(sizes[q]) * (q * blk + int(sizes[q])) for q in range(nb)))
    H = cnt.shape[0]
    active = cnt.sum(axis=1)
    return FlopReport(
        active_blocks=int(active.sum()),
        causal_blocks=H * mask.causal_count(),
        block_density=float(active.sum()) / (H * mask.causal_count()),
        estimated_flops_sparse=int(per_head_sparse.sum()),
        estimated_flops_dense=H * dense_one,
        per_head_active=active,
        per_head_flops_sparse=per_head_sparse,
    )


def _check_buffer(name: str, t: torch.Tensor, shape: tuple, dtype, device) -> None:
    if not isinstance(t, torch.Tensor) or tuple(t.shape) != tuple(shape) or t.dtype != dtype \
            or t.device != device or not t.is_contiguous():
        got = (tuple(t.shape), t.dtype, str(t.device), t.is_contiguous()) if isinstance(t, torch.Tensor) else type(t)
        raise InputError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)} on {device}, got {got}")


def sparse_attention(heads, mask: BlockMask, out: torch.Tensor | None = None,
                     lse: torch.Tensor | None = None, report: bool = True, check: bool | None = None,
                     peer_out: list | None = None):
    """Block-sparse causal attention over the mask's active blocks
    (executor.py:104-158).  Returns (out [H, S, d] in the input dtype,
    FlopReport with the kernel's touched-block count and wall_time_sparse,
    the kernel's CUDA-event time) — or (out, None) with report=False, which
    keeps the call free of host synchronisation.  check (default: report)
    reads the device status word and raises the reference's errors for an
    empty query block / broken mask invariants / empty normaliser.
    peer_out: device addresses (peer-mapped, parallel.PeerGather) of the same
    rows in other ranks' gather buffers; the kernel stores every output row
    there too, tile by tile (sa_sparse_forward_peers, bf16 only)."""
    b = as_batch(heads)
    if check is None:
        check = report
    if mask.n_heads != b.Hq:
        raise InputError(f"mask covers {mask.n_heads} heads, batch has {b.Hq}")
    nb = n_blocks(b.S, mask.blk)
    if mask.n_qblocks != nb:
        raise InputError(f"mask has {mask.n_qblocks} blocks of {mask.blk}, head needs {nb} for S={b.S}")
    if out is None:
        out = torch.empty_like(b.q)
    else:
        _check_buffer("out", out, b.q.shape, b.q.dtype, b.q.device)
    if lse is not None:
        _check_buffer("lse", lse, (b.Hq, b.S), torch.float32, b.q.device)
    touched = torch.zeros(b.Hq, dtype=torch.int64, device=b.q.device) if report else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if report else None
    if ev:
        ev[0].record()
    args = (b.q.data_ptr(), b.k.data_ptr(), b.v.data_ptr(), b.dtype_code, b.S, b.Hq, b.Hkv, b.d, mask.blk, b.group,
            b.q_head0, mask.kv_cnt.data_ptr(), mask.kv_idx.data_ptr(), mask.order(b.group, b.q_head0).data_ptr(),
            out.data_ptr(), None if lse is None else lse.data_ptr(), None if touched is None else touched.data_ptr())
    if peer_out:
        arr = (ctypes.c_void_p * len(peer_out))(*[int(p) for p in peer_out])
        dcall(b.q.device, "sa_sparse_forward_peers", *args, arr, len(peer_out), b.stream)
    else:
        dcall(b.q.device, "sa_sparse_forward", *args, b.stream)
    if ev:
        ev[1].record()
    if check:
        check_status(b.q.device)
    if not report:
        return out, None
    rep = flop_accounting(mask, b.S, b.d)
    rep.active_blocks = int(touched.sum().item())
    rep.wall_time_sparse = ev[0].elapsed_time(ev[1]) / 1e3
    return out, rep
