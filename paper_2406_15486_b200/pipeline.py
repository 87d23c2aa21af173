"""End-to-end composition: the reference's run_pipeline (pipeline.py:149-217)
and the batched drop-in `sample_attention(q, k, v, ...)`.

Both run all heads of a batch through stage 1 -> stage 2 -> stage 3 on the
GPU with no host synchronisation inside the hot path; stage times are CUDA
events on the launching stream.  Accuracy metrics (sampled-row CRA, and with
want_oracle the full CRA and dense output error) are computed afterwards with
torch on the device; they are harness, not hot path, exactly as the
reference's oracle module is.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import ChunkPlan, SparseConfig, n_blocks, plan_chunks, resolve_config
from .errors import InputError
from .heads import HeadBatch, HeadSet, check_finite_async, check_status, raise_on_flags, scan_inputs_async
from .masks import BlockMask
from .stages import (FlopReport, block_reduce, flop_accounting, merge_index, sample_scores, sampled_retained,
                     select, sparse_attention)

__all__ = ["ORACLE_CAP", "HeadMetrics", "MetricsReport", "cra_full", "run_pipeline", "sample_attention",
           "SampleAttentionResult", "dense_attention"]

ORACLE_CAP = 8192


@dataclass
class SampleAttentionResult:
    """Everything sample_attention produced besides the output."""

    cfg: SparseConfig
    plan: ChunkPlan
    mask: BlockMask
    rescored: torch.Tensor | None          # guard flags [H*cn] (device)
    events: list | None = None             # CUDA events: start, stage1, stage2, stage3
    lse: torch.Tensor | None = None

    def stage_ms(self) -> dict:
        if not self.events:
            return {}
        e = self.events
        torch.cuda.synchronize(e[0].device if hasattr(e[0], "device") else None)
        return {"stage1_ms": e[0].elapsed_time(e[1]), "stage2_ms": e[1].elapsed_time(e[2]),
                "stage3_ms": e[2].elapsed_time(e[3]), "total_ms": e[0].elapsed_time(e[3])}

    def n_rescored(self) -> int:
        return 0 if self.rescored is None else int(self.rescored.sum().item())


def sample_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, alpha: float = 0.95,
                     alpha_c: float | None = None, alpha_s: float | None = None, chunk_n: int | None = None,
                     sample_ratio: float | None = None, blk: int = 128, sink_blocks: int = 0,
                     local_blocks: int = 1, guard: str = "auto", check_inputs: bool = True,
                     return_lse: bool = False, timings: bool = False, q_head0: int = 0,
                     group: int | None = None, out: torch.Tensor | None = None, peer_out: list | None = None):
    """SampleAttention prefill for q [Hq,S,d], k/v [Hkv,S,d] (bf16 or fp32, CUDA).

    alpha: CRA threshold (alpha_c = alpha_s = alpha unless given);
    sample_ratio / chunk_n: how many 128-row query windows stage 1 scores;
    sink_blocks / local_blocks: optional forced key blocks (defaults reproduce
    the reference, which forces only the diagonal).  Returns (out, result).

    check_inputs: scan q/k/v for NaN/Inf (InputError, ref core.py:30-37) and
    read the stage-3 invariant status (ref executor.py:131-132, 150-153); both
    are device flags read with ONE host sync after every stage is enqueued.
    check_inputs=False leaves the call free of host synchronisation.
    peer_out: the output gather fused into stage 3 (parallel.sample_attention_sharded)."""
    batch = HeadBatch.from_tensors(q, k, v, group=group, q_head0=q_head0)
    flag = None
    rescan = None
    if check_inputs:
        flag = torch.zeros(1, dtype=torch.int32, device=batch.q.device)
        if scan_inputs_async(batch.q, batch.k, batch.v, flag, batch.stream):
            rescan = batch.q
    cfg = resolve_config(batch.S, alpha, alpha_c, alpha_s, chunk_n, sample_ratio, blk)
    plan = plan_chunks(batch.S, cfg)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timings else None
    if ev:
        ev[0].record()
    reduced = block_reduce(sample_scores(batch, plan), cfg.blk)
    if ev:
        ev[1].record()
    sel = select(reduced, cfg, guard=guard)
    mask = merge_index(sel, plan, cfg.blk, batch.S, sink_blocks, local_blocks)
    mask.order(batch.group, batch.q_head0)
    if ev:
        ev[2].record()
    lse = torch.empty((batch.Hq, batch.S), dtype=torch.float32, device=batch.q.device) if return_lse else None
    o, _ = sparse_attention(batch, mask, out=out, lse=lse, report=False, peer_out=peer_out)
    if ev:
        ev[3].record()
    if check_inputs:
        raise_on_flags(flag, batch.q.device, rescan)
    return o, SampleAttentionResult(cfg, plan, mask, sel.flags, ev, lse)


def dense_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, blk: int = 128,
                    out: torch.Tensor | None = None, group: int | None = None):
    """Dense causal attention through the same stage-3 kernel (full mask)."""
    batch = HeadBatch.from_tensors(q, k, v, group=group)
    mask = BlockMask.full(batch.Hq, batch.S, blk, device=batch.q.device)
    o, _ = sparse_attention(batch, mask, out=out, report=False)
    return o


# ---------------------------------------------------------------- metrics
@dataclass
class HeadMetrics:
    head_id: int
    cra_sampled_min: float
    cra_sampled_mean: float
    block_density: float
    sparsity_ratio: float
    active_blocks: int
    flop_ratio: float
    wall_time_sample: float
    wall_time_filter: float
    wall_time_sparse: float
    cra_full_min: float | None = None
    cra_full_mean: float | None = None
    output_error: float | None = None
    wall_time_dense: float | None = None


@dataclass
class MetricsReport:
    """Same flat-serializable document as the reference (pipeline.py:79-146).
    Wall times are the batched stage times (CUDA events) split evenly across
    heads, since all heads run in one launch per stage."""

    S: int
    d: int
    n_heads: int
    alpha_c: float
    alpha_s: float
    chunk_n: int
    effective_chunk_n: int
    blk: int
    oracle: bool
    heads: list
    seed: int | None = None
    masks: tuple = field(default=(), repr=False)
    outputs: object = field(default=None, repr=False)
    n_rescored: int = 0

    def to_flat_dict(self) -> dict:
        out = {"S": self.S, "d": self.d, "n_heads": self.n_heads, "alpha_c": self.alpha_c,
               "alpha_s": self.alpha_s, "chunk_n": self.chunk_n, "effective_chunk_n": self.effective_chunk_n,
               "blk": self.blk, "oracle": self.oracle}
        if self.seed is not None:
            out["seed"] = self.seed
        for h in self.heads:
            p = f"head_{h.head_id}_"
            for key in ("cra_sampled_min", "cra_sampled_mean", "block_density", "sparsity_ratio",
                        "active_blocks", "flop_ratio", "wall_time_sample", "wall_time_filter",
                        "wall_time_sparse"):
                out[p + key] = getattr(h, key)
            if self.oracle:
                for key in ("cra_full_min", "cra_full_mean", "output_error", "wall_time_dense"):
                    out[p + key] = getattr(h, key)
        hs = self.heads
        out["cra_sampled_min"] = min(h.cra_sampled_min for h in hs)
        out["cra_sampled_mean"] = sum(h.cra_sampled_mean for h in hs) / len(hs)
        out["block_density_mean"] = sum(h.block_density for h in hs) / len(hs)
        out["sparsity_ratio_mean"] = sum(h.sparsity_ratio for h in hs) / len(hs)
        out["flop_ratio_mean"] = sum(h.flop_ratio for h in hs) / len(hs)
        out["wall_time_total"] = sum(h.wall_time_sample + h.wall_time_filter + h.wall_time_sparse for h in hs)
        if self.oracle:
            out["cra_full_min"] = min(h.cra_full_min for h in hs)
            out["cra_full_mean"] = sum(h.cra_full_mean for h in hs) / len(hs)
            out["output_error_max"] = max(h.output_error for h in hs)
        return out

    def to_json(self) -> str:
        return json.dumps(self.to_flat_dict(), sort_keys=True, indent=2) + "\n"


def _causal_probs(qr: torch.Tensor, k: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
    s = (qr.double() @ k.double().T) / float(np.sqrt(k.shape[1]))
    keep = torch.arange(k.shape[0], device=k.device)[None, :] <= rows[:, None]
    s = torch.where(keep, s, torch.tensor(float("-inf"), device=k.device, dtype=s.dtype))
    return torch.softmax(s, dim=1)


def _retained(p: torch.Tensor, rows: torch.Tensor, dense_mask: torch.Tensor, blk: int) -> torch.Tensor:
    S = p.shape[1]
    nb = dense_mask.shape[0]
    pad = nb * blk - S
    bs = torch.nn.functional.pad(p, (0, pad)).view(p.shape[0], nb, blk).sum(dim=2)
    return (bs * dense_mask[rows // blk]).sum(dim=1)


def cra_full(batch: HeadBatch, mask: BlockMask, row_chunk: int = 1024) -> tuple:
    """Entry-level CRA of every query row (ref oracle.py:86-99 / pipeline.py:37-58,
    the reference's `cra_full`), on the GPU in fp64 and for any S -- the
    reference caps it at ORACLE_CAP because it materialises S x S on the CPU;
    here rows are processed `row_chunk` at a time.  Returns
    per-head (min, mean) numpy arrays of the retained causal probability mass."""
    S, blk = batch.S, mask.blk
    dense = torch.from_numpy(mask.to_dense()).to(batch.q.device)
    mins, means = [], []
    for h in range(batch.Hq):
        kh = batch.k[(batch.q_head0 + h) // batch.group - batch.q_head0 // batch.group]
        kept = []
        for r0 in range(0, S, row_chunk):
            rows = torch.arange(r0, min(S, r0 + row_chunk), device=batch.q.device)
            kept.append(_retained(_causal_probs(batch.q[h, rows], kh, rows), rows, dense[h], blk))
        k_all = torch.cat(kept)
        mins.append(float(k_all.min()))
        means.append(float(k_all.mean()))
    return np.array(mins), np.array(means)


def run_pipeline(head_set, cfg: SparseConfig, want_oracle: bool = False, seed: int | None = None,
                 dtype=torch.bfloat16, guard: str = "auto", device=None) -> MetricsReport:
    """Run every head through the GPU pipeline and collect the reference's metrics."""
    batch = head_set if isinstance(head_set, HeadBatch) else HeadBatch.from_heads(
        head_set if isinstance(head_set, HeadSet) else HeadSet(list(head_set)), dtype=dtype, device=device)
    S, d, H = batch.S, batch.d, batch.Hq
    if want_oracle and S > ORACLE_CAP:
        raise InputError(f"oracle metrics need S <= {ORACLE_CAP}, got {S}; run without --oracle")
    flag = torch.zeros(1, dtype=torch.int32, device=batch.q.device)
    check_finite_async((batch.q, batch.k, batch.v), flag, batch.stream)
    plan = plan_chunks(S, cfg)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    reduced = block_reduce(sample_scores(batch, plan), cfg.blk)
    ev[1].record()
    sel = select(reduced, cfg, guard=guard)
    mask = merge_index(sel, plan, cfg.blk, S)
    ev[2].record()
    kept_sampled = sampled_retained(reduced, mask, sel.flags)  # cra_sampled from stage 1's partials
    out, flop = sparse_attention(batch, mask, check=False)
    ev[3].record()
    raise_on_flags(flag, batch.q.device)
    flop.wall_time_sparse = ev[2].elapsed_time(ev[3]) / 1e3
    t_s, t_f, t_x = (ev[i].elapsed_time(ev[i + 1]) / 1e3 / H for i in range(3))
    dense = torch.from_numpy(mask.to_dense()).to(batch.q.device)  # [H, nb, nb]
    kv_of = [(batch.q_head0 + h) // batch.group - batch.q_head0 // batch.group for h in range(H)]
    total_causal = S * (S + 1) // 2
    cnt = mask.kv_cnt.to(torch.int64)
    nb, blk = mask.n_qblocks, cfg.blk
    sizes = torch.clamp(S - torch.arange(nb, device=cnt.device) * blk, max=blk)
    entries = ((cnt - 1) * sizes * blk + sizes * (sizes + 1) // 2).sum(dim=1).cpu().numpy()
    heads = []
    dense_out = None
    t_dense = None
    if want_oracle:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dense_out = dense_attention(batch.q, batch.k, batch.v, blk=blk, group=batch.group)
        e1.record()
        torch.cuda.synchronize(batch.q.device)
        t_dense = e0.elapsed_time(e1) / 1e3 / H
    for h in range(H):
        kh = batch.k[kv_of[h]]
        kept = kept_sampled[h]
        hm = HeadMetrics(
            head_id=batch.head_ids[h] if batch.head_ids else batch.q_head0 + h,
            cra_sampled_min=float(kept.min()), cra_sampled_mean=float(kept.mean()),
            block_density=float(flop.per_head_active[h]) / mask.causal_count(),
            sparsity_ratio=1.0 - float(entries[h]) / total_causal,
            active_blocks=int(flop.per_head_active[h]),
            flop_ratio=float(flop.per_head_flops_sparse[h]) / (flop.estimated_flops_dense / H),
            wall_time_sample=t_s, wall_time_filter=t_f, wall_time_sparse=t_x)
        if want_oracle:
            rows = torch.arange(S, device=batch.q.device)
            kept_full = torch.cat([
                _retained(_causal_probs(batch.q[h, r0:r0 + 512], kh, rows[r0:r0 + 512]), rows[r0:r0 + 512],
                          dense[h], blk) for r0 in range(0, S, 512)])
            hm.cra_full_min, hm.cra_full_mean = float(kept_full.min()), float(kept_full.mean())
            o_s, o_d = out[h].double(), dense_out[h].double()
            num = torch.linalg.norm(o_s - o_d, dim=1)
            den = torch.clamp(torch.linalg.norm(o_d, dim=1), min=1e-12)
            hm.output_error = float((num / den).max())
            hm.wall_time_dense = t_dense
        heads.append(hm)
    return MetricsReport(S=S, d=d, n_heads=H, alpha_c=cfg.alpha_c, alpha_s=cfg.alpha_s, chunk_n=cfg.chunk_n,
                         effective_chunk_n=plan.chunk_n, blk=cfg.blk, oracle=want_oracle, heads=heads, seed=seed,
                         masks=tuple(mask.head(h) for h in range(H)), outputs=out,
                         n_rescored=sel.n_rescored())
