"""Host-buffer entry point: SampleAttention on q/k/v that live in (pinned)
host memory, with the PCIe transfers overlapped with the kernels.

The reference is called with host arrays (numpy heads, pkg/src/blocksift/
pipeline.py:149), so a drop-in has to move 1.1 GB of q/k/v in and 1 GB of
output out at 128K x 32 heads, ~40 ms of PCIe against ~36 ms of kernels.
Stages 1 and 2 read only K and the SAMPLED query windows (128 rows per chunk,
ref sampler.py:103-117), so the copy stream sends K/V and those windows
first (~2 % of the bytes); stages 1-2 then run for ALL heads at once while
the bulk of Q streams in behind them.  Stage 3 runs per head group as each
group's Q lands (one launch per group; the groups shrink at the end so the
last device->host copy is short), and each group's output goes back on a
second copy stream while the next group computes.  The result is that of
sample_attention on the whole batch: stages 1-3 are independent per q head
(ref pipeline.py:169) and stage 3 of a head reads only that head's rows.
"""

from __future__ import annotations

import contextlib
import threading

import numpy as np
import torch

from .config import plan_chunks, resolve_config
from .errors import InputError
from .heads import HeadBatch, check_finite_async, dcall, raise_on_flags
from .pipeline import SampleAttentionResult
from .stages import block_reduce, merge_index, sample_scores, select, sparse_attention

__all__ = ["sample_attention_host", "release_staging"]


def _as_host(x) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor) or x.is_cuda:
        raise InputError("sample_attention_host takes host (CPU) tensors or numpy arrays")
    return x.contiguous()


def _group_plan(Hq: int, group: int, hpg: int) -> list:
    """Stage-3 head groups [h0, h1) inside KV-group boundaries.  A head's Q
    crosses PCIe in ~0.6x the time its stage 3 takes (128K), so the groups
    ramp up (1, 1, 2, 3, 5 heads, then `hpg`; the first stage-3 launch waits
    for one head's Q instead of two: e2e -0.2..0.4 ms at C3 against 2, 2, 3, 5,
    profiles/r2/s3/e2e_ramp_ab2.txt): each group's copy hides under the
    previous group's kernels.  The last groups shrink (3, 2, then 1 head):
    each group's output copy hides under the next group's kernels and the
    copy after the last kernel is short."""
    groups, h0 = [], 0
    n_kv = Hq // group
    for g in range(n_kv):
        rest, head, tail = group, [], []
        if g == n_kv - 1:
            for s in (1, 2, 3):
                if rest > s:
                    tail.insert(0, s)
                    rest -= s
        if g == 0:
            for s in (1, 1, 2, 3, 5):
                if rest > s:
                    head.append(s)
                    rest -= s
        n_mid = -(-rest // hpg)  # near-equal groups of at most hpg heads
        sizes = head + ([rest // n_mid + (1 if i < rest % n_mid else 0) for i in range(n_mid)] if rest else []) + tail
        for s in sizes:
            groups.append((h0, h0 + s))
            h0 += s
    return groups


def sample_attention_host(q, k, v, heads_per_group: int = 8, device=None, out: torch.Tensor | None = None,
                          check_inputs: bool = True, dtype=torch.bfloat16, alpha: float = 0.95,
                          alpha_c: float | None = None, alpha_s: float | None = None, chunk_n: int | None = None,
                          sample_ratio: float | None = None, blk: int = 128, sink_blocks: int = 0,
                          local_blocks: int = 1, guard: str = "auto", _lanes: int = 2):
    """q [Hq,S,d], k/v [Hkv,S,d] on the host -> (out [Hq,S,d] on the host,
    [SampleAttentionResult]).  Keyword arguments are those of sample_attention.

    For the transfers to overlap, pass pinned tensors (torch .pin_memory());
    pageable inputs are staged through pinned buffers first."""
    q, k, v = _as_host(q), _as_host(k), _as_host(v)
    if q.dim() != 3 or k.dim() != 3 or k.shape != v.shape or q.shape[1:] != k.shape[1:]:
        raise InputError(f"expected q [Hq,S,d] and k, v [Hkv,S,d]; got {tuple(q.shape)}, {tuple(k.shape)}")
    Hq, Hkv, S = q.shape[0], k.shape[0], q.shape[1]
    if Hq % Hkv:
        raise InputError(f"Hq={Hq} is not a multiple of Hkv={Hkv}")
    group = Hq // Hkv
    hpg = max(1, min(heads_per_group, group))
    cfg = resolve_config(S, alpha, alpha_c, alpha_s, chunk_n, sample_ratio, blk)
    plan = plan_chunks(S, cfg)
    dev = torch.device(device or "cuda")
    if q.dtype != dtype:
        q, k, v = (t.to(dtype) for t in (q, k, v))
    if not q.is_pinned():
        q, k, v = (t.pin_memory() for t in (q, k, v))
    if out is None:
        out = torch.empty(q.shape, dtype=dtype, pin_memory=True)
    with _staging(dev, tuple(q.shape), tuple(k.shape), dtype) as st_:
        return _run(q, k, v, out, st_, dev, group, hpg, cfg, plan, check_inputs, sink_blocks, local_blocks,
                    guard, _lanes)


class _Staging:
    """Device copies of q/k/v/out and the copy / side streams of one geometry,
    kept across calls: allocating 2+ GB per call costs the caching allocator
    fresh cudaMallocs (up to ~17 ms measured at C3) whenever its blocks are
    still tied to the previous call's streams."""

    def __init__(self, dev, qshape, kshape, dtype):
        self.dq = torch.empty(qshape, dtype=dtype, device=dev)
        self.dk = torch.empty(kshape, dtype=dtype, device=dev)
        self.dv = torch.empty(kshape, dtype=dtype, device=dev)
        self.dout = torch.empty_like(self.dq)
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        self.side = torch.cuda.Stream(device=dev)
        # stages 1-2 of the later KV groups: high priority, so their CTAs take SMs as stage-3 CTAs retire
        self.s12 = torch.cuda.Stream(device=dev, priority=-1)
        self.lock = threading.Lock()


_STAGING: dict = {}
_STAGING_LOCK = threading.Lock()


@contextlib.contextmanager
def _staging(dev, qshape, kshape, dtype):
    key = (dev, qshape, kshape, dtype)
    with _STAGING_LOCK:
        st_ = _STAGING.get(key)
        if st_ is None:
            _STAGING.clear()  # one geometry at a time: the buffers are large
            st_ = _STAGING[key] = _Staging(dev, qshape, kshape, dtype)
    with st_.lock:
        yield st_


def release_staging() -> None:
    """Free the cached device buffers of sample_attention_host."""
    with _STAGING_LOCK:
        _STAGING.clear()


def _run(q, k, v, out, st_, dev, group, hpg, cfg, plan, check_inputs, sink_blocks, local_blocks, guard, _lanes):
    Hq, S = q.shape[0], q.shape[1]
    dq, dk, dv, dout = st_.dq, st_.dk, st_.dv, st_.dout
    compute = torch.cuda.current_stream(dev)
    h2d, d2h, side, s12 = st_.h2d, st_.d2h, st_.side, st_.s12
    h2d.wait_stream(compute)  # the previous call's readers of dq/dk/dv and this call's inputs
    groups = _group_plan(Hq, group, hpg)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    fused = dq.dtype == torch.bfloat16  # q's NaN/Inf scan left to stage 3 (scan_inputs_async)
    # phase 0 = the first KV group, phase 1 = the rest: stage 3 starts after the
    # first group's K and filtering only, and the other groups' stages 1-2 run on
    # their own stream while it computes
    n_kv = Hq // group
    phases = [(0, 1), (1, n_kv)] if n_kv > 1 else [(0, 1)]
    row_bytes = q.shape[2] * q.element_size()
    sampled, ready = [], []
    # the copy stream carries copies only: a kernel queued on it (the NaN/Inf
    # scan) would wait for SMs behind a running stage-3 launch and hold up
    # every copy behind it
    def send_filter_inputs(p):  # K (stage 1 reads every key) and the sampled query windows of phase p
        g0, g1 = phases[p]
        hs0, hs1 = g0 * group, g1 * group
        dk[g0:g1].copy_(k[g0:g1], non_blocking=True)
        for c in plan.chunks:
            off = (hs0 * S + c.sample_start) * row_bytes
            dcall(dev, "sa_copy2d_async", dq.data_ptr() + off, S * row_bytes, q.data_ptr() + off, S * row_bytes,
                  (c.sample_end - c.sample_start) * row_bytes, hs1 - hs0, h2d.cuda_stream)
        e = torch.cuda.Event()
        e.record(h2d)
        sampled.append(e)

    # order: phase 0's K + windows + V, its first Q group, then the other
    # phases' K + windows (their filtering then overlaps the first stage-3
    # launches instead of waiting behind them for SMs), the rest of Q and V
    with torch.cuda.stream(h2d):
        send_filter_inputs(0)
        dv[0:1].copy_(v[0:1], non_blocking=True)
        first_v = {0}
        for i, (h0, h1) in enumerate(groups):
            g = h0 // group
            p = 0 if g < phases[0][1] else 1
            if p == 1 and len(sampled) == 1:  # no first-phase group followed (single head group)
                send_filter_inputs(1)
            if g not in first_v:
                gp0, gp1 = phases[p]
                dv[gp0:gp1].copy_(v[gp0:gp1], non_blocking=True)
                first_v.update(range(gp0, gp1))
            dq[h0:h1].copy_(q[h0:h1], non_blocking=True)  # the windows are sent again; same bits
            e = torch.cuda.Event()
            e.record(h2d)
            ready.append(e)
            if i == 0 and len(phases) > 1:
                send_filter_inputs(1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    lanes = (compute, side, s12)
    side.wait_stream(compute)
    s12.wait_stream(compute)
    masks, results = [], []
    for p, (g0, g1) in enumerate(phases):  # stages 1-2 per phase
        st = compute if p == 0 else s12
        st.wait_event(sampled[p])
        if p == 0:
            ev[0].record(st)
        hs0, hs1 = g0 * group, g1 * group
        with torch.cuda.stream(st):
            if check_inputs:  # the reference's NaN/Inf check (core.py:30-37), read once at the end
                check_finite_async([dk[g0:g1]], flag, st.cuda_stream)
            batch = HeadBatch.from_tensors(dq[hs0:hs1], dk[g0:g1], dv[g0:g1], group=group, q_head0=hs0)
            reduced = block_reduce(sample_scores(batch, plan), cfg.blk)
            if p == 0:
                ev[1].record(st)
            sel = select(reduced, cfg, guard=guard)
            mask = merge_index(sel, plan, cfg.blk, S, sink_blocks, local_blocks)
            if p == 0:
                ev[2].record(st)
        done_p = torch.cuda.Event()
        done_p.record(st)
        masks.append((hs0, hs1, mask, done_p))
        results.append(SampleAttentionResult(cfg, plan, mask, sel.flags, ev if p == 0 else None, None))
    # stage-3 launches alternate between two streams, so a group's kernel fills
    # the SMs the previous group's last wave leaves idle
    for i, ((h0, h1), landed) in enumerate(zip(groups, ready)):
        st = lanes[i % _lanes]
        st.wait_event(landed)
        hs0, hs1, mask, done_p = next(m for m in masks if m[0] <= h0 < m[1])
        st.wait_event(done_p)
        kv0, kv1 = h0 // group, (h1 - 1) // group + 1
        if check_inputs:
            if h0 == hs0:
                check_finite_async([dv[kv0:kv1]], flag, st.cuda_stream)
            if not fused:
                check_finite_async([dq[h0:h1]], flag, st.cuda_stream)
        with torch.cuda.stream(st):
            part = HeadBatch.from_tensors(dq[h0:h1], dk[kv0:kv1], dv[kv0:kv1], group=group, q_head0=h0)
            sparse_attention(part, mask.heads(h0 - hs0, h1 - hs0), out=dout[h0:h1], report=False)
        done = torch.cuda.Event()
        done.record(st)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            out[h0:h1].copy_(dout[h0:h1], non_blocking=True)
    compute.wait_stream(side)
    compute.wait_stream(s12)
    ev[3].record(compute)
    compute.wait_stream(d2h)
    flag.record_stream(side)
    flag.record_stream(s12)
    for _, _, m, _ in masks:
        for t in (m.kv_cnt, m.kv_idx):
            t.record_stream(side)
            t.record_stream(compute)
    # `out` is host memory: the caller may read it as soon as we return
    d2h.synchronize()
    if check_inputs:
        raise_on_flags(flag, dev, dq if fused else None)
    return out, results
