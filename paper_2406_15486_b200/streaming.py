"""Host-buffer entry point: SampleAttention on q/k/v that live in (pinned)
host memory, with the PCIe transfers overlapped with the kernels.

The reference is called with host arrays (numpy heads, pkg/src/blocksift/
pipeline.py:149), so a drop-in has to move 1.1 GB of q/k/v in and 1 GB of
output out at 128K x 32 heads.  Done naively (copy in, compute, copy out)
the copies cost more than the attention itself.  Here the q heads are split
into groups inside their KV group; all host->device copies are queued up
front on one copy stream (each KV head ahead of its first q group), each
group's three stages run on the compute stream as soon as its inputs land,
and its output goes back on a second copy stream while the next group
computes.  The result is the same as sample_attention on the whole batch:
stages 1-3 are independent per q head (ref pipeline.py:169).
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import InputError
from .heads import check_finite_async, raise_on_flags
from .pipeline import sample_attention

__all__ = ["sample_attention_host"]


def _as_host(x) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor) or x.is_cuda:
        raise InputError("sample_attention_host takes host (CPU) tensors or numpy arrays")
    return x.contiguous()


def _group_plan(Hq: int, group: int, hpg: int) -> list:
    """Head groups [h0, h1) inside KV-group boundaries.  The first groups of
    the batch are small (1, then 2 heads) so the first kernels start after a
    short copy, and the last groups shrink again (2, then 1) so the final
    device->host copy after the last kernel is short; the rest use `hpg`."""
    sizes_per_kv = []
    n_kv = Hq // group
    for g in range(n_kv):
        head, tail = [], []
        rest = group
        if g == 0:
            for s in (1, 2):
                if rest > s:
                    head.append(s)
                    rest -= s
        if g == n_kv - 1:
            for s in (1, 2):
                if rest > s:
                    tail.insert(0, s)
                    rest -= s
        n_mid = -(-rest // hpg)  # near-equal middle groups of at most hpg heads
        mid = [rest // n_mid + (1 if i < rest % n_mid else 0) for i in range(n_mid)] if rest else []
        sizes_per_kv.append(head + mid + tail)
    groups, h0 = [], 0
    for sizes in sizes_per_kv:
        for s in sizes:
            groups.append((h0, h0 + s))
            h0 += s
    return groups


def sample_attention_host(q, k, v, heads_per_group: int = 4, device=None, out: torch.Tensor | None = None,
                          check_inputs: bool = True, dtype=torch.bfloat16, **kw):
    """q [Hq,S,d], k/v [Hkv,S,d] on the host -> (out [Hq,S,d] on the host,
    list of per-group SampleAttentionResult).  Keyword arguments are those of
    sample_attention (alpha, chunk_n / sample_ratio, guard, ...).

    For the transfers to overlap, pass pinned tensors (torch .pin_memory());
    pageable inputs are staged through pinned buffers first."""
    q, k, v = _as_host(q), _as_host(k), _as_host(v)
    if q.dim() != 3 or k.dim() != 3 or k.shape != v.shape or q.shape[1:] != k.shape[1:]:
        raise InputError(f"expected q [Hq,S,d] and k, v [Hkv,S,d]; got {tuple(q.shape)}, {tuple(k.shape)}")
    Hq, Hkv = q.shape[0], k.shape[0]
    if Hq % Hkv:
        raise InputError(f"Hq={Hq} is not a multiple of Hkv={Hkv}")
    group = Hq // Hkv
    hpg = max(1, min(heads_per_group, group))
    while group % hpg:
        hpg -= 1
    dev = torch.device(device or "cuda")
    if q.dtype != dtype:
        q, k, v = (t.to(dtype) for t in (q, k, v))
    if not q.is_pinned():
        q, k, v = (t.pin_memory() for t in (q, k, v))
    dq = torch.empty(q.shape, dtype=dtype, device=dev)
    dk = torch.empty(k.shape, dtype=dtype, device=dev)
    dv = torch.empty(v.shape, dtype=dtype, device=dev)
    dout = torch.empty_like(dq)
    if out is None:
        out = torch.empty(q.shape, dtype=dtype, pin_memory=True)
    compute = torch.cuda.current_stream(dev)
    h2d = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    h2d.wait_stream(compute)  # dq/dk/dv were allocated on the compute stream
    groups = _group_plan(Hq, group, hpg)
    ready = []
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    with torch.cuda.stream(h2d):
        copied_kv = set()
        for h0, h1 in groups:
            kv = h0 // group
            fresh = []
            if kv not in copied_kv:
                dk[kv].copy_(k[kv], non_blocking=True)
                dv[kv].copy_(v[kv], non_blocking=True)
                copied_kv.add(kv)
                fresh = [dk[kv], dv[kv]]
            dq[h0:h1].copy_(q[h0:h1], non_blocking=True)
            if check_inputs:  # the reference's NaN/Inf check (core.py:30-37), read once at the end
                check_finite_async([dq[h0:h1]] + fresh, flag, h2d.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(h2d)
            ready.append(ev)
    results = []
    for (h0, h1), ev in zip(groups, ready):
        compute.wait_event(ev)
        kv = h0 // group
        _, res = sample_attention(dq[h0:h1], dk[kv:kv + 1], dv[kv:kv + 1], q_head0=h0, group=group,
                                  out=dout[h0:h1], check_inputs=False, **kw)
        results.append(res)
        done = torch.cuda.Event()
        done.record(compute)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            out[h0:h1].copy_(dout[h0:h1], non_blocking=True)
    compute.wait_stream(d2h)
    for t in (dq, dk, dv, dout, flag):
        t.record_stream(h2d)
        t.record_stream(d2h)
    # `out` is host memory: the caller may read it as soon as we return
    d2h.synchronize()
    if check_inputs:
        raise_on_flags(flag, dev)
    return out, results
