"""Attention-head containers: the reference's AttentionHead / HeadSet
(pkg/src/blocksift/core.py:40-107) plus the device-resident batch the
kernels consume.

The reference stores each head as fp64 numpy [S, d] with its own k and v.
Here a `HeadBatch` holds q [Hq, S, d] and k, v [Hkv, S, d] on one CUDA device
in the compute dtype (bf16 for the tensor-core path, fp32 for the exact
path), with GQA/MQA grouping (q head h reads kv head h // group).  A
reference-style HeadSet becomes a batch with Hkv == Hq.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InputError, InternalInvariantError

__all__ = ["AttentionHead", "HeadSet", "HeadBatch", "check_finite", "check_finite_async", "check_status", "dcall",
           "raise_on_flags", "scan_inputs_async"]

_DTYPES = {torch.bfloat16: _lib.SA_BF16, torch.float32: _lib.SA_FP32}


def _as_2d(a, name):
    if isinstance(a, torch.Tensor):
        if a.dim() != 2:
            raise InputError(f"{name} must be 2-D, got shape {tuple(a.shape)}")
        return a
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise InputError(f"{name} must be 2-D, got shape {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise InputError(f"{name} contains NaN or Inf")
    return arr


class AttentionHead:
    """Q/K/V of one causal self-attention head, each S x d (core.py:40-75:
    equal shapes, S and d >= 1, finite values)."""

    def __init__(self, q, k, v, head_id: int = 0):
        q, k, v = _as_2d(q, "q"), _as_2d(k, "k"), _as_2d(v, "v")
        if not (tuple(q.shape) == tuple(k.shape) == tuple(v.shape)):
            raise InputError(f"head {head_id}: q/k/v must share one S x d shape, got "
                             f"{tuple(q.shape)}/{tuple(k.shape)}/{tuple(v.shape)}")
        if q.shape[0] < 1 or q.shape[1] < 1:
            raise InputError(f"head {head_id}: S and d must be >= 1")
        self.q, self.k, self.v, self.head_id = q, k, v, head_id

    @property
    def S(self) -> int:
        return int(self.q.shape[0])

    @property
    def d(self) -> int:
        return int(self.q.shape[1])


class HeadSet:
    """Heads sharing S and d (core.py:77-107)."""

    def __init__(self, heads):
        heads = tuple(heads)
        if not heads:
            raise InputError("HeadSet needs at least one head")
        S, d = heads[0].S, heads[0].d
        for h in heads:
            if h.S != S or h.d != d:
                raise InputError(f"head {h.head_id} has shape {h.S}x{h.d}, expected {S}x{d}")
        self.heads = heads

    @property
    def S(self) -> int:
        return self.heads[0].S

    @property
    def d(self) -> int:
        return self.heads[0].d

    def __len__(self):
        return len(self.heads)

    def __iter__(self):
        return iter(self.heads)


def dcall(device: torch.device, name: str, *args) -> int:
    """_lib.call with `device` current: kernels launch on the device that owns
    the tensors (and the per-device shared-memory opt-ins apply to it), whatever
    the caller's current device is."""
    if device.index is not None and device.index != torch.cuda.current_device():
        with torch.cuda.device(device):
            return _lib.call(name, *args)
    return _lib.call(name, *args)


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def check_finite_async(tensors, flag: torch.Tensor, stream: int) -> None:
    """Queue the NaN/Inf scan of `tensors` on `stream`, OR-ing into the int32
    device flag; the caller reads the flag later (no synchronisation here)."""
    for t in tensors:
        dcall(t.device, "sa_check_finite", t.data_ptr(), _DTYPES[t.dtype], t.numel(), flag.data_ptr(), stream)


def check_finite(*tensors: torch.Tensor) -> None:
    """Device-side NaN/Inf scan (sa_check_finite, replacing as_matrix's check,
    core.py:30-37); raises InputError.  One host sync."""
    dev = tensors[0].device
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    for t in tensors:
        dcall(t.device, "sa_check_finite", t.data_ptr(), _DTYPES[t.dtype], t.numel(), flag.data_ptr(), _stream(t))
    if int(flag.item()) != 0:
        raise InputError("q/k/v contain NaN or Inf")


def _read_status(device: torch.device) -> list:
    import ctypes

    buf = (ctypes.c_uint * 4)()
    with torch.cuda.device(device):
        _lib.call("sa_status", buf, 1)
    return list(buf)


def check_status(device: torch.device) -> None:
    """Read (and reset) the device status word the stage-3 kernels fill
    (sa_status; synchronises the device) and raise the reference's exception
    for the first violation: InputError for a query block without active key
    blocks (ref executor.py:131-132), InternalInvariantError for a mask that
    breaks the BlockMask invariants (filtering.py:97-106) or an empty softmax
    normaliser (executor.py:150-153)."""
    _raise_status(_read_status(device))


def _raise_status(status: list) -> None:
    bits, h, qb, n = status
    if not bits:
        return
    where = f"head {h} query block {qb}" + (f" (and {n - 1} more)" if n > 1 else "")
    if bits & _lib.SA_STATUS_EMPTY_BLOCK:
        raise InputError(f"query block {qb} has no active key blocks ({where})")
    if bits & _lib.SA_STATUS_MASK:
        raise InternalInvariantError(f"block mask violates its invariants (kb <= qb, ascending, diagonal kept) "
                                     f"at {where}")
    raise InternalInvariantError(f"query block {qb} produced an empty softmax normalizer ({where})")


def scan_inputs_async(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, flag: torch.Tensor, stream: int) -> bool:
    """Queue the NaN/Inf scan of the inputs (core.py:30-37).  Returns True when
    q was left out: on the bf16 path every query row runs through stage 3, and
    a NaN/Inf anywhere in a row makes that row's softmax normaliser non-finite
    (every logit of the row is NaN or +-Inf), which the kernel reports in the
    status word -- so the 1 GB scan of q at 128K is skipped and q is rescanned
    only when that status bit comes back (raise_on_flags)."""
    fused = q.dtype == torch.bfloat16
    check_finite_async((k, v) if fused else (q, k, v), flag, stream)
    return fused


def raise_on_flags(finite_flag: torch.Tensor | None, device: torch.device, rescan_q: torch.Tensor | None = None) -> None:
    """One host sync for everything a call checked on the device: the NaN/Inf
    flag of its inputs (InputError, core.py:30-37) first, then the stage-3
    status word (a non-finite input also poisons the normaliser, so the input
    error wins and the status is cleared).  With `rescan_q` (q's scan was left
    to stage 3, scan_inputs_async) a non-finite normaliser triggers the scan of
    q, so a NaN/Inf in q still raises InputError."""
    bad_input = finite_flag is not None and int(finite_flag.item()) != 0
    if bad_input:
        _read_status(device)
        raise InputError("q/k/v contain NaN or Inf")
    if rescan_q is not None:
        bits = _read_status(device)
        if bits[0] & _lib.SA_STATUS_NORMALISER:
            f = torch.zeros(1, dtype=torch.int32, device=rescan_q.device)
            check_finite_async((rescan_q,), f, _stream(rescan_q))
            if int(f.item()) != 0:
                raise InputError("q/k/v contain NaN or Inf")
        _raise_status(bits)
        return
    check_status(device)


@dataclass
class HeadBatch:
    """Device tensors q [Hq,S,d], k/v [Hkv,S,d] (contiguous, same dtype).

    q_head0 / group describe the GQA mapping for head-sharded runs: local q
    head h reads local kv head (q_head0 + h)//group - q_head0//group."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    group: int = 1
    q_head0: int = 0
    head_ids: tuple | None = None  # reference head ids (AttentionHead.head_id) when built from heads

    def __post_init__(self):
        q, k, v = self.q, self.k, self.v
        if not (isinstance(q, torch.Tensor) and isinstance(k, torch.Tensor) and isinstance(v, torch.Tensor)):
            raise InputError("HeadBatch needs torch tensors")
        if q.dim() != 3 or k.dim() != 3 or v.dim() != 3:
            raise InputError("q must be [Hq,S,d], k and v [Hkv,S,d]")
        if k.shape != v.shape or q.shape[1:] != k.shape[1:]:
            raise InputError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
        if not (q.dtype == k.dtype == v.dtype) or q.dtype not in _DTYPES:
            raise InputError("q/k/v must share dtype bfloat16 or float32")
        if not (q.is_cuda and k.device == q.device and v.device == q.device):
            raise InputError("q/k/v must live on one CUDA device")
        self.q, self.k, self.v = q.contiguous(), k.contiguous(), v.contiguous()
        if self.group < 1:
            raise InputError("group must be >= 1")

    @property
    def Hq(self) -> int:
        return int(self.q.shape[0])

    @property
    def Hkv(self) -> int:
        return int(self.k.shape[0])

    @property
    def S(self) -> int:
        return int(self.q.shape[1])

    @property
    def d(self) -> int:
        return int(self.q.shape[2])

    @property
    def dtype_code(self) -> int:
        return _DTYPES[self.q.dtype]

    @property
    def stream(self) -> int:
        return _stream(self.q)

    @classmethod
    def from_tensors(cls, q, k, v, group: int | None = None, q_head0: int = 0) -> "HeadBatch":
        """q [Hq,S,d] (or [S,d]), k/v [Hkv,S,d]; group defaults to Hq // Hkv."""
        if q.dim() == 2:
            q, k, v = q[None], k[None], v[None]
        if group is None:
            if q.shape[0] % k.shape[0] != 0:
                raise InputError(f"Hq={q.shape[0]} is not a multiple of Hkv={k.shape[0]}")
            group = q.shape[0] // k.shape[0]
        return cls(q, k, v, group=group, q_head0=q_head0)

    @classmethod
    def from_heads(cls, heads, dtype=torch.bfloat16, device=None) -> "HeadBatch":
        """Stack reference-style heads (each with its own k, v) onto the device."""
        if isinstance(heads, AttentionHead):
            heads = HeadSet([heads])
        elif not isinstance(heads, HeadSet):
            heads = HeadSet(list(heads))
        device = torch.device(device or "cuda")

        def stack(attr):
            parts = []
            for h in heads:
                a = getattr(h, attr)
                t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
                parts.append(t.to(device=device, dtype=dtype))
            return torch.stack(parts).contiguous()

        return cls(stack("q"), stack("k"), stack("v"), group=1, q_head0=0,
                   head_ids=tuple(int(h.head_id) for h in heads))
