"""QKV container I/O (the reference's flat binary format, ref tensor_io.py:1-80),
with a loader that goes straight to the GPU.

Layout (unchanged): one ASCII header line `QKV 1 <heads> <S> <d>`, the 4-byte
endianness probe 1.0f written little-endian, then little-endian float32
values, per head Q, K, V, each row-major [S, d].

`load_tensors(path)` returns a reference-style HeadSet (fp64 numpy) with the
reference's validation and error messages.  `load_tensors_device(path)`
validates the same header, maps the payload without a host copy, uploads the
fp32 cube once, runs the NaN/Inf scan on the device (sa_check_finite) and
returns a HeadBatch in the compute dtype; the host only re-reads the file to
name the first bad element when that scan fails.
"""

from __future__ import annotations

import struct
import warnings

import numpy as np
import torch

from . import _lib
from .errors import InputError
from .heads import AttentionHead, HeadBatch, HeadSet, dcall

__all__ = ["MAGIC", "load_tensors", "load_tensors_device", "save_tensors"]

MAGIC = 0x3F800000  # float32 1.0 (ref tensor_io.py:20)
_MAGIC_SWAPPED = 0x0000803F
_MAX_HEADER = 128


def save_tensors(heads, path) -> None:
    """Write a HeadSet / list of AttentionHead, or a (q, k, v) tuple of
    [n, S, d] tensors or arrays (one k, v per head), as QKV v1 (ref :25-32)."""
    if isinstance(heads, tuple) and len(heads) == 3:
        q, k, v = (t.detach().float().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
                   for t in heads)
        if not (q.shape == k.shape == v.shape) or q.ndim != 3:
            raise InputError("save_tensors needs q, k, v of one [n, S, d] shape")
        triples = [(q[i], k[i], v[i]) for i in range(q.shape[0])]
    else:
        hs = heads if isinstance(heads, HeadSet) else HeadSet(list(heads))
        triples = [tuple(np.asarray(a.cpu() if isinstance(a, torch.Tensor) else a) for a in (h.q, h.k, h.v))
                   for h in hs]
    n, (S, d) = len(triples), triples[0][0].shape
    with open(path, "wb") as f:
        f.write(f"QKV 1 {n} {S} {d}\n".encode("ascii"))
        f.write(struct.pack("<I", MAGIC))
        for tri in triples:
            for arr in tri:
                f.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())


def _parse(path, raw: memoryview):
    """Header / magic / size checks of ref tensor_io.py:35-68; returns
    (n, S, d, payload offset)."""
    head = bytes(raw[:_MAX_HEADER])
    nl = head.find(b"\n")
    if nl < 0:
        raise InputError(f"{path}: no header line within {_MAX_HEADER} bytes")
    fields = head[:nl].decode("ascii", errors="replace").split()
    if len(fields) != 5 or fields[0] != "QKV":
        raise InputError(f"{path}: malformed header {head[:nl]!r}")
    if fields[1] != "1":
        raise InputError(f"{path}: unsupported version {fields[1]!r}")
    try:
        n, S, d = (int(x) for x in fields[2:])
    except ValueError as e:
        raise InputError(f"{path}: malformed header {head[:nl]!r}") from e
    if n < 1 or S < 1 or d < 1:
        raise InputError(f"{path}: header counts must be positive, got {n}, {S}, {d}")
    body = nl + 1
    if len(raw) < body + 4:
        raise InputError(f"{path}: truncated before the magic value at byte {body}")
    (magic,) = struct.unpack("<I", bytes(raw[body: body + 4]))
    if magic != MAGIC:
        if magic == _MAGIC_SWAPPED:
            raise InputError(f"{path}: magic value is byte-swapped; file was written big-endian")
        raise InputError(f"{path}: bad magic value 0x{magic:08X} at byte {body}")
    payload = body + 4
    expected = n * 3 * S * d * 4
    got = len(raw) - payload
    if got != expected:
        raise InputError(f"{path}: payload at byte {payload} holds {got} bytes, expected {expected}")
    return n, S, d, payload


def _first_bad(path, values: np.ndarray, payload: int):
    finite = np.isfinite(values)
    if not finite.all():
        bad = int(np.flatnonzero(~finite)[0])
        raise InputError(f"{path}: non-finite value at byte {payload + 4 * bad} (element {bad})")


def load_tensors(path) -> HeadSet:
    """Host loader with the reference's semantics (ref tensor_io.py:35-80)."""
    raw = np.fromfile(path, dtype=np.uint8)
    n, S, d, payload = _parse(path, memoryview(raw))
    values = raw[payload:].view("<f4")
    _first_bad(path, values, payload)
    cube = values.astype(np.float64).reshape(n, 3, S, d)
    return HeadSet(tuple(AttentionHead(cube[i, 0], cube[i, 1], cube[i, 2], head_id=i) for i in range(n)))


def load_tensors_device(path, device=None, dtype=torch.bfloat16) -> HeadBatch:
    """Load straight to the GPU: q, k, v as [n, S, d] in `dtype` (each head
    its own k, v, as in the file).  Same validation and messages as
    load_tensors."""
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    n, S, d, payload = _parse(path, memoryview(mm))
    dev = torch.device(device or "cuda")
    with warnings.catch_warnings():  # the map is read-only; torch only reads it for the copy
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(np.asarray(mm[payload:]).view("<f4").reshape(n, 3, S, d))
    cube = host.to(dev)  # fp32, one H2D copy
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    dcall(cube.device, "sa_check_finite", cube.data_ptr(), _lib.SA_FP32, cube.numel(), flag.data_ptr(),
          torch.cuda.current_stream(cube.device).cuda_stream)
    if int(flag.item()) != 0:  # diagnostics only: name the first bad element like the reference
        _first_bad(path, np.asarray(mm[payload:]).view("<f4"), payload)
        raise InputError(f"{path}: non-finite value in the payload")
    q, k, v = (cube[:, j].to(dtype).contiguous() for j in range(3))
    del cube
    return HeadBatch(q, k, v, group=1)
