"""Head sharding across GPUs (one process per GPU) and the output gather.

Stages 1-3 are independent per q head (the reference loops heads
independently, pkg/src/blocksift/pipeline.py:169; the paper partitions heads
beyond 256K), so a job of Hq heads over N ranks gives rank r
the contiguous q heads [r*Hq/N, (r+1)*Hq/N) plus the KV heads they read, and
nothing crosses GPUs on the hot path.  The only exchange is the optional
gather of the per-rank outputs (the 1M-token configuration).  On GPUs it is
fused into stage 3: the ranks map each other's gather buffers (CUDA IPC over
NVLink / NVSwitch, PeerGather) and the K3 epilogue stores every finished
output row into all of them, so the transfer overlaps the attention tile by
tile (sa_sparse_forward_peers).  Elsewhere (CPU tensors, the gloo tests) the
rows are broadcast from their owner after each head chunk.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .errors import InputError

__all__ = ["HeadShard", "shard_heads", "sample_attention_sharded", "PeerGather"]


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    q_heads: tuple      # global q head indices owned by this rank
    kv_heads: tuple     # global kv heads they read
    group: int          # q heads per kv head (GQA group size)

    @property
    def q_head0(self) -> int:
        return self.q_heads[0]

    def local_kv(self, h_global: int) -> int:
        """Local kv index of global q head h (the C ABI's mapping
        (q_head0 + h)/group - q_head0/group)."""
        return h_global // self.group - self.q_heads[0] // self.group


def shard_heads(Hq: int, Hkv: int, world: int, rank: int) -> HeadShard:
    if Hq < 1 or Hkv < 1 or Hq % Hkv:
        raise InputError(f"Hq={Hq} must be a positive multiple of Hkv={Hkv}")
    if world < 1 or not 0 <= rank < world:
        raise InputError(f"bad rank {rank} of {world}")
    if Hq % world:
        raise InputError(f"{Hq} q heads do not split evenly over {world} ranks")
    per = Hq // world
    group = Hq // Hkv
    q = tuple(range(rank * per, (rank + 1) * per))
    kv = tuple(sorted({h // group for h in q}))
    return HeadShard(rank, world, q, kv, group)


class PeerGather:
    """Every rank's gather buffer mapped into this process.  Built
    collectively: each rank exports the CUDA IPC handle (+ byte offset) of its
    buffer, all ranks exchange them, and the peers' handles are opened once per
    allocation (cached, since opening an IPC mapping costs milliseconds).
    addr[r] is the device address of rank r's buffer (this rank's own pointer
    for r == rank)."""

    _opened: dict = {}  # (peer handle bytes) -> mapped base address

    def __init__(self, full: torch.Tensor, rank: int, world: int, process_group=None):
        import torch.distributed as dist

        handle = (ctypes.c_char * _lib.SA_IPC_HANDLE_BYTES)()
        off = ctypes.c_ulonglong(0)
        with torch.cuda.device(full.device):
            _lib.call("sa_ipc_export", ctypes.c_void_p(full.data_ptr()), handle, ctypes.byref(off))
        got = [None] * world
        dist.all_gather_object(got, (bytes(handle), int(off.value)), group=process_group)
        self.addr = []
        for r, (h, o) in enumerate(got):
            if r == rank:
                self.addr.append(full.data_ptr())
                continue
            base = PeerGather._opened.get(h)
            if base is None:
                ptr = ctypes.c_void_p()
                with torch.cuda.device(full.device):
                    _lib.call("sa_ipc_open", ctypes.create_string_buffer(h, len(h)), ctypes.byref(ptr))
                base = PeerGather._opened[h] = int(ptr.value)
            self.addr.append(base + o)
        self.rank, self.world = rank, world

    def peers_at(self, byte_offset: int) -> list:
        """The other ranks' addresses of the same element of their buffers."""
        return [a + byte_offset for r, a in enumerate(self.addr) if r != self.rank]

    @classmethod
    def close_all(cls) -> None:
        for base in cls._opened.values():
            _lib.call("sa_ipc_close", ctypes.c_void_p(base))
        cls._opened.clear()


def sample_attention_sharded(q_local: torch.Tensor, k_local: torch.Tensor, v_local: torch.Tensor,
                             shard: HeadShard, heads_per_chunk: int = 1, gather: bool = True,
                             process_group=None, compute_fn=None, out: torch.Tensor | None = None,
                             transport: str = "auto", **kw):
    """Run this rank's heads in chunks of `heads_per_chunk`.  With gather, the
    job's output [Hq,S,d] is allocated once and this rank computes straight
    into its own head rows; every rank's rows reach every other rank's buffer:
      transport "p2p" (the default for bf16 CUDA tensors): stage 3 stores each
        finished output row into the peers' buffers too (PeerGather, CUDA IPC
        over NVLink), so the gather overlaps the attention tile by tile and no
        collective runs on the data path; the call ends with a stream sync and
        a barrier, after which every buffer holds every rank's rows (it also
        starts with one, so no rank writes into a buffer a peer still reads);
      transport "collective": after each chunk every rank's rows of that chunk
        are broadcast in place from their owner (one broadcast per rank, on a
        side stream for CUDA tensors, overlapping the next chunk's compute;
        nothing synchronises the host).
    No temporaries, no copies: a head's rows are a contiguous slice of the
    final buffer.

    compute_fn(q, k, v, q_head0=, group=, out=, **kw) defaults to
    sample_attention with check_inputs=False (no host sync per chunk); the CPU
    multi-process tests inject the oracle here.
    Returns (local_out [H_local,S,d], gathered [Hq,S,d] or None); local_out is
    a view of gathered when gathering."""
    import torch.distributed as dist

    if compute_fn is None:
        from .pipeline import sample_attention

        def compute_fn(*a, **k2):
            k2.setdefault("check_inputs", False)
            return sample_attention(*a, **k2)
    H, S, d = q_local.shape
    if H != len(shard.q_heads):
        raise InputError(f"shard owns {len(shard.q_heads)} heads, got {H}")
    world = shard.world
    do_gather = gather and world > 1
    if do_gather:
        full = out if out is not None else torch.empty((world * H, S, d), dtype=q_local.dtype,
                                                       device=q_local.device)
        if tuple(full.shape) != (world * H, S, d) or not full.is_contiguous():
            raise InputError(f"out must be a contiguous [{world * H},{S},{d}] tensor")
        mine = full[shard.rank * H:(shard.rank + 1) * H]
    else:
        full = None
        mine = out if out is not None else torch.empty_like(q_local)
    on_gpu = q_local.is_cuda
    if transport == "auto":
        transport = "p2p" if (on_gpu and q_local.dtype == torch.bfloat16) else "collective"
    if transport not in ("p2p", "collective"):
        raise InputError(f"unknown transport {transport!r}")
    if do_gather and transport == "p2p":
        if not on_gpu:
            raise InputError("the p2p gather needs CUDA tensors")
        if world - 1 > _lib.SA_MAX_PEERS:
            raise InputError(f"the p2p gather supports up to {_lib.SA_MAX_PEERS + 1} ranks")
        return _sharded_p2p(q_local, k_local, v_local, shard, heads_per_chunk, full, mine, process_group,
                            compute_fn, kw)
    comm = torch.cuda.Stream(device=q_local.device) if (do_gather and on_gpu) else None
    main = torch.cuda.current_stream(q_local.device) if on_gpu else None
    works = []
    for h0 in range(0, H, heads_per_chunk):
        h1 = min(H, h0 + heads_per_chunk)
        g0 = shard.q_heads[h0]
        kv0 = shard.local_kv(g0)
        kv1 = shard.local_kv(shard.q_heads[h1 - 1]) + 1
        compute_fn(q_local[h0:h1], k_local[kv0:kv1], v_local[kv0:kv1], q_head0=g0, group=shard.group,
                   out=mine[h0:h1], **kw)
        if not do_gather:
            continue
        if comm is not None:
            ev = torch.cuda.Event()
            ev.record(main)
            comm.wait_event(ev)
        with (torch.cuda.stream(comm) if comm is not None else _null()):
            for r in range(world):
                works.append(dist.broadcast(full[r * H + h0:r * H + h1], src=r, group=process_group,
                                            async_op=True))
    if not do_gather:
        return mine, None
    with (torch.cuda.stream(comm) if comm is not None else _null()):
        for w in works:
            w.wait()
    if comm is not None:
        main.wait_stream(comm)
        full.record_stream(comm)
    return mine, full


def _sharded_p2p(q_local, k_local, v_local, shard, heads_per_chunk, full, mine, process_group, compute_fn, kw):
    import torch.distributed as dist

    H, S, d = q_local.shape
    dev = q_local.device
    torch.cuda.current_stream(dev).synchronize()  # no rank writes into a buffer a peer may still be reading
    peers = PeerGather(full, shard.rank, shard.world, process_group)  # collective: also the entry barrier
    row_bytes = S * d * full.element_size()
    for h0 in range(0, H, heads_per_chunk):
        h1 = min(H, h0 + heads_per_chunk)
        g0 = shard.q_heads[h0]
        kv0 = shard.local_kv(g0)
        kv1 = shard.local_kv(shard.q_heads[h1 - 1]) + 1
        compute_fn(q_local[h0:h1], k_local[kv0:kv1], v_local[kv0:kv1], q_head0=g0, group=shard.group,
                   out=mine[h0:h1], peer_out=peers.peers_at((shard.rank * H + h0) * row_bytes), **kw)
    torch.cuda.current_stream(dev).synchronize()  # this rank's remote stores have landed
    dist.barrier(group=process_group)              # ... and every peer's
    return mine, full


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
