"""Head sharding across GPUs (one process per GPU) and the output gather.

Stages 1-3 are independent per q head (the reference loops heads
independently, pkg/src/blocksift/pipeline.py:169; the paper partitions heads
beyond 256K), so a job of Hq heads over N ranks gives rank r
the contiguous q heads [r*Hq/N, (r+1)*Hq/N) plus the KV heads they read, and
nothing crosses GPUs on the hot path.  The only collective is the optional
gather of the per-rank outputs (the 1M-token configuration), done with NCCL
all-gather over NVLink and overlapped with the next head chunk's compute.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import InputError

__all__ = ["HeadShard", "shard_heads", "sample_attention_sharded"]


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


def sample_attention_sharded(q_local: torch.Tensor, k_local: torch.Tensor, v_local: torch.Tensor,
                             shard: HeadShard, heads_per_chunk: int = 1, gather: bool = True,
                             process_group=None, compute_fn=None, out: torch.Tensor | None = None, **kw):
    """Run this rank's heads in chunks of `heads_per_chunk`.  With gather, the
    job's output [Hq,S,d] is allocated once and this rank computes straight
    into its own head rows; after each chunk every rank's rows of that chunk
    are broadcast in place from their owner (one NCCL broadcast per rank, on a
    side stream for CUDA tensors, so the NVLink transfer overlaps the next
    chunk's compute).  No temporaries, no copies: a head's rows are a
    contiguous slice of the final buffer.  Nothing synchronises the host.

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


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
