"""CUDA-graph executor for repeated SampleAttention prefills on fixed buffers.

A serving loop calls the same attention shape over and over.  Launching the
~15 kernels of one sample_attention call from Python costs ~0.6 ms of host
time per call, and any host hiccup (a GC pause, a page fault) in the middle of
a call leaves the GPU idle, because stage 2 is enqueued only after the host
has finished the Python of stage 1.  Here the three stages are captured once
as CUDA graphs on static device buffers; a call is three graph launches that
the host enqueues in microseconds, so the GPU runs the whole pipeline back to
back.  Inputs are written into `q`, `k`, `v` (the captured buffers), the
result appears in `out`.

The captured work is exactly sample_attention's (stage 1 block_reduce, stage 2
select + guard + merge + schedule, stage 3 sparse_attention); only the NaN/Inf
check becomes asynchronous (a device flag and the stage-3 status read by
`check()`).
"""

from __future__ import annotations

import torch

from . import _lib
from .config import plan_chunks, resolve_config
from .errors import InputError
from .heads import HeadBatch, raise_on_flags, scan_inputs_async
from .stages import block_reduce, merge_index, private_workspace, sample_scores, select, sparse_attention

__all__ = ["SampleAttentionGraph"]


class SampleAttentionGraph:
    """Captured stage-1 / stage-2 / stage-3 graphs of one sample_attention
    configuration on the given device tensors q [Hq,S,d], k/v [Hkv,S,d]
    (which become the graph's input buffers).  Keyword arguments are those of
    sample_attention: alpha, alpha_c, alpha_s, chunk_n, sample_ratio, blk,
    sink_blocks, local_blocks, guard, group, q_head0."""

    def __init__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, alpha: float = 0.95,
                 alpha_c: float | None = None, alpha_s: float | None = None, chunk_n: int | None = None,
                 sample_ratio: float | None = None, blk: int = 128, sink_blocks: int = 0, local_blocks: int = 1,
                 guard: str = "auto", group: int | None = None, q_head0: int = 0, warmup: int = 2):
        self.batch = HeadBatch.from_tensors(q, k, v, group=group, q_head0=q_head0)
        b = self.batch
        self.cfg = resolve_config(b.S, alpha, alpha_c, alpha_s, chunk_n, sample_ratio, blk)
        self.plan = plan_chunks(b.S, self.cfg)
        self.guard, self.sink_blocks, self.local_blocks = guard, sink_blocks, local_blocks
        self.q, self.k, self.v = b.q, b.k, b.v
        self.out = torch.empty_like(b.q)
        self.flag = torch.zeros(1, dtype=torch.int32, device=b.q.device)
        dev = b.q.device
        with private_workspace(b, self.cfg.blk, self.plan.chunk_n) as ws:
            self._ws = ws  # the graphs hold its address: it lives as long as they do
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):  # warm-up: kernel attributes, TMA descriptors, allocator pools
                for _ in range(max(1, warmup)):
                    self._stage3(self._stage2(self._stage1()))
            torch.cuda.current_stream(dev).wait_stream(side)
            torch.cuda.synchronize(dev)
            self.graphs = [torch.cuda.CUDAGraph() for _ in range(3)]
            pool = torch.cuda.graph_pool_handle()
            n0 = _lib.launch_count()
            with torch.cuda.graph(self.graphs[0], pool=pool):
                self.reduced = self._stage1()
            with torch.cuda.graph(self.graphs[1], pool=pool):
                self.mask, self.selection = self._stage2(self.reduced)
            with torch.cuda.graph(self.graphs[2], pool=pool):
                self._stage3((self.mask, self.selection))
            # library kernels per replay (the C ABI counts launches as they are captured)
            self.kernels_per_replay = _lib.launch_count() - n0

    # ---- captured bodies
    def _stage1(self):
        b = self.batch
        self.flag.zero_()
        self._rescan = b.q if scan_inputs_async(b.q, b.k, b.v, self.flag, b.stream) else None
        return block_reduce(sample_scores(b, self.plan), self.cfg.blk)

    def _stage2(self, reduced):
        b = self.batch
        sel = select(reduced, self.cfg, guard=self.guard)
        mask = merge_index(sel, self.plan, self.cfg.blk, b.S, self.sink_blocks, self.local_blocks)
        mask.order(b.group, b.q_head0)
        return mask, sel

    def _stage3(self, mask_sel):
        mask, _ = mask_sel
        sparse_attention(self.batch, mask, out=self.out, report=False)

    # ---- replay
    def replay_stage(self, i: int) -> None:
        self.graphs[i].replay()

    def replay(self) -> torch.Tensor:
        """Run stages 1-3 on the current contents of q/k/v; returns `out`
        (stream-ordered on the current stream; no host synchronisation)."""
        for g in self.graphs:
            g.replay()
        return self.out

    def check(self) -> None:
        """Raise InputError if the last replay saw NaN/Inf in q/k/v, or the
        reference's stage-3 errors from the device status word (host sync)."""
        raise_on_flags(self.flag, self.batch.q.device, self._rescan)

    def n_rescored(self) -> int:
        return self.selection.n_rescored()
