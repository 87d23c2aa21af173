"""Stage-1 (tensor-core block_reduce) time alone, median of many launches.

    python tools/stage1_bench.py [--config c4] [--chunk-n 77] [--reps 20]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--chunk-n", type=int, default=None)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
S, Hq, Hkv, alpha, cn, _ = bench.CONFIGS[a.config]
cn = a.chunk_n or cn
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=0, device="cuda")
b = sa.HeadBatch.from_tensors(q, k, v)
plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=cn))
ts = []
for i in range(a.reps + 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sa.block_reduce(sa.sample_scores(b, plan), 128, mode="tensor")
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"{a.config} cn={cn}: stage 1 median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f}  max {ts[-1]:.3f}")
