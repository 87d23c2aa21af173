"""Per-call timing of one sample_attention step (device events between every
host call, plus host timestamps) to find GPU idle gaps inside the step.

    python tools/stage_diag.py [--config c3] [--alpha 0.95] [--steps 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import stages, synth  # noqa: E402
from paper_2406_15486_b200.config import plan_chunks, resolve_config  # noqa: E402
from paper_2406_15486_b200.heads import HeadBatch, check_finite  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    S, Hq, Hkv, alpha, cn, _ = bench.CONFIGS[a.config]
    alpha = a.alpha or alpha
    dev = torch.device("cuda:0")
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=0, heads=list(range(Hq)), device=dev)
    out = torch.empty_like(q)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for it in range(3 + a.steps):
        flush.zero_()
        marks = []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e, time.perf_counter()))

        mark("start")
        b = HeadBatch.from_tensors(q, k, v, group=Hq // Hkv)
        check_finite(b.q, b.k, b.v)
        mark("check_finite")
        cfg = resolve_config(S, alpha, None, None, cn, None, 128)
        plan = plan_chunks(S, cfg)
        red = stages.block_reduce(stages.sample_scores(b, plan), 128)
        mark("stage1")
        sel = stages.select(red, cfg, guard="auto")
        mark("select+guard")
        mask = stages.merge_index(sel, plan, 128, S)
        mark("merge")
        mask.order(b.group, 0)
        mark("schedule")
        stages.sparse_attention(b, mask, out=out, report=False)
        mark("stage3")
        torch.cuda.synchronize()
        if it >= 3:
            t0 = marks[0][2]
            row = {n: {"gpu_ms": round(marks[i - 1][1].elapsed_time(e), 3), "host_ms": round((h - t0) * 1e3, 3)}
                   for i, (n, e, h) in enumerate(marks) if i > 0}
            row["rescored"] = sel.n_rescored()
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
