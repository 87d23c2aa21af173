"""Stage-1 (K1) work that is exactly zero: per 32-row warp of a sampled window
and key block, are all exp2 arguments below -127 (ex2.approx.ftz returns 0),
measured against the running max K1 would hold (ascending key blocks inside a
CTA's key split of `kpc` blocks)?  Diagnostic only.

    python tools/k1_dead_blocks.py [--config c4] [--chunk-n 77] [--heads 0 5] [--kpc 64]
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
ap.add_argument("--chunk-n", type=int, default=77)
ap.add_argument("--heads", type=int, nargs="+", default=[0, 5, 17])
ap.add_argument("--kpc", type=int, default=64)
ap.add_argument("--chunks", type=int, default=12, help="chunks sampled per head (evenly spread)")
a = ap.parse_args()
S, Hq, Hkv, alpha, _, _ = bench.CONFIGS[a.config]
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=a.chunk_n))
group = Hq // Hkv
sl2 = 1.4426950408889634 / 128 ** 0.5
cs = sorted(set(int(round(i * (plan.chunk_n - 1) / max(1, a.chunks - 1))) for i in range(a.chunks)))
for h in a.heads:
    tot = dead = dead_global = 0
    for c in cs:
        ch = plan.chunks[c]
        ss, se = ch.sample_start, ch.sample_end
        rows = torch.arange(ss, se, device="cuda")
        s = (q[h, ss:se].float() @ k[h // group, :se].float().T) * sl2          # [128, se] log2 units
        s = s.masked_fill(torch.arange(se, device="cuda")[None, :] > rows[:, None], float("-inf"))
        nkb = (se + 127) // 128
        pad = nkb * 128 - se
        if pad:
            s = torch.nn.functional.pad(s, (0, pad), value=float("-inf"))
        bmax = s.view(128, nkb, 128).amax(dim=2)                                # [rows, nkb]
        gmax = bmax.amax(dim=1, keepdim=True)
        # running max inside each key split, ascending blocks
        run = torch.empty_like(bmax)
        for k0 in range(0, nkb, a.kpc):
            run[:, k0:k0 + a.kpc] = torch.cummax(bmax[:, k0:k0 + a.kpc], dim=1).values
        gap = (bmax - run).view(4, 32, nkb).amax(dim=1)                         # warp x block: closest row
        gapg = (bmax - gmax).view(4, 32, nkb).amax(dim=1)
        tot += gap.numel()
        dead += int((gap < -127).sum().item())
        dead_global += int((gapg < -127).sum().item())
    print(f"head {h}: {dead} of {tot} (warp, key block) tiles exactly zero under the split running max "
          f"({100.0 * dead / max(1, tot):.2f} %), {100.0 * dead_global / max(1, tot):.2f} % against the row max")
