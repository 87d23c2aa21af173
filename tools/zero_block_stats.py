"""How many kept (query block, key block) pairs of the stage-3 mask carry no
probability mass at all in fp32 (every row's block max logit at least 134
log2 units below the row max over its kept blocks: exp2 underflows to 0 even
against a reference max lagging by the lazy-rescale threshold of 8)?  Those
blocks' PV MMAs add exact zeros.  Diagnostic only.

    python tools/zero_block_stats.py [--config c3] [--heads 0 17]
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
ap.add_argument("--config", default="c3")
ap.add_argument("--heads", type=int, nargs="+", default=[0, 17])
ap.add_argument("--gap", type=float, default=134.0)
a = ap.parse_args()
S, Hq, Hkv, alpha, cn, _ = bench.CONFIGS[a.config]
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
_, res = sa.sample_attention(q, k, v, alpha=alpha, chunk_n=cn)
mask = res.mask
group = Hq // Hkv
sl2 = 1.4426950408889634 / 128 ** 0.5
cnt = mask.kv_cnt.cpu()
for h in a.heads:
    kvh = h // group
    tot = zero = 0
    for qb in range(S // 128):
        n = int(cnt[h, qb])
        lst = mask.kv_idx[h, qb * (qb + 1) // 2: qb * (qb + 1) // 2 + n].long()
        qq = q[h, qb * 128:(qb + 1) * 128].float()
        keys = k[kvh].view(-1, 128, 128)[lst].float()          # [n, 128 keys, d]
        s = torch.einsum("rd,nkd->nrk", qq, keys) * sl2         # [n, 128 rows, 128 keys], log2 units
        if lst[-1].item() == qb:  # causal mask on the diagonal block
            tri = torch.triu(torch.ones(128, 128, dtype=torch.bool, device=s.device), 1)
            s[-1].masked_fill_(tri, float("-inf"))
        bmax = s.amax(dim=2)                                     # [n, rows]
        rmax = bmax.amax(dim=0, keepdim=True)                    # [1, rows]
        gap = (bmax - rmax).amax(dim=1)                          # [n]: the closest row
        tot += n
        zero += int((gap < -a.gap).sum().item())
    print(f"head {h}: {zero} of {tot} kept blocks carry no fp32 mass ({100.0 * zero / max(1, tot):.2f} %)")
