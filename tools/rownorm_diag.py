"""Relative error of the tensor-core stage-1 row normalisers (log-sum-exp of
each sampled row) against the fp64 exact pass: the error that a band-only
exact refinement inherits from reusing them.

    python tools/rownorm_diag.py S chunk_n Hkv [scale sink]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402
from paper_2406_15486_b200.stages import _workspace  # noqa: E402

S = int(sys.argv[1]); cn = int(sys.argv[2]); Hkv = int(sys.argv[3]); Hq = 32
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
b = sa.HeadBatch.from_tensors(q, k, v)
plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=cn))
nb = -(-S // 128)
rows = Hq * plan.chunk_n * 128
align = lambda x: (x + 255) & ~255  # noqa: E731
off = align(3 * Hq * plan.chunk_n * 128 * nb * 4)
ws = _workspace(b, 128, plan.chunk_n)


def rowstat():
    return ws[off: off + rows * 16].view(torch.float64).view(rows, 2).clone().cpu().numpy()


sa.block_reduce(sa.sample_scores(b, plan), 128, mode="tensor")
torch.cuda.synchronize()
rt = rowstat()
sa.block_reduce(sa.sample_scores(b, plan), 128, mode="exact")
torch.cuda.synchronize()
rx = rowstat()
lse_t = np.log(rt[:, 1]) + rt[:, 0] * math.log(2.0)   # TC: max in log2 units
lse_x = np.log(rx[:, 1]) + rx[:, 0]                   # exact: natural units
ok = np.isfinite(lse_t) & np.isfinite(lse_x)
rel = np.abs(np.expm1(lse_t[ok] - lse_x[ok]))
print(f"S {S} cn {plan.chunk_n}: row normaliser relative error  median {np.median(rel):.3e}  "
      f"p99.9 {np.quantile(rel, 0.999):.3e}  max {rel.max():.3e}  rows {ok.sum()}")
