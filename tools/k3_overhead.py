"""Per-unit fixed cost of stage 3: K3 on a diagonal-only mask (every item one
block) at the C3 shape, against the same units with 16 and 64 blocks each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402

S, Hq, Hkv = 131072, 32, 2
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
nb = S // 128
b = sa.HeadBatch.from_tensors(q, k, v)
for width in (1, 16, 64):
    grid = np.zeros((Hq, nb, nb), dtype=bool)
    for qb in range(nb):
        grid[:, qb, max(0, qb - width + 1): qb + 1] = True
    mask = sa.BlockMask.from_dense(128, grid, S=S, device="cuda")
    for _ in range(2):
        sa.sparse_attention(b, mask, report=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sa.sparse_attention(b, mask, report=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    blocks = int(grid.sum())
    t = float(np.median(ts))
    units = Hq * nb // 2
    print(f"width {width}: {t:.3f} ms, {blocks} item-blocks, {units} units -> "
          f"{t * 1e3 * 148 / units:.2f} us per unit per SM, {t * 1e6 * 148 / blocks:.1f} ns per item-block per SM", flush=True)
