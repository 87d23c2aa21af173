"""How many guard decisions a per-row certificate of the tie would settle.

The band refinement normalises the exact (fp64) block numerators with stage 1's
tensor-core row normalisers Z_r (1 + d_r), |d_r| <= dmax.  The order of the two
cut blocks a, b is then certain when

    |s_a - s_b| > dmax * (s_a + s_b)            (the product's test, BAND_EPS), or
    |s_a - s_b| > dmax * sum_r |x_ra - x_rb|    (per-row: the d_r act on both blocks of a row alike),

x_rb being row r's exact mass in block b.  This prints, per alpha, how many
decisions pass each test on exact fp64 scores of the given inputs.

    python tools/band_w_diag.py S Hkv [ref]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2406_15486_b200 import synth  # noqa: E402
from paper_2406_15486_b200.stages import BAND_EPS, GUARD_EPS  # noqa: E402

S = int(sys.argv[1]); Hkv = int(sys.argv[2]); Hq = 32; blk = 128; nb = S // blk
if len(sys.argv) > 3 and sys.argv[3] == "ref":
    import bench
    q, k, v, _, _ = bench.workload_inputs("c2ref", S, Hq, Hkv, 128, 0, list(range(Hq)), "cuda")
else:
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
rows = torch.arange(S - blk, S, device="cuda")  # chunk_n = 1: the last query block is the sampled window
key = torch.arange(S, device="cuda")
off = ((rows[:, None] - key[None, :]).clamp(min=0) // blk).clamp(max=nb - 1)
res = {a: [0, 0, 0, 0] for a in (0.90, 0.95, 0.98)}
ratios = []
for h in range(Hq):
    qr = q[h, S - blk:].double()
    kk = k[h // (Hq // Hkv)].double()
    s = (qr @ kk.T) / np.sqrt(128)
    s = s.masked_fill(key[None, :] > rows[:, None], float("-inf"))
    p = torch.softmax(s, dim=1)
    xc = p.view(blk, nb, blk).sum(2)  # [row, col block]
    xs = torch.zeros(blk, nb, dtype=torch.float64, device="cuda").scatter_add_(1, off, p)
    for X in (xc, xs):
        sc = X.sum(0).cpu().numpy()
        Xn = X.cpu().numpy()
        order = np.lexsort((np.arange(nb), -sc))
        cum = np.cumsum(sc[order])
        for alpha in res:
            kq = int(np.searchsorted(cum, alpha * cum[-1], side="left")) + 1
            if kq >= nb:
                continue
            a, b = order[kq - 1], order[kq]
            D = sc[a] - sc[b]
            W = np.abs(Xn[:, a] - Xn[:, b]).sum()
            r = res[alpha]
            r[0] += 1
            r[1] += D > BAND_EPS * (sc[a] + sc[b])
            r[2] += D > BAND_EPS * W
            r[3] += D < GUARD_EPS * cum[-1]
            ratios.append((alpha, D / (sc[a] + sc[b]), D / max(W, 1e-300)))
for alpha, r in res.items():
    print(f"alpha {alpha}: decisions {r[0]}; tie certified by BAND_EPS*(a+b): {r[1]}, by BAND_EPS*sum|x_a-x_b|: {r[2]}; "
          f"gap below GUARD_EPS*total: {r[3]}")
for alpha in res:
    rr = np.array([(x, y) for a, x, y in ratios if a == alpha])
    print(f"alpha {alpha}: gap/(a+b) quantiles {np.quantile(rr[:, 0], [0, .1, .5]).round(8)}, "
          f"gap/W quantiles {np.quantile(rr[:, 1], [0, .1, .5]).round(8)}")
