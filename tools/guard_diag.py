"""Diagnostics for the selection guard: tensor-core vs exact stage-1 score
error and the decision margins of every (head, chunk, direction)."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_15486_b200 as sa
from paper_2406_15486_b200 import synth

S = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cn = int(sys.argv[2]) if len(sys.argv) > 2 else 1
Hq, Hkv = 32, 2
q, k, v, kv = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
b = sa.HeadBatch.from_tensors(q, k, v)
plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=cn))
for _ in range(2):
    rt = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="tensor")
torch.cuda.synchronize()
t0 = time.time(); rt = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="tensor"); torch.cuda.synchronize(); t_tc = time.time() - t0
rx = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="exact"); torch.cuda.synchronize()
t0 = time.time(); rx = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="exact"); torch.cuda.synchronize(); t_x = time.time() - t0
print(f"stage1 tensor {t_tc*1e3:.2f} ms  exact {t_x*1e3:.2f} ms for {Hq*plan.chunk_n} pairs")
ct, cx = rt.col.cpu().numpy(), rx.col.cpu().numpy()
st_, sx = rt.slash.cpu().numpy(), rx.slash.cpu().numpy()
rows = []
for alpha in (0.9, 0.95, 0.98):
    worst_err, min_margin = 0.0, 1.0
    for h in range(Hq):
        for c in range(plan.chunk_n):
            for a_t, a_x in ((ct[h, c], cx[h, c]), (st_[h, c], sx[h, c])):
                srt = -np.sort(-a_x); cum = np.cumsum(srt); tot = cum[-1]
                err = np.abs(a_t - a_x).max() / tot
                cum_err = np.abs(np.cumsum(-np.sort(-a_t)) - cum).max() / tot
                tgt = alpha * tot
                kk = int(np.searchsorted(cum, tgt, side="left")) + 1
                m1 = (cum[kk - 1] - tgt) / tot
                m2 = (tgt - cum[kk - 2]) / tot if kk >= 2 else 1.0
                gap = (srt[kk - 1] - srt[kk]) / tot if kk < len(srt) else 1.0
                worst_err = max(worst_err, err, cum_err)
                min_margin = min(min_margin, m1, m2, gap)
                rows.append((alpha, h, c, err, cum_err, m1, m2, gap))
    print(f"alpha {alpha}: worst |tc-exact|/total {worst_err:.3e}  smallest decision margin {min_margin:.3e}")
arr = np.array([r[3:] for r in rows])
print("error quantiles (per-block max / total):", np.quantile(arr[:, 0], [0.5, 0.9, 1.0]))
print("prefix-sum error quantiles:", np.quantile(arr[:, 1], [0.5, 0.9, 1.0]))
mm = np.min(arr[:, 2:], axis=1)
for eps in (1e-5, 2e-6, 1e-6, 5e-7, 2e-7, 1e-7):
    print(f"eps {eps:.0e}: would flag {(mm < eps).sum()} of {len(mm)}")

# relative error of individual block scores (blocks above 1e-6 of total)
rel = []
for h in range(Hq):
    for c in range(plan.chunk_n):
        for a_t, a_x in ((ct[h, c], cx[h, c]), (st_[h, c], sx[h, c])):
            m = a_x > 1e-6 * a_x.sum()
            rel.append((np.abs(a_t - a_x)[m] / a_x[m]).max())
print("per-block relative error quantiles:", np.quantile(rel, [0.5, 0.9, 1.0]))

# error against the per-pair logit bound (sa_stage1's guard scale)
bnd = rt.logit_bound.cpu().numpy()
errs = []
for h in range(Hq):
    for c in range(plan.chunk_n):
        e = 0.0
        for a_t, a_x in ((ct[h, c], cx[h, c]), (st_[h, c], sx[h, c])):
            tot = a_x.sum()
            e = max(e, np.abs(np.cumsum(-np.sort(-a_t)) - np.cumsum(-np.sort(-a_x))).max() / tot)
        errs.append((bnd[h, c], e))
errs = np.array(errs)
print("logit bound quantiles:", np.quantile(errs[:, 0], [0.0, 0.5, 1.0]))
print("prefix-sum error / bound quantiles:", np.quantile(errs[:, 1] / errs[:, 0], [0.5, 0.9, 1.0]))
print(json.dumps({"S": S, "cn": cn, "bound_max": float(errs[:, 0].max()), "err_max": float(errs[:, 1].max()),
                  "err_over_bound_max": float((errs[:, 1] / errs[:, 0]).max())}))
