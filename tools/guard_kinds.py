"""Which margin flags the guard's pairs (alpha cut vs boundary tie) and how
many blocks sit in the tie band -- sizing a band-only exact refinement.

    python tools/guard_kinds.py S chunk_n Hkv
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402
from paper_2406_15486_b200.stages import GUARD_EPS, GUARD_LOGIT_REF  # noqa: E402

S = int(sys.argv[1]); cn = int(sys.argv[2]); Hkv = int(sys.argv[3]); Hq = 32
if len(sys.argv) > 4 and sys.argv[4] == "ref":  # the reference's calibrated generator (bench --config c2ref)
    import bench
    q, k, v, _, _ = bench.workload_inputs("c2ref", S, Hq, Hkv, 128, 0, list(range(Hq)), "cuda")
else:
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
b = sa.HeadBatch.from_tensors(q, k, v)
plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=cn))
rt = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="tensor")
rx = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="exact")
torch.cuda.synchronize()
bnd = rt.logit_bound.cpu().numpy().reshape(Hq, plan.chunk_n)
T = (rt.col.cpu().numpy(), rt.slash.cpu().numpy())
X = (rx.col.cpu().numpy(), rx.slash.cpu().numpy())


def select(s, alpha):
    order = np.lexsort((np.arange(len(s)), -s))
    cum = np.cumsum(s[order])
    kk = int(np.searchsorted(cum, alpha * cum[-1], side="left")) + 1
    return order, cum, kk


for alpha in (0.90, 0.95, 0.98):
    n_dec = n_cut = n_tie_only = 0
    bands = []
    chains = []
    hybrid_ok = 0
    for h in range(Hq):
        for c in range(plan.chunk_n):
            E_rel = GUARD_EPS * max(1.0, bnd[h, c] / GUARD_LOGIT_REF)
            for d in range(2):
                st, sx = T[d][h, c], X[d][h, c]
                n_dec += 1
                order, cum, kk = select(st, alpha)
                tot = cum[-1]
                E = E_rel * tot
                m1 = cum[kk - 1] - alpha * tot
                m2 = alpha * tot - cum[kk - 2] if kk >= 2 else np.inf
                gap = st[order[kk - 1]] - st[order[kk]] if kk < len(st) else np.inf
                cut = m1 < E or m2 < E
                tie = gap < E
                if cut:
                    n_cut += 1
                elif tie:
                    n_tie_only += 1
                    srt = st[order]
                    a_, b_ = kk - 1, kk  # the chain of consecutive gaps < 2E around the cut (k2_select's run)
                    while a_ > 0 and srt[a_ - 1] - srt[a_] < 2 * E:
                        a_ -= 1
                    while b_ + 1 < len(srt) and srt[b_] - srt[b_ + 1] < 2 * E:
                        b_ += 1
                    chains.append(b_ - a_ + 1)
                    hi, lo = st[order[kk - 1]], st[order[kk]]
                    band = np.flatnonzero((st >= lo - 2 * E) & (st <= hi + 2 * E))
                    bands.append(len(band))
                    # band-only refinement: exact scores inside the band, tensor-core scores elsewhere
                    hyb = st.copy()
                    hyb[band] = sx[band]
                    above = np.flatnonzero(st > hi + 2 * E)
                    ob = band[np.lexsort((band, -hyb[band]))]
                    pick = np.sort(np.concatenate([above, ob[: kk - len(above)]]))
                    ox, _, kx = select(sx, alpha)
                    hybrid_ok += int(kx == kk and np.array_equal(pick, np.sort(ox[:kx])))
    print(f"alpha {alpha}: decisions {n_dec}, flagged by the cut {n_cut}, by the tie only {n_tie_only}; "
          f"tie band sizes {sorted(bands)[:5]}..{sorted(bands)[-5:] if bands else []} "
          f"(max {max(bands) if bands else 0}); band refinement reproduces the exact selection in "
          f"{hybrid_ok}/{n_tie_only}; k2_select runs: max {max(chains) if chains else 0}, "
          f"> 16: {sum(c > 16 for c in chains)}, > 64: {sum(c > 64 for c in chains)}", flush=True)
