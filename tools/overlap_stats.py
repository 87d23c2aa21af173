"""How much K/V traffic would pairing two (head, query block) work items in
one CTA save?  For the bench workload's masks, compares the summed list
lengths with the union lengths for two pairings:
  gqa : (h, qb) with (h', qb), h and h' adjacent q heads of one KV group
  adj : (h, qb) with (h, qb+1)

    python tools/overlap_stats.py [--config c3] [--alpha 0.95]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--alpha", type=float, default=None)
    a = ap.parse_args()
    S, Hq, Hkv, alpha, cn, _ = bench.CONFIGS[a.config]
    alpha = a.alpha or alpha
    dev = torch.device("cuda:0")
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=0, heads=list(range(Hq)), device=dev)
    _, res = sa.sample_attention(q, k, v, alpha=alpha, chunk_n=cn, group=Hq // Hkv)
    m = res.mask
    cnt = m.kv_cnt.cpu().numpy()
    idx = m.kv_idx.cpu().numpy()
    nb = cnt.shape[1]

    def lst(h, qb):
        o = qb * (qb + 1) // 2
        return idx[h, o:o + cnt[h, qb]]

    total = int(cnt.sum())
    g = Hq // Hkv
    u_gqa = 0
    for h in range(0, Hq, 2):
        assert h // g == (h + 1) // g
        for qb in range(nb):
            u_gqa += np.union1d(lst(h, qb), lst(h + 1, qb)).size
    u_adj = 0
    for h in range(Hq):
        for qb in range(0, nb, 2):
            a_ = lst(h, qb)
            b_ = lst(h, qb + 1) if qb + 1 < nb else np.array([], dtype=np.int32)
            u_adj += np.union1d(a_, b_).size
    # 4-way: heads (h..h+3) same qb
    u_g4 = 0
    for h in range(0, Hq, 4):
        for qb in range(nb):
            u_g4 += np.unique(np.concatenate([lst(h + i, qb) for i in range(4)])).size
    print(json.dumps({"config": a.config, "alpha": alpha, "density": round(m.block_density(), 4),
                      "blocks": total, "union_gqa2": u_gqa, "ratio_gqa2": round(u_gqa / total, 4),
                      "union_adj2": u_adj, "ratio_adj2": round(u_adj / total, 4),
                      "union_gqa4": u_g4, "ratio_gqa4": round(u_g4 / total, 4)}))


if __name__ == "__main__":
    main()
