"""Dump the stage-2 block mask of a bench workload as packed bits (analysis aid).

Writes gpurun_out/<name>.npz with bits [H, nb, nb/8] (np.packbits of the
(query block x key block) grid per head).  Usage:
  python tools/dump_mask.py --config c3 --alpha 0.95 --out gpurun_out/mask_c3.npz
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402

CONFIGS = {"c2": (32768, 32, 2, 1), "c3": (131072, 32, 2, 1), "c4": (98304, 32, 8, 15)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--alpha", type=float, default=0.95)
    ap.add_argument("--chunk-n", type=int, default=None)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    S, Hq, Hkv, cn = CONFIGS[a.config]
    cn = a.chunk_n or cn
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=0, device="cuda")
    _, res = sa.sample_attention(q, k, v, alpha=a.alpha, chunk_n=cn)
    m = res.mask
    nb = m.n_qblocks
    bits = np.zeros((Hq, nb, nb // 8), dtype=np.uint8)
    for h in range(Hq):
        dense = m.head(h).to_dense()[0]
        bits[h] = np.packbits(dense.astype(bool), axis=1)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    np.savez_compressed(a.out, bits=bits, S=S, Hq=Hq, Hkv=Hkv, alpha=a.alpha, cn=cn)
    print("density", m.block_density(), "saved", a.out)


if __name__ == "__main__":
    main()
