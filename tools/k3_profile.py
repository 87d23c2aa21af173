"""Cycle accounting of the stage-3 kernel k3_share (library built with
-DSA_K3_PROF=1, e.g. SA_NVCC_EXTRA=-DSA_K3_PROF=1 python -m
paper_2406_15486_b200.build --out=paper_2406_15486_b200/exp/libsa_PROF.so and
SA_LIB_PATH pointing at it): per processed (item, key block), the cycles each
role spends in each phase, on the bench workload (default C3, alpha 0.95).

    python tools/k3_profile.py [--config c3] [--dense]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import _lib, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--dense", action="store_true")
a = ap.parse_args()
S, Hq, Hkv, alpha, cn, _ = bench.CONFIGS[a.config]
dev = torch.device("cuda:0")
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=0, heads=list(range(Hq)), device=dev)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 16)()


def run():
    if a.dense:
        sa.dense_attention(q, k, v, group=Hq // Hkv)
    else:
        sa.sample_attention(q, k, v, alpha=alpha, chunk_n=cn, group=Hq // Hkv)
    torch.cuda.synchronize()


run()
reader = lib.sa_debug_k3s_profile
reader(buf, 1)
run()
reader(buf, 1)
c = list(buf)
blocks = max(1, c[13])
names = {0: "softmax: wait S", 1: "softmax: pass 1 (max)", 2: "softmax: rescale", 3: "softmax: pass 2 (exp, P)",
         4: "softmax: wait O (epilogue)", 5: "mma: wait P part", 6: "mma: wait P full", 7: "mma: wait V",
         8: "mma: wait K", 9: "mma: wait Q", 10: "tma: wait K slot", 11: "tma: wait V slot",
         12: "mma: loop total"}
print(f"{a.config} {'dense' if a.dense else 'sparse'}: {blocks} (item, block) pairs")
for i, nm in names.items():
    # softmax slots are summed over 4 warps of a tile (lane 0 each); others once per CTA
    div = blocks * (4 if i <= 4 else 1)
    print(f"{nm:28s} {c[i] / div:10.1f} cycles per (item, block)")
