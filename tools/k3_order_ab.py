"""Interleaved A/B of stage-3 unit pairings (and optionally library builds).

Orders compared on the same mask (all group-major, longest-first):
  product  the library's sa_schedule
  greedy   per (KV group, query block), heads paired greedily by the smallest
           symmetric difference of their key-block lists (host-computed)
    python tools/k3_order_ab.py --libs a.so b.so [--config c3] [--reps 8]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def greedy_order(grid, Hq, Hkv, cnt):
    H, nb, _ = grid.shape
    G = Hq // Hkv
    units = []
    for g in range(Hkv):
        hs = np.arange(g * G, (g + 1) * G)
        us = []
        for qb in range(nb):
            X = grid[hs, qb].astype(np.int32)
            c = X.sum(1)
            sym = c[:, None] + c[None, :] - 2 * (X @ X.T)
            np.fill_diagonal(sym, 1 << 30)
            left = list(range(G))
            while len(left) > 1:
                sub = sym[np.ix_(left, left)]
                i, j = np.unravel_index(np.argmin(sub), sub.shape)
                a, b = left[i], left[j]
                us.append((int(hs[a]) * nb + qb, int(hs[b]) * nb + qb))
                left = [x for x in left if x not in (a, b)]
        us.sort(key=lambda u: -(cnt.flat[u[0]] + cnt.flat[u[1]]))
        units += us
    return np.array(units, dtype=np.int32).reshape(-1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    import torch
    import paper_2406_15486_b200 as sa
    from paper_2406_15486_b200 import _lib, synth
    from bench import CONFIGS
    S, Hq, Hkv, alpha, cn, _ = CONFIGS[args.config]
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
    batch = sa.HeadBatch.from_tensors(q, k, v)
    _, res = sa.sample_attention(q, k, v, alpha=alpha, chunk_n=cn)
    mask = res.mask
    grid = mask.to_dense()
    cnt = mask.kv_cnt.cpu().numpy()
    orders = {"product": mask.order(batch.group, 0),
              "greedy": torch.from_numpy(greedy_order(grid, Hq, Hkv, cnt)).cuda()}
    assert orders["product"].numel() == orders["greedy"].numel()
    libs = []
    for p in args.libs:
        lib = ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL)
        fn = lib.sa_sparse_forward
        fn.restype, fn.argtypes = _lib.SIGNATURES["sa_sparse_forward"]
        libs.append((os.path.basename(p), fn))
    combos = [(li, on) for li in range(len(libs)) for on in orders]
    outs = {c: torch.empty_like(q) for c in combos}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def launch(c):
        li, on = c
        rc = libs[li][1](q.data_ptr(), k.data_ptr(), v.data_ptr(), _lib.SA_BF16, S, Hq, Hkv, 128, 128,
                         batch.group, 0, mask.kv_cnt.data_ptr(), mask.kv_idx.data_ptr(), orders[on].data_ptr(),
                         outs[c].data_ptr(), None, None, st)
        assert rc == 0, rc

    for c in combos:
        launch(c)
    torch.cuda.synchronize()
    times = {c: [] for c in combos}
    for r in range(args.reps):
        for j in range(len(combos)):
            c = combos[(j + r) % len(combos)]
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launch(c)
            e1.record()
            torch.cuda.synchronize()
            times[c].append(e0.elapsed_time(e1))
    base = outs[combos[0]].float()
    for c in combos:
        ts = times[c]
        print(json.dumps({"lib": libs[c[0]][0], "order": c[1], "median_ms": round(statistics.median(ts), 3),
                          "min_ms": round(min(ts), 3), "maxdiff": float((outs[c].float() - base).abs().max()),
                          "config": args.config}), flush=True)


if __name__ == "__main__":
    main()
