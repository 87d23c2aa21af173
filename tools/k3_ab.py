"""Interleaved A/B timing of stage-3 (K3) builds on one workload, in ONE
process: every build's libsampleattn.so is dlopen'ed side by side (RTLD_LOCAL,
so their symbols do not clash) and the launches alternate between builds, so
all see the same clocks, power state and L2 conditions.

    python tools/k3_ab.py --libs a.so b.so ... [--config c3] [--alpha A] [--dense] [--reps 12]

The mask, schedule and inputs come from the product library; each build's
sa_sparse_forward runs on them, L2 flushed before every launch.  Prints per
build the median / min stage-3 ms and the max |out - out(first build)|.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--chunk-n", type=int, default=None)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--reps", type=int, default=12)
    args = ap.parse_args()
    import torch
    import paper_2406_15486_b200 as sa
    from paper_2406_15486_b200 import _lib, synth
    from bench import CONFIGS
    S, Hq, Hkv, alpha, cn, _ = CONFIGS[args.config]
    alpha = args.alpha or alpha
    cn = args.chunk_n or cn
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
    batch = sa.HeadBatch.from_tensors(q, k, v)
    if args.dense:
        mask = sa.BlockMask.full(Hq, S, 128)
    else:
        _, res = sa.sample_attention(q, k, v, alpha=alpha, chunk_n=cn)
        mask = res.mask
    order = mask.order(batch.group, 0)
    libs = []
    for p in args.libs:
        lib = ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL)
        fn = lib.sa_sparse_forward
        fn.restype, fn.argtypes = _lib.SIGNATURES["sa_sparse_forward"]
        libs.append((os.path.basename(p), fn))
    outs = [torch.empty_like(q) for _ in libs]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def launch(i):
        rc = libs[i][1](q.data_ptr(), k.data_ptr(), v.data_ptr(), _lib.SA_BF16, S, Hq, Hkv, 128, 128,
                        batch.group, 0, mask.kv_cnt.data_ptr(), mask.kv_idx.data_ptr(), order.data_ptr(),
                        outs[i].data_ptr(), None, None, st)
        assert rc == 0, rc

    for i in range(len(libs)):  # warm-up (kernel attributes, TMA descriptors)
        launch(i)
    torch.cuda.synchronize()
    times = [[] for _ in libs]
    for r in range(args.reps):
        for j in range(len(libs)):
            i = (j + r) % len(libs)  # rotate the order every round
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            launch(i)
            e1.record()
            torch.cuda.synchronize()
            times[i].append(e0.elapsed_time(e1))
    base = outs[0].float()
    for (name, _), ts, o in zip(libs, times, outs):
        print(json.dumps({"lib": name, "median_ms": round(statistics.median(ts), 3), "min_ms": round(min(ts), 3),
                          "max_ms": round(max(ts), 3), "maxdiff_vs_first": float((o.float() - base).abs().max()),
                          "config": args.config, "alpha": alpha, "dense": args.dense}), flush=True)


if __name__ == "__main__":
    main()
