"""Stage-1 pass over every (head, chunk) pair -- exact (fp64, DMMA) or tensor
(tcgen05) mode -- timed per library build (interleaved), plus the max
relative |col - col(first build)|.

    python tools/exact_bench.py --libs a.so b.so [--config c2] [--chunk-n 77] [--mode tensor] [--reps 5]
"""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", nargs="+")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--mode", choices=["exact", "tensor"], default="exact")
    ap.add_argument("--chunk-n", type=int, default=None)
    a = ap.parse_args()
    import torch
    import bench
    import paper_2406_15486_b200 as sa
    from paper_2406_15486_b200 import _lib, synth
    from paper_2406_15486_b200.stages import _workspace
    S, Hq, Hkv, alpha, cn, _ = bench.CONFIGS[a.config]
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=0, device="cuda")
    b = sa.HeadBatch.from_tensors(q, k, v)
    plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=a.chunk_n or cn))
    mode = _lib.SA_STAGE1_EXACT if a.mode == "exact" else _lib.SA_STAGE1_TENSOR
    nb = -(-S // 128)
    ws = _workspace(b, 128, plan.chunk_n)
    st = torch.cuda.current_stream().cuda_stream
    libs = []
    for p in a.libs:
        lib = ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL)
        fn = lib.sa_stage1
        fn.restype, fn.argtypes = _lib.SIGNATURES["sa_stage1"]
        libs.append((os.path.basename(p), fn))
    cols = [torch.zeros(Hq * plan.chunk_n * nb, dtype=torch.float64, device="cuda") for _ in libs]
    slash = torch.zeros_like(cols[0])

    def run(i):
        rc = libs[i][1](q.data_ptr(), k.data_ptr(), _lib.SA_BF16, S, Hq, Hkv, 128, 128, b.group, 0, plan.chunk_n,
                        plan.itv, cols[i].data_ptr(), slash.data_ptr(), None, mode, None,
                        ws.data_ptr(), ws.numel(), st)
        assert rc == 0, rc

    for i in range(len(libs)):
        run(i)
    torch.cuda.synchronize()
    ts = [[] for _ in libs]
    for r in range(a.reps):
        for j in range(len(libs)):
            i = (j + r) % len(libs)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(i)
            e1.record()
            torch.cuda.synchronize()
            ts[i].append(e0.elapsed_time(e1))
    for (name, _), t, c in zip(libs, ts, cols):
        rel = float(((c - cols[0]).abs() / cols[0].abs().clamp(min=1e-300)).max())
        print(name, "median ms %.3f min %.3f" % (statistics.median(t), min(t)), "max rel diff vs first %.3g" % rel,
              "pairs", Hq * plan.chunk_n, flush=True)


if __name__ == "__main__":
    main()
