"""Time the round-1 single-item stage-3 kernel (k3_tc, selected with
SA_K3_IMPL=single) in dense mode under its runtime SA_K3_EXP variants
(0 full, 1 no softmax math, 2 no MMA, 3 neither) in subprocesses.  The product
kernel k3_share takes its experiment variants at build time instead
(SA_NVCC_EXTRA=-DSA_K3_EXP=..., see tools/k3_variants.sh)."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import torch, json, sys
sys.path.insert(0, ".")
import paper_2406_15486_b200 as sa
H, S = 32, 32768
torch.manual_seed(0)
q, k, v = (torch.randn(n, S, 128, device="cuda", dtype=torch.bfloat16) for n in (H, 2, 2))
o = torch.empty_like(q)
for _ in range(3): sa.dense_attention(q, k, v, out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record(); sa.dense_attention(q, k, v, out=o); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
fl = 4 * 128 * sum(128 * (qb * 128 + 128) for qb in range(S // 128)) * H
print(json.dumps({"ms": min(ts), "tflops": fl / min(ts) / 1e9}))
'''
libs = sys.argv[1:] or [""]
modes = [int(m) for m in os.environ.get("MODES", "0,1,2,3").split(",")]
for lib in libs:
    for mode in modes:
        env = dict(os.environ, SA_K3_EXP=str(mode), SA_K3_IMPL="single")
        if lib:
            env["SA_LIB_PATH"] = os.path.abspath(lib)
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        print(lib or "default", mode, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:])
