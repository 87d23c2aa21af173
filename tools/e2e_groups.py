"""e2e (host-buffer path) time at C3 for several head-group sizes of
sample_attention_host (the default, 4, measured best: ~45 ms; 2: ~47.5, 8: ~47, 16: ~52).

    python tools/e2e_groups.py
"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2406_15486_b200 as sa
from paper_2406_15486_b200 import synth
q, k, v, _ = synth.make_inputs(131072, 32, 2, 128, seed=0, device="cuda")
hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
ho = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
for hpg in (2, 4, 6, 8, 16):
    ts = []
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sa.sample_attention_host(hq, hk, hv, alpha=0.95, chunk_n=1, out=ho, heads_per_group=hpg)
        e1.record(); torch.cuda.synchronize()
        if i: ts.append(e0.elapsed_time(e1))
    print(hpg, [round(t, 2) for t in ts])
