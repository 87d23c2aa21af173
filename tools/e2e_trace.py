"""Kineto trace of one host-buffer call (sample_attention_host) at C3: the
timeline of copies and kernels (start/end ms, relative to the first event)."""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402

S, Hq, Hkv = 131072, 32, 2
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
ho = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
kw = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
for _ in range(2):
    sa.sample_attention_host(hq, hk, hv, alpha=0.95, chunk_n=1, out=ho, **kw)
torch.cuda.synchronize()
for rep in range(3):
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        sa.sample_attention_host(hq, hk, hv, alpha=0.95, chunk_n=1, out=ho, **kw)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    t0 = min(e.time_range.start for e in evs)
    rows = []
    for e in evs:
        n = e.name
        if "emcpy" in n or "k3_share" in n or "xf_pass" in n or "k1_tc" in n or "Memset" in n:
            rows.append((round((e.time_range.start - t0) / 1e3, 2), round((e.time_range.end - t0) / 1e3, 2), n[:60]))
    rows.sort()
    end = max(e.time_range.end for e in evs)
    print(f"rep {rep}: span {(end - t0) / 1e3:.2f} ms", flush=True)
    for r in rows:
        print("  ", r)
    cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda")]
    slow = sorted(cpu, key=lambda e: -e.cpu_time_total)[:8]
    print("   slowest host CUDA API calls:", [(e.name, round(e.cpu_time_total / 1e3, 2)) for e in slow], flush=True)
