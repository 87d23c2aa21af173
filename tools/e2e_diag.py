"""Timing of the host-buffer path (sample_attention_host) variants at C3."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import synth  # noqa: E402

S, Hq, Hkv = int(os.environ.get("S", 131072)), 32, 2
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, seed=0, device="cuda")
hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
ho = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
for name, kw in [("default", {}), ("one_lane", {"_lanes": 1}), ("hpg16", {"heads_per_group": 16}),
                 ("hpg4", {"heads_per_group": 4}), ("no_check", {"check_inputs": False})]:
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, res = sa.sample_attention_host(hq, hk, hv, alpha=0.95, chunk_n=1, out=ho, **kw)
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r = res[0]
        print(name, rep, "event ms %.2f host ms %.2f" % (e0.elapsed_time(e1), (t1 - t0) * 1e3),
              {k_: round(v_, 2) for k_, v_ in r.stage_ms().items()}, flush=True)
