"""e2e (host-buffer path) at C3 for several stage-3 head-group ramps of
sample_attention_host, interleaved (monkeypatches streaming._group_plan's
first-KV-group ramp).  Diagnostic / A-B only.

    [REPS=n] python tools/e2e_ramp_ab.py [2,2,3,5 1,1,2,3,5 ...]
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2406_15486_b200 as sa  # noqa: E402
from paper_2406_15486_b200 import streaming, synth  # noqa: E402

# a variant is "head ramp[/tail ramp]", e.g. 1,1,2,3,5/1,2,3 (the tail ramp lists the last groups from the end)
def _parse(a):
    h, _, t = a.partition("/")
    return (tuple(int(x) for x in h.split(",")), tuple(int(x) for x in t.split(",")) if t else (1, 2, 3))


RAMPS = [_parse(r) for r in sys.argv[1:]] or [((2, 2, 3, 5), (1, 2, 3)), ((1, 2, 3, 5), (1, 2, 3)),
                                              ((1, 1, 2, 3, 5), (1, 2, 3)), ((1, 2, 2, 3, 5), (1, 2, 3))]
REPS = int(os.environ.get('REPS', '7'))
orig = streaming._group_plan


def plan_with(ramp, tail_ramp=(1, 2, 3)):
    def plan(Hq, group, hpg):
        groups, h0 = [], 0
        n_kv = Hq // group
        for g in range(n_kv):
            rest, head, tail = group, [], []
            if g == n_kv - 1:
                for s in tail_ramp:
                    if rest > s:
                        tail.insert(0, s)
                        rest -= s
            if g == 0:
                for s in ramp:
                    if rest > s:
                        head.append(s)
                        rest -= s
            n_mid = -(-rest // hpg)
            sizes = head + ([rest // n_mid + (1 if i < rest % n_mid else 0) for i in range(n_mid)] if rest else []) + tail
            for s in sizes:
                groups.append((h0, h0 + s))
                h0 += s
        return groups
    return plan


assert plan_with((1, 1, 2, 3, 5))(32, 16, 4) == orig(32, 16, 4)
q, k, v, _ = synth.make_inputs(131072, 32, 2, 128, seed=0, device="cuda")
hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
ho = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
res = {r: [] for r in RAMPS}
for rep in range(REPS):
    for r in RAMPS:
        streaming._group_plan = plan_with(*r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sa.sample_attention_host(hq, hk, hv, alpha=0.95, chunk_n=1, out=ho)
        e1.record()
        torch.cuda.synchronize()
        if rep:
            res[r].append(e0.elapsed_time(e1))
for r, ts in res.items():
    ts.sort()
    print(r, "median", round(ts[len(ts) // 2], 3), "min", round(ts[0], 3))
