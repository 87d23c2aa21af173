"""Prefix-sum error of the tensor-core stage-1 scores against the exact fp64
ones on large-logit heads (the guard's error model: error / total grows with
the per-pair logit bound max||q|| max||k|| / sqrt(d))."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_15486_b200 as sa

rows = []
for seed, scale, sink in [(0, 1.0, 0.0), (0, 2.0, 30.0), (1, 3.0, 60.0), (2, 2.5, 120.0), (3, 4.0, 0.0), (4, 5.0, 200.0)]:
    S, cn = 8192, 8
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((S, 128)) * scale
    k = rng.standard_normal((S, 128)) * scale
    if sink:
        u = rng.standard_normal(128); u /= np.linalg.norm(u)
        q += np.sqrt(sink) * u
        pos = rng.choice(S, size=24, replace=False)
        k[pos] += np.outer(rng.uniform(0.3, 1.0, size=24), u) * np.sqrt(sink) * np.sqrt(128)
    qt = torch.from_numpy(q).to("cuda", torch.bfloat16)[None]
    kt = torch.from_numpy(k).to("cuda", torch.bfloat16)[None]
    b = sa.HeadBatch.from_tensors(qt, kt, kt)
    plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=cn))
    rt = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="tensor")
    rx = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="exact")
    bnd = rt.logit_bound.cpu().numpy()[0]
    for c in range(cn):
        e = 0.0
        for a_t, a_x in ((rt.col[0, c], rx.col[0, c]), (rt.slash[0, c], rx.slash[0, c])):
            a_t, a_x = a_t.cpu().numpy(), a_x.cpu().numpy()
            e = max(e, np.abs(np.cumsum(-np.sort(-a_t)) - np.cumsum(-np.sort(-a_x))).max() / a_x.sum())
        rows.append({"seed": seed, "scale": scale, "sink": sink, "chunk": c, "bound": float(bnd[c]), "err": float(e)})
for r in rows:
    print(json.dumps(r))
arr = np.array([(r["bound"], r["err"]) for r in rows])
print("max err/bound:", (arr[:, 1] / arr[:, 0]).max(), " max err:", arr[:, 1].max())
