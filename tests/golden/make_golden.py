"""Generate golden fixtures from the UNMODIFIED reference (run in the build
container only; /root/reference does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src.  Inputs are
either regenerated on the fly from a seed (`random_head` below, numpy
default_rng -> deterministic) or stored (the calibrated C1 head, produced by
the reference's own generator, which cannot travel).  Outputs of the
reference's stage functions are stored so that the oracle port
(`oracle/blocksift_port.py`) and the GPU path can be checked against them.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import blocksift as bs  # noqa: E402
from tests.golden.inputs import (random_qkv, C1_SPEC, RANDOM_CASES, PIPELINE_CASES, TUNE_GRID,  # noqa: E402
                                 TUNE_TEMPLATE, WALL_KEYS)


def run_reference(q, k, v, alpha_c, alpha_s, chunk_n, blk, with_output):
    head = bs.AttentionHead(q, k, v)
    cfg = bs.SparseConfig(alpha_c, alpha_s, chunk_n=chunk_n, blk=blk)
    plan = bs.plan_chunks(head.S, cfg)
    samples = bs.sample_scores(head, plan)
    reduced = bs.block_reduce(samples, blk)
    mask = bs.select_and_merge(reduced, plan, cfg)
    rec = {
        "windows": np.array([[c.sample_start, c.sample_end, c.region_start, c.region_end]
                             for c in plan.chunks], dtype=np.int64),
        "chunk_n_eff": np.int64(plan.chunk_n),
        "col": np.stack([c.col_scores for c in reduced.chunks]),
        "slash": np.stack([c.slash_scores for c in reduced.chunks]),
        "total": np.array([c.total_mass for c in reduced.chunks]),
        "k_c": np.array([s.k_c for s in mask.provenance.chunks], dtype=np.int64),
        "k_s": np.array([s.k_s for s in mask.provenance.chunks], dtype=np.int64),
        "mask_text": np.array(mask.serialize()),
        "density": np.float64(mask.block_density()),
    }
    nb = mask.n_qblocks
    ic = np.full((len(plan.chunks), nb), -1, dtype=np.int64)
    is_ = np.full((len(plan.chunks), nb), -1, dtype=np.int64)
    for c, s in enumerate(mask.provenance.chunks):
        ic[c, : s.k_c] = s.i_c
        is_[c, : s.k_s] = s.i_s
    rec["i_c"], rec["i_s"] = ic, is_
    if with_output:
        out, rep = bs.sparse_attention(head, mask)
        rec["out"] = out.astype(np.float32)
        rec["touched"] = np.int64(rep.active_blocks)
        rec["flops_sparse"] = np.int64(rep.estimated_flops_sparse)
        rec["flops_dense"] = np.int64(rep.estimated_flops_dense)
    return rec


def kats() -> dict:
    """Known-answer values straight from the reference functions (the inputs
    are the ones its own tests use, tests/test_filtering.py:43-143,
    tests/test_sampler.py:86-166)."""
    out = {}
    out["find_k"] = [
        (s, a, bs.find_k(s, a)) for s, a in [
            ([0.5, 0.3, 0.2], 0.7), ([3.0, 1.0], 0.0), ([0.4, 0.0, 0.3, 0.0, 0.3], 1.0),
            ([0.0, 0.0], 0.9), ([0.25, 0.25, 0.25, 0.25], 0.5), ([0.25, 0.25, 0.25, 0.25], 0.75),
            ([1e-300, 1.0, 1e-300], 1.0), ([5.0, 5.0, 5.0, 1.0], 0.95),
        ]
    ]
    out["arg_topk"] = [
        (s, kk, list(bs.arg_topk(s, kk))) for s, kk in [
            ([0.1, 0.9, 0.5], 2), ([0.5, 0.5, 0.5], 1), ([0.5, 0.5, 0.5], 2),
            ([0.0, 0.3, 0.3, 0.0, 0.3], 2), ([1.0, 0.0, 0.0, 1.0], 3),
        ]
    ]
    plans = []
    for S, cn, blk in [(8, 2, 2), (1024, 1, 128), (300, 4, 128), (50, 3, 128),
                       (65536, 2, 128), (98304, 15, 128), (98304, 77, 128),
                       (131072, 1, 128), (1048576, 1, 128), (1024, 3, 128), (4096, 2, 128)]:
        p = bs.plan_chunks(S, bs.SparseConfig(chunk_n=cn, blk=blk))
        plans.append((S, cn, blk, p.chunk_n, p.itv,
                      [[c.sample_start, c.sample_end, c.region_start, c.region_end] for c in p.chunks]))
    out["plans"] = plans
    # merge_index worked examples (tests/test_filtering.py:109-143 + SURVEY 8c straddle)
    merges = []
    for S, cn, blk, sels in [
        (8, 2, 2, [((0,), (0,)), ((), (0, 1))]),
        (16, 1, 2, [((), (0,))]),
        (1024, 3, 128, [((0,), (0,)), ((1,), ()), ((), (2,))]),
        (16, 2, 2, [(tuple(range(8)), tuple(range(8)))] * 2),
    ]:
        plan = bs.plan_chunks(S, bs.SparseConfig(chunk_n=cn, blk=blk))
        selected = bs.SelectedIndices(tuple(
            bs.ChunkSelection(i_c=a, i_s=b, k_c=len(a), k_s=len(b)) for a, b in sels))
        merges.append((S, cn, blk, [[list(a), list(b)] for a, b in sels],
                       bs.merge_index(selected, plan, blk, S).serialize()))
    out["merges"] = merges
    # block_reduce hand case (tests/test_sampler.py:127-132)
    smp = bs.SampledScores(4, (bs.sampler.ChunkSample(np.array([3]), np.array([[0.1, 0.2, 0.3, 0.4]])),))
    red = bs.block_reduce(smp, 2)
    out["block_reduce_hand"] = [list(red.chunks[0].col_scores), list(red.chunks[0].slash_scores)]
    return out


def pipeline_goldens() -> dict:
    out = {}
    for name, ((ac, as_, cn, blk), heads) in PIPELINE_CASES.items():
        hs = []
        for case, hid in heads:
            q, k, v = random_qkv(case)
            hs.append(bs.AttentionHead(q, k, v, head_id=hid))
        rep = bs.run_pipeline(bs.HeadSet(hs), bs.SparseConfig(ac, as_, chunk_n=cn, blk=blk), want_oracle=True)
        flat = {kk: vv for kk, vv in rep.to_flat_dict().items() if not kk.endswith(WALL_KEYS)}
        out[name] = flat
    return out


def tune_golden():
    import blocksift.tuning as bt

    tasks = []
    orig = bt.generate_synthetic

    def rounded(spec):
        hset = orig(spec)
        heads = [bs.AttentionHead(h.q.astype(np.float32).astype(np.float64), h.k.astype(np.float32).astype(np.float64),
                                  h.v.astype(np.float32).astype(np.float64), head_id=h.head_id) for h in hset]
        tasks.append((spec.S, np.stack([np.stack([h.q, h.k, h.v]) for h in heads]).astype(np.float32)))
        return bs.HeadSet(heads)

    bt.generate_synthetic = rounded
    try:
        res = bt.tune(bs.TuneGrid(**TUNE_GRID), bs.SyntheticSpec(**TUNE_TEMPLATE))
    finally:
        bt.generate_synthetic = orig
    arrays = {f"task{i}_S{S}": a for i, (S, a) in enumerate(tasks)}
    return res.to_json_dict(), arrays


def main():
    if "--only-new" in sys.argv:  # the step-4/5 goldens alone (the older fixtures stay byte-identical)
        return main_new()
    # 1. KATs as JSON
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats(), f, indent=1)
    # 2. seeded random heads (inputs regenerated from the seed on both sides)
    recs = {}
    for case in RANDOM_CASES:
        q, k, v = random_qkv(case)
        rec = run_reference(q, k, v, case["alpha_c"], case["alpha_s"], case["chunk_n"],
                            case["blk"], with_output=case["S"] <= 2048)
        for key, val in rec.items():
            recs[f"{case['name']}/{key}"] = val
        print("case", case["name"], "density", float(rec["density"]))
    np.savez_compressed(os.path.join(HERE, "random_cases.npz"), **recs)
    # 3. the calibrated C1 head (reference generator; inputs stored as fp32)
    spec = bs.SyntheticSpec(**C1_SPEC)
    head = bs.generate_synthetic(spec).heads[0]
    q, k, v = (head.q.astype(np.float32), head.k.astype(np.float32), head.v.astype(np.float32))
    rec = run_reference(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64),
                        0.95, 0.95, 2, 128, with_output=True)
    np.savez_compressed(os.path.join(HERE, "c1_head.npz"), q=q, k=k, v=v, **rec)
    print("C1 density", float(rec["density"]), "k_c", rec["k_c"], "k_s", rec["k_s"])
    # 4. run_pipeline metrics (MetricsReport.to_flat_dict, wall times dropped)
    with open(os.path.join(HERE, "pipeline_metrics.json"), "w") as f:
        json.dump(pipeline_goldens(), f, indent=1, sort_keys=True)
    # 5. the reference tuner on its own generator (tasks recorded as fp32)
    res, arrays = tune_golden()
    with open(os.path.join(HERE, "tune_result.json"), "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "tune_tasks.npz"), **arrays)
    print("tune:", [(r["lo"], r["feasible"], r["best"]) for r in res["ranges"]])


def main_new():
    with open(os.path.join(HERE, "pipeline_metrics.json"), "w") as f:
        json.dump(pipeline_goldens(), f, indent=1, sort_keys=True)
    res, arrays = tune_golden()
    with open(os.path.join(HERE, "tune_result.json"), "w") as f:
        json.dump(res, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "tune_tasks.npz"), **arrays)
    print("tune:", [(r["lo"], r["feasible"], r["best"]) for r in res["ranges"]])


if __name__ == "__main__":
    main()
