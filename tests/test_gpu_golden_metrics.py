"""run_pipeline's MetricsReport and the tuner's result document against the
UNMODIFIED reference's own (tests/golden/make_golden.py, steps 4-5): same
inputs (bf16- or fp32-rounded, upcast as the reference sees them), same
config, same flat keys.

Tolerances: counts, flags and the config exactly; mask-derived ratios
(block_density, sparsity_ratio, flop_ratio) 1e-12; CRA 1e-10 when computed
in fp64 from fp64-exact partials (fp32 mode, and cra_full, which is a torch
fp64 recompute on the device) and 1e-6 for cra_sampled from the bf16
tensor-core partials (their fp32 accumulation, ~1e-7 relative);
output_error (sparse vs dense output, both from the kernels) 2e-2 in bf16
(the outputs' own tolerance) and 1e-4 in fp32."""

import json
import os

import numpy as np
import pytest
import torch

from tests.golden.inputs import PIPELINE_CASES, TUNE_GRID, WALL_KEYS, random_qkv

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def sa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_15486_b200 as m
    return m


@pytest.mark.parametrize("name", sorted(PIPELINE_CASES))
def test_run_pipeline_matches_reference_metrics(sa, name):
    golden = json.load(open(os.path.join(HERE, "pipeline_metrics.json")))[name]
    (ac, as_, cn, blk), heads = PIPELINE_CASES[name]
    bf16 = heads[0][0]["dtype"] == "bf16"
    hs = sa.HeadSet([sa.AttentionHead(*random_qkv(case), head_id=hid) for case, hid in heads])
    rep = sa.run_pipeline(hs, sa.SparseConfig(ac, as_, chunk_n=cn, blk=blk), want_oracle=True,
                          dtype=torch.bfloat16 if bf16 else torch.float32)
    got = {k: v for k, v in rep.to_flat_dict().items() if not k.endswith(WALL_KEYS)}
    assert sorted(got) == sorted(golden)
    for key, want in golden.items():
        have = got[key]
        if isinstance(want, (bool, str)) or key.endswith("active_blocks") or key in (
                "S", "d", "n_heads", "chunk_n", "effective_chunk_n", "blk"):
            assert have == want, key
        elif "output_error" in key:
            assert abs(have - want) <= (2e-2 if bf16 else 1e-4), (key, have, want)
        elif "cra_sampled" in key:
            assert abs(have - want) <= (1e-6 if bf16 else 1e-10), (key, have, want)
        elif "cra_full" in key:
            assert abs(have - want) <= 1e-10, (key, have, want)
        else:  # block_density, sparsity_ratio, flop_ratio and their means, alphas
            assert abs(have - want) <= 1e-12, (key, have, want)


def test_tune_matches_reference_on_its_tasks(sa):
    """The reference's tune() on its own calibrated generator (each head
    rounded to fp32 and recorded): the GPU tuner on the same tasks reports the
    same feasibility, the same winner and the same per-cell values."""
    from paper_2406_15486_b200.tuning import TuneGrid, tune
    golden = json.load(open(os.path.join(HERE, "tune_result.json")))
    arrays = np.load(os.path.join(HERE, "tune_tasks.npz"))
    grid = TuneGrid(**TUNE_GRID)
    keys = sorted(arrays.files, key=lambda k: int(k.split("_")[0][4:]))  # generation order
    assert len(keys) == len(grid.length_ranges) * grid.trials_per_cell
    tasks, it = [], iter(keys)
    for lo, hi in grid.length_ranges:
        per = []
        for _ in range(grid.trials_per_cell):
            a = torch.from_numpy(arrays[next(it)]).to("cuda")  # [heads, 3, S, d] fp32
            assert a.shape[2] == hi
            per.append(sa.HeadBatch.from_tensors(a[:, 0].contiguous(), a[:, 1].contiguous(), a[:, 2].contiguous()))
        tasks.append(per)
    got = tune(grid, tasks=tasks, seed=golden["seed"]).to_json_dict()
    assert got["recall_target"] == golden["recall_target"] and got["trials_per_cell"] == golden["trials_per_cell"]
    for rg, rw in zip(got["ranges"], golden["ranges"]):
        assert (rg["lo"], rg["hi"], rg["feasible"]) == (rw["lo"], rw["hi"], rw["feasible"])
        assert (rg["best"] is None) == (rw["best"] is None)
        if rw["best"] is not None:
            for key in ("alpha_c", "alpha_s", "chunk_n", "cra_metric"):
                assert rg["best"][key] == rw["best"][key], key
        for cg, cw in zip(rg["grid"], rw["grid"]):
            assert (cg["alpha_c"], cg["alpha_s"], cg["chunk_n"], cg["feasible"]) == \
                (cw["alpha_c"], cw["alpha_s"], cw["chunk_n"], cw["feasible"])
            assert abs(cg["mean_density"] - cw["mean_density"]) <= 1e-12
            assert abs(cg["mean_cra"] - cw["mean_cra"]) <= 1e-10, (cg, cw)
