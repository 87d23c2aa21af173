"""Pin the CPU oracle (oracle/blocksift_port.py) to the reference's own outputs.

Fixtures were produced by tests/golden/make_golden.py from the unmodified
reference; the oracle must reproduce index sets and masks bit-exactly and the
fp64 scores/outputs to rounding.
"""

import json
import os

import numpy as np
import pytest

from oracle import blocksift_port as O
from tests.golden.inputs import RANDOM_CASES, random_qkv


@pytest.fixture(scope="module")
def random_fx(golden_dir):
    return np.load(os.path.join(golden_dir, "random_cases.npz"))


@pytest.fixture(scope="module")
def kats(golden_dir):
    with open(os.path.join(golden_dir, "kats.json")) as f:
        return json.load(f)


def picks(fx, name):
    k_c, k_s = fx[f"{name}/k_c"], fx[f"{name}/k_s"]
    ic, is_ = fx[f"{name}/i_c"], fx[f"{name}/i_s"]
    return [(tuple(int(x) for x in ic[c, : k_c[c]]), tuple(int(x) for x in is_[c, : k_s[c]]))
            for c in range(len(k_c))]


def test_find_k_kats(kats):
    for s, a, want in kats["find_k"]:
        assert O.find_k(s, a) == want, (s, a)


def test_arg_topk_kats(kats):
    for s, k, want in kats["arg_topk"]:
        assert list(O.arg_topk(s, k)) == want, (s, k)


def test_plan_kats(kats):
    for S, cn, blk, cn_eff, itv, wins in kats["plans"]:
        p = O.plan_chunks(S, cn, blk)
        assert p.chunk_n == cn_eff and p.itv == itv
        assert [list(w) for w in p.windows] == wins


def test_merge_kats(kats):
    for S, cn, blk, sels, text in kats["merges"]:
        plan = O.plan_chunks(S, cn, blk)
        grid = O.merge_index([(tuple(a), tuple(b)) for a, b in sels], plan)
        assert O.serialize_mask(grid, blk) == text


def test_block_reduce_hand(kats):
    col, slash = kats["block_reduce_hand"]
    cols, slashes, _ = O.block_reduce([(np.array([3]), np.array([[0.1, 0.2, 0.3, 0.4]]))], 4, 2)
    np.testing.assert_allclose(cols[0], col, rtol=0, atol=1e-15)
    np.testing.assert_allclose(slashes[0], slash, rtol=0, atol=1e-15)


@pytest.mark.parametrize("case", RANDOM_CASES, ids=[c["name"] for c in RANDOM_CASES])
def test_pipeline_matches_reference(case, random_fx):
    name = case["name"]
    q, k, v = random_qkv(case)
    with_out = f"{name}/out" in random_fx
    r = O.run_head(q, k, v, case["alpha_c"], case["alpha_s"], case["chunk_n"], case["blk"],
                   with_output=with_out)
    assert np.array_equal(np.array(r["plan"].windows), random_fx[f"{name}/windows"])
    tot = np.asarray(r["totals"])[:, None]
    np.testing.assert_allclose(np.stack(r["cols"]) / tot, random_fx[f"{name}/col"] / tot, rtol=0, atol=1e-13)
    np.testing.assert_allclose(np.stack(r["slashes"]) / tot, random_fx[f"{name}/slash"] / tot, rtol=0, atol=1e-13)
    assert r["selection"] == picks(random_fx, name)
    assert O.serialize_mask(r["grid"], case["blk"]) == str(random_fx[f"{name}/mask_text"])
    if with_out:
        np.testing.assert_allclose(r["out"], random_fx[f"{name}/out"], rtol=0, atol=2e-6)
        assert r["touched"] == int(random_fx[f"{name}/touched"])
        fl = O.flop_accounting(r["grid"], case["S"], case["d"], case["blk"])
        assert fl["estimated_flops_sparse"] == int(random_fx[f"{name}/flops_sparse"])
        assert fl["estimated_flops_dense"] == int(random_fx[f"{name}/flops_dense"])


def test_c1_head_matches_reference(golden_dir):
    fx = np.load(os.path.join(golden_dir, "c1_head.npz"))
    q, k, v = (fx[n].astype(np.float64) for n in "qkv")
    r = O.run_head(q, k, v, 0.95, 0.95, 2, 128, with_output=True)
    assert r["selection"] == picks({f"c1/{n}": fx[n] for n in ("k_c", "k_s", "i_c", "i_s")}, "c1")
    assert O.serialize_mask(r["grid"], 128) == str(fx["mask_text"])
    np.testing.assert_allclose(r["out"], fx["out"], rtol=0, atol=2e-6)
