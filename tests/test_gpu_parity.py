"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures) and the pinned CPU oracle on identical inputs.

Bars: selected (i_c, i_s) index sets and the merged
block mask bit-identical; outputs within 2e-2 max-abs for bf16 and 1e-4 for
fp32, both against the reference's sparse_attention on the reference mask.
"""

import os

import numpy as np
import pytest
import torch

from oracle import blocksift_port as O
from tests.golden.inputs import RANDOM_CASES, random_qkv

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
FP32_TOL = 1e-4


@pytest.fixture(scope="module")
def sa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_15486_b200 as m
    return m


@pytest.fixture(scope="module")
def fx(golden_dir):
    return np.load(os.path.join(golden_dir, "random_cases.npz"))


def golden_picks(fx, name):
    k_c, k_s = fx[f"{name}/k_c"], fx[f"{name}/k_s"]
    ic, is_ = fx[f"{name}/i_c"], fx[f"{name}/i_s"]
    return [(tuple(int(x) for x in ic[c, : k_c[c]]), tuple(int(x) for x in is_[c, : k_s[c]]))
            for c in range(len(k_c))]


def to_dev(arrs, dtype):
    return [torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)[None] for a in arrs]


def gpu_run(sa, q, k, v, case, guard="auto", mode=None):
    dtype = torch.bfloat16 if case["dtype"] == "bf16" else torch.float32
    qt, kt, vt = to_dev((q, k, v), dtype)
    cfg = sa.SparseConfig(case["alpha_c"], case["alpha_s"], case["chunk_n"], case["blk"])
    plan = sa.plan_chunks(q.shape[0], cfg)
    batch = sa.HeadBatch.from_tensors(qt, kt, vt)
    red = sa.block_reduce(sa.sample_scores(batch, plan), cfg.blk, mode=mode)
    mask = sa.select_and_merge(red, plan, cfg, guard=guard)
    out, rep = sa.sparse_attention(batch, mask)
    torch.cuda.synchronize()
    sel = [(c.i_c, c.i_s) for c in mask.selections()[0].chunks]
    return red, mask, sel, out[0].float().cpu().numpy(), rep


@pytest.mark.parametrize("case", RANDOM_CASES, ids=[c["name"] for c in RANDOM_CASES])
def test_case_matches_reference(sa, fx, case):
    name = case["name"]
    q, k, v = random_qkv(case)
    red, mask, sel, out, rep = gpu_run(sa, q, k, v, case)
    assert sel == golden_picks(fx, name)
    assert mask.serialize() == str(fx[f"{name}/mask_text"])
    tot = fx[f"{name}/total"][:, None]
    tol = 1e-5 if case["dtype"] == "bf16" else 1e-12
    np.testing.assert_allclose(red.col[0].cpu().numpy() / tot, fx[f"{name}/col"] / tot, rtol=0, atol=tol)
    np.testing.assert_allclose(red.slash[0].cpu().numpy() / tot, fx[f"{name}/slash"] / tot, rtol=0, atol=tol)
    if f"{name}/out" in fx:
        err = np.abs(out - fx[f"{name}/out"]).max()
        assert err <= (BF16_TOL if case["dtype"] == "bf16" else FP32_TOL), err
        assert rep.active_blocks == int(fx[f"{name}/touched"])
        assert rep.estimated_flops_sparse == int(fx[f"{name}/flops_sparse"])
        assert rep.estimated_flops_dense == int(fx[f"{name}/flops_dense"])


def test_c1_head_fp32(sa, golden_dir):
    """Config 1: single head, S=4096, d=128, fp32, alpha 0.95, 5% sampling (chunk_n 2)."""
    f = np.load(os.path.join(golden_dir, "c1_head.npz"))
    case = dict(dtype="fp32", alpha_c=0.95, alpha_s=0.95, chunk_n=2, blk=128)
    red, mask, sel, out, rep = gpu_run(sa, f["q"], f["k"], f["v"], case)
    want = golden_picks({f"c/{n}": f[n] for n in ("k_c", "k_s", "i_c", "i_s")}, "c")
    assert sel == want
    assert mask.serialize() == str(f["mask_text"])
    assert np.abs(out - f["out"]).max() <= FP32_TOL


@pytest.mark.parametrize("case", [c for c in RANDOM_CASES if c["dtype"] == "bf16"], ids=lambda c: c["name"])
def test_tensor_scores_close_to_exact(sa, case):
    """tcgen05 stage-1 scores vs the fp64 path on the same bf16 inputs."""
    q, k, v = random_qkv(case)
    qt, kt, vt = to_dev((q, k, v), torch.bfloat16)
    cfg = sa.SparseConfig(case["alpha_c"], case["alpha_s"], case["chunk_n"], case["blk"])
    plan = sa.plan_chunks(q.shape[0], cfg)
    b = sa.HeadBatch.from_tensors(qt, kt, vt)
    rt = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="tensor")
    rx = sa.block_reduce(sa.sample_scores(b, plan), 128, mode="exact")
    tot = rx.col.sum(dim=2, keepdim=True)
    for a, bb in ((rt.col, rx.col), (rt.slash, rx.slash)):
        err = ((a - bb).abs() / tot).max().item()
        assert err < 2e-6, err
    # exact zeros stay exact zeros
    assert torch.equal(rt.col == 0, rx.col == 0)


def test_guard_policies_agree(sa):
    case = dict(RANDOM_CASES[-2])
    q, k, v = random_qkv(case)
    _, m_auto, s_auto, o_auto, _ = gpu_run(sa, q, k, v, case, guard="auto")
    _, m_all, s_all, o_all, _ = gpu_run(sa, q, k, v, case, guard="always")
    assert s_auto == s_all
    assert m_auto.serialize() == m_all.serialize()


@pytest.mark.parametrize("seed,S,density", [(1, 512, 0.4), (2, 1024, 0.3), (3, 2048, 0.15), (4, 1000, 0.5)])
def test_sparse_kernel_random_masks(sa, seed, S, density):
    """Stage 3 alone on random causal masks (ref tests/conftest.py:28-34 recipe)."""
    rng = np.random.default_rng(seed)
    q, k, v = (O_bf16(rng.standard_normal((S, 128))) for _ in range(3))
    nb = -(-S // 128)
    grid = np.tril(rng.random((nb, nb)) < density)
    np.fill_diagonal(grid, True)
    mask = sa.BlockMask.from_dense(128, grid, S=S)
    qt, kt, vt = to_dev((q, k, v), torch.bfloat16)
    out, rep = sa.sparse_attention(sa.HeadBatch.from_tensors(qt, kt, vt), mask)
    ref, touched = O.sparse_attention(q, k, v, grid, 128)
    assert rep.active_blocks == touched == int(grid.sum())
    assert np.abs(out[0].float().cpu().numpy() - ref).max() <= BF16_TOL


def O_bf16(a):
    return torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).double().numpy()


def test_dense_mode_matches_sdpa(sa):
    torch.manual_seed(0)
    H, S = 4, 2048
    q, k, v = (torch.randn(H, S, 128, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = sa.dense_attention(q, k, v)
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), is_causal=True)
    assert (o.float() - ref).abs().max().item() <= BF16_TOL


def test_gqa_grouping(sa):
    """Hq=4 q heads over Hkv=2 kv heads vs the oracle on repeated K/V."""
    rng = np.random.default_rng(5)
    S = 1024
    qs = [O_bf16(rng.standard_normal((S, 128)) * 1.5) for _ in range(4)]
    ks = [O_bf16(rng.standard_normal((S, 128)) * 1.5) for _ in range(2)]
    vs = [O_bf16(rng.standard_normal((S, 128))) for _ in range(2)]
    qt = torch.from_numpy(np.stack(qs)).to("cuda", torch.bfloat16)
    kt = torch.from_numpy(np.stack(ks)).to("cuda", torch.bfloat16)
    vt = torch.from_numpy(np.stack(vs)).to("cuda", torch.bfloat16)
    out, res = sa.sample_attention(qt, kt, vt, alpha=0.9, chunk_n=2)
    sels = res.mask.selections()
    for h in range(4):
        r = O.run_head(qs[h], ks[h // 2], vs[h // 2], 0.9, 0.9, 2, 128)
        assert [(c.i_c, c.i_s) for c in sels[h].chunks] == r["selection"]
        assert np.abs(out[h].float().cpu().numpy() - r["out"]).max() <= BF16_TOL


def test_sink_and_local_blocks(sa):
    """Forced blocks are added on top of the reference mask; defaults add nothing."""
    case = dict(RANDOM_CASES[-3])
    q, k, v = random_qkv(case)
    qt, kt, vt = to_dev((q, k, v), torch.bfloat16)
    _, r0 = sa.sample_attention(qt, kt, vt, alpha=0.5, chunk_n=2)
    _, r1 = sa.sample_attention(qt, kt, vt, alpha=0.5, chunk_n=2, sink_blocks=2, local_blocks=3)
    g0, g1 = r0.mask.to_dense()[0], r1.mask.to_dense()[0]
    assert (g1 | g0).sum() == g1.sum()  # superset
    nb = g1.shape[0]
    for qb in range(nb):
        assert g1[qb, : min(2, qb + 1)].all()
        assert g1[qb, max(0, qb - 2): qb + 1].all()


def test_find_k_arg_topk_kats(sa, golden_dir):
    import json
    kats = json.load(open(os.path.join(golden_dir, "kats.json")))
    for s, a, want in kats["find_k"]:
        assert sa.find_k(s, a) == want, (s, a)
    for s, kk, want in kats["arg_topk"]:
        assert list(sa.arg_topk(s, kk)) == want


def test_merge_kats(sa, golden_dir):
    import json
    kats = json.load(open(os.path.join(golden_dir, "kats.json")))
    for S, cn, blk, sels, text in kats["merges"]:
        plan = sa.plan_chunks(S, sa.SparseConfig(chunk_n=cn, blk=blk))
        selected = sa.SelectedIndices(tuple(sa.ChunkSelection(tuple(a), tuple(b), len(a), len(b)) for a, b in sels))
        assert sa.merge_index(selected, plan, blk, S).serialize() == text


def test_input_errors(sa):
    q = torch.zeros(1, 256, 128, device="cuda", dtype=torch.bfloat16)
    bad = q.clone()
    bad[0, 3, 4] = float("nan")
    with pytest.raises(sa.InputError):
        sa.sample_attention(bad, q, q)
    with pytest.raises(sa.InputError):
        sa.sample_attention(q[:, :, :64].contiguous(), q[:, :, :64].contiguous(), q[:, :, :64].contiguous())
    with pytest.raises(sa.InputError):
        sa.sample_attention(q, q, q, alpha=1.5)


def test_determinism(sa):
    case = dict(RANDOM_CASES[-4])
    q, k, v = random_qkv(case)
    qt, kt, vt = to_dev((q, k, v), torch.bfloat16)
    o1, r1 = sa.sample_attention(qt, kt, vt, alpha=0.95, chunk_n=3)
    o2, r2 = sa.sample_attention(qt, kt, vt, alpha=0.95, chunk_n=3)
    assert torch.equal(o1, o2)
    assert r1.mask.n_heads == 1
    assert r1.mask.serialize() == r2.mask.serialize()
    assert r1.mask.selections() == r2.mask.selections()
    assert torch.equal(r1.mask.kv_cnt, r2.mask.kv_cnt)


@pytest.mark.parametrize("growth", [0.0, 40.0, 400.0])
def test_sparse_kernel_extreme_and_growing_logits(sa, growth):
    """Logits that grow by `growth` nats along the key axis force the stage-3
    softmax to move its reference max mid-tile (the overflow rebase path);
    the outputs must stay finite and match the oracle (ref
    tests/test_executor.py:101-108 checks extreme logits stay finite)."""
    rng = np.random.default_rng(7)
    S = 1024
    q = np.ones((S, 128)) * 0.25 + 0.01 * rng.standard_normal((S, 128))
    k = 0.01 * rng.standard_normal((S, 128))
    k[:, 0] += np.linspace(0.0, growth, S) * np.sqrt(128) / (0.25 * 1)  # logit_j ~ growth * j / S
    v = rng.standard_normal((S, 128))
    q, k, v = (O_bf16(a) for a in (q, k, v))
    nb = S // 128
    grid = np.tril(np.ones((nb, nb), dtype=bool))
    mask = sa.BlockMask.from_dense(128, grid, S=S)
    qt, kt, vt = to_dev((q, k, v), torch.bfloat16)
    out, _ = sa.sparse_attention(sa.HeadBatch.from_tensors(qt, kt, vt), mask)
    got = out[0].float().cpu().numpy()
    assert np.isfinite(got).all()
    ref, _ = O.sparse_attention(q, k, v, grid, 128)
    assert np.abs(got - ref).max() <= BF16_TOL


def test_host_streaming_matches_device_path(sa):
    """sample_attention_host (pinned host buffers, overlapped copies) gives the
    same output and selections as sample_attention on device tensors."""
    from paper_2406_15486_b200 import synth
    q, k, v, _ = synth.make_inputs(2048, 8, 2, seed=3, device="cuda")
    o_dev, r_dev = sa.sample_attention(q, k, v, alpha=0.95, chunk_n=2)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    o_host, res = sa.sample_attention_host(hq, hk, hv, alpha=0.95, chunk_n=2, heads_per_group=2)
    assert torch.equal(o_host, o_dev.cpu())
    sel_dev = r_dev.mask.selections()
    sel_host = [s for r in res for s in r.mask.selections()]
    assert [[(c.i_c, c.i_s) for c in s.chunks] for s in sel_dev] == [[(c.i_c, c.i_s) for c in s.chunks] for s in sel_host]
    bad = hq.clone()
    bad[3, 5, 7] = float("inf")
    with pytest.raises(sa.InputError):
        sa.sample_attention_host(bad, hk, hv, alpha=0.95, chunk_n=2)


@pytest.mark.gpu
def test_graph_executor_matches_eager(sa):
    """SampleAttentionGraph (stages captured as CUDA graphs) reproduces the
    eager call bit for bit, including after the inputs change in place."""
    import torch

    from paper_2406_15486_b200 import synth

    dev = torch.device("cuda:0")
    q, k, v, _ = synth.make_inputs(4096, 4, 2, 128, seed=3, heads=list(range(4)), device=dev)
    g = sa.SampleAttentionGraph(q, k, v, alpha=0.95, chunk_n=2, group=2)
    for seed in (3, 4):
        if seed == 4:  # new inputs written into the captured buffers
            q2, k2, v2, _ = synth.make_inputs(4096, 4, 2, 128, seed=4, heads=list(range(4)), device=dev)
            g.q.copy_(q2)
            g.k.copy_(k2)
            g.v.copy_(v2)
        out = g.replay().clone()
        g.check()
        ref, res = sa.sample_attention(g.q.clone(), g.k.clone(), g.v.clone(), alpha=0.95, chunk_n=2, group=2)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        assert torch.equal(g.mask.kv_cnt, res.mask.kv_cnt)
    assert g.kernels_per_replay > 0
    g.q[0, 5, 3] = float("nan")
    g.replay()
    with pytest.raises(sa.InputError):
        g.check()


@pytest.mark.gpu
@pytest.mark.parametrize("Hq,Hkv,world", [(32, 2, 8), (32, 2, 4), (8, 8, 2), (6, 2, 2)])
def test_head_shards_match_full_batch(sa, Hq, Hkv, world):
    """Every rank's shard (q_head0 / group through the C ABI, work units built
    per shard, odd heads pairing adjacent query blocks) reproduces its slice of
    the unsharded batch bit for bit -- the N-GPU bench path on one GPU."""
    import torch

    from paper_2406_15486_b200 import synth
    from paper_2406_15486_b200.parallel import shard_heads

    S, group = 4096, Hq // Hkv
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=5, device="cuda")
    full, res = sa.sample_attention(q, k, v, alpha=0.95, chunk_n=2, group=group)
    for r in range(world):
        s = shard_heads(Hq, Hkv, world, r)
        qs = q[s.q_heads[0]: s.q_heads[-1] + 1].contiguous()
        ks = k[s.kv_heads[0]: s.kv_heads[-1] + 1].contiguous()
        vs = v[s.kv_heads[0]: s.kv_heads[-1] + 1].contiguous()
        o, rs = sa.sample_attention(qs, ks, vs, alpha=0.95, chunk_n=2, group=group, q_head0=s.q_head0)
        g = sa.SampleAttentionGraph(qs, ks, vs, alpha=0.95, chunk_n=2, group=group, q_head0=s.q_head0)
        og = g.replay()
        torch.cuda.synchronize()
        assert torch.equal(o, full[s.q_heads[0]: s.q_heads[-1] + 1])
        assert torch.equal(og, o)
        assert torch.equal(rs.mask.kv_cnt, res.mask.kv_cnt[s.q_heads[0]: s.q_heads[-1] + 1])


@pytest.mark.parametrize("S,Hq,Hkv,cn", [(100, 2, 1, 1), (129, 3, 1, 2), (777, 5, 1, 3)])
def test_short_and_mqa_sequences(sa, S, Hq, Hkv, cn):
    """bf16 tensor-core path on S < 128 (one window [0, S), ref sampler.py:99-101),
    S = 129 (a one-key trailing block), ragged S, MQA (one KV head for all q
    heads) and odd head counts (the unit schedule pairs adjacent query blocks)."""
    rng = np.random.default_rng(S)
    qs = [O_bf16(rng.standard_normal((S, 128)) * 1.5) for _ in range(Hq)]
    ks = [O_bf16(rng.standard_normal((S, 128)) * 1.5) for _ in range(Hkv)]
    vs = [O_bf16(rng.standard_normal((S, 128))) for _ in range(Hkv)]
    qt = torch.from_numpy(np.stack(qs)).to("cuda", torch.bfloat16)
    kt = torch.from_numpy(np.stack(ks)).to("cuda", torch.bfloat16)
    vt = torch.from_numpy(np.stack(vs)).to("cuda", torch.bfloat16)
    out, res = sa.sample_attention(qt, kt, vt, alpha=0.9, chunk_n=cn)
    sels = res.mask.selections()
    g = Hq // Hkv
    for h in range(Hq):
        r = O.run_head(qs[h], ks[h // g], vs[h // g], 0.9, 0.9, cn, 128)
        assert [(c.i_c, c.i_s) for c in sels[h].chunks] == r["selection"], h
        assert np.array_equal(res.mask.to_dense()[h], r["grid"]), h
        assert np.abs(out[h].float().cpu().numpy() - r["out"]).max() <= BF16_TOL, h


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_lse_matches_masked_logsumexp(sa, dtype):
    """return_lse: per row log(sum over the mask's active causal keys of
    exp(q.k/sqrt(d))), against an fp64 torch computation on the same mask."""
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    S, Hq, Hkv = 1000, 2, 1
    g = torch.Generator(device="cuda").manual_seed(3)
    q = (torch.randn((Hq, S, 128), generator=g, device="cuda") * 1.2).to(tdt)
    k = (torch.randn((Hkv, S, 128), generator=g, device="cuda") * 1.2).to(tdt)
    v = torch.randn((Hkv, S, 128), generator=g, device="cuda").to(tdt)
    out, res = sa.sample_attention(q, k, v, alpha=0.9, chunk_n=2, return_lse=True)
    grids = torch.from_numpy(res.mask.to_dense()).cuda()  # [H, nb, nb]
    nb = grids.shape[1]
    rows = torch.arange(S, device="cuda")
    for h in range(Hq):
        s = (q[h].double() @ k[0].double().T) / np.sqrt(128)
        keep = grids[h][rows // 128][:, rows // 128] & (rows[None, :] <= rows[:, None])
        s = torch.where(keep, s, torch.tensor(float("-inf"), device="cuda", dtype=torch.float64))
        ref = torch.logsumexp(s, dim=1)
        err = (res.lse[h].double() - ref).abs().max().item()
        assert err <= (2e-3 if dtype == "bf16" else 1e-5), (h, err)  # fp32 math: ~1e-7 relative on |lse| ~ 10
    assert nb == 8


def test_cra_full_beyond_the_oracle_cap(sa):
    """cra_full (entry-level retained mass of every row) on the GPU: equals
    run_pipeline's oracle metric below ORACLE_CAP, runs beyond it, and is
    exactly 1 for a full mask."""
    from paper_2406_15486_b200 import synth

    q, k, v, _ = synth.make_inputs(4096, 2, 1, 128, seed=2, device="cuda")
    b = sa.HeadBatch.from_tensors(q, k, v)
    cfg = sa.SparseConfig(0.9, 0.9, chunk_n=2)
    rep = sa.run_pipeline(b, cfg, want_oracle=True)
    _, res = sa.sample_attention(q, k, v, alpha=0.9, chunk_n=2)  # the same stages 1-2 as run_pipeline
    mins, means = sa.cra_full(b, res.mask)
    for h in range(2):
        assert abs(mins[h] - rep.heads[h].cra_full_min) < 1e-12
        assert abs(means[h] - rep.heads[h].cra_full_mean) < 1e-12
    full_min, _ = sa.cra_full(b, sa.BlockMask.full(2, 4096, 128))
    assert np.allclose(full_min, 1.0, atol=1e-12)
    q2, k2, v2, _ = synth.make_inputs(16384, 1, 1, 128, seed=3, device="cuda")
    _, res = sa.sample_attention(q2, k2, v2, alpha=0.95, chunk_n=1)
    m16, a16 = sa.cra_full(sa.HeadBatch.from_tensors(q2, k2, v2), res.mask)
    assert 0.0 < m16[0] <= a16[0] <= 1.0 + 1e-12


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_device_invariant_errors(sa, dtype):
    """The stage-3 kernels check the mask invariants the reference's BlockMask
    enforces (filtering.py:97-106) and the executor's errors (executor.py:
    131-132 InputError for a query block without active key blocks, 150-153
    InternalInvariantError for an empty normaliser) on the device; the host
    raises them from the status word, which is then clear for the next call."""
    S, nb = 1024, 8
    rng = np.random.default_rng(0)
    q, k, v = (O_bf16(rng.standard_normal((S, 128))) for _ in range(3))
    qt, kt, vt = to_dev((q, k, v), dtype)
    batch = sa.HeadBatch.from_tensors(qt, kt, vt)
    grid = np.tril(np.ones((nb, nb), dtype=bool))

    def fresh():
        return sa.BlockMask.from_dense(128, grid, S=S, device="cuda")

    out, _ = sa.sparse_attention(batch, fresh())  # valid: no error
    m = fresh()
    m.kv_cnt[0, 3] = 0  # query block 3 without any key block
    with pytest.raises(sa.InputError, match="no active key blocks"):
        sa.sparse_attention(batch, m)
    m = fresh()
    m.kv_cnt[0, 5] = 5  # list 0..4: the diagonal is missing
    with pytest.raises(sa.InternalInvariantError, match="invariants"):
        sa.sparse_attention(batch, m)
    m = fresh()
    m.kv_idx[0, 3 + 1] = 3  # query block 2 lists [0, 3, 2]: kb > qb and unsorted
    with pytest.raises(sa.InternalInvariantError, match="invariants"):
        sa.sparse_attention(batch, m)
    bad = qt.clone()
    bad[0, 200, 5] = float("nan")
    with pytest.raises(sa.InternalInvariantError, match="normalizer"):
        sa.sparse_attention(sa.HeadBatch.from_tensors(bad, kt, vt), fresh())
    with pytest.raises(sa.InputError, match="NaN"):  # the input check wins over the normaliser
        sa.sample_attention(bad, kt, vt, alpha=0.95, chunk_n=2)
    out2, _ = sa.sparse_attention(batch, fresh())  # status was reset
    assert torch.equal(out, out2)


def test_out_buffer_validation(sa):
    qt, kt, vt = to_dev([O_bf16(np.random.default_rng(1).standard_normal((512, 128)))] * 3, torch.bfloat16)
    with pytest.raises(sa.InputError, match="out must be"):
        sa.sample_attention(qt, kt, vt, out=torch.empty(qt.shape, dtype=torch.float32, device="cuda"))
    with pytest.raises(sa.InputError, match="out must be"):
        sa.sample_attention(qt, kt, vt, out=torch.empty((1, 256, 128), dtype=torch.bfloat16, device="cuda"))


@pytest.mark.parametrize("seed,scale,sink", [(0, 2.0, 30.0), (1, 3.0, 60.0), (2, 2.5, 120.0), (3, 4.0, 0.0)])
def test_guard_auto_matches_always_at_large_logits(sa, seed, scale, sink):
    """High-magnitude logits (q, k scaled so q.k/sqrt(d) has std scale^2, plus
    attention-sink keys with logits up to `sink`): the tensor-core stage-1
    error grows with the logit magnitude, so the guard margin scales with a
    per-(head, chunk) logit bound; guard='auto' must select exactly what the
    all-fp64 guard='always' selects, which must equal the oracle's."""
    S, cn = 4096, 4
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((S, 128)) * scale
    k = rng.standard_normal((S, 128)) * scale
    v = rng.standard_normal((S, 128))
    if sink:
        u = rng.standard_normal(128)
        u /= np.linalg.norm(u)
        q += np.outer(np.full(S, 1.0), u) * np.sqrt(sink)
        pos = rng.choice(S, size=24, replace=False)
        k[pos] += np.outer(rng.uniform(0.3, 1.0, size=24), u) * np.sqrt(sink) * np.sqrt(128)
    q, k, v = (O_bf16(a) for a in (q, k, v))
    qt, kt, vt = to_dev((q, k, v), torch.bfloat16)
    for alpha in (0.9, 0.95, 0.98):
        _, ra = sa.sample_attention(qt, kt, vt, alpha=alpha, chunk_n=cn, guard="auto")
        _, rw = sa.sample_attention(qt, kt, vt, alpha=alpha, chunk_n=cn, guard="always")
        assert ra.mask.selections() == rw.mask.selections(), (alpha, ra.n_rescored())
        ref = O.run_head(q, k, None, alpha, alpha, cn, 128, with_output=False)
        assert [(c.i_c, c.i_s) for c in rw.mask.selections()[0].chunks] == ref["selection"], alpha


@pytest.mark.parametrize("Hq,Hkv,S", [(32, 2, 16384), (12, 2, 4096), (10, 2, 4096), (16, 4, 8192)])
def test_schedule_overlap_pairing(sa, Hq, Hkv, S):
    """sa_schedule's overlap pairing: every (head, query block) item appears in
    exactly one unit, both items of a unit read the same KV head (same query
    block for head pairs; adjacent query blocks for an odd group's last head),
    costs descend inside each KV group, no pairing leaves more one-item union
    steps than the fixed (2p, 2p+1) pairing, and the stage-3 output is the
    same whichever order runs it."""
    from paper_2406_15486_b200 import _lib
    from paper_2406_15486_b200 import synth
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=7, device="cuda")
    out, res = sa.sample_attention(q, k, v, alpha=0.95, chunk_n=2)
    m = res.mask
    nb, G = m.n_qblocks, Hq // Hkv
    order = m.order(G, 0).cpu().numpy().reshape(-1, 2)
    cnt = m.kv_cnt.cpu().numpy()
    grid = m.to_dense()
    items = order[order >= 0]
    assert np.array_equal(np.sort(items), np.arange(Hq * nb))
    last = None
    singles = 0
    for a, b in order:
        ha, qa = divmod(int(a), nb)
        g = ha // G
        if b >= 0:
            hb, qbb = divmod(int(b), nb)
            assert hb // G == g
            assert qa == qbb or (ha == hb and ha % G == G - 1 and G % 2 == 1 and qbb == qa + 1)
            singles += int((grid[ha, qa] ^ grid[hb, qbb]).sum())
        c = cnt.flat[a] + (cnt.flat[b] if b >= 0 else 0)
        if last is not None and last[0] == g:
            assert c <= last[1]
        last = (g, c)
    fixed = sum(int((grid[g * G + 2 * p, qb] ^ grid[g * G + 2 * p + 1, qb]).sum())
                for g in range(Hkv) for p in range(G // 2) for qb in range(nb))
    fixed += sum(int((grid[g * G + G - 1, 2 * j] ^ grid[g * G + G - 1, 2 * j + 1]).sum())
                 for g in range(Hkv) if G % 2 for j in range(nb // 2))
    assert singles <= fixed
    # the same mask through the natural (fixed) unit order gives the same output
    b = sa.HeadBatch.from_tensors(q, k, v)
    o2 = torch.empty_like(q)
    st = torch.cuda.current_stream().cuda_stream
    rc = _lib.load().sa_sparse_forward(q.data_ptr(), k.data_ptr(), v.data_ptr(), _lib.SA_BF16, S, Hq, Hkv, 128, 128,
                                       b.group, 0, m.kv_cnt.data_ptr(), m.kv_idx.data_ptr(), None, o2.data_ptr(),
                                       None, None, st)
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(out, o2)


@pytest.mark.parametrize("where,val", [((0, 0, 0), float("nan")), ((1, 700, 5), float("inf")),
                                       ((2, 1023, 127), float("-inf")), ((3, 129, 64), float("nan"))])
def test_nonfinite_q_raises_input_error_on_every_path(sa, where, val):
    """On the bf16 path q's NaN/Inf scan is left to stage 3 (a non-finite
    element poisons its row's normaliser; heads.scan_inputs_async), so a single
    bad element of q -- first row, last row, any dim -- must still raise
    InputError, through sample_attention, the graph executor and the host path;
    a bad k or v element is caught by their own scans; and a clean call after a
    failed one is unaffected."""
    from paper_2406_15486_b200 import synth
    q, k, v, _ = synth.make_inputs(1024, 4, 2, 128, seed=11, device="cuda")
    bad = q.clone()
    bad[where] = val
    with pytest.raises(sa.InputError):
        sa.sample_attention(bad, k, v, alpha=0.95, chunk_n=2)
    o, _ = sa.sample_attention(q, k, v, alpha=0.95, chunk_n=2)
    assert torch.isfinite(o.float()).all()
    g = sa.SampleAttentionGraph(bad, k, v, alpha=0.95, chunk_n=2)
    g.replay()
    with pytest.raises(sa.InputError):
        g.check()
    with pytest.raises(sa.InputError):
        sa.sample_attention_host(bad.cpu(), k.cpu(), v.cpu(), alpha=0.95, chunk_n=2)
    kb = k.clone()
    kb[1, 1000, 3] = val
    with pytest.raises(sa.InputError):
        sa.sample_attention(q, kb, v, alpha=0.95, chunk_n=2)
    vb = v.clone()
    vb[0, 5, 100] = val
    with pytest.raises(sa.InputError):
        sa.sample_attention(q, k, vb, alpha=0.95, chunk_n=2)


@pytest.mark.parametrize("S,Hq,Hkv,cn,hpg", [(1000, 3, 1, 2, 2), (777, 6, 2, 3, 1), (4096, 4, 4, 2, 8),
                                            (2048, 16, 2, 1, 3)])
def test_host_path_shapes(sa, S, Hq, Hkv, cn, hpg):
    """sample_attention_host over ragged S, MQA, MHA and odd group splits (one
    or two filtering phases, ramped head groups, pageable inputs) gives the
    device path's output and masks bit for bit."""
    from paper_2406_15486_b200 import synth
    q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=S + Hq, device="cuda")
    o_dev, r_dev = sa.sample_attention(q, k, v, alpha=0.95, chunk_n=cn)
    o_host, res = sa.sample_attention_host(q.cpu(), k.cpu(), v.cpu(), alpha=0.95, chunk_n=cn, heads_per_group=hpg)
    assert torch.equal(o_host, o_dev.cpu())
    grid = np.concatenate([r.mask.to_dense() for r in res])
    assert np.array_equal(grid, r_dev.mask.to_dense())
    sa.release_staging()


def test_band_refinement_survives_a_later_stage1(sa):
    """The guard's band refinement normalises with stage 1's row statistics,
    which later stage-1 calls of the same geometry overwrite in the shared
    workspace (the tuner scores many tasks before selecting): they travel with
    the ReducedScores, so selecting task A after scoring task B equals
    selecting A right after scoring it -- and both equal the all-fp64 guard."""
    from paper_2406_15486_b200 import synth
    from paper_2406_15486_b200.config import SparseConfig, plan_chunks
    S, Hq, Hkv, cn = 32768, 8, 2, 31
    qa, ka, va, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=21, device="cuda")
    qb, kb, vb, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=22, device="cuda")
    cfg = SparseConfig(0.98, 0.98, chunk_n=cn)
    plan = plan_chunks(S, cfg)
    A, B = sa.HeadBatch.from_tensors(qa, ka, va), sa.HeadBatch.from_tensors(qb, kb, vb)
    ra_fresh = sa.block_reduce(sa.sample_scores(A, plan), 128)
    sel_fresh = sa.select(ra_fresh, cfg)
    ra = sa.block_reduce(sa.sample_scores(A, plan), 128)
    sa.block_reduce(sa.sample_scores(B, plan), 128)  # overwrites the workspace's row statistics
    sel_late = sa.select(ra, cfg)
    rx = sa.block_reduce(sa.sample_scores(A, plan), 128)
    sel_exact = sa.select(rx, cfg, guard="always")
    for s_ in (sel_fresh, sel_late):
        assert torch.equal(s_.k_sel, sel_exact.k_sel)
        for h in range(Hq):
            for c in range(cn):
                for d in range(2):
                    k_ = int(s_.k_sel[h, c, d])
                    assert torch.equal(s_.idx_sel[h, c, d, :k_], sel_exact.idx_sel[h, c, d, :k_])
    assert sel_late.n_band_refined() + sel_late.n_rescored() > 0  # the guard had work to do
