"""CPU-side checks: the C-ABI library loads and exports every declared
symbol, and the host integer logic (config, plan) matches the pinned oracle."""

import ctypes
import os
import re

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2406_15486_b200 as sa
from oracle import blocksift_port as O
from paper_2406_15486_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sampleattn.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|long long|const char\*)\s+(sa_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 10
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == syms
    assert lib.sa_version() >= 100


def test_workspace_bytes_positive():
    lib = _lib.load()
    assert lib.sa_workspace_bytes(131072, 32, 2, 128, 128, 1, _lib.SA_BF16) > 0
    assert lib.sa_workspace_bytes(0, 32, 2, 128, 128, 1, _lib.SA_BF16) == 0


def test_config_defaults_and_validation():
    cfg = sa.SparseConfig()
    assert (cfg.alpha_c, cfg.alpha_s, cfg.chunk_n, cfg.blk) == (0.95, 0.95, 1, 128)
    for kw in ({"alpha_c": -0.1}, {"alpha_s": 1.5}, {"chunk_n": 0}, {"blk": 0}):
        with pytest.raises(sa.InputError):
            sa.SparseConfig(**kw)


def test_resolve_config_shorthands():
    c = sa.resolve_config(98304, alpha=0.9, sample_ratio=0.02)
    assert (c.alpha_c, c.alpha_s, c.chunk_n) == (0.9, 0.9, 15)
    c = sa.resolve_config(4096, alpha=0.95, sample_ratio=0.05)
    assert c.chunk_n == 2
    c = sa.resolve_config(4096, alpha=0.9, alpha_s=0.98)
    assert (c.alpha_c, c.alpha_s) == (0.9, 0.98)
    with pytest.raises(sa.InputError):
        sa.resolve_config(4096, chunk_n=2, sample_ratio=0.1)


@given(S=st.integers(1, 5000), chunk_n=st.integers(1, 16), blk=st.integers(1, 512))
@settings(max_examples=300, deadline=None)
def test_plan_matches_oracle(S, chunk_n, blk):
    p = sa.plan_chunks(S, sa.SparseConfig(chunk_n=chunk_n, blk=blk))
    o = O.plan_chunks(S, chunk_n, blk)
    assert (p.chunk_n, p.itv) == (o.chunk_n, o.itv)
    assert [(c.sample_start, c.sample_end, c.region_start, c.region_end) for c in p.chunks] == list(o.windows)


def test_plan_kats():
    p = sa.plan_chunks(300, sa.SparseConfig(chunk_n=4, blk=128))
    assert p.chunk_n == 2 and p.itv == 150
    assert [(c.sample_start, c.sample_end) for c in p.chunks] == [(22, 150), (172, 300)]
    assert sa.plan_chunks(65536, sa.SparseConfig(chunk_n=2)).sampled_rows() == 256


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2406_15486_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, re.M), fn


def _err(lib):
    return lib.sa_last_error().decode()


def test_c_abi_rejects_bad_arguments_without_touching_the_gpu():
    """Argument validation of the C ABI runs before any CUDA call (so it is
    testable on a CPU host) and maps to the reference's exception classes."""
    lib = _lib.load()
    fake = 0x1000  # never dereferenced: every call below fails validation first
    # stage 1: unsupported tensor-core shape (d != 128), bad plan layout, too small workspace
    rc = lib.sa_stage1(fake, fake, _lib.SA_BF16, 4096, 2, 1, 64, 128, 2, 0, 1, 4096, fake, fake, None,
                       _lib.SA_STAGE1_TENSOR, None, fake, 1 << 30, None)
    assert rc == _lib.SA_ERR_UNSUPPORTED and "d == 128" in _err(lib)
    rc = lib.sa_stage1(fake, fake, _lib.SA_BF16, 4096, 2, 1, 128, 128, 2, 0, 3, 4000, fake, fake, None,
                       _lib.SA_STAGE1_TENSOR, None, fake, 1 << 30, None)
    assert rc == _lib.SA_ERR_INVALID and "plan_chunks" in _err(lib)
    rc = lib.sa_stage1(fake, fake, _lib.SA_BF16, 4096, 2, 1, 128, 128, 2, 0, 1, 4096, fake, fake, None,
                       _lib.SA_STAGE1_TENSOR, None, fake, 16, None)
    assert rc == _lib.SA_ERR_INVALID and "workspace" in _err(lib)
    # GQA mapping past the supplied kv heads
    rc = lib.sa_stage1(fake, fake, _lib.SA_BF16, 4096, 4, 1, 128, 128, 2, 0, 1, 4096, fake, fake, None,
                       _lib.SA_STAGE1_TENSOR, None, fake, 1 << 30, None)
    assert rc == _lib.SA_ERR_INVALID and "kv heads" in _err(lib)
    # stage 2: alpha outside [0, 1] (ref sampler.py:52-56), guard without flags
    assert lib.sa_select(fake, fake, 1, 1, 8, 1.5, 0.9, 0.0, None, 1.0, None, None, None, fake, fake, None, 0.0, None) == _lib.SA_ERR_INVALID
    assert "alpha_c" in _err(lib)
    assert lib.sa_select(fake, fake, 1, 1, 8, 0.9, 0.9, 1e-7, None, 1.0, None, None, None, fake, fake, None, 0.0, None) == _lib.SA_ERR_INVALID
    assert lib.sa_select(fake, fake, 1, 1, 8, 0.9, 0.9, 1e-7, fake, 0.0, fake, None, None, fake, fake, None, 0.0, None) \
        == _lib.SA_ERR_INVALID and "bound_ref" in _err(lib)
    assert lib.sa_merge(fake, fake, 1, 1, 7, 1024, 128, 1024, 0, 1, fake, fake, None, None, None) == _lib.SA_ERR_INVALID
    # band guard: the per-row tie certificate checks its pointers, eps and workspace before any launch
    ws_bytes = lib.sa_workspace_bytes(4096, 2, 1, 128, 128, 1, _lib.SA_BF16)
    assert lib.sa_certify_band_ties(_lib.SA_BF16, 4096, 2, 1, 128, 128, 1, 4096, None, fake, fake, fake, fake, None,
                                    320.0, 3e-5, fake, ws_bytes, None) == _lib.SA_ERR_INVALID and "null" in _err(lib)
    assert lib.sa_certify_band_ties(_lib.SA_BF16, 4096, 2, 1, 128, 128, 1, 4096, fake, fake, fake, fake, fake, None,
                                    320.0, 0.0, fake, ws_bytes, None) == _lib.SA_ERR_INVALID and "band_eps" in _err(lib)
    assert lib.sa_certify_band_ties(_lib.SA_BF16, 4096, 2, 1, 128, 128, 1, 4096, fake, fake, fake, fake, fake, None,
                                    320.0, 3e-5, fake, 16, None) == _lib.SA_ERR_INVALID and "workspace" in _err(lib)
    assert lib.sa_certify_band_ties(_lib.SA_FP32, 4096, 2, 1, 128, 128, 1, 4096, fake, fake, fake, fake, fake, None,
                                    320.0, 3e-5, fake, 1 << 30, None) == _lib.SA_ERR_UNSUPPORTED
    assert lib.sa_schedule_len(0, 8, 1, 0) < 0
    assert lib.sa_schedule_len(32, 1024, 16, 0) == 2 * 32 * 1024 // 2
    assert lib.sa_schedule_len(3, 5, 3, 0) == 2 * (5 + 3)  # one head pair + the odd head's adjacent-block pairs
    # stage 3: fp32 path limits
    rc = lib.sa_sparse_forward(fake, fake, fake, _lib.SA_FP32, 512, 1, 1, 256, 128, 1, 0, fake, fake, None, fake,
                               None, None, None)
    assert rc == _lib.SA_ERR_UNSUPPORTED
    # stage 3 with the fused gather: peer count, peer pointers and dtype are checked before any launch
    P = ctypes.c_void_p
    peers8 = (P * 8)(*([fake] * 8))
    assert lib.sa_sparse_forward_peers(fake, fake, fake, _lib.SA_BF16, 4096, 2, 1, 128, 128, 2, 0, fake, fake, None,
                                       fake, None, None, peers8, 8, None) == _lib.SA_ERR_INVALID
    assert "n_peer" in _err(lib)
    assert lib.sa_sparse_forward_peers(fake, fake, fake, _lib.SA_BF16, 4096, 2, 1, 128, 128, 2, 0, fake, fake, None,
                                       fake, None, None, (P * 1)(None), 1, None) == _lib.SA_ERR_INVALID
    assert "null peer" in _err(lib)
    assert lib.sa_sparse_forward_peers(fake, fake, fake, _lib.SA_FP32, 4096, 2, 1, 128, 128, 2, 0, fake, fake, None,
                                       fake, None, None, peers8, 1, None) == _lib.SA_ERR_UNSUPPORTED
    assert lib.sa_ipc_export(None, None, None) == _lib.SA_ERR_INVALID
    assert lib.sa_ipc_open(None, None) == _lib.SA_ERR_INVALID
    assert lib.sa_ipc_close(None) == _lib.SA_ERR_INVALID
    # the Python wrapper turns these codes into the reference's exception types
    with pytest.raises(sa.InputError):
        _lib.call("sa_schedule", None, None, 1, 1, 1, 0, None, None, None)


@pytest.mark.parametrize("Hq,group,hpg", [(32, 16, 4), (32, 4, 4), (32, 32, 4), (8, 8, 2), (4, 1, 4), (32, 16, 16)])
def test_host_path_group_plan(Hq, group, hpg):
    """Stage-3 head groups of the host-buffer path: contiguous, cover every
    head once, never straddle a KV group, at most max(hpg, 5) heads, and the
    first group of the job is a single head when the KV group has several."""
    from paper_2406_15486_b200.streaming import _group_plan

    groups = _group_plan(Hq, group, hpg)
    assert groups[0][0] == 0 and groups[-1][1] == Hq
    for (a0, a1), (b0, _) in zip(groups, groups[1:]):
        assert a1 == b0
    for h0, h1 in groups:
        assert 0 < h1 - h0 <= max(hpg, 5)
        assert h0 // group == (h1 - 1) // group  # one KV group per launch
    if group > 1:
        assert groups[0] == (0, 1)
