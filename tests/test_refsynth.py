"""The device restatement of the reference's calibrated generator
(paper_2406_15486_b200/refsynth.py) against the UNMODIFIED reference's
`generate_synthetic` (fixtures: tests/golden/make_refsynth_golden.py).

Runs on whatever device torch has (CPU here, the GPU box under -m gpu): the
draws are the reference's bits, so heads built from the same calibrated
parameters agree to fp64 rounding; only the summation order of the mass
measurements differs (calibration steps are continuous in them).
"""

import json
import os

import numpy as np
import pytest
import torch

from paper_2406_15486_b200 import refsynth
from paper_2406_15486_b200.errors import GeneratorError, InputError

HERE = os.path.dirname(os.path.abspath(__file__))
FX = json.load(open(os.path.join(HERE, "golden", "refsynth.json")))
DEV = "cpu"  # the CPU suite; test_generator_on_the_gpu repeats the check on the device path


def _spec(kw):
    return refsynth.SyntheticSpec(**kw)


@pytest.mark.parametrize("case", FX["specs"], ids=lambda c: f"S{c['spec']['S']}_seed{c['spec'].get('seed', 0)}")
def test_generator_matches_reference(case):
    spec = _spec(case["spec"])
    heads = refsynth.generate_synthetic(spec, device=DEV)
    assert len(heads) == len(case["heads"])
    for h, want in zip(heads, case["heads"]):
        q, k, v = (t.cpu().numpy() for t in (h.q, h.k, h.v))
        rows = np.array(want["rows"])
        np.testing.assert_allclose(q[rows], np.array(want["q_rows"]), rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(k[rows], np.array(want["k_rows"]), rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose([q.sum(), k.sum(), v.sum()], want["sums"], rtol=1e-9, atol=1e-6)
        np.testing.assert_allclose([np.abs(q).sum(), np.abs(k).sum()], want["abs_sums"], rtol=1e-10)
        np.testing.assert_allclose([k[p, i] for i, (p, _) in enumerate(spec.sink_columns)], want["sink_k"],
                                   rtol=1e-9)
        # the final full-row planted masses, the quantity calibration drives
        np.testing.assert_allclose(h.sink_mass, want["sink_mass"], rtol=1e-9)
        np.testing.assert_allclose(h.band_mass, want["band_mass"], rtol=1e-9, atol=1e-12)
        t = spec.targets()
        got = np.concatenate([h.sink_mass, h.band_mass])
        assert np.all(np.abs(got / t - 1.0) <= refsynth.FINAL_REL_TOL)


@pytest.mark.parametrize("case", FX["bad"], ids=lambda c: str(c["error"]))
def test_generator_errors_match_reference(case):
    if case["error"] is None:
        refsynth.generate_synthetic(_spec(case["spec"]), device=DEV)
        return
    exc = {"InputError": InputError, "GeneratorError": GeneratorError}[case["error"]]
    with pytest.raises(exc) as ei:
        refsynth.generate_synthetic(_spec(case["spec"]), device=DEV)
    assert type(ei.value) is exc
    assert str(ei.value) == case["message"]


def test_control_offsets_match_reference():
    for case in FX["specs"]:
        spec = _spec(case["spec"])
        assert (refsynth._control_offsets(spec) if spec.slash_offsets else []) == case["controls"]


def test_gqa_inputs_share_planted_dims():
    spec = refsynth.SyntheticSpec(S=1024, d=64, sink_columns=((0, 0.2), (300, 0.1)), slash_offsets=((0, 0.5),),
                                  seed=3)
    q, k, v, heads = refsynth.calibrated_gqa_inputs(spec, Hq=4, Hkv=2, dtype=torch.float64, device=DEV)
    assert q.shape == (4, 1024, 64) and k.shape == (2, 1024, 64) and v.shape == (2, 1024, 64)
    r = spec.reserved_dims()
    assert torch.equal(q[0], heads[0].q) and torch.equal(q[2], heads[1].q)
    assert torch.equal(q[1, :, :r], q[0, :, :r]) and not torch.equal(q[1, :, r:], q[0, :, r:])
    # a redrawn-noise head of the group still carries the calibrated masses (+-20 %)
    sm, bm = refsynth.planted_masses(q[1], k[0], spec, torch.arange(1024, device=q.device),
                                    refsynth._control_offsets(spec))
    got = np.concatenate([sm, bm])
    assert np.all(np.abs(got / spec.targets() - 1.0) <= 0.2)


@pytest.mark.gpu
@pytest.mark.parametrize("case", FX["specs"][:2], ids=lambda c: f"S{c['spec']['S']}")
def test_generator_on_the_gpu(case):
    """The same reference comparison with the mass measurements on the GPU
    (fp64 matmuls / exp / cumsum on the device)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    spec = _spec(case["spec"])
    heads = refsynth.generate_synthetic(spec, device="cuda")
    for h, want in zip(heads, case["heads"]):
        rows = np.array(want["rows"])
        np.testing.assert_allclose(h.q.cpu().numpy()[rows], np.array(want["q_rows"]), rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(h.k.cpu().numpy()[rows], np.array(want["k_rows"]), rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(h.sink_mass, want["sink_mass"], rtol=1e-9)
        np.testing.assert_allclose(h.band_mass, want["band_mass"], rtol=1e-9, atol=1e-12)
