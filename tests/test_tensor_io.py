"""QKV container I/O against fixtures written and judged by the reference
(tests/golden/make_qkv_golden.py): same payload, same error messages."""
import json
import os

import numpy as np
import pytest

from paper_2406_15486_b200 import InputError, tensor_io

QKV = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "qkv")
CASES = json.load(open(os.path.join(QKV, "qkv_cases.json")))["cases"]


def test_load_reference_file():
    ref = np.load(os.path.join(QKV, "ref_small.npz"))
    hs = tensor_io.load_tensors(os.path.join(QKV, "ref_small.qkv"))
    assert len(hs) == 2 and hs.S == 8 and hs.d == 4
    for i, h in enumerate(hs):
        np.testing.assert_array_equal(h.q, ref["q"][i].astype(np.float32).astype(np.float64))
        np.testing.assert_array_equal(h.v, ref["v"][i].astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("name", sorted(CASES))
def test_error_messages_match_reference(name):
    path = os.path.join(QKV, name)
    with pytest.raises(InputError) as e:
        tensor_io.load_tensors(path)
    assert str(e.value) == CASES[name].replace(name, path, 1)


def test_save_roundtrip_is_byte_identical(tmp_path):
    src = os.path.join(QKV, "ref_small.qkv")
    hs = tensor_io.load_tensors(src)
    out = tmp_path / "again.qkv"
    tensor_io.save_tensors(hs, out)
    assert open(out, "rb").read() == open(src, "rb").read()
    ref = np.load(os.path.join(QKV, "ref_small.npz"))
    out2 = tmp_path / "tuple.qkv"
    tensor_io.save_tensors((ref["q"], ref["k"], ref["v"]), out2)
    assert open(out2, "rb").read() == open(src, "rb").read()


@pytest.mark.gpu
def test_device_loader_matches_host_loader():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    src = os.path.join(QKV, "ref_small.qkv")
    b = tensor_io.load_tensors_device(src, dtype=torch.float32)
    hs = tensor_io.load_tensors(src)
    for i, h in enumerate(hs):
        np.testing.assert_array_equal(b.q[i].cpu().numpy(), h.q.astype(np.float32))
        np.testing.assert_array_equal(b.k[i].cpu().numpy(), h.k.astype(np.float32))
    for name in ("nan.qkv", "bad_magic.qkv", "truncated.qkv"):
        path = os.path.join(QKV, name)
        with pytest.raises(InputError) as e:
            tensor_io.load_tensors_device(path)
        assert str(e.value) == CASES[name].replace(name, path, 1)
