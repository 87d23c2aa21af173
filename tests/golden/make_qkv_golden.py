"""QKV container fixtures from the UNMODIFIED reference (build container only):
a small file written by the reference's save_tensors, corrupted variants, and
the reference loader's error message for each (tests/golden/qkv/).

    cd tests/golden/qkv && PYTHONDONTWRITEBYTECODE=1 python ../make_qkv_golden.py
"""
import json
import struct
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import blocksift as bs  # noqa: E402
from blocksift import tensor_io as T  # noqa: E402

rng = np.random.default_rng(11)
heads = [bs.AttentionHead(rng.standard_normal((8, 4)), rng.standard_normal((8, 4)), rng.standard_normal((8, 4)),
                          head_id=i) for i in range(2)]
T.save_tensors(bs.HeadSet(tuple(heads)), "ref_small.qkv")
raw = open("ref_small.qkv", "rb").read()
cases = {}


def check(name, data):
    open(name, "wb").write(data)
    try:
        T.load_tensors(name)
        cases[name] = None
    except bs.InputError as e:
        cases[name] = str(e)


body = raw.index(b"\n") + 1
check("bad_magic.qkv", raw[:body] + struct.pack("<I", 0x12345678) + raw[body + 4:])
check("swapped.qkv", raw[:body] + struct.pack("<I", 0x0000803F) + raw[body + 4:])
check("truncated.qkv", raw[:-4])
check("no_header.qkv", b"x" * 200)
check("bad_version.qkv", raw.replace(b"QKV 1", b"QKV 2", 1))
check("bad_counts.qkv", b"QKV 1 0 8 4\n" + raw[body:])
check("malformed.qkv", b"QKV 1 a 8 4\n" + raw[body:])
vals = bytearray(raw)
struct.pack_into("<f", vals, body + 4 + 4 * 37, float("nan"))
check("nan.qkv", bytes(vals))
check("short_magic.qkv", raw[:body + 2])
json.dump({"cases": cases}, open("qkv_cases.json", "w"), indent=1, sort_keys=True)
np.savez("ref_small.npz", q=np.stack([h.q for h in heads]), k=np.stack([h.k for h in heads]),
         v=np.stack([h.v for h in heads]))
