"""Golden fixtures for the device restatement of the reference's calibrated
generator (paper_2406_15486_b200/refsynth.py), produced by the UNMODIFIED
reference `generate_synthetic` (run in the build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_refsynth_golden.py

Per spec and head: the calibrated parameters are not exposed by the reference,
so the fixture stores what identifies them -- the planted sink entries of k,
the staircase / band entries of q and k at seeded positions -- together with
sums and sampled rows of q, k, v, and the reference's own planted-mass
measurement on every row.  Specs that the reference rejects store the
exception type and message.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from blocksift import synth as ref  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden.inputs import REFSYNTH_SPECS, REFSYNTH_BAD_SPECS  # noqa: E402


def main():
    out = {"specs": [], "bad": []}
    for kw in REFSYNTH_SPECS:
        spec = ref.SyntheticSpec(**kw)
        hs = ref.generate_synthetic(spec)
        controls = ref._control_offsets(spec) if spec.slash_offsets else []
        rows = np.arange(spec.S)
        rng = np.random.default_rng(123)
        sample = rng.choice(spec.S, size=min(16, spec.S), replace=False)
        heads = []
        for h in hs:
            sink_m, band_m = ref._planted_masses(h.q, h.k, spec, rows, controls)
            heads.append({
                "sums": [float(h.q.sum()), float(h.k.sum()), float(h.v.sum())],
                "abs_sums": [float(np.abs(h.q).sum()), float(np.abs(h.k).sum())],
                "rows": sample.tolist(),
                "q_rows": h.q[sample].tolist(),
                "k_rows": h.k[sample].tolist(),
                "sink_k": [float(h.k[p, i]) for i, (p, _) in enumerate(spec.sink_columns)],
                "sink_mass": sink_m.tolist(),
                "band_mass": band_m.tolist(),
            })
        out["specs"].append({"spec": kw, "controls": controls, "heads": heads})
        print("spec", kw["S"], kw.get("seed"), "done", flush=True)
    for kw in REFSYNTH_BAD_SPECS:
        try:
            ref.generate_synthetic(ref.SyntheticSpec(**kw))
            out["bad"].append({"spec": kw, "error": None, "message": None})
        except Exception as e:  # noqa: BLE001 -- the type and message are the fixture
            out["bad"].append({"spec": kw, "error": type(e).__name__, "message": str(e)})
    with open(os.path.join(HERE, "refsynth.json"), "w") as f:
        json.dump(out, f)
    print("wrote refsynth.json")


if __name__ == "__main__":
    main()
