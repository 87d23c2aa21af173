"""Seeded input recipes shared by the golden generator and the tests.

Inputs are regenerated bit-identically from the seed on any box (numpy's
default_rng is platform-stable); bf16 cases are rounded with torch's RNE cast
and then upcast to fp64, which is exactly what the reference sees
(parity = reference on the bf16-rounded inputs).
"""

from __future__ import annotations

import numpy as np

# C1: acceptance-04 family (ref tests/test_acceptance.py:156-165), fp32 mode.
C1_SPEC = dict(S=4096, d=128, n_heads=1, sink_columns=[(0, 0.18), (1500, 0.14)],
               slash_offsets=[(0, 0.60)], noise_scale=1.0, seed=0)

# name, seed, S, d, blk, chunk_n, alpha_c, alpha_s, scale, dtype
RANDOM_CASES = [
    dict(name="r1024_cn1", seed=11, S=1024, d=128, blk=128, chunk_n=1, alpha_c=0.9, alpha_s=0.9, scale=1.5, dtype="bf16"),
    dict(name="r2048_cn2", seed=12, S=2048, d=128, blk=128, chunk_n=2, alpha_c=0.95, alpha_s=0.95, scale=1.5, dtype="bf16"),
    dict(name="r1000_cn3", seed=13, S=1000, d=128, blk=128, chunk_n=3, alpha_c=0.95, alpha_s=0.9, scale=1.5, dtype="bf16"),
    dict(name="r3072_cn5", seed=14, S=3072, d=128, blk=128, chunk_n=5, alpha_c=0.9, alpha_s=0.95, scale=2.0, dtype="bf16"),
    dict(name="r4096_cn4", seed=15, S=4096, d=128, blk=128, chunk_n=4, alpha_c=0.98, alpha_s=0.98, scale=2.0, dtype="bf16"),
    dict(name="r2048_a1", seed=16, S=2048, d=128, blk=128, chunk_n=2, alpha_c=1.0, alpha_s=1.0, scale=1.0, dtype="bf16"),
    dict(name="r2048_a0", seed=17, S=2048, d=128, blk=128, chunk_n=2, alpha_c=0.0, alpha_s=0.0, scale=1.0, dtype="bf16"),
    dict(name="r512_f32", seed=18, S=512, d=64, blk=128, chunk_n=1, alpha_c=0.95, alpha_s=0.95, scale=1.0, dtype="fp32"),
    dict(name="r96_blk16", seed=19, S=96, d=8, blk=16, chunk_n=3, alpha_c=0.9, alpha_s=0.9, scale=1.0, dtype="fp32"),
    dict(name="r200_blk32", seed=20, S=200, d=16, blk=32, chunk_n=3, alpha_c=0.8, alpha_s=0.95, scale=1.0, dtype="fp32"),
    # structured heads: planted graded sinks + a smooth local band (nontrivial picks)
    dict(name="s2048_cn1", seed=31, S=2048, d=128, blk=128, chunk_n=1, alpha_c=0.95, alpha_s=0.95, scale=0.5, dtype="bf16",
         sinks=[(0, 10.5), (700, 9.5), (1500, 9.0)], band=5.0),
    dict(name="s2048_cn3", seed=32, S=2048, d=128, blk=128, chunk_n=3, alpha_c=0.98, alpha_s=0.98, scale=0.5, dtype="bf16",
         sinks=[(i * 200 + 3, 11 - 0.5 * i) for i in range(8)], band=5.0),
    dict(name="s4096_cn2", seed=33, S=4096, d=128, blk=128, chunk_n=2, alpha_c=0.9, alpha_s=0.9, scale=0.6, dtype="bf16",
         sinks=[(i * 390 + 3, 11.5 - 0.5 * i) for i in range(10)], band=5.0),
    dict(name="s4096_cn7", seed=34, S=4096, d=128, blk=128, chunk_n=7, alpha_c=0.95, alpha_s=0.9, scale=0.6, dtype="bf16",
         sinks=[(i * 390 + 3, 11.5 - 0.5 * i) for i in range(10)], band=4.0),
    dict(name="s1900_cn2", seed=35, S=1900, d=128, blk=128, chunk_n=2, alpha_c=0.9, alpha_s=0.95, scale=0.5, dtype="bf16",
         sinks=[(0, 10.0), (640, 9.0)], band=5.0),
]


# run_pipeline metric goldens (ref pipeline.py:149-217, want_oracle=True):
# name -> (cfg (alpha_c, alpha_s, chunk_n, blk), [(case recipe, head_id), ...])
PIPELINE_CASES = {
    "p2048_bf16": ((0.95, 0.95, 2, 128), [
        (dict(seed=41, S=2048, d=128, scale=0.5, dtype="bf16", sinks=[(0, 10.5), (700, 9.5)], band=5.0), 4),
        (dict(seed=42, S=2048, d=128, scale=1.5, dtype="bf16"), 1),
        (dict(seed=43, S=2048, d=128, scale=0.6, dtype="bf16", sinks=[(i * 300 + 3, 11 - 0.5 * i) for i in range(6)],
              band=4.0), 7)]),
    "p1000_fp32": ((0.9, 0.95, 3, 128), [
        (dict(seed=44, S=1000, d=64, scale=1.0, dtype="fp32"), 0),
        (dict(seed=45, S=1000, d=64, scale=0.5, dtype="fp32", sinks=[(0, 9.0), (333, 8.0)], band=4.0), 2)]),
}
WALL_KEYS = ("wall_time_sample", "wall_time_filter", "wall_time_sparse", "wall_time_dense", "wall_time_total")

# tuner golden (ref tuning.py:156-231): the reference's own tune() on its own
# generator, each generated head rounded to fp32 (recorded, so the GPU tuner
# can run on the same bits)
TUNE_TEMPLATE = dict(S=2048, d=32, n_heads=1, sink_columns=[(0, 0.25), (700, 0.15)],
                     slash_offsets=[(0, 0.3)], noise_scale=2.5, seed=21)
TUNE_GRID = dict(alphas_c=(0.6, 0.9), alphas_s=(0.6, 0.9), chunk_ns=(1, 3),
                 length_ranges=((1024, 2048), (9216, 9216)), recall_target=0.8, trials_per_cell=2)



def bf16_round(x: np.ndarray) -> np.ndarray:
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def _smooth(rng, length, dims, sigma):
    x = np.arange(-4 * sigma, 4 * sigma + 1, dtype=np.float64)
    ker = np.exp(-(x ** 2) / (2.0 * sigma ** 2))
    ker /= np.sqrt((ker ** 2).sum())
    w = rng.standard_normal((length, dims))
    return np.column_stack([np.convolve(w[:, a], ker, mode="same") for a in range(dims)])


def random_qkv(case: dict):
    """q, k scaled N(0,1), v N(0,1) (the reference fixture recipe,
    ref tests/conftest.py:7-14), rounded to the case's dtype, as fp64.

    Structured cases additionally plant sink columns (one reserved dim per
    sink: q = 1, k[pos] = shift * sqrt(d), the construction of ref
    synth.py:210-214) and a local band from a shared smooth topic process
    (ref synth.py:170-180, 232-237 at offset 0)."""
    rng = np.random.default_rng(case["seed"])
    S, d, sc = case["S"], case["d"], case["scale"]
    q = sc * rng.standard_normal((S, d))
    k = sc * rng.standard_normal((S, d))
    v = rng.standard_normal((S, d))
    slot = 0
    for pos, shift in case.get("sinks", []):
        q[:, slot] = 1.0
        k[:, slot] = 0.0
        k[pos, slot] = shift * np.sqrt(d)
        slot += 1
    if case.get("band"):
        topics = _smooth(rng, S, 16, 24)
        beta = np.sqrt(case["band"] * np.sqrt(d) / 16)
        q[:, slot:slot + 16] = beta * topics
        k[:, slot:slot + 16] = beta * topics
    if case["dtype"] == "bf16":
        q, k, v = (bf16_round(a) for a in (q, k, v))
    else:
        q, k, v = (a.astype(np.float32) for a in (q, k, v))
    return q.astype(np.float64), k.astype(np.float64), v.astype(np.float64)


# ---- calibrated generator (ref synth.py): specs for tests/golden/refsynth.json
REFSYNTH_SPECS = [
    dict(S=1024, d=64, n_heads=2, sink_columns=((0, 0.2), (300, 0.1)), slash_offsets=((0, 0.5),), seed=3),
    dict(S=2048, d=128, n_heads=2, sink_columns=((0, 0.18), (1500, 0.14)), slash_offsets=((0, 0.60),), seed=0),
    dict(S=1536, d=128, n_heads=1, sink_columns=((0, 0.15),), slash_offsets=((0, 0.4), (300, 0.1)), seed=5),
    dict(S=3000, d=96, n_heads=1, sink_columns=((10, 0.1), (2000, 0.05)), slash_offsets=((0, 0.3), (700, 0.15)),
         noise_scale=1.5, seed=11),
]
REFSYNTH_BAD_SPECS = [
    dict(S=1024, d=64, sink_columns=((1020, 0.2),)),                   # no measurement rows past the sink
    dict(S=1024, d=64, sink_columns=((0, 0.6),), slash_offsets=((0, 0.6),)),   # masses sum past 1
    dict(S=1024, d=64, slash_offsets=((0, 0.3), (10, 0.2))),           # offsets too close to separate
    dict(S=1024, d=8, sink_columns=((0, 0.2),), slash_offsets=((0, 0.3),)),    # reserved dims exceed d
    dict(S=1024, d=64, sink_columns=((5, 0.2), (5, 0.1))),             # duplicate sink
    dict(S=64, d=64, sink_columns=((0, 0.9),), noise_scale=3.0, seed=1),  # calibration target out of reach?
]
