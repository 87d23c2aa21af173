"""Seeded GPU generator for long-context benchmark inputs.

The reference's generator (pkg/src/blocksift/synth.py:183-238 _HeadBuilder,
calibrated by :290-438) plants column sinks in reserved head dimensions
(q = 1, k[pos] = shift * sqrt(d)), an offset-0 local band and offset bands from
a smooth random "topic" process shared by q and (shifted) k, over seeded
noise.  Its calibration loop measures dense probability rows and is
quadratic in S (minutes per head at 128K on the CPU), so this module keeps the
construction but sets the amplitudes analytically for the last sampled row:
with noise logit std s_n, the noise partition of a row at position r is about
r * exp(s_n^2 / 2); a sink with target mass m gets logit ln(m * Z_ref), a band
with target mass m gets the amplitude whose summed kernel weight equals
m * Z_ref (solved by bisection).  Heads of one KV group share K/V and differ
in q (their own noise and per-head amplitude jitter), as GQA heads do.

Everything is generated directly on the device with torch (plumbing, not the
measured path); the recipe is deterministic for a given seed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

__all__ = ["LongContextSpec", "make_inputs", "GLM_128K", "spec_for"]

_TOPIC_DIMS = 16


@dataclass(frozen=True)
class LongContextSpec:
    n_sinks: int = 1024          # column "heavy hitters" at seeded key positions
    sink_mass: float = 0.55      # total planted column mass at the reference row
    sink_zipf: float = 1.1       # masses m_i ~ i^-zipf (a long graded tail)
    band_mass: float = 0.30      # offset-0 local band
    band_sigma: int = 32         # topic-process smoothing (keys)
    slash_mass: float = 0.07     # one extra slash band at offset S // 16
    noise_std: float = 1.0       # noise logit std
    head_jitter: float = 0.10    # per-q-head amplitude spread
    extra: dict = field(default_factory=dict)


GLM_128K = LongContextSpec()


def spec_for(S: int) -> LongContextSpec:
    return GLM_128K


def _smooth(gen, S: int, dims: int, sigma: int, device) -> torch.Tensor:
    """Unit-variance process with Gaussian autocorrelation exp(-D^2/(4 sigma^2))
    (the reference's _smooth_process, synth.py:170-180), via a 1-D convolution."""
    radius = 4 * sigma
    x = torch.arange(-radius, radius + 1, device=device, dtype=torch.float32)
    ker = torch.exp(-(x ** 2) / (2.0 * sigma ** 2))
    ker = ker / ker.square().sum().sqrt()
    white = torch.randn((dims, 1, S + 2 * radius), generator=gen, device=device)
    with torch.backends.cudnn.flags(enabled=True, benchmark=False, deterministic=True):
        out = torch.nn.functional.conv1d(white, ker.view(1, 1, -1))  # [dims, 1, S]
    return out[:, 0, :].T.contiguous()  # [S, dims]


def _band_amplitude(target: float, sigma: int) -> float:
    """B such that sum_{D>=0} exp(B * rho(D)) = target, rho = exp(-D^2/(4 sigma^2))."""
    D = torch.arange(0, 16 * sigma, dtype=torch.float64)
    rho = torch.exp(-(D ** 2) / (4.0 * sigma ** 2))
    lo, hi = 0.0, 60.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if torch.exp(mid * rho).sum().item() > target:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def make_inputs(S: int, Hq: int, Hkv: int, d: int = 128, seed: int = 0, spec: LongContextSpec | None = None,
                heads=None, device="cuda", dtype=torch.bfloat16):
    """q [len(heads), S, d], k/v [kv heads needed, S, d] for the given global q
    heads (default: all), GQA group = Hq // Hkv.  Returns (q, k, v, kv_heads)."""
    spec = spec or spec_for(S)
    device = torch.device(device)
    group = Hq // Hkv
    heads = list(range(Hq)) if heads is None else list(heads)
    kv_heads = sorted({h // group for h in heads})
    # all column sinks share ONE reserved dim: q = const there, k carries a
    # per-key logit bias (the reference uses one dim per sink, synth.py:210-214;
    # a shared dim plants any number of sinks at the same cost)
    n_res = 1 + 2 * _TOPIC_DIMS
    n_noise = d - n_res
    if n_noise < 8:
        raise ValueError("head dimension too small for the planted structure")
    # noise entries so that q.k/sqrt(d) over the noise dims has std noise_std
    c = (spec.noise_std ** 2 * d / n_noise) ** 0.25
    z_ref = S * math.exp(spec.noise_std ** 2 / 2) / max(1e-6, 1.0 - spec.sink_mass - spec.band_mass - spec.slash_mass)
    rd = math.sqrt(d)
    w = [(i + 1) ** -spec.sink_zipf for i in range(spec.n_sinks)]
    sink_logit = [math.log(spec.sink_mass * wi / sum(w) * z_ref) for wi in w]
    band_B = _band_amplitude(spec.band_mass * z_ref, spec.band_sigma)
    slash_B = _band_amplitude(spec.slash_mass * z_ref, spec.band_sigma)
    slash_off = S // 16
    qs, ks, vs = [], [], []
    for g in kv_heads:
        gen = torch.Generator(device=device)
        gen.manual_seed(seed * 1000003 + 7919 * g)
        k = torch.empty((S, d), device=device)
        k[:, :n_noise] = c * torch.randn((S, n_noise), generator=gen, device=device)
        # sinks: position 0 plus seeded positions spread over the sequence
        pos = torch.randint(0, int(S * 0.97), (spec.n_sinks,), generator=gen, device=device)
        pos[0] = 0
        bias = torch.zeros((S,), device=device)
        # colliding positions keep the larger logit (order-independent, so the
        # generator is bit-deterministic; a plain index_put picks a random writer)
        bias.scatter_reduce_(0, pos, torch.tensor(sink_logit, device=device), reduce="amax", include_self=False)
        k[:, n_noise] = bias * rd
        t0 = _smooth(gen, S, _TOPIC_DIMS, spec.band_sigma, device)
        t1 = _smooth(gen, S + slash_off, _TOPIC_DIMS, spec.band_sigma, device)
        b0 = math.sqrt(band_B * rd / _TOPIC_DIMS)
        b1 = math.sqrt(slash_B * rd / _TOPIC_DIMS)
        o = n_noise + 1
        k[:, o: o + _TOPIC_DIMS] = b0 * t0
        k[:, o + _TOPIC_DIMS: o + 2 * _TOPIC_DIMS] = b1 * t1[slash_off: slash_off + S]  # k_j ~ t1[j + off]
        v = torch.randn((S, d), generator=gen, device=device)
        ks.append(k.to(dtype))
        vs.append(v.to(dtype))
        for h in heads:
            if h // group != g:
                continue
            hg = torch.Generator(device=device)
            hg.manual_seed(seed * 1000003 + 104729 * (h + 1))
            jit = 1.0 + spec.head_jitter * (2 * torch.rand((3,), generator=hg, device=device) - 1)
            q = torch.empty((S, d), device=device)
            q[:, :n_noise] = c * torch.randn((S, n_noise), generator=hg, device=device)
            q[:, n_noise] = jit[0]
            q[:, o: o + _TOPIC_DIMS] = b0 * jit[1] * t0
            # q_i ~ t1[i]: q_i . k_j over the slash dims peaks at i - j = slash_off
            q[:, o + _TOPIC_DIMS:] = b1 * jit[2] * t1[:S]
            qs.append((h, q.to(dtype)))
    qs.sort(key=lambda t: heads.index(t[0]))
    q = torch.stack([t[1] for t in qs]).contiguous()
    return q, torch.stack(ks).contiguous(), torch.stack(vs).contiguous(), kv_heads
