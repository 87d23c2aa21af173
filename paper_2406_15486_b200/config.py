"""Tunable knobs and the chunk plan (host-side integer logic).

Restates SparseConfig / plan_chunks of the reference
(pkg/src/blocksift/sampler.py:33-118) with the same validation and clamping,
plus the north-star shorthands the reference does not have: a single
`alpha` for both directions and a `sample_ratio` that maps to chunk_n.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InputError

__all__ = ["SparseConfig", "SampledRange", "ChunkPlan", "n_blocks", "plan_chunks", "resolve_config"]


def n_blocks(s: int, blk: int) -> int:
    """Blocks covering s positions; the trailing one may be narrower (sampler.py:33-35)."""
    return -(-s // blk)


@dataclass(frozen=True)
class SparseConfig:
    """alpha_c / alpha_s CRA thresholds, chunk count and block size
    (sampler.py:38-56; same defaults and InputError checks)."""

    alpha_c: float = 0.95
    alpha_s: float = 0.95
    chunk_n: int = 1
    blk: int = 128

    def __post_init__(self):
        if not 0.0 <= self.alpha_c <= 1.0:
            raise InputError(f"alpha_c must be in [0, 1], got {self.alpha_c}")
        if not 0.0 <= self.alpha_s <= 1.0:
            raise InputError(f"alpha_s must be in [0, 1], got {self.alpha_s}")
        if self.chunk_n < 1:
            raise InputError(f"chunk_n must be >= 1, got {self.chunk_n}")
        if self.blk < 1:
            raise InputError(f"blk must be >= 1, got {self.blk}")


def resolve_config(S: int, alpha: float = 0.95, alpha_c: float | None = None,
                   alpha_s: float | None = None, chunk_n: int | None = None,
                   sample_ratio: float | None = None, blk: int = 128) -> SparseConfig:
    """North-star keyword form -> SparseConfig.

    `alpha` is shorthand for alpha_c = alpha_s; `sample_ratio` (fraction of
    query rows to score exactly) maps to chunk_n = max(1, round(ratio*S/blk)),
    after which plan_chunks applies the reference's own clamping.  Giving both
    chunk_n and sample_ratio is an error."""
    if chunk_n is not None and sample_ratio is not None:
        raise InputError("give chunk_n or sample_ratio, not both")
    if sample_ratio is not None:
        if not 0.0 < sample_ratio <= 1.0:
            raise InputError(f"sample_ratio must be in (0, 1], got {sample_ratio}")
        chunk_n = max(1, int(round(sample_ratio * S / blk)))
    return SparseConfig(
        alpha_c=alpha if alpha_c is None else alpha_c,
        alpha_s=alpha if alpha_s is None else alpha_s,
        chunk_n=1 if chunk_n is None else int(chunk_n),
        blk=blk,
    )


@dataclass(frozen=True)
class SampledRange:
    """One chunk: sampled rows [sample_start, sample_end) and governed
    region [region_start, region_end) (sampler.py:59-66)."""

    sample_start: int
    sample_end: int
    region_start: int
    region_end: int


@dataclass(frozen=True)
class ChunkPlan:
    """sampler.py:69-85: effective chunk_n after clamping, requested kept."""

    S: int
    blk: int
    requested_chunk_n: int
    chunk_n: int
    itv: int
    chunks: tuple

    def sampled_rows(self) -> int:
        return sum(c.sample_end - c.sample_start for c in self.chunks)

    def sample_ratio(self) -> float:
        return self.sampled_rows() / self.S


def plan_chunks(S: int, cfg: SparseConfig) -> ChunkPlan:
    """Sampling layout (sampler.py:88-118).

    S < blk: one window [0, S).  Otherwise itv = S // chunk_n, clamping
    chunk_n to max(1, S // blk) when a segment would be shorter than blk;
    window i samples [i*itv - blk, i*itv) and governs [(i-1)*itv, i*itv),
    the last region extending to S."""
    if S < 1:
        raise InputError(f"S must be >= 1, got {S}")
    blk = cfg.blk
    if S < blk:
        cn, itv = 1, S
    else:
        cn = cfg.chunk_n
        itv = S // cn
        if itv < blk:
            cn = max(1, S // blk)
            itv = S // cn
    chunks = tuple(
        SampledRange(max(0, i * itv - blk), i * itv, (i - 1) * itv, S if i == cn else i * itv)
        for i in range(1, cn + 1)
    )
    return ChunkPlan(S, blk, cfg.chunk_n, cn, itv, chunks)
