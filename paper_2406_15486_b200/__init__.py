"""B200-native SampleAttention: the hot path of the reference package
`blocksift` (arxiv 2406.15486) as hand-written sm_100a CUDA behind the
reference's own Python entry points.

    stage 1  sample_scores + block_reduce  -> tcgen05/TMA fused sampled attention
    stage 2  find_k / arg_topk / merge     -> block-wide sort + sequential fp64 cumsum + CSR merge
    stage 3  sparse_attention              -> tcgen05/TMEM block-sparse prefill (GQA-aware)

Names, argument meaning and exceptions follow `blocksift` (see the per-module
docstrings for the file:line each one mirrors).  There is no CPU fallback:
every compute call goes through libsampleattn.so and raises if it is missing.
"""

from .config import ChunkPlan, SampledRange, SparseConfig, n_blocks, plan_chunks, resolve_config
from .errors import GeneratorError, InfeasibleGridError, InputError, InternalInvariantError
from .heads import AttentionHead, HeadBatch, HeadSet, check_finite
from .masks import BlockMask, ChunkSelection, SelectedIndices
from .pipeline import (ORACLE_CAP, HeadMetrics, MetricsReport, SampleAttentionResult, cra_full, dense_attention,
                       run_pipeline, sample_attention)
from . import tensor_io
from .graph import SampleAttentionGraph
from . import refsynth, streaming
from .refsynth import SyntheticSpec, generate_synthetic
from .streaming import release_staging, sample_attention_host
from .stages import (GUARD_EPS, ChunkScores, FlopReport, ReducedScores, SampledScores, arg_topk, block_reduce,
                     find_k, flop_accounting, merge_index, sample_scores, select, select_and_merge,
                     sparse_attention)

__version__ = "0.1.0"

__all__ = [
    "AttentionHead", "BlockMask", "ChunkPlan", "ChunkScores", "ChunkSelection", "FlopReport",
    "GUARD_EPS", "GeneratorError", "HeadBatch", "HeadMetrics", "HeadSet", "InfeasibleGridError", "InputError",
    "InternalInvariantError", "MetricsReport", "SampleAttentionGraph", "ORACLE_CAP", "ReducedScores", "SampleAttentionResult",
    "SampledRange", "SampledScores", "SelectedIndices", "SparseConfig", "arg_topk", "block_reduce",
    "check_finite", "cra_full", "dense_attention", "find_k", "flop_accounting", "merge_index", "n_blocks", "plan_chunks",
    "release_staging", "resolve_config", "run_pipeline", "sample_attention", "sample_attention_host", "sample_scores",
    "select", "select_and_merge", "sparse_attention", "SyntheticSpec", "generate_synthetic",
]
