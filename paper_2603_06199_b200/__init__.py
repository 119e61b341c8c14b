"""paper_2603_06199_b200 — B200-native FlashPrefill (arxiv 2603.06199) sparse-prefill hot path.

Drop-in for the reference's ``bsattn::`` C++ API (discover / max_threshold_mask /
compress_indices / block_sparse_attention / dense_attention) on hand-written sm_100a kernels
behind the C ABI in include/fpb200.h.  See DESIGN.md.
"""
from .bsattn import (  # noqa: F401
    ActiveMask, AttentionOutput, AttentionStats, BlockEnergies, BlockGrid, BlockScoreMap,
    ConfigError, CudaError, FormatError, IoError, PipelineConfig, PlanError, PooledKeys,
    PrefillRunner,
    SelectionStats, SparseBlockPlan, ValidationError, approx_block_scores, block_sparse_attention,
    compress_indices, dense_attention, density, discover, discover_exact, discover_pool_both,
    discover_select, flops_dense_causal, topk_select, topp_select,
    flops_sparse, full_causal_plan, make_block_grid, make_sequence_batch, max_threshold_mask,
    normalize_block_scores, pool_keys, prefill, prefill_host, visit_count,
)
from . import workload  # noqa: F401,E402  (synthetic inputs for bench / tests)
from . import shard  # noqa: F401,E402  (multi-GPU partitions and gathers)
