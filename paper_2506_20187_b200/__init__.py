"""paper_2506_20187_b200 -- B200-native (sm_100a) LeoAM KV selection + sparse decode path.

Drop-in for the hot path of the reference package `kvtier` (importance / chunk_tree /
engine.attention_output), plus a batched decode API (`decode`) used by bench.py.
All compute runs in hand-written CUDA kernels behind the C ABI in include/kvtier_b200.h;
there is no CPU fallback.
"""

from .chunk_tree import (
    CANDIDATE, DESERT, IMPORTANT, PAD, ChunkNode, ChunkPlanConfig, ChunkSource, Partition, SelectionResult,
    build_partition, chunk_cost, dump_partition, merge_desert, next_pow2, plan_chunk_count, select_top_k,
)
from .engine import attention_output, cosine_similarity, desert_rate_on_grid, oracle_output, token_runs
from .importance import (
    ChunkAbstract, ChunkBounds, attention_logits, bound_chunk, bound_chunks_batch, make_abstract,
    merge_abstracts, score_tokens, softmax,
)

__version__ = "0.1.0"
