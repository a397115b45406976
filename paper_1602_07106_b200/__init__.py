"""B200-native Barabasi-Albert edge generator (Sanders & Schulz, arXiv 1602.07106).

Drop-in for the hot path of the reference package ``parba``: same names,
argument meaning, return types and error behaviour for the generator (uniform
degree or degree sequence, option flags) and the degree API; the chains and
the degree-sequence index run in hand-written sm_100a CUDA kernels
(``libparba_b200.so``, C ABI in include/parba_b200.h).  There is no CPU
fallback: without the library or a CUDA device every compute call raises
``GenerationError``.
"""

from .analytics import (
    DegreeCounter,
    DegreeCountConsumer,
    count_block,
    count_edge,
    count_seed_edges,
    degree_counts,
    merge,
)
from .driver import (
    DEFAULT_BATCH_SIZE,
    Batch,
    CollectConsumer,
    Consumer,
    DiscardConsumer,
    Granularity,
    RunStats,
    WorkerStats,
    plan_batches,
    run,
)
from . import degreeseq, io, parallel
from .degreeseq import (
    PrefixIndex,
    RankBits,
    build_prefix,
    build_rank_bits,
    first_half_pos,
    node_of_edge,
    node_of_edge_bisect,
    read_degree_file,
    resolve_targets_deferred,
)
from .errors import GenerationError, InfeasibleTargetsError, ParameterError, SeedGraphFormatError
from .generator import (
    MAX_EDGES,
    ChainResult,
    Edge,
    GenParams,
    edge_count,
    edges_at,
    generate_block,
    generate_block_device,
    generate_edge,
    generate_node_edges,
    resolve_chain,
    resolve_chain_block,
)
from .io import EdgeFileWriter, write_edges_binary
from .hashing import (
    CRC32C_TABLE,
    DEFAULT_MULTIPLIER,
    HashConfig,
    HashKind,
    crc32c_u64,
    crc32c_u64_many,
    h_crc,
    h_crc_many,
    h_simple,
    h_simple_many,
    hash_many,
    hash_value,
    mulhi_u64,
)
from .oracle_compat import bb_generate, edge_list

__version__ = "0.1.0"

__all__ = [
    "CRC32C_TABLE", "crc32c_u64", "crc32c_u64_many", "h_crc_many", "h_simple_many", "mulhi_u64",
    "Batch", "ChainResult", "CollectConsumer", "Consumer", "DEFAULT_BATCH_SIZE",
    "DEFAULT_MULTIPLIER", "DegreeCountConsumer", "EdgeFileWriter", "write_edges_binary", "DegreeCounter", "DiscardConsumer", "Edge",
    "GenParams", "GenerationError", "Granularity", "HashConfig", "HashKind",
    "InfeasibleTargetsError", "MAX_EDGES", "ParameterError", "PrefixIndex", "RankBits", "RunStats",
    "SeedGraphFormatError", "build_prefix", "build_rank_bits", "first_half_pos", "node_of_edge",
    "node_of_edge_bisect", "read_degree_file", "resolve_targets_deferred",
    "WorkerStats", "bb_generate", "count_block", "count_edge", "count_seed_edges", "degree_counts",
    "edge_count", "edge_list", "edges_at",
    "generate_block", "generate_block_device", "generate_edge", "generate_node_edges", "h_crc",
    "h_simple", "hash_many", "hash_value", "merge", "plan_batches", "resolve_chain",
    "resolve_chain_block", "run",
]
