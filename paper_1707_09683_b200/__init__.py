"""B200-native MSV/SSV filter scan (HMMER3 filters per arxiv 1707.09683),
a drop-in for the reference lanehmm filter path.

Native library: _lib/liblhmm_b200.so (C ABI in include/lhmm_b200.h); no CPU
fallback exists -- calls raise NativeLibraryError if it is missing.
"""
from .lanehmm import (  # noqa: F401
    Algorithm, ContractError, CudaError, ParseError, CostMatrix, DataError, HitResult, PipelineReport, ProfileHMM,
    QuantParams, Rng, filter_pipeline,
    ScanOptions, ScanReport, Scanner, SequenceDB, Variant, engine_sequence_base, finalize_hit,
    hits_from, move_cost, quantize_emissions, scan_database, scan_sequences_s1, select_geometry)
from .seqdb import (  # noqa: F401
    BalanceStats, BlockSet, IdTable, balance_stats, ingest_fasta, ingest_fasta_file, pack_blocks,
    parse_profile, read_block_db, read_profile_file, serialize_profile, to_fasta, write_block_db)
from ._native import LIB_PATH, NativeLibraryError, lib  # noqa: F401
