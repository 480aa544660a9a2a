"""ctypes binding of the C ABI (include/lhmm_b200.h) -> _lib/liblhmm_b200.so.

The product path has no fallback: if the native library is missing or cannot
load, every call raises NativeLibraryError.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# LHMM_LIB selects an experimental side build (tuning sweeps only)
LIB_PATH = os.environ.get("LHMM_LIB") or os.path.join(PKG, "_lib", "liblhmm_b200.so")


class NativeLibraryError(RuntimeError):
    pass


class Quant(C.Structure):
    _fields_ = [("scale", C.c_double), ("base", C.c_uint8), ("dbias", C.c_uint8),
                ("tec", C.c_uint8), ("tjb", C.c_uint8)]


class ScanOptionsC(C.Structure):
    _fields_ = [("alg", C.c_int), ("variant", C.c_int), ("lanes", C.c_uint32),
                ("rows", C.c_uint32), ("threshold", C.c_double), ("fault_injection", C.c_int),
                ("reorder_mode", C.c_int)]


class ScanStatsC(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("gcups", C.c_double), ("sequences", C.c_uint64),
                ("residues", C.c_uint64), ("cells", C.c_uint64), ("lanes", C.c_uint32),
                ("rows", C.c_uint32), ("variant", C.c_uint32), ("launches", C.c_uint32),
                ("grid", C.c_uint32), ("threads", C.c_uint32), ("smem_bytes", C.c_uint32),
                ("recomputed", C.c_uint32), ("saturated", C.c_uint64),
                ("mode_rows", C.c_uint64), ("lazy_rows", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class BalanceC(C.Structure):
    _fields_ = [("avg_m", C.c_double), ("sd_m", C.c_double), ("avg_endings", C.c_double),
                ("sd_endings", C.c_double), ("prr", C.c_double), ("total_seqs", C.c_uint64),
                ("total_residues", C.c_uint64)]


u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p

# name -> (restype, argtypes); every symbol include/lhmm_b200.h declares
SIGNATURES = {
    "lhmm_abi_version": (C.c_int, []),
    "lhmm_last_error": (C.c_char_p, []),
    "lhmm_quantize_emissions": (C.c_int, [f64p, C.c_uint32, C.POINTER(Quant), u8p]),
    "lhmm_move_cost": (C.c_uint8, [C.c_uint64, C.POINTER(Quant)]),
    "lhmm_sequence_base": (C.c_uint8, [C.c_uint64, C.POINTER(Quant)]),
    "lhmm_finalize_hit": (C.c_int, [C.c_uint8, C.c_uint64, C.c_double, C.c_double,
                                    C.POINTER(Quant), C.c_int, f64p, f64p,
                                    C.POINTER(C.c_int)]),
    "lhmm_select_geometry": (C.c_int, [C.c_uint32, C.c_int, C.c_int, u32p, u32p]),
    "lhmm_length_tables": (C.c_int, [C.POINTER(Quant), C.c_double, C.c_double, C.c_int,
                                     C.c_double, C.c_uint32, u8p, u8p]),
    "lhmm_shard_plan": (C.c_int, [u64p, C.c_uint64, C.c_uint32, C.c_uint32, u64p, u64p]),
    "lhmm_context_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "lhmm_context_destroy": (C.c_int, [vp]),
    "lhmm_context_set_stream": (C.c_int, [vp, vp]),
    "lhmm_context_set_db_budget": (C.c_int, [vp, C.c_uint64]),
    "lhmm_database_resident": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "lhmm_context_device_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                           C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "lhmm_set_profile": (C.c_int, [vp, u8p, C.c_uint32, C.POINTER(Quant), C.c_double,
                                   C.c_double]),
    "lhmm_add_profile": (C.c_int, [vp, u8p, C.c_uint32, C.POINTER(Quant), C.c_double,
                                   C.c_double, u32p]),
    "lhmm_select_profile": (C.c_int, [vp, C.c_uint32]),
    "lhmm_update_profile": (C.c_int, [vp, C.c_uint32, u8p, C.c_uint32, C.POINTER(Quant), C.c_double,
                                      C.c_double]),
    "lhmm_set_database": (C.c_int, [vp, u8p, u64p, C.c_uint64, C.c_uint32, C.c_uint32, u64p]),
    "lhmm_shard_indices": (C.c_int, [vp, u64p]),
    "lhmm_database_stats": (C.c_int, [vp, u64p, u64p, u64p, u64p]),
    "lhmm_upload_database": (C.c_int, [vp]),
    "lhmm_scan": (C.c_int, [vp, C.POINTER(ScanOptionsC), u8p, u8p, C.POINTER(ScanStatsC)]),
    "lhmm_scan_device": (C.c_int, [vp, C.POINTER(ScanOptionsC), vp, vp,
                                   C.POINTER(ScanStatsC)]),
    "lhmm_scan_device_global": (C.c_int, [vp, C.POINTER(ScanOptionsC), vp, vp,
                                          C.POINTER(ScanStatsC)]),
    "lhmm_peer_buffer_create": (C.c_int, [vp, C.c_uint64, vp, C.POINTER(vp)]),
    "lhmm_peer_buffer_open": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "lhmm_peer_buffers_release": (C.c_int, [vp]),
    "lhmm_device_fill": (C.c_int, [vp, vp, C.c_uint8, C.c_uint64]),
    "lhmm_device_to_host": (C.c_int, [vp, vp, vp, C.c_uint64]),
    "lhmm_device_copy": (C.c_int, [vp, vp, vp, C.c_uint64]),
    "lhmm_scatter_results": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_uint64]),
    "lhmm_context_synchronize": (C.c_int, [vp]),
    "lhmm_scan_streamed": (C.c_int, [vp, C.POINTER(ScanOptionsC), C.c_int, u8p, u8p,
                                     C.POINTER(ScanStatsC)]),
    "lhmm_scan_streamed_jobs": (C.c_int, [vp, C.c_int, u32p, C.POINTER(ScanOptionsC), C.c_int,
                                          C.POINTER(u8p), C.POINTER(u8p), C.POINTER(ScanStatsC)]),
    "lhmm_filter_pipeline": (C.c_int, [vp, C.c_double, C.c_int, u8p, u8p, u8p, u64p,
                                       C.POINTER(ScanStatsC), C.POINTER(ScanStatsC)]),
    "lhmm_rng_create": (C.c_int, [C.c_uint64, C.POINTER(vp)]),
    "lhmm_rng_destroy": (C.c_int, [vp]),
    "lhmm_rng_next": (C.c_uint64, [vp]),
    "lhmm_synth_random_profile": (C.c_int, [vp, C.c_uint32, f64p, f64p, f64p]),
    "lhmm_synth_random_records": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    "lhmm_synth_lognormal_records": (C.c_int, [vp, C.c_uint64, C.c_double, C.c_double,
                                               C.c_uint64, u64p]),
    "lhmm_synth_plant_motifs": (C.c_int, [vp, f64p, C.c_uint32, C.c_double]),
    "lhmm_synth_take": (C.c_int, [vp, u8p, u64p]),
    "lhmm_seqset_create": (C.c_int, [u8p, u64p, C.c_uint64, C.c_char_p, u64p, C.POINTER(vp)]),
    "lhmm_seqset_destroy": (C.c_int, [vp]),
    "lhmm_seqset_view": (C.c_int, [vp, u64p, u64p, C.POINTER(u8p), C.POINTER(u64p),
                                   C.POINTER(C.c_void_p), C.POINTER(u64p)]),
    "lhmm_seqset_layout": (C.c_int, [vp, u32p, u64p, C.POINTER(u64p), C.POINTER(u32p)]),
    "lhmm_seqset_set_layout": (C.c_int, [vp, C.c_uint32, C.c_uint64, u64p, u32p]),
    "lhmm_ingest_fasta": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(vp)]),
    "lhmm_ingest_fasta_file": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "lhmm_read_block_db": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "lhmm_write_block_db": (C.c_int, [vp, C.c_char_p]),
    "lhmm_pack_blocks": (C.c_int, [vp, C.c_uint64, C.c_uint32, C.POINTER(vp)]),
    "lhmm_balance_stats": (C.c_int, [vp, C.POINTER(BalanceC)]),
    "lhmm_parse_profile": (C.c_int, [C.c_char_p, C.c_size_t, u32p, f64p, f64p, f64p, C.c_size_t,
                                     C.c_char_p, C.c_size_t]),
    "lhmm_serialize_profile": (C.c_int, [C.c_char_p, C.c_uint32, f64p, C.c_double, C.c_double,
                                         C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
}

_lib = None


def lib():
    """Load (once) and return the native library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    try:
        L = C.CDLL(LIB_PATH)
    except OSError as e:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.lhmm_abi_version() != 2:
        raise NativeLibraryError("ABI version mismatch")
    _lib = L
    return L
