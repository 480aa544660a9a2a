"""Host-side mirror of the reference's filter interface (lanehmm engine.hpp)
over the B200 C ABI.

Names, argument meaning and errors follow /root/reference/proj/include/lanehmm:
  QuantParams, ProfileHMM, CostMatrix     profile.hpp:14-52
  Algorithm, ScanOptions, HitResult,
  ScanReport, finalize_hit,
  engine_sequence_base, scan_database,
  scan_sequences_s1, filter_pipeline      engine.hpp:13-132
  ContractError / DataError               errors.hpp:23-32
  synth.*                                 synth.hpp:13-27

The database argument is a ``SequenceDB`` (flat residue codes + offsets, the
input a length-binned B200 packer wants) instead of a BlockSet; pack_blocks'
job is done by the native tile packer behind lhmm_set_database.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import NativeLibraryError  # noqa: F401  (re-export)

AMINO = "ACDEFGHIKLMNPQRSTVWY"
UNKNOWN_CODE, ENDING_CODE, PADDING_CODE = 20, 21, 22


class ContractError(ValueError):
    """A caller broke a documented precondition (errors.hpp:29-32)."""


class DataError(RuntimeError):
    """Structurally invalid data (errors.hpp:23-27)."""


class ParseError(RuntimeError):
    """Malformed input text, "line N: ..." (errors.hpp:10-20)."""


class CudaError(RuntimeError):
    pass


def _check(rc):
    if rc == 0:
        return
    msg = _native.lib().lhmm_last_error().decode()
    if rc == 1:
        raise ContractError(msg)
    if rc == 2:
        raise DataError(msg)
    if rc == 4:
        raise MemoryError(msg)
    if rc == 5:
        raise ParseError(msg)
    raise CudaError(msg)


class Algorithm(enum.IntEnum):
    Msv = 0
    Ssv = 1


class Variant(enum.IntEnum):
    Auto = 0
    Dpx16 = 1
    Fp16 = 2
    Swar8 = 3
    Fp16x = 4
    Fp16xAlt = 5   # MSV only: FP16X with a quarter of the cost steps on the FP16 pipe
    Fp16xMixed = 6  # FP16X with a mixed 16-bit / byte table (1.6 B per cell)
    Fp16xHybrid = 7  # MSV: FP16X exact rows + FP16XM lazy rows (two tables)
    Fp16xRelaxed = 8  # MSV: no 255 cap (subnormal f16), flagged sequences rescored exactly
    Fp16xRelaxedFixedB = 9  # MSV: relaxed with B fixed at base, FP16XM table, flags rescored


@dataclass
class QuantParams:
    scale: float = 3.0
    base: int = 195
    dbias: int = 3
    tec: int = 3
    tjb: int = 3

    kNegInfMsv = 0x00
    kNegInfSsv = 0x80

    def c(self):
        return _native.Quant(self.scale, self.base, self.dbias, self.tec, self.tjb)


def neg_inf(alg):
    return QuantParams.kNegInfMsv if alg == Algorithm.Msv else QuantParams.kNegInfSsv


@dataclass
class ProfileHMM:
    name: str
    length: int
    match_scores: np.ndarray  # length x 20 float64
    lambda_: float = 0.69
    tau: float = 2.0


@dataclass
class CostMatrix:
    model_length: int
    bytes: np.ndarray  # model_length x 21 uint8

    def at(self, node1, code):
        if code > UNKNOWN_CODE:
            return 0xFF
        return int(self.bytes[(node1 - 1) * 21 + code])


@dataclass
class SequenceDB:
    residues: np.ndarray  # uint8 codes 0..20
    offsets: np.ndarray   # uint64, n+1
    ids: list | None = None

    def __post_init__(self):
        self.residues = np.ascontiguousarray(self.residues, dtype=np.uint8)
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.uint64)

    @property
    def count(self):
        return self.offsets.size - 1

    def lengths(self):
        return np.diff(self.offsets).astype(np.uint64)

    def total_residues(self):
        return int(self.offsets[-1])

    def sequence(self, k):
        return self.residues[int(self.offsets[k]):int(self.offsets[k + 1])]

    @staticmethod
    def from_sequences(seqs):
        seqs = [np.asarray(s, dtype=np.uint8) for s in seqs]
        off = np.zeros(len(seqs) + 1, dtype=np.uint64)
        off[1:] = np.cumsum([s.size for s in seqs])
        res = np.concatenate(seqs) if seqs and off[-1] > 0 else np.zeros(0, np.uint8)
        return SequenceDB(res, off)

    def subset(self, idx):
        return SequenceDB.from_sequences([self.sequence(int(k)) for k in idx])


def encode_residue(ch):
    """alphabet.cpp:29-31: the 20 canonical letters (any case), else unknown."""
    i = AMINO.find(ch.upper())
    return i if i >= 0 else UNKNOWN_CODE


@dataclass
class ScanOptions:
    alg: Algorithm = Algorithm.Msv
    variant: Variant = Variant.Auto
    lanes: int = 0      # 0 = auto geometry
    rows: int = 0
    threshold: float = 0.02
    fault_injection: bool = False
    paper_wrap: bool = False  # ReorderMode::PaperWrap (non-normative study mode)
    workers: int = 1    # accepted for interface parity; must be >= 1

    def c(self):
        if self.workers < 1:
            raise ContractError("worker count must be >= 1")
        return _native.ScanOptionsC(int(self.alg), int(self.variant), self.lanes, self.rows,
                                    float(self.threshold), int(bool(self.fault_injection)),
                                    int(bool(self.paper_wrap)))


@dataclass
class HitResult:
    seq_index: int
    raw: int
    bits: float
    p_value: float
    overflow: bool
    seq_len: int


@dataclass
class ScanReport:
    alg: Algorithm
    lanes: int
    rows: int
    variant: int
    total_sequences: int
    total_residues: int
    elapsed_seconds: float  # device (CUDA-event) time of the scan
    gcups: float
    raw: np.ndarray
    passed: np.ndarray
    stats: dict = field(default_factory=dict)


@dataclass
class PipelineReport:
    """engine.hpp:118-126: SSV stage over everything, MSV over the survivors."""
    threshold: float
    ssv_scanned: int
    msv_rescored: int
    ssv_seconds: float
    msv_seconds: float
    survivors: np.ndarray   # local indices with pValue <= t or SSV overflow
    ssv_raw: np.ndarray     # all sequences
    passed: np.ndarray
    msv_raw: np.ndarray     # survivors' MSV bytes, 0 elsewhere
    ssv_stats: dict = field(default_factory=dict)
    msv_stats: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# byte-space helpers (host, bit-identical to the reference)

def quantize_emissions(hmm: ProfileHMM, q: QuantParams) -> CostMatrix:
    scores = np.ascontiguousarray(hmm.match_scores, dtype=np.float64).reshape(-1)
    m = hmm.length
    if scores.size != m * 20:
        raise ContractError("match score table must be length x 20")
    out = np.zeros(m * 21, dtype=np.uint8)
    qc = q.c()
    _check(_native.lib().lhmm_quantize_emissions(
        scores.ctypes.data_as(_native.f64p), m, C.byref(qc),
        out.ctypes.data_as(_native.u8p)))
    return CostMatrix(m, out)


def move_cost(seq_len, q: QuantParams):
    qc = q.c()
    return _native.lib().lhmm_move_cost(seq_len, C.byref(qc))


def engine_sequence_base(seq_len, q: QuantParams):
    qc = q.c()
    return _native.lib().lhmm_sequence_base(seq_len, C.byref(qc))


def finalize_hit(raw, seq_len, lambda_, tau, q: QuantParams, alg) -> HitResult:
    bits, p, ovf = C.c_double(), C.c_double(), C.c_int()
    qc = q.c()
    _check(_native.lib().lhmm_finalize_hit(raw, seq_len, lambda_, tau, C.byref(qc), int(alg),
                                           C.byref(bits), C.byref(p), C.byref(ovf)))
    return HitResult(-1, raw, bits.value, p.value, bool(ovf.value), seq_len)


def select_geometry(model_length, alg, variant=Variant.Auto):
    L, H = C.c_uint32(), C.c_uint32()
    _check(_native.lib().lhmm_select_geometry(model_length, int(alg), int(variant), C.byref(L),
                                              C.byref(H)))
    return L.value, H.value


# ---------------------------------------------------------------------------
# device scanner

class Scanner:
    """One device context: a resident profile and database (or shard)."""

    def __init__(self, device=0):
        self._ctx = C.c_void_p()
        _check(_native.lib().lhmm_context_create(device, C.byref(self._ctx)))
        self.device = device
        self.n_local = 0
        self.m = 0

    def close(self):
        if self._ctx:
            _native.lib().lhmm_context_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def device_info(self):
        sm, clk, ma, mi = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_native.lib().lhmm_context_device_info(self._ctx, C.byref(sm), C.byref(clk),
                                                      C.byref(ma), C.byref(mi)))
        return {"sm_count": sm.value, "sm_clock_khz": clk.value, "cc": (ma.value, mi.value)}

    def set_db_budget(self, device_bytes):
        """Out-of-core mode: databases whose packed image exceeds this many
        device bytes stay in pinned host memory and are streamed through a
        ring of device slots on every scan (0 = unlimited)."""
        _check(_native.lib().lhmm_context_set_db_budget(self._ctx, int(device_bytes)))

    def database_resident(self):
        on = C.c_int()
        _check(_native.lib().lhmm_database_resident(self._ctx, C.byref(on)))
        return bool(on.value)

    def set_stream(self, stream_handle):
        _check(_native.lib().lhmm_context_set_stream(self._ctx, C.c_void_p(stream_handle)))

    def set_profile(self, costs: CostMatrix, q: QuantParams, lambda_=0.69, tau=2.0):
        b = np.ascontiguousarray(costs.bytes, dtype=np.uint8)
        qc = q.c()
        _check(_native.lib().lhmm_set_profile(self._ctx, b.ctypes.data_as(_native.u8p),
                                              costs.model_length, C.byref(qc), lambda_, tau))
        self.m = costs.model_length

    def add_profile(self, costs: CostMatrix, q: QuantParams, lambda_=0.69, tau=2.0):
        """Keep another model resident; returns its id (now current)."""
        b = np.ascontiguousarray(costs.bytes, dtype=np.uint8)
        qc = q.c()
        pid = C.c_uint32()
        _check(_native.lib().lhmm_add_profile(self._ctx, b.ctypes.data_as(_native.u8p),
                                              costs.model_length, C.byref(qc), lambda_, tau,
                                              C.byref(pid)))
        self.m = costs.model_length
        self._models = getattr(self, "_models", {})
        self._models[pid.value] = costs.model_length
        return pid.value

    def select_profile(self, pid):
        _check(_native.lib().lhmm_select_profile(self._ctx, pid))
        self.m = getattr(self, "_models", {}).get(pid, self.m)

    def set_database(self, db: SequenceDB, shard_rank=0, shard_count=1):
        n = C.c_uint64()
        res = db.residues if db.residues.size else np.zeros(1, np.uint8)
        _check(_native.lib().lhmm_set_database(
            self._ctx, res.ctypes.data_as(_native.u8p), db.offsets.ctypes.data_as(_native.u64p),
            db.count, shard_rank, shard_count, C.byref(n)))
        self.n_local = n.value
        return self.n_local

    def shard_indices(self):
        out = np.zeros(max(self.n_local, 1), dtype=np.uint64)
        _check(_native.lib().lhmm_shard_indices(self._ctx, out.ctypes.data_as(_native.u64p)))
        return out[:self.n_local]

    def database_stats(self):
        r, p, t, b = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_native.lib().lhmm_database_stats(self._ctx, C.byref(r), C.byref(p), C.byref(t),
                                                 C.byref(b)))
        return {"residues": r.value, "padded_cells": p.value, "tiles": t.value,
                "packed_bytes": b.value}

    def upload_database(self):
        _check(_native.lib().lhmm_upload_database(self._ctx))

    def _outputs(self, out):
        """Caller-provided (raw, passed) uint8 arrays of >= n_local bytes
        (reused across scans; page-locked ones are copied into directly),
        or fresh ones."""
        n = max(self.n_local, 1)
        if out is None:
            return np.empty(n, dtype=np.uint8), np.empty(n, dtype=np.uint8)
        raw, passed = out
        for a in (raw, passed):
            if a.dtype != np.uint8 or a.size < self.n_local or not a.flags.c_contiguous:
                raise ContractError("outputs must be contiguous uint8 arrays of n_local bytes")
        return raw, passed

    def scan(self, opt: ScanOptions, out=None):
        raw, passed = self._outputs(out)
        st = _native.ScanStatsC()
        oc = opt.c()
        _check(_native.lib().lhmm_scan(self._ctx, C.byref(oc), raw.ctypes.data_as(_native.u8p),
                                       passed.ctypes.data_as(_native.u8p), C.byref(st)))
        n = self.n_local
        return ScanReport(opt.alg, st.lanes, st.rows, st.variant, st.sequences, st.residues,
                          st.device_ms * 1e-3, st.gcups, raw[:n], passed[:n].view(bool),
                          st.as_dict())

    def scan_streamed(self, opt: ScanOptions, segments=8, out=None):
        """End-to-end scan from the packed host image with the H2D copy
        overlapped with the kernels (lhmm_scan_streamed)."""
        raw, passed = self._outputs(out)
        st = _native.ScanStatsC()
        oc = opt.c()
        _check(_native.lib().lhmm_scan_streamed(self._ctx, C.byref(oc), segments,
                                                raw.ctypes.data_as(_native.u8p),
                                                passed.ctypes.data_as(_native.u8p), C.byref(st)))
        n = self.n_local
        return ScanReport(opt.alg, st.lanes, st.rows, st.variant, st.sequences, st.residues,
                          st.device_ms * 1e-3, st.gcups, raw[:n], passed[:n].view(bool),
                          st.as_dict())

    def scan_streamed_jobs(self, jobs, segments=64, outs=None):
        """Several scans over ONE streamed upload of the packed host image
        (lhmm_scan_streamed_jobs): `jobs` = [(profile_id, ScanOptions)], each
        piece scanned by every job as it lands.  `outs`: optional [(raw,
        passed)] per job.  Returns one ScanReport per job."""
        k = len(jobs)
        if k < 1:
            raise ContractError("no jobs")
        outs = [self._outputs(None if outs is None else outs[j]) for j in range(k)]
        ids = (C.c_uint32 * k)(*[int(p) for p, _ in jobs])
        opts = (_native.ScanOptionsC * k)(*[o.c() for _, o in jobs])
        raws = (_native.u8p * k)(*[r.ctypes.data_as(_native.u8p) for r, _ in outs])
        passes = (_native.u8p * k)(*[p.ctypes.data_as(_native.u8p) for _, p in outs])
        sts = (_native.ScanStatsC * k)()
        _check(_native.lib().lhmm_scan_streamed_jobs(self._ctx, k, ids, opts, int(segments), raws,
                                                     passes, sts))
        n = self.n_local
        reps = []
        for j, (_, o) in enumerate(jobs):
            st = sts[j]
            raw, passed = outs[j]
            reps.append(ScanReport(o.alg, st.lanes, st.rows, st.variant, st.sequences,
                                   st.residues, st.device_ms * 1e-3, st.gcups, raw[:n],
                                   passed[:n].view(bool), st.as_dict()))
        return reps

    def filter_pipeline(self, threshold, variant=Variant.Auto):
        """SSV over the resident database, survivors (pValue <= t or overflow)
        compacted on the device, MSV over the survivors (lhmm_filter_pipeline).
        Returns a PipelineReport."""
        n = max(self.n_local, 1)
        ssv = np.zeros(n, np.uint8)
        passed = np.zeros(n, np.uint8)
        msv = np.zeros(n, np.uint8)
        resc = C.c_uint64()
        s1, s2 = _native.ScanStatsC(), _native.ScanStatsC()
        _check(_native.lib().lhmm_filter_pipeline(
            self._ctx, float(threshold), int(variant), ssv.ctypes.data_as(_native.u8p),
            passed.ctypes.data_as(_native.u8p), msv.ctypes.data_as(_native.u8p), C.byref(resc),
            C.byref(s1), C.byref(s2)))
        k = self.n_local
        return PipelineReport(float(threshold), k, resc.value, s1.device_ms * 1e-3,
                              s2.device_ms * 1e-3, np.flatnonzero(passed[:k]), ssv[:k],
                              passed[:k].astype(bool), msv[:k], s1.as_dict(), s2.as_dict())

    def scan_device_global(self, opt: ScanOptions, raw_ptr: int, pass_ptr: int):
        """Outputs addressed by GLOBAL sequence index into full-length device
        buffers -- typically rank 0's, mapped through CUDA IPC (the fused
        gather, shard.PeerOutputs)."""
        st = _native.ScanStatsC()
        oc = opt.c()
        _check(_native.lib().lhmm_scan_device_global(self._ctx, C.byref(oc), C.c_void_p(raw_ptr),
                                                     C.c_void_p(pass_ptr), C.byref(st)))
        return st.as_dict()

    def peer_buffer_create(self, nbytes):
        """A device buffer whose CUDA IPC handle other processes can map;
        returns (device pointer, 64-byte handle)."""
        h = (C.c_uint8 * 64)()
        ptr = C.c_void_p()
        _check(_native.lib().lhmm_peer_buffer_create(self._ctx, int(nbytes), h, C.byref(ptr)))
        return ptr.value, bytes(h)

    def peer_buffer_open(self, handle: bytes):
        h = (C.c_uint8 * 64).from_buffer_copy(handle)
        ptr = C.c_void_p()
        _check(_native.lib().lhmm_peer_buffer_open(self._ctx, h, C.byref(ptr)))
        return ptr.value

    def peer_buffers_release(self):
        _check(_native.lib().lhmm_peer_buffers_release(self._ctx))

    def device_fill(self, ptr, value, nbytes):
        _check(_native.lib().lhmm_device_fill(self._ctx, C.c_void_p(ptr), value, int(nbytes)))

    def device_to_host(self, ptr, nbytes):
        out = np.zeros(max(int(nbytes), 1), np.uint8)
        _check(_native.lib().lhmm_device_to_host(self._ctx, C.c_void_p(ptr),
                                                 out.ctypes.data_as(C.c_void_p), int(nbytes)))
        return out[:int(nbytes)]

    def device_copy(self, dst_ptr, src_ptr, nbytes):
        """Asynchronous device-to-device copy on the context's stream (local,
        peer or IPC-mapped pointers): the block gather's bulk NVLink copy."""
        _check(_native.lib().lhmm_device_copy(self._ctx, C.c_void_p(dst_ptr), C.c_void_p(src_ptr),
                                              int(nbytes)))

    def scatter_results(self, raw_dst, pass_dst, raw_src, pass_src, index_ptr, n):
        """dst[index[k]] = src[k] for k < n (device pointers; index u64)."""
        _check(_native.lib().lhmm_scatter_results(
            self._ctx, C.c_void_p(raw_dst), C.c_void_p(pass_dst), C.c_void_p(raw_src),
            C.c_void_p(pass_src), C.c_void_p(index_ptr), int(n)))

    def synchronize(self):
        _check(_native.lib().lhmm_context_synchronize(self._ctx))

    def scan_device(self, opt: ScanOptions, raw_ptr: int, pass_ptr: int):
        """Outputs stay on the device (e.g. torch.uint8 tensors' data_ptr())."""
        st = _native.ScanStatsC()
        oc = opt.c()
        _check(_native.lib().lhmm_scan_device(self._ctx, C.byref(oc), C.c_void_p(raw_ptr),
                                              C.c_void_p(pass_ptr), C.byref(st)))
        return st.as_dict()


def hits_from(report: ScanReport, db: SequenceDB, hmm: ProfileHMM, q: QuantParams):
    """Per-sequence HitResults in input order (the reference's hit list)."""
    lens = db.lengths()
    out = []
    for k in range(db.count):
        h = finalize_hit(int(report.raw[k]), int(lens[k]), hmm.lambda_, hmm.tau, q, report.alg)
        h.seq_index = k
        out.append(h)
    return out


def scan_database(hmm: ProfileHMM, costs: CostMatrix, db: SequenceDB, q: QuantParams,
                  opt: ScanOptions, device=0) -> ScanReport:
    """engine.hpp:94-95 -- scan every sequence of `db` with MSV or SSV."""
    if opt.workers < 1:
        raise ContractError("worker count must be >= 1")
    with Scanner(device) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(db)
        return s.scan(opt)


def filter_pipeline(hmm: ProfileHMM, costs: CostMatrix, db: SequenceDB, threshold: float,
                    q: QuantParams, opt: ScanOptions = None, device=0) -> PipelineReport:
    """engine.hpp:130-132 -- SSV over `db`, then MSV rescoring of every
    sequence with pValue <= threshold or SSV overflow, on the device."""
    if threshold < 0.0 or threshold > 1.0:
        raise ContractError("pipeline threshold must lie in [0,1]")
    variant = opt.variant if opt is not None else Variant.Auto
    with Scanner(device) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(db)
        return s.filter_pipeline(threshold, variant)


def scan_sequences_s1(hmm, costs, db, q, opt, device=0) -> ScanReport:
    """engine.hpp:99-101 -- the reference's S=1 path (one warp per sequence):
    here the whole warp cooperates on one sequence (lanes = 32)."""
    if db.count == 0:
        raise DataError("no sequences to scan")
    o = ScanOptions(**{**opt.__dict__, "lanes": 32, "rows": 0})
    return scan_database(hmm, costs, db, q, o, device)


# ---------------------------------------------------------------------------
# seeded synthetic inputs (src/synth.cpp:8-81, same streams)

class Rng:
    def __init__(self, seed):
        self._h = C.c_void_p()
        _check(_native.lib().lhmm_rng_create(seed, C.byref(self._h)))
        self._pending = 0

    def __del__(self):
        try:
            _native.lib().lhmm_rng_destroy(self._h)
        except Exception:
            pass

    def next(self):
        return _native.lib().lhmm_rng_next(self._h)

    def random_profile(self, m, name=None) -> ProfileHMM:
        s = np.zeros(m * 20, dtype=np.float64)
        lam, tau = C.c_double(), C.c_double()
        _check(_native.lib().lhmm_synth_random_profile(self._h, m,
                                                       s.ctypes.data_as(_native.f64p),
                                                       C.byref(lam), C.byref(tau)))
        return ProfileHMM(name or f"synth{m}", m, s.reshape(m, 20), lam.value, tau.value)

    def _take(self, count, total):
        res = np.zeros(max(total, 1), dtype=np.uint8)
        off = np.zeros(count + 1, dtype=np.uint64)
        _check(_native.lib().lhmm_synth_take(self._h, res.ctypes.data_as(_native.u8p),
                                             off.ctypes.data_as(_native.u64p)))
        return SequenceDB(res[:total], off)

    def random_records(self, count, len_lo, len_hi, plant: tuple | None = None) -> SequenceDB:
        """synth::random_records; plant=(hmm, fraction) then applies
        synth::plant_motifs on the same generator."""
        tot = C.c_uint64()
        _check(_native.lib().lhmm_synth_random_records(self._h, count, len_lo, len_hi,
                                                       C.byref(tot)))
        self._plant(plant)
        return self._take(count, tot.value)

    def lognormal_records(self, count, median, sigma, min_len=1, plant=None) -> SequenceDB:
        tot = C.c_uint64()
        _check(_native.lib().lhmm_synth_lognormal_records(self._h, count, median, sigma, min_len,
                                                          C.byref(tot)))
        self._plant(plant)
        return self._take(count, tot.value)

    def _plant(self, plant):
        if plant is None:
            return
        hmm, fraction = plant
        s = np.ascontiguousarray(hmm.match_scores, dtype=np.float64).reshape(-1)
        _check(_native.lib().lhmm_synth_plant_motifs(self._h, s.ctypes.data_as(_native.f64p),
                                                     hmm.length, fraction))
