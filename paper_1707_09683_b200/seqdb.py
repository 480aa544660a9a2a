"""Mirror of the reference's sequence-database and profile-text I/O
(include/lanehmm/seqdb.hpp, profile.hpp) over the native C ABI
(csrc/seqdb_io.cpp).  Names, argument meaning and error types follow the
reference:

  ingest_fasta / ingest_fasta_file / to_fasta     src/seqdb.cpp:35-98
  pack_blocks (Algorithm 1)                       src/seqdb.cpp:109-188
  balance_stats                                   src/seqdb.cpp:190-227
  write_block_db / read_block_db                  src/seqdb.cpp:252-385
  parse_profile / serialize_profile               src/profile.cpp:49-142

A ``BlockSet`` here is a ``SequenceDB`` in (block, column, ordinal) order plus
its block layout -- the information the reference's BlockSet carries minus
the '@'/'#' bytes, which are implied (the native reader verifies every column
is exactly (sequence '@')* '#'*).  Scanning it with ``Scanner.set_database``
yields scores in the reference's hit order.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .lanehmm import AMINO, ProfileHMM, SequenceDB, _check


class IdTable:
    """Sequence ids as one byte blob + offsets (list-like, str items)."""

    def __init__(self, blob: bytes, offsets: np.ndarray):
        self.blob = blob
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)

    def __len__(self):
        return self.offsets.size - 1

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        return self.blob[int(self.offsets[k]):int(self.offsets[k + 1])].decode("latin-1")

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    def __eq__(self, other):
        return list(self) == list(other)

    @staticmethod
    def from_list(ids):
        enc = [i.encode("latin-1") for i in ids]
        off = np.zeros(len(enc) + 1, np.uint64)
        off[1:] = np.cumsum([len(e) for e in enc]) if enc else []
        return IdTable(b"".join(enc), off)


@dataclass
class BlockSet:
    """Sequences in (block, column, ordinal) order + block layout
    (seqdb.hpp:25-53)."""
    lanes: int
    block_rows: np.ndarray     # uint64 [blocks]
    column_counts: np.ndarray  # uint32 [blocks, lanes]
    db: SequenceDB

    @property
    def block_count(self):
        return int(self.block_rows.size)

    def container_width(self):
        return 128 // self.lanes

    def total_sequences(self):
        return self.db.count

    def total_residues(self):
        return self.db.total_residues()

    def columns(self, b):
        """Block b's container columns as the reference stores them:
        sequences each followed by '@' (21), padded with '#' (22) to rows."""
        rows = int(self.block_rows[b])
        first = int(self.column_counts[:b].sum())
        out = []
        for c in range(self.lanes):
            col = np.full(rows, 22, np.uint8)
            pos = 0
            for _ in range(int(self.column_counts[b, c])):
                s = self.db.sequence(first)
                col[pos:pos + s.size] = s
                col[pos + s.size] = 21
                pos += s.size + 1
                first += 1
            out.append(col)
        return out


@dataclass
class BalanceStats:
    avg_m: float
    sd_m: float
    avg_endings: float
    sd_endings: float
    prr: float
    total_seqs: int
    total_residues: int


class _SeqSet:
    """Owns a native lhmm_seqset handle."""

    def __init__(self, h=None):
        self.h = h if h is not None else C.c_void_p()

    def __del__(self):
        try:
            if self.h:
                _native.lib().lhmm_seqset_destroy(self.h)
        except Exception:
            pass

    @staticmethod
    def from_db(db: SequenceDB):
        s = _SeqSet()
        res = db.residues if db.residues.size else np.zeros(1, np.uint8)
        ids = db.ids
        if ids is not None and not isinstance(ids, IdTable):
            ids = IdTable.from_list(list(ids))
        if ids is not None:
            blob = ids.blob if ids.blob else b"\0"
            _check(_native.lib().lhmm_seqset_create(
                res.ctypes.data_as(_native.u8p), db.offsets.ctypes.data_as(_native.u64p),
                db.count, blob, ids.offsets.ctypes.data_as(_native.u64p), C.byref(s.h)))
        else:
            _check(_native.lib().lhmm_seqset_create(
                res.ctypes.data_as(_native.u8p), db.offsets.ctypes.data_as(_native.u64p),
                db.count, None, None, C.byref(s.h)))
        return s

    def to_db(self) -> SequenceDB:
        n, nr = C.c_uint64(), C.c_uint64()
        rp, op, ip, iop = _native.u8p(), _native.u64p(), C.c_void_p(), _native.u64p()
        _check(_native.lib().lhmm_seqset_view(self.h, C.byref(n), C.byref(nr), C.byref(rp),
                                              C.byref(op), C.byref(ip), C.byref(iop)))
        n, nr = n.value, nr.value
        off = np.ctypeslib.as_array(op, shape=(n + 1,)).copy()
        res = np.ctypeslib.as_array(rp, shape=(nr,)).copy() if nr else np.zeros(0, np.uint8)
        ioff = np.ctypeslib.as_array(iop, shape=(n + 1,)).copy()
        blob = C.string_at(ip, int(ioff[-1])) if int(ioff[-1]) else b""
        return SequenceDB(res, off, IdTable(blob, ioff))

    def to_blockset(self) -> BlockSet:
        lanes, nb = C.c_uint32(), C.c_uint64()
        rows_p, cc_p = _native.u64p(), _native.u32p()
        _check(_native.lib().lhmm_seqset_layout(self.h, C.byref(lanes), C.byref(nb),
                                                C.byref(rows_p), C.byref(cc_p)))
        L, B = lanes.value, nb.value
        rows = np.ctypeslib.as_array(rows_p, shape=(B,)).copy() if B else np.zeros(0, np.uint64)
        cc = (np.ctypeslib.as_array(cc_p, shape=(B * L,)).copy() if B
              else np.zeros(0, np.uint32)).reshape(B, L)
        return BlockSet(L, rows, cc, self.to_db())

    @staticmethod
    def from_blockset(bs: BlockSet):
        s = _SeqSet.from_db(bs.db)
        rows = np.ascontiguousarray(bs.block_rows, dtype=np.uint64)
        cc = np.ascontiguousarray(bs.column_counts, dtype=np.uint32).reshape(-1)
        _check(_native.lib().lhmm_seqset_set_layout(
            s.h, bs.lanes, rows.size, rows.ctypes.data_as(_native.u64p),
            cc.ctypes.data_as(_native.u32p)))
        return s


# ---------------------------------------------------------------------------
# FASTA

def ingest_fasta(text) -> SequenceDB:
    """seqdb.cpp:35-76: records with ids; DataError on malformed input."""
    b = text.encode("latin-1") if isinstance(text, str) else bytes(text)
    s = _SeqSet()
    _check(_native.lib().lhmm_ingest_fasta(b, len(b), C.byref(s.h)))
    return s.to_db()


def ingest_fasta_file(path) -> SequenceDB:
    s = _SeqSet()
    _check(_native.lib().lhmm_ingest_fasta_file(os.fsencode(path), C.byref(s.h)))
    return s.to_db()


def to_fasta(db: SequenceDB) -> str:
    """seqdb.cpp:85-98: 60 residues per line."""
    letters = np.frombuffer((AMINO + "X@#").encode() + b"X" * 233, dtype=np.uint8)
    ids = db.ids if db.ids is not None else [f"s{k}" for k in range(db.count)]
    out = []
    for k in range(db.count):
        seq = letters[np.minimum(db.sequence(k), 255)].tobytes().decode()
        # decode_residue: 0..19 letters, 21 '@', 22 '#', else 'X'
        out.append(f">{ids[k]}\n")
        out.extend(seq[i:i + 60] + "\n" for i in range(0, len(seq), 60))
    return "".join(out)


# ---------------------------------------------------------------------------
# block database

def pack_blocks(db: SequenceDB, block_count: int, lanes: int) -> BlockSet:
    """Algorithm 1 (seqdb.cpp:109-188)."""
    src = _SeqSet.from_db(db)
    out = _SeqSet()
    _check(_native.lib().lhmm_pack_blocks(src.h, int(block_count), int(lanes), C.byref(out.h)))
    return out.to_blockset()


def balance_stats(bs: BlockSet) -> BalanceStats:
    s = _SeqSet.from_blockset(bs)
    st = _native.BalanceC()
    _check(_native.lib().lhmm_balance_stats(s.h, C.byref(st)))
    return BalanceStats(st.avg_m, st.sd_m, st.avg_endings, st.sd_endings, st.prr,
                        st.total_seqs, st.total_residues)


def write_block_db(bs: BlockSet, path) -> None:
    s = _SeqSet.from_blockset(bs)
    _check(_native.lib().lhmm_write_block_db(s.h, os.fsencode(path)))


def read_block_db(path) -> BlockSet:
    s = _SeqSet()
    _check(_native.lib().lhmm_read_block_db(os.fsencode(path), C.byref(s.h)))
    return s.to_blockset()


# ---------------------------------------------------------------------------
# profile text

def parse_profile(text) -> ProfileHMM:
    """profile.cpp:49-123; ParseError("line N: ...") on malformed text."""
    b = text.encode("latin-1") if isinstance(text, str) else bytes(text)
    m, lam, tau = C.c_uint32(), C.c_double(), C.c_double()
    _check(_native.lib().lhmm_parse_profile(b, len(b), C.byref(m), None, None, None, 0, None, 0))
    scores = np.zeros(max(m.value, 1) * 20, np.float64)
    name = C.create_string_buffer(len(b) + 1)
    _check(_native.lib().lhmm_parse_profile(b, len(b), C.byref(m), C.byref(lam), C.byref(tau),
                                            scores.ctypes.data_as(_native.f64p), scores.size,
                                            name, len(b) + 1))
    return ProfileHMM(name.value.decode("latin-1"), m.value,
                      scores[:m.value * 20].reshape(m.value, 20), lam.value, tau.value)


def read_profile_file(path) -> ProfileHMM:
    with open(path, "rb") as f:
        return parse_profile(f.read())


def serialize_profile(hmm: ProfileHMM) -> str:
    s = np.ascontiguousarray(hmm.match_scores, dtype=np.float64).reshape(-1)
    need = C.c_size_t()
    name = hmm.name.encode("latin-1")
    _check(_native.lib().lhmm_serialize_profile(name, hmm.length, s.ctypes.data_as(_native.f64p),
                                                hmm.lambda_, hmm.tau, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value + 1)
    _check(_native.lib().lhmm_serialize_profile(name, hmm.length, s.ctypes.data_as(_native.f64p),
                                                hmm.lambda_, hmm.tau, buf, need.value + 1,
                                                C.byref(need)))
    return buf.raw[:need.value].decode("latin-1")
