"""Database and profile I/O against the reference.

The native readers/writers (csrc/seqdb_io.cpp) must reproduce the
reference's ingest_fasta, pack_blocks, balance_stats, write/read_block_db
and parse/serialize_profile (src/seqdb.cpp, src/profile.cpp): same records,
same ids, byte-identical files, same statistics and the same error
messages.  Transcribes proj/tests/test_seqdb.cpp and test_profile.cpp:10-70,
then compares with the reference library (oracle/_ref) on random inputs.
Host-only: no GPU needed."""
import os

import numpy as np
import pytest

import paper_1707_09683_b200 as P
from paper_1707_09683_b200 import seqdb


def rec_db(spec, code=0):
    """[(id, len)] -> SequenceDB of constant residues (test_seqdb.cpp:20-22)."""
    db = P.SequenceDB.from_sequences([np.full(n, code, np.uint8) for _, n in spec])
    db.ids = [i for i, _ in spec]
    return db


def random_db(seed, n, lo, hi, prefix="r"):
    rng = np.random.default_rng(seed)
    lens = rng.integers(lo, hi + 1, n)
    seqs = [rng.integers(0, 21, L).astype(np.uint8) for L in lens]
    db = P.SequenceDB.from_sequences(seqs)
    db.ids = [f"{prefix}{k}" for k in range(n)]
    return db


# --- ingest_fasta (test_seqdb.cpp:29-66) -------------------------------------

def test_fasta_basics():
    db = P.ingest_fasta(">a\nACD")
    assert db.count == 1 and list(db.ids) == ["a"]
    assert db.sequence(0).tolist() == [0, 1, 2]
    assert (P.ingest_fasta(">a\nac d\n").sequence(0) == P.ingest_fasta(">a\nACD").sequence(0)).all()
    assert P.ingest_fasta(">a\nABXZ*").sequence(0).tolist() == [0, 20, 20, 20, 20]


def test_fasta_errors():
    with pytest.raises(P.DataError, match="empty FASTA input"):
        P.ingest_fasta("")
    with pytest.raises(P.DataError, match="empty FASTA input"):
        P.ingest_fasta("\n\r\n\n")
    with pytest.raises(P.DataError, match="'a'"):
        P.ingest_fasta(">a\n>b\nACD\n")
    with pytest.raises(P.DataError, match="FASTA record 'b' has an empty body"):
        P.ingest_fasta(">a\nAC\n>b\n")
    with pytest.raises(P.DataError, match="FASTA record 'seq2' has an empty body"):
        P.ingest_fasta(">a\nAC\n>\n>c\nW\n")
    with pytest.raises(P.DataError, match="FASTA body before any '>' header"):
        P.ingest_fasta("AC\n>a\nW\n")


def test_fasta_round_trip_through_serializer():
    db = random_db(4, 3, 5, 80, "rt")
    back = P.ingest_fasta(P.to_fasta(db))
    assert list(back.ids) == list(db.ids)
    assert (back.residues == db.residues).all() and (back.offsets == db.offsets).all()


def quirky_fasta(seed, nrec, big=False):
    """FASTA text with CRLF, blank lines, lowercase, inner whitespace,
    headers with descriptions, leading blanks and missing ids."""
    rng = np.random.default_rng(seed)
    letters = "ACDEFGHIKLMNPQRSTVWYacdefghiklmnpqrstvwyBXZUO*-."
    out = []
    for k in range(nrec):
        r = rng.random()
        if r < 0.05:
            hdr = ">"
        elif r < 0.1:
            hdr = ">  \tlead%d desc" % k
        else:
            hdr = ">id%d some description\twith tab" % k
        out.append(hdr + ("\r\n" if rng.random() < 0.3 else "\n"))
        n = int(rng.integers(1, 400 if big else 90))
        body = "".join(letters[i] for i in rng.integers(0, len(letters), n))
        pos = 0
        while pos < n:
            w = int(rng.integers(1, 70))
            line = body[pos:pos + w]
            if rng.random() < 0.1:
                line = line[:len(line) // 2] + " \t" + line[len(line) // 2:]
            out.append(line + ("\r\n" if rng.random() < 0.3 else "\n"))
            if rng.random() < 0.05:
                out.append("\n")
            pos += w
    return "".join(out).encode()


@pytest.mark.parametrize("seed,nrec,big", [(1, 50, False), (2, 500, False), (3, 12000, True)])
def test_fasta_matches_reference(ref, seed, nrec, big):
    text = quirky_fasta(seed, nrec, big)
    if big:
        assert len(text) > (2 << 20)  # exercises the parallel record split
    res, off, ids = ref.ingest_fasta(text)
    db = P.ingest_fasta(text)
    assert list(db.ids) == ids
    assert (db.offsets == off).all() and (db.residues == res).all()


@pytest.mark.parametrize("text", [b"", b"\n\n", b"AC\n>a\nW\n", b">a\n>b\nW\n", b">a\nW\n>b\n",
                                  b">a\nW\n>\r\n\n>c\nY\n", b">a b\nW\r\n>  \n  \n"])
def test_fasta_error_messages_match_reference(ref, text):
    with pytest.raises(RuntimeError) as want:
        ref.ingest_fasta(text)
    with pytest.raises(P.DataError) as got:
        P.ingest_fasta(text)
    assert str(got.value) == str(want.value)


def test_fasta_file(tmp_path):
    p = tmp_path / "x.fa"
    p.write_bytes(b">q1 x\nMKV\n>q2\nwy\n")
    db = P.ingest_fasta_file(str(p))
    assert list(db.ids) == ["q1", "q2"] and db.residues.tolist() == [10, 8, 17, 18, 19]
    with pytest.raises(P.DataError, match="cannot open FASTA file"):
        P.ingest_fasta_file(str(tmp_path / "missing.fa"))


# --- pack_blocks / balance_stats (test_seqdb.cpp:68-200) ---------------------

def test_pack_blocks_hand_traced_case():
    bs = P.pack_blocks(rec_db([("s0", 5), ("s1", 3), ("s2", 2)]), 1, 2)
    assert bs.block_rows.tolist() == [7]
    assert bs.column_counts.tolist() == [[1, 2]]
    cols = bs.columns(0)
    assert cols[0].tolist() == [0, 0, 0, 0, 0, 21, 22]
    assert cols[1].tolist() == [0, 0, 0, 21, 0, 0, 21]
    assert list(bs.db.ids) == ["s0", "s1", "s2"]


def test_pack_blocks_equal_lengths_zero_padding():
    bs = P.pack_blocks(rec_db([(f"e{i}", 40) for i in range(128)]), 1, 128)
    assert bs.block_rows.tolist() == [41]
    st = P.balance_stats(bs)
    assert st.prr == 0.0 and st.total_seqs == 128 and st.total_residues == 128 * 40


def test_pack_blocks_edge_cases():
    with pytest.raises(P.DataError, match="pack_blocks: no sequences to pack"):
        P.pack_blocks(P.SequenceDB.from_sequences([]), 1, 2)
    with pytest.raises(P.ContractError, match="block count must be >= 1"):
        P.pack_blocks(rec_db([("a", 4)]), 0, 2)
    with pytest.raises(P.ContractError, match="power of two"):
        P.pack_blocks(rec_db([("a", 4)]), 1, 3)
    with pytest.raises(P.DataError, match="pack_blocks: sequence 'b' is empty"):
        P.pack_blocks(rec_db([("a", 4), ("b", 0)]), 1, 2)
    bs = P.pack_blocks(rec_db([("a", 4)]), 1, 128)
    assert bs.block_rows.tolist() == [5]
    assert int((bs.column_counts > 0).sum()) == 1
    assert bs.columns(0)[100].tolist() == [22] * 5


def test_balance_stats_hand_cases():
    st = P.balance_stats(P.pack_blocks(rec_db([("a", 6), ("b", 8)]), 2, 1))
    assert (st.avg_m, st.sd_m, st.avg_endings, st.sd_endings, st.prr) == (8.0, 1.0, 1.0, 0.0, 0.0)
    assert (st.total_seqs, st.total_residues) == (2, 14)
    st = P.balance_stats(P.pack_blocks(rec_db([(f"z{i}", 25) for i in range(8)]), 4, 2))
    assert st.sd_m == 0.0 and st.sd_endings == 0.0


def test_packer_balance_lognormal_regime():
    """test_seqdb.cpp:288-300: sd(M)/avg(M) <= 1% and PRR <= 1e-3."""
    db = P.Rng(16).lognormal_records(100000, 200.0, 0.25)
    st = P.balance_stats(P.pack_blocks(db, 24, 32))
    assert st.sd_m / st.avg_m <= 0.01 and st.prr <= 1e-3


@pytest.mark.parametrize("n,blocks,lanes", [(3, 1, 2), (64, 2, 16), (200, 2, 32), (40, 8, 128),
                                            (500, 4, 32), (7, 5, 4), (1000, 3, 1)])
def test_pack_write_byte_identical_to_reference(ref, tmp_path, n, blocks, lanes):
    db = random_db(100 + n, n, 1, 120)
    want_path, got_path = str(tmp_path / "ref.lhmm"), str(tmp_path / "b200.lhmm")
    want_stats = ref.pack_write(db.residues, db.offsets, list(db.ids), blocks, lanes, want_path)
    bs = P.pack_blocks(db, blocks, lanes)
    P.write_block_db(bs, got_path)
    assert open(got_path, "rb").read() == open(want_path, "rb").read()
    st = P.balance_stats(bs)
    assert (st.avg_m, st.sd_m, st.avg_endings, st.sd_endings, st.prr,
            float(st.total_seqs), float(st.total_residues)) == want_stats


def test_read_reference_file_matches_reconstruct(ref, tmp_path):
    db = random_db(7, 777, 1, 300)
    path = str(tmp_path / "db.lhmm")
    ref.pack_write(db.residues, db.offsets, list(db.ids), 6, 32, path)
    res, off, ids, stats = ref.read_block_db(path)
    bs = P.read_block_db(path)
    assert list(bs.db.ids) == ids
    assert (bs.db.offsets == off).all() and (bs.db.residues == res).all()
    st = P.balance_stats(bs)
    assert (st.avg_m, st.sd_m, st.avg_endings, st.sd_endings, st.prr,
            float(st.total_seqs), float(st.total_residues)) == stats


def test_block_db_round_trip_byte_exact(tmp_path):
    bs = P.pack_blocks(random_db(14, 64, 1, 90, "db"), 2, 16)
    p1, p2 = str(tmp_path / "a.lhmm"), str(tmp_path / "b.lhmm")
    P.write_block_db(bs, p1)
    back = P.read_block_db(p1)
    assert back.lanes == bs.lanes and (back.block_rows == bs.block_rows).all()
    assert (back.column_counts == bs.column_counts).all() and list(back.db.ids) == list(bs.db.ids)
    P.write_block_db(back, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()


def test_empty_block_set_round_trips(tmp_path):
    bs = seqdb.BlockSet(32, np.zeros(0, np.uint64), np.zeros((0, 32), np.uint32),
                        P.SequenceDB.from_sequences([]))
    p = str(tmp_path / "e.lhmm")
    P.write_block_db(bs, p)
    back = P.read_block_db(p)
    assert back.lanes == 32 and back.block_count == 0 and back.db.count == 0


def _ref_error(ref, path):
    with pytest.raises(RuntimeError) as e:
        ref.read_block_db(path)
    return str(e.value)


def test_corrupted_payload_names_block(ref, tmp_path):
    bs = P.pack_blocks(random_db(15, 40, 1, 60, "crc"), 2, 8)
    p = str(tmp_path / "c.lhmm")
    P.write_block_db(bs, p)
    data = bytearray(open(p, "rb").read())
    pos = len(data) - int(bs.block_rows[1]) * 4
    data[pos] ^= 0x7
    open(p, "wb").write(bytes(data))
    with pytest.raises(P.DataError, match="checksum failure in block 1"):
        P.read_block_db(p)
    assert _ref_error(ref, p) == "checksum failure in block 1"


def test_bad_magic_version_truncation(ref, tmp_path):
    p = str(tmp_path / "bad.lhmm")
    open(p, "wb").write(b"NOPE" + b"x" * 19)
    with pytest.raises(P.DataError, match="magic"):
        P.read_block_db(p)
    open(p, "wb").write(b"LHMM" + (9).to_bytes(2, "little") + b"\0" * 20)
    with pytest.raises(P.DataError, match="unsupported block database version 9"):
        P.read_block_db(p)
    open(p, "wb").write(b"LHMM")
    with pytest.raises(P.DataError, match="truncated"):
        P.read_block_db(p)
    with pytest.raises(P.DataError, match="cannot open block database"):
        P.read_block_db(str(tmp_path / "missing.lhmm"))


def test_every_truncation_point_matches_reference(ref, tmp_path):
    bs = P.pack_blocks(random_db(21, 12, 1, 9, "t"), 2, 4)
    full = str(tmp_path / "full.lhmm")
    P.write_block_db(bs, full)
    data = open(full, "rb").read()
    p = str(tmp_path / "cut.lhmm")
    for cut in range(len(data)):
        open(p, "wb").write(data[:cut])
        want = _ref_error(ref, p)
        with pytest.raises(P.DataError) as got:
            P.read_block_db(p)
        assert str(got.value) == want, cut


def test_structural_column_errors(tmp_path):
    """A set that reads is scannable: columns must be (seq '@')* '#'*, with
    the engine's messages (src/engine.cpp:404-440)."""
    import struct
    import zlib

    def file_with(cols, meta, rows):
        body = struct.pack("<QI", rows, len(cols))
        for m in meta:
            body += struct.pack("<I", len(m))
            for sid, L in m:
                body += struct.pack("<I", len(sid)) + sid.encode() + struct.pack("<Q", L)
        pay = b"".join(bytes(c) for c in cols)
        body += pay + struct.pack("<I", zlib.crc32(pay))
        head = b"LHMM" + struct.pack("<HHIQ", 1, 0, len(cols), 1) + struct.pack("<Q", 28)
        return head + body

    cases = [
        ([[0, 21, 22, 0]], [[("a", 1)]], "block 0 column 0: residues after padding"),
        ([[0, 22, 21, 22]], [[("a", 1)]], "block 0 column 0: ending byte after padding"),
        ([[0, 21, 1, 21]], [[("a", 1)]], "block 0 column 0: more sequences than metadata entries"),
        ([[0, 0, 21, 22]], [[("a", 1)]], "block 0 column 0: sequence length does not match metadata"),
        ([[0, 21, 0, 0]], [[("a", 1)]], "block 0 column 0: column ended with an unterminated sequence"),
        ([[0, 21, 22, 22]], [[("a", 1), ("b", 1)]],
         "block 0 column 0: column ended with an unterminated sequence"),
        ([[0, 30, 21, 22]], [[("a", 2)]], "block 0 column 0: invalid residue code 30"),
    ]
    p = str(tmp_path / "s.lhmm")
    for cols, meta, msg in cases:
        open(p, "wb").write(file_with(cols, meta, 4))
        with pytest.raises(P.DataError) as e:
            P.read_block_db(p)
        assert str(e.value) == msg
    # a well-formed two-column file reads back its sequences
    open(p, "wb").write(file_with([[0, 21, 1, 21], [22] * 4], [[("a", 1), ("b", 1)], []], 4))
    bs = P.read_block_db(p)
    assert list(bs.db.ids) == ["a", "b"] and bs.db.residues.tolist() == [0, 1]
    assert bs.column_counts.tolist() == [[2, 0]]


def test_invalid_lane_count(tmp_path):
    import struct
    p = str(tmp_path / "l.lhmm")
    open(p, "wb").write(b"LHMM" + struct.pack("<HHIQ", 1, 0, 3, 0))
    with pytest.raises(P.DataError, match="block database has invalid lane count"):
        P.read_block_db(p)


def test_layout_contract(tmp_path):
    db = rec_db([("a", 3), ("b", 2)])
    bs = seqdb.BlockSet(2, np.array([3], np.uint64), np.array([[1, 1]], np.uint32), db)
    with pytest.raises(P.ContractError, match="column longer than the block rows"):
        P.write_block_db(bs, str(tmp_path / "x.lhmm"))
    bs = seqdb.BlockSet(2, np.array([4], np.uint64), np.array([[1, 0]], np.uint32), db)
    with pytest.raises(P.ContractError, match="does not cover every sequence"):
        P.write_block_db(bs, str(tmp_path / "x.lhmm"))


# --- profile text (test_profile.cpp:12-70; docs/formats.md) -------------------

def one_node_profile():
    return "NAME t1\nLENG 1\nSTATS 0.7 2.0\n1" + " 0.0" * 20 + "\n//\n"


def test_parse_one_node_profile():
    h = P.parse_profile(one_node_profile())
    assert h.name == "t1" and h.length == 1 and h.lambda_ == 0.7 and h.tau == 2.0
    assert (h.match_scores == 0.0).all()


def _rows(n, val="1.5"):
    return "".join(f"{j}" + f" {val}" * 20 + "\n" for j in range(1, n + 1))


BAD_PROFILES = [
    "NAME x\nLENG 3\nSTATS 0.7 2\n" + _rows(2) + "//\n",
    "LENG 1\n//\n",
    "NAME x\nLENG 0\nSTATS 0.7 2\n//\n",
    "NAME x\nLENG 1\nSTATS 0.7 2\n1" + " 0.5" * 19 + " oops\n//\n",
    "NAME x y\nLENG 1\n",
    "NAME x\nLENG -1\n",
    "NAME x\nLENG 1 2\n",
    "NAME x\nLENG 1\nSTATS 0 2\n",
    "NAME x\nLENG 1\nSTATS nan 2\n",
    "NAME x\nLENG 1\nSTATS 0.7\n",
    "NAME x\nLENG 1\nSTATS 0.7 2x\n",
    "NAME x\n" + _rows(1) + "LENG 1\n",
    "NAME x\nLENG 1\nSTATS 0.7 2\n1 1 2\n//\n",
    "NAME x\nLENG 2\nSTATS 0.7 2\n2" + " 0" * 20 + "\n//\n",
    "NAME x\nLENG 1\nSTATS 0.7 2\n" + _rows(2) + "//\n",
    "NAME x\nLENG 1\nSTATS 0.7 2\n1" + " inf" * 20 + "\n//\n",
    "NAME x\nLENG 1\nSTATS 0.7 2\n1" + " 1e999" * 20 + "\n//\n",
    "NAME x\nLENG 1\nSTATS 0.7 2\n+1" + " 0" * 20 + "\n//\n",
    "NAME x\nLENG 1\nSTATS 0.7 2\n" + _rows(1),
    "LENG 1\nSTATS 0.7 2\n" + _rows(1) + "//\n",
    "NAME x\nSTATS 0.7 2\n//\n",
    "NAME x\nLENG 1\n" + _rows(1) + "//\n",
    "",
    "NAME x\r\nLENG 1\r\nSTATS 0.7 2\r\n" + _rows(1).replace("\n", "\r\n") + "//\r\n",
    "\n\n  NAME   x  \nLENG 1\n\tSTATS 0.7 -3.5\n" + _rows(1, "-0.25") + "  //  trailing\nignored\n",
    "NAME x\nLENG 1\nSTATS 0x1p-1 2\n1" + " 1e-3" * 20 + "\n//\n",
]


@pytest.mark.parametrize("k", range(len(BAD_PROFILES)))
def test_profile_parse_matches_reference(ref, k):
    text = BAD_PROFILES[k].encode()
    try:
        want = ref.parse_profile(text)
    except RuntimeError as e:
        with pytest.raises(P.ParseError) as got:
            P.parse_profile(text)
        assert str(got.value) == str(e)
        return
    h = P.parse_profile(text)
    name, m, scores, lam, tau = want
    assert (h.name, h.length, h.lambda_, h.tau) == (name, m, lam, tau)
    assert (h.match_scores == scores).all()


def test_profile_round_trip_and_serializer_matches_reference(ref):
    for m in (1, 45, 400):
        hmm = P.Rng(45 + m).random_profile(m)
        text = P.serialize_profile(hmm)
        assert text == ref.serialize_profile(hmm.name, hmm.match_scores, hmm.lambda_, hmm.tau)
        back = P.parse_profile(text)
        assert back.name == hmm.name and back.length == m
        assert back.lambda_ == hmm.lambda_ and back.tau == hmm.tau
        assert (back.match_scores == hmm.match_scores).all()


def test_profile_file(tmp_path):
    p = tmp_path / "p.txt"
    p.write_text(one_node_profile())
    assert P.read_profile_file(str(p)).name == "t1"


# --- scanning a block database (GPU) -----------------------------------------

@pytest.mark.gpu
def test_block_db_scan_in_reference_hit_order(ora, tmp_path):
    """LHMM file -> native reader -> device scan: scores in (block, column,
    ordinal) order equal the oracle's on the same sequences, and follow the
    ids back to the original records."""
    import oracle
    rng = P.Rng(0x1BD)
    hmm = rng.random_profile(150)
    db = rng.random_records(4000, 20, 500, plant=(hmm, 0.05))
    db.ids = [f"q{k}" for k in range(db.count)]
    path = str(tmp_path / "scan.lhmm")
    P.write_block_db(P.pack_blocks(db, 8, 32), path)
    back = P.read_block_db(path)
    pos = {i: k for k, i in enumerate(db.ids)}
    order = np.array([pos[i] for i in back.db.ids])
    qp = P.QuantParams(3.0, 120, 3, 20, 20)
    costs = P.quantize_emissions(hmm, qp)
    oq = oracle.QuantParams(qp.scale, qp.base, qp.dbias, qp.tec, qp.tjb)
    with P.Scanner(0) as s:
        s.set_profile(costs, qp, hmm.lambda_, hmm.tau)
        s.set_database(back.db)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            got = s.scan(P.ScanOptions(alg=alg)).raw
            want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq)
            assert (got == want[order]).all()
