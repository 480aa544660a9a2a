"""Property-based checks (hypothesis) of the host-side pieces against the
reference library: Algorithm 1 packing, balance statistics, LHMM files and
FASTA on generated inputs, and the shard plan's invariants.  Host-only."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_1707_09683_b200 as P

SET = settings(max_examples=60, deadline=None,
               suppress_health_check=[HealthCheck.function_scoped_fixture])

lengths = st.lists(st.integers(min_value=1, max_value=60), min_size=1, max_size=120)


def make_db(lens, seed):
    rng = np.random.default_rng(seed)
    db = P.SequenceDB.from_sequences([rng.integers(0, 21, n).astype(np.uint8) for n in lens])
    db.ids = [f"p{k}_{n}" for k, n in enumerate(lens)]
    return db


@SET
@given(lens=lengths, blocks=st.integers(1, 6), lanes=st.sampled_from([1, 2, 4, 8, 32, 128]),
       seed=st.integers(0, 2**31))
def test_pack_write_equals_reference(ref, tmp_path_factory, lens, blocks, lanes, seed):
    """pack_blocks + write_block_db: byte-identical to the reference for any
    length multiset, block count and lane count; balance_stats identical."""
    db = make_db(lens, seed)
    d = tmp_path_factory.mktemp("pk")
    want_stats = ref.pack_write(db.residues, db.offsets, list(db.ids), blocks, lanes,
                                str(d / "ref.lhmm"))
    bs = P.pack_blocks(db, blocks, lanes)
    P.write_block_db(bs, str(d / "b200.lhmm"))
    assert open(d / "b200.lhmm", "rb").read() == open(d / "ref.lhmm", "rb").read()
    s = P.balance_stats(bs)
    assert (s.avg_m, s.sd_m, s.avg_endings, s.sd_endings, s.prr, float(s.total_seqs),
            float(s.total_residues)) == want_stats
    # conservation: every record once, in (block, column, ordinal) order
    assert sorted(bs.db.ids) == sorted(db.ids)
    assert bs.db.total_residues() == db.total_residues()
    back = P.read_block_db(str(d / "b200.lhmm"))
    assert list(back.db.ids) == list(bs.db.ids)
    assert (back.db.residues == bs.db.residues).all()


letters = st.text(alphabet="ACDEFGHIKLMNPQRSTVWYacdxz*BXZ -", min_size=0, max_size=80)


@SET
@given(recs=st.lists(st.tuples(st.text(alphabet="abcXYZ019_.|", min_size=0, max_size=8),
                                st.lists(letters, min_size=0, max_size=4)),
                      min_size=0, max_size=25),
       crlf=st.booleans(), blank=st.booleans())
def test_fasta_equals_reference(ref, recs, crlf, blank):
    """ingest_fasta on generated texts (empty ids, empty bodies, odd letters,
    CRLF, blank lines): same records and ids, or the same error."""
    nl = "\r\n" if crlf else "\n"
    out = []
    for rid, lines in recs:
        out.append(">" + rid + nl)
        for line in lines:
            out.append(line + nl)
            if blank:
                out.append(nl)
    text = "".join(out).encode()
    try:
        want = ref.ingest_fasta(text)
    except RuntimeError as e:
        with pytest.raises(P.DataError) as got:
            P.ingest_fasta(text)
        assert str(got.value) == str(e)
        return
    db = P.ingest_fasta(text)
    res, off, ids = want
    assert list(db.ids) == ids
    assert (db.offsets == off).all() and (db.residues == res).all()


@SET
@given(lens=st.lists(st.integers(0, 3000), min_size=1, max_size=400),
       world=st.integers(1, 8))
def test_shard_plan_invariants(lens, world):
    """Every sequence is owned by exactly one shard; shards are balanced by
    residue count within one tile's worth of the mean."""
    import ctypes as C
    from paper_1707_09683_b200 import _native
    off = np.zeros(len(lens) + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    owned = []
    loads = []
    for r in range(world):
        n = C.c_uint64()
        lib = _native.lib()
        assert lib.lhmm_shard_plan(off.ctypes.data_as(_native.u64p), len(lens), r, world,
                                   None, C.byref(n)) == 0
        out = np.zeros(max(n.value, 1), np.uint64)
        assert lib.lhmm_shard_plan(off.ctypes.data_as(_native.u64p), len(lens), r, world,
                                   out.ctypes.data_as(_native.u64p), C.byref(n)) == 0
        idx = out[:n.value]
        assert (np.diff(idx.astype(np.int64)) > 0).all()
        owned.extend(idx.tolist())
        loads.append(int(np.asarray(lens)[idx.astype(np.int64)].sum()) if n.value else 0)
    assert sorted(owned) == list(range(len(lens)))
    tile_max = max(lens) * 32
    assert max(loads) - min(loads) <= tile_max


@SET
@given(m=st.integers(1, 30), scores=st.data())
def test_profile_text_round_trip_equals_reference(ref, m, scores):
    vals = scores.draw(st.lists(st.floats(-50, 50, allow_nan=False, allow_infinity=False),
                                min_size=m * 20, max_size=m * 20))
    hmm = P.ProfileHMM("h" + str(m), m, np.array(vals).reshape(m, 20), 0.5 + m / 10, -m / 3)
    text = P.serialize_profile(hmm)
    assert text == ref.serialize_profile(hmm.name, hmm.match_scores, hmm.lambda_, hmm.tau)
    try:
        ref.parse_profile(text.encode())
    except RuntimeError as e:
        # e.g. a subnormal score: std::stod reports ERANGE, so the reference
        # rejects its own serialization -- the parser must agree
        with pytest.raises(P.ParseError) as got:
            P.parse_profile(text)
        assert str(got.value) == str(e)
        return
    back = P.parse_profile(text)
    assert (back.match_scores == hmm.match_scores).all()
    assert (back.lambda_, back.tau, back.length) == (hmm.lambda_, hmm.tau, m)
