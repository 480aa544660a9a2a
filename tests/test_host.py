"""Host-side logic of the B200 build, checked on CPU (no GPU calls): the C ABI
exports, the seeded generators, byte-space helpers, the pass-decision
tables, the shard plan and the geometry policy."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_1707_09683_b200 as P
from paper_1707_09683_b200 import _native
from paper_1707_09683_b200.shard import shard_plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def oq(q):
    return oracle.QuantParams(q.scale, q.base, q.dbias, q.tec, q.tjb)


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "lhmm_b200.h")).read()
    names = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(lhmm_[a-z_0-9]+)\s*\(", hdr,
                           re.M))
    assert len(names) >= 30
    L = C.CDLL(_native.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(_native.SIGNATURES) == names


def test_synth_matches_reference_golden():
    """The product generators reproduce the reference synth:: streams (the
    golden file records the reference's residue / cost checksums)."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_golden.json")))
    for case in g["cases"]:
        rng = P.Rng(case["seed"])
        hmm = rng.random_profile(case["m"])
        plant = (hmm, case["plant"]) if case["plant"] else None
        if case["gen"] == "uniform":
            db = rng.random_records(case["count"], case["lo"], case["hi"], plant=plant)
        else:
            db = rng.lognormal_records(case["count"], case["median"], case["sigma"], 2, plant=plant)
        assert int(db.residues.astype(np.uint64).sum()) == case["residue_sum"]
        c = P.quantize_emissions(hmm, P.QuantParams(*case["quant"]))
        assert int(c.bytes.astype(np.uint64).sum()) == case["cost_sum"]


def test_synth_matches_reference_library(ref):
    for seed in (1, 99):
        g = ref.rng(seed)
        s, lam, tau = g.random_profile(123)
        res, off = g.random_records(300, 1, 500, plant=(s, 0.3))
        r2, o2 = g.lognormal_records(2000, 290, 0.65, 2)
        mine = P.Rng(seed)
        h = mine.random_profile(123)
        db = mine.random_records(300, 1, 500, plant=(h, 0.3))
        db2 = mine.lognormal_records(2000, 290, 0.65, 2)
        np.testing.assert_array_equal(h.match_scores.reshape(-1), s)
        assert (h.lambda_, h.tau) == (lam, tau)
        np.testing.assert_array_equal(db.residues, res)
        np.testing.assert_array_equal(db.offsets, off)
        np.testing.assert_array_equal(db2.residues, r2)
        np.testing.assert_array_equal(db2.offsets, o2)
        assert mine.next() == g.next()


def test_quantize_and_helpers_match_oracle(ora):
    rng = P.Rng(4)
    for q in (P.QuantParams(), P.QuantParams(2.0, 240, 10, 1, 5), P.QuantParams(0.7, 10, 0, 0, 0)):
        hmm = rng.random_profile(300)
        np.testing.assert_array_equal(P.quantize_emissions(hmm, q).bytes,
                                      ora.quantize(hmm.match_scores.reshape(-1), oq(q)))
        for n in list(range(0, 2000, 7)) + [35000, 10**6]:
            assert P.move_cost(n, q) == ora.move_cost(n, oq(q))
            assert P.engine_sequence_base(n, q) == ora.sequence_base(n, oq(q))
        for raw in range(0, 256, 17):
            for n in (0, 1, 290, 40000):
                for alg in (0, 1):
                    h = P.finalize_hit(raw, n, 0.69, 2.0, q, alg)
                    assert (h.bits, h.p_value, h.overflow) == ora.finalize(raw, n, 0.69, 2.0,
                                                                           oq(q), alg)


def test_quant_errors():
    with pytest.raises(P.ContractError):
        P.quantize_emissions(P.ProfileHMM("x", 1, np.zeros((1, 20))), P.QuantParams(scale=0.0))
    with pytest.raises(P.ContractError):
        P.quantize_emissions(P.ProfileHMM("x", 1, np.zeros((1, 20))),
                             P.QuantParams(base=254, dbias=4))


def length_tables(q, lam, tau, alg, t, max_len):
    base = np.zeros(max_len + 1, np.uint8)
    rawmin = np.zeros(max_len + 1, np.uint8)
    qc = q.c()
    rc = _native.lib().lhmm_length_tables(C.byref(qc), lam, tau, alg, t, max_len,
                                          base.ctypes.data_as(_native.u8p),
                                          rawmin.ctypes.data_as(_native.u8p))
    return rc, base, rawmin


@pytest.mark.parametrize("alg", [0, 1])
def test_pass_table_equals_finalize_rule(ora, alg):
    """Device pass bit raw==255 || raw>=rawmin[len] == (p <= t || overflow)
    for every raw byte (SURVEY §7 hard part 2)."""
    for q in (P.QuantParams(), P.QuantParams(3.0, 120, 3, 20, 20)):
        for lam, tau in ((0.69, 2.0), (0.3, -1.0), (1.2, 5.0)):
            for t in (0.0, 0.022, 0.103, 0.3, 0.458, 1.0):
                rc, base, rawmin = length_tables(q, lam, tau, alg, t, 3000)
                assert rc == 0
                for n in list(range(0, 3001, 97)) + [1, 2, 3]:
                    assert base[n] == ora.sequence_base(n, oq(q))
                    for raw in range(256):
                        want = ora.passes(raw, n, lam, tau, oq(q), alg, t)
                        assert (raw == 255 or raw >= rawmin[n]) == want, (n, raw, t)


def test_pass_table_rejects_bad_threshold():
    rc, _, _ = length_tables(P.QuantParams(), 0.69, 2.0, 0, 1.5, 10)
    assert rc == 1


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_partitions_by_residue_count(world):
    db = P.Rng(8).lognormal_records(20000, 290, 0.65, 2)
    lens = np.diff(db.offsets).astype(np.int64)
    parts = [shard_plan(db.offsets, r, world) for r in range(world)]
    allidx = np.concatenate(parts)
    assert np.array_equal(np.sort(allidx), np.arange(db.count))
    loads = np.array([lens[p.astype(np.int64)].sum() for p in parts])
    assert loads.max() / loads.mean() < 1.02
    for p in parts:
        assert np.all(np.diff(p.astype(np.int64)) > 0)


def test_geometry_policy_covers_every_model_length():
    for alg in (0, 1):
        for variant in (P.Variant.Dpx16, P.Variant.Fp16, P.Variant.Swar8):
            cpw = 4 if variant == P.Variant.Swar8 else 2
            for m in list(range(1, 300)) + list(range(300, 2406, 37)) + [2405]:
                L, H = P.select_geometry(m, alg, variant)
                assert cpw * L * H >= m
                assert L in (1, 2, 4, 8, 16, 32)


def test_reference_geometry_points():
    assert P.select_geometry(48, 1, P.Variant.Dpx16) == (1, 24)
    L, H = P.select_geometry(2405, 0, P.Variant.Dpx16)
    assert 2 * L * H >= 2405
