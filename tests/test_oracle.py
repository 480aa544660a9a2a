"""Pins the CPU oracle (oracle/oracle.c) before it is trusted as the checker:
the reference's known-answer tests (proj/tests/test_oracle.cpp:22-128,
test_profile.cpp:75-129, test_engine.cpp:280-335), an exhaustive path
enumeration for tiny shapes (brute_force.hpp:31-99), the golden vectors the
reference produced (tests/golden/), and -- where oracle/_ref is built -- the
reference library itself on random instances."""
import json
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "oracle_golden.json")
Q = oracle.QuantParams


def direct_costs(m, fill):
    return np.full(m * 21, fill, dtype=np.uint8)


# --- test_oracle.cpp:22-65 hand cases ---------------------------------------

def test_empty_sequence_scores_floor(ora):
    c = direct_costs(4, 3)
    assert ora.msv(c, [], Q()) == 0
    assert ora.ssv(c, [], Q()) == 0x80


def test_one_node_one_residue(ora):
    c = direct_costs(1, 3)
    assert ora.msv(c, [0], Q()) == 194
    assert ora.msv(direct_costs(1, 197), [0], Q()) == 0


def test_ssv_two_step_diagonal(ora):
    c = direct_costs(2, 0xFF)
    c[0 * 21 + 0] = 0
    c[1 * 21 + 1] = 0
    assert ora.ssv(c, [0, 1], Q()) == 0x86


def test_ssv_all_invalid(ora):
    assert ora.ssv(direct_costs(3, 0xFF), [0, 5, 11, 19, 2], Q()) == 0x80


def test_move_cost_and_base(ora):
    q = Q()
    assert ora.move_cost(0, q) == 0
    assert ora.sequence_base(0, q) == q.base
    assert ora.move_cost(1, q) == 1
    assert ora.move_cost(100, q) == 15
    assert ora.sequence_base(100, q) == q.base - 15
    # len 290 -> 175, len 35,000 -> 154
    assert ora.sequence_base(290, q) == 175
    assert ora.sequence_base(35000, q) == 154


def test_rejects_sentinel_codes(ora):
    with pytest.raises(ValueError):
        ora.msv(direct_costs(2, 3), [0, 21], Q())


# --- exhaustive path enumeration (brute_force.hpp semantics) ------------------

def _adds(a, b):
    return min(255, a + b)


def _subs(a, b):
    return a - b if a > b else 0


def _cost(c, node, code):
    return 0xFF if code > 20 else int(c[(node - 1) * 21 + code])


def msv_enum(c, seq, q, base):
    m = c.size // 21
    best = 0

    def extend(min_row, scJ, scB):
        nonlocal best
        for i in range(min_row, len(seq)):
            for j in range(1, m + 1):
                v, row, node = scB, i, j
                while row < len(seq) and node <= m:
                    v = _subs(_adds(v, q.dbias), _cost(c, node, seq[row]))
                    best = max(best, v)
                    j2 = max(scJ, _subs(v, q.tec))
                    b2 = max(base, _subs(j2, q.tjb))
                    extend(row + 1, j2, b2)
                    row += 1
                    node += 1

    extend(0, 0, base)
    return best


def ssv_enum(c, seq, q):
    m = c.size // 21
    best = 0x80
    for i in range(len(seq)):
        for j in range(1, m + 1):
            v, row, node = 0x80, i, j
            while row < len(seq) and node <= m:
                v = max(_subs(_adds(v, q.dbias), _cost(c, node, seq[row])), 0x80)
                best = max(best, v)
                row += 1
                node += 1
    return best


@pytest.mark.parametrize("q", [Q(), Q(2.0, 240, 10, 1, 5), Q(3.0, 0, 0, 0, 0)], ids=repr)
def test_oracle_equals_path_enumeration(ora, q):
    rs = np.random.default_rng(555)
    n = 0
    for m in range(1, 4):
        for length in range(0, 6):
            for t in range(6):
                c = (rs.integers(0, 25, m * 21) * (10 if t % 3 == 1 else 1)).astype(np.uint8) \
                    if t % 3 != 2 else rs.integers(0, 256, m * 21).astype(np.uint8)
                seq = list(rs.integers(0, 20, length))
                base = ora.sequence_base(length, q)
                assert ora.msv(c, seq, q) == msv_enum(c, seq, q, base)
                assert ora.ssv(c, seq, q) == ssv_enum(c, seq, q)
                n += 1
    assert n == 3 * 6 * 6


# --- quantization KATs (test_profile.cpp:75-129) ------------------------------

def test_quantize_formula_and_clamping(ora):
    s = np.zeros(3 * 20)
    s[0], s[1], s[2] = 0.0, -10.0, 2.0
    c = ora.quantize(s, Q())
    assert (c[0], c[1], c[2]) == (3, 33, 0)


def test_unknown_cost_is_mean_rounded_up(ora):
    s = np.array([(-1.0 if a % 2 else 0.0) for a in range(20)])
    assert ora.quantize(s, Q())[20] == 5


def test_quant_validation(ora):
    with pytest.raises(ValueError):
        ora.quantize(np.zeros(20), Q(scale=0.0))
    with pytest.raises(ValueError):
        ora.quantize(np.zeros(20), Q(base=254, dbias=4))


def test_finalize_kats(ora):
    q = Q()
    bits, p, ovf = ora.finalize(q.base, 0, 0.69, 2.0, q, 0)
    assert bits == pytest.approx(0.0) and p == pytest.approx(min(1.0, np.exp(0.69 * 2.0)))
    bits, p, ovf = ora.finalize(255, 100, 0.69, 2.0, q, 0)
    assert ovf and p == 0.0
    bits, p, ovf = ora.finalize(0x80, 0, 0.69, 2.0, q, 1)
    assert bits == pytest.approx(0.0)
    for length in (1, 10, 500):
        prev = 2.0
        for raw in range(255):
            _, p, _ = ora.finalize(raw, length, 0.69, 2.0, q, 0)
            assert 0.0 < p <= prev
            prev = p


# --- golden vectors produced by the reference --------------------------------

def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_golden_vectors(ora):
    import paper_1707_09683_b200 as P  # product generators reproduce the inputs
    g = _golden()
    assert g["cases"], "empty golden file"
    for case in g["cases"]:
        rng = P.Rng(case["seed"])
        hmm = rng.random_profile(case["m"])
        plant = (hmm, case["plant"]) if case["plant"] else None
        if case["gen"] == "uniform":
            db = rng.random_records(case["count"], case["lo"], case["hi"], plant=plant)
        else:
            db = rng.lognormal_records(case["count"], case["median"], case["sigma"], 2, plant=plant)
        assert int(db.residues.astype(np.uint64).sum()) == case["residue_sum"]
        q = Q(*case["quant"])
        costs = ora.quantize(hmm.match_scores.reshape(-1), q)
        assert int(costs.astype(np.uint64).sum()) == case["cost_sum"]
        for alg, key in ((0, "msv"), (1, "ssv")):
            got = ora.scan_flat(alg, costs, db.residues, db.offsets, q)
            np.testing.assert_array_equal(got, np.array(case[key], dtype=np.uint8),
                                          err_msg=f"seed {case['seed']} {key}")
        lens = np.diff(db.offsets)
        for alg, key in ((0, "msv"), (1, "ssv")):
            for t, want in case[f"pass_{key}"].items():
                got = [ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, q, alg, float(t))
                       for r, n in zip(case[key], lens)]
                assert got == want


def test_oracle_matches_reference_library(ora, ref):
    """The restatement vs the unmodified reference on random instances."""
    for seed, m in ((1, 7), (2, 91), (3, 400), (4, 1216)):
        g = ref.rng(seed)
        s, lam, tau = g.random_profile(m)
        res, off = g.random_records(40, 1, max(8, 200000 // m), plant=(s, 0.2))
        for q in (Q(), Q(3.0, 120, 3, 20, 20), Q(2.0, 240, 10, 1, 5)):
            c = ref.quantize(s, q)
            np.testing.assert_array_equal(c, ora.quantize(s, q))
            for alg in (0, 1):
                want = [ref.scalar(alg, c, res[off[k]:off[k + 1]], q) for k in range(40)]
                np.testing.assert_array_equal(ora.scan_flat(alg, c, res, off, q), want)
            for raw in (0, 100, 180, 254, 255):
                for n in (0, 1, 290, 35000):
                    assert ora.finalize(raw, n, lam, tau, q, 0) == ref.finalize(raw, n, lam, tau, q, 0)
                    assert ora.finalize(raw, n, lam, tau, q, 1) == ref.finalize(raw, n, lam, tau, q, 1)
