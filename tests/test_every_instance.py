"""Every compiled kernel instance against the oracle, bit-exact.

The library instantiates one kernel per (variant, algorithm, lanes L, rows H)
(csrc/gen_instances.py) plus the K-warp long-model kernels; the parity tests
in test_gpu_parity.py reach a sample of them through the geometry policy.
Here each instance is pinned explicitly (ScanOptions lanes/rows/variant) and
scored on a small database whose model fills the instance's top row group
(full, and one stripe short), with the reference's QuantParams sets rotated
through (proj/tests/test_oracle.cpp:95-96 and SURVEY §8(c) signal sets), so
a wrong constant in any single template specialisation is caught."""
import os
import sys
import zlib

import numpy as np
import pytest

import oracle
import paper_1707_09683_b200 as P

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(P.__file__), "csrc"))
import gen_instances as G  # noqa: E402

VARIANT = {"dpx16": P.Variant.Dpx16, "fp16": P.Variant.Fp16, "swar8": P.Variant.Swar8,
           "fp16x": P.Variant.Fp16x, "fp16xalt": P.Variant.Fp16xAlt,
           "fp16xm": P.Variant.Fp16xMixed, "fp16xh": P.Variant.Fp16xHybrid,
           "fp16xr": P.Variant.Fp16xRelaxed, "fp16xrm": P.Variant.Fp16xRelaxedFixedB}
QUANTS = [P.QuantParams(), P.QuantParams(3.0, 120, 3, 20, 20), P.QuantParams(2.0, 240, 10, 1, 5),
          P.QuantParams(3.0, 0, 0, 0, 0)]
# cells per case: keeps the scalar oracle at a few ms per instance
CELL_BUDGET = 1_500_000


def oq(q):
    return oracle.QuantParams(q.scale, q.base, q.dbias, q.tec, q.tjb)


def cases():
    for v, rows in G.ROWS.items():
        for a in ("msv", "ssv"):
            if (v, a) in G.SKIP:
                continue
            yield pytest.param(v, a, id=f"{v}-{a}")


def check(s, ora, rng, alg, variant, L, H, m, q, seed_tag):
    hmm = rng.random_profile(m)
    nseq = 40
    maxlen = int(max(6, min(260, CELL_BUDGET // (nseq * m))))
    db = rng.random_records(nseq, 1, maxlen, plant=(hmm, 0.25))
    costs = P.quantize_emissions(hmm, q)
    s.set_profile(costs, q, hmm.lambda_, hmm.tau)
    s.set_database(db)
    try:
        rep = s.scan(P.ScanOptions(alg=alg, variant=variant, lanes=L, rows=H, threshold=0.2))
    except P.DataError as e:
        # geometries whose table exceeds the shared-memory budget are not
        # instantiated for scans (the policy never picks them)
        assert "table" in str(e) or "geometry" in str(e), str(e)
        return False
    assert (rep.lanes, rep.rows) == (L, H), seed_tag
    if L <= 32:
        # the widest register rows run 12-warp CTAs (lhmm_kernel.cuh threads_for)
        assert rep.stats["threads"] == (384 if H >= 54 else 512), seed_tag
    want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
    np.testing.assert_array_equal(rep.raw, want, err_msg=f"{seed_tag} m={m} q={q}")
    lens = db.lengths()
    wp = np.array([ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, oq(q), int(alg), 0.2)
                   for r, n in zip(want, lens)])
    np.testing.assert_array_equal(rep.passed, wp, err_msg=f"{seed_tag} pass bits")
    return True


@pytest.mark.parametrize("vname,aname", list(cases()))
def test_every_standard_instance(ora, vname, aname):
    variant = VARIANT[vname]
    alg = P.Algorithm.Msv if aname == "msv" else P.Algorithm.Ssv
    cpw = 4 if vname == "swar8" else 2
    ran = total = 0
    with P.Scanner(0) as s:
        for L in G.LANES:
            for i, H in enumerate(G.ROWS[vname]):
                rng = P.Rng(zlib.crc32(f"{vname}/{aname}/{L}/{H}".encode()))
                cap = cpw * L * H
                # full capacity, then one stripe short of it (partial top group)
                for k, m in enumerate((cap, max(1, cap - cpw * L + 1 + int(rng.next() % (cpw * L))))):
                    q = QUANTS[(i + k + L) % len(QUANTS)]
                    total += 1
                    ran += check(s, ora, rng, alg, variant, L, H, m, q, f"{vname}/{aname} L={L} H={H}")
    print(f"{vname}/{aname}: {ran} of {total} (instance, model) cases scanned")
    assert ran >= total * 3 // 4


@pytest.mark.parametrize("aname", ["msv", "ssv"])
def test_every_long_instance(ora, aname):
    """scan_kernel_long<V, K, H> for every K (warps per sequence) and H."""
    alg = P.Algorithm.Msv if aname == "msv" else P.Algorithm.Ssv
    with P.Scanner(0) as s:
        for K in G.LONG_K:
            for i, H in enumerate(G.LONG_ROWS):
                rng = P.Rng(0x10A6 + 131 * K + H + int(alg))
                cap = 2 * 32 * K * H
                m = cap - int(rng.next() % 64)
                q = QUANTS[(i + K) % 2]  # saturating and non-saturating parameters
                assert check(s, ora, rng, alg, P.Variant.Auto, 32 * K, H, m, q,
                             f"long {aname} K={K} H={H}")
