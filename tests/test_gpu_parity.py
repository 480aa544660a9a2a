"""GPU parity: every kernel variant / lane count / algorithm against the CPU
oracle, bit-exact (integer byte scores and pass bits), through the C ABI.

Mirrors the reference's engine tests (proj/tests/test_engine.cpp) and the
acceptance criteria 1, 5 and 6 (proj/tests/acceptance_main.cpp)."""
import numpy as np
import pytest

import oracle
import paper_1707_09683_b200 as P

pytestmark = pytest.mark.gpu

VARIANTS = [P.Variant.Dpx16, P.Variant.Fp16, P.Variant.Swar8, P.Variant.Fp16x, P.Variant.Fp16xAlt]
QUANTS = [P.QuantParams(), P.QuantParams(3.0, 120, 3, 20, 20), P.QuantParams(2.0, 240, 10, 1, 5),
          P.QuantParams(3.0, 0, 0, 0, 0)]


def oq(q):
    return oracle.QuantParams(q.scale, q.base, q.dbias, q.tec, q.tjb)


def rows_list(variant):
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(P.__file__), "csrc"))
    import gen_instances
    return gen_instances.ROWS[{P.Variant.Swar8: "swar8", P.Variant.Dpx16: "dpx16",
                               P.Variant.Fp16: "fp16", P.Variant.Fp16x: "fp16x",
                               P.Variant.Fp16xAlt: "fp16xalt",
                               P.Variant.Fp16xMixed: "fp16xm",
                               P.Variant.Fp16xHybrid: "fp16xh",
                               P.Variant.Fp16xRelaxed: "fp16xr",
                               P.Variant.Fp16xRelaxedFixedB: "fp16xrm"}[variant]]


def rows_for(variant, L, m):
    cpw = 4 if variant == P.Variant.Swar8 else 2
    for h in rows_list(variant):
        if cpw * L * h >= m:
            return h
    return None


def scan(costs, q, db, hmm, **kw):
    with P.Scanner(0) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(db)
        return s.scan(P.ScanOptions(**kw))


@pytest.mark.parametrize("variant", VARIANTS, ids=lambda v: v.name)
@pytest.mark.parametrize("alg", [P.Algorithm.Msv, P.Algorithm.Ssv], ids=lambda a: a.name)
@pytest.mark.parametrize("L", [1, 2, 4, 8, 16, 32])
def test_every_lane_count_matches_oracle(ora, variant, alg, L):
    rng = P.Rng(1000 + 97 * L + int(alg) + 7 * int(variant))
    cpw = 4 if variant == P.Variant.Swar8 else 2
    maxcap = cpw * L * {P.Variant.Swar8: 32, P.Variant.Dpx16: 64}.get(variant, 72)
    for t, q in enumerate(QUANTS):
        m = int(7 + rng.next() % max(1, min(maxcap, 2405) - 6))
        hmm = rng.random_profile(m)
        db = rng.random_records(64, 1, max(8, min(400, 3_000_000 // (64 * m))),
                                plant=(hmm, 0.2))
        costs = P.quantize_emissions(hmm, q)
        H = rows_for(variant, L, m)
        rep = scan(costs, q, db, hmm, alg=alg, variant=variant, lanes=L, rows=H, threshold=0.3)
        want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
        assert rep.lanes == L and rep.rows == H
        np.testing.assert_array_equal(rep.raw, want, err_msg=f"m={m} q={q} L={L} H={H}")


@pytest.mark.parametrize("variant", VARIANTS, ids=lambda v: v.name)
def test_pass_bits_match_finalize_hit(ora, variant):
    rng = P.Rng(0xC1)
    hmm = rng.random_profile(200)
    db = rng.random_records(500, 50, 650, plant=(hmm, 0.05))
    for q in QUANTS[:2]:
        costs = P.quantize_emissions(hmm, q)
        lens = np.diff(db.offsets)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            for t in (0.0, 0.022, 0.103, 0.307, 0.458, 1.0):
                rep = scan(costs, q, db, hmm, alg=alg, variant=variant, threshold=t)
                want = np.array([ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, oq(q), int(alg), t)
                                 for r, n in zip(rep.raw, lens)])
                np.testing.assert_array_equal(rep.passed, want, err_msg=f"{alg} t={t}")


@pytest.mark.parametrize("variant", VARIANTS, ids=lambda v: v.name)
def test_edge_lengths_and_empty_sequences(ora, variant):
    """Empty sequences score the floor (test_oracle.cpp:22-28); lengths around
    the 16-row chunk boundary; a single residue; long sequences."""
    rng = P.Rng(5)
    hmm = rng.random_profile(61)
    q = P.QuantParams(3.0, 120, 3, 20, 20)
    costs = P.quantize_emissions(hmm, q)
    lens = [0, 1, 2, 15, 16, 17, 31, 32, 33, 0, 47, 48, 49, 255, 256, 257, 1000, 3001, 0, 5]
    seqs = [np.frombuffer(np.random.default_rng(n + 1).integers(0, 21, n).astype(np.uint8).tobytes(),
                          np.uint8) for n in lens]
    db = P.SequenceDB.from_sequences(seqs)
    for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
        for L in (1, 4, 32):
            rep = scan(costs, q, db, hmm, alg=alg, variant=variant, lanes=L)
            want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
            np.testing.assert_array_equal(rep.raw, want)
            assert rep.raw[0] == (0 if alg == P.Algorithm.Msv else 0x80)


@pytest.mark.parametrize("variant", VARIANTS, ids=lambda v: v.name)
def test_floor_profiles(variant):
    """Flat profile with zero base pins MSV at 0 (test_engine.cpp:112-134);
    all-invalid emissions keep SSV at 0x80 (test_engine.cpp:386-404)."""
    rng = P.Rng(3)
    db = rng.random_records(40, 1, 50)
    flat = P.ProfileHMM("flat", 1, np.zeros((1, 20)), 0.7, 2.0)
    q0 = P.QuantParams(base=0)
    rep = scan(P.quantize_emissions(flat, q0), q0, db, flat, alg=P.Algorithm.Msv, variant=variant)
    assert (rep.raw == 0).all()
    inv = P.ProfileHMM("inv", 5, np.full((5, 20), -100.0), 0.7, 2.0)
    q = P.QuantParams()
    rep = scan(P.quantize_emissions(inv, q), q, db, inv, alg=P.Algorithm.Ssv, variant=variant)
    assert (rep.raw == 0x80).all()


def test_largest_pfam_model_2405(ora):
    rng = P.Rng(2405)
    hmm = rng.random_profile(2405)
    db = rng.random_records(96, 1, 300)
    for q in QUANTS[:2]:
        costs = P.quantize_emissions(hmm, q)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            for variant in (P.Variant.Dpx16, P.Variant.Fp16):
                rep = scan(costs, q, db, hmm, alg=alg, variant=variant)
                want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
                np.testing.assert_array_equal(rep.raw, want)


def test_fault_injection_is_detected(ora):
    rng = P.Rng(37)
    hmm = rng.random_profile(64)
    db = rng.random_records(16, 40, 80)
    q = P.QuantParams(3.0, 120, 3, 20, 20)
    costs = P.quantize_emissions(hmm, q)
    rep = scan(costs, q, db, hmm, alg=P.Algorithm.Msv, lanes=32, fault_injection=True)
    want = ora.scan_flat(0, costs.bytes, db.residues, db.offsets, oq(q))
    assert (rep.raw != want).any()


def test_shards_cover_the_database(ora):
    rng = P.Rng(77)
    hmm = rng.random_profile(150)
    db = rng.lognormal_records(3000, 290, 0.65, 2)
    q = P.QuantParams(3.0, 120, 3, 20, 20)
    costs = P.quantize_emissions(hmm, q)
    want = ora.scan_flat(0, costs.bytes, db.residues, db.offsets, oq(q))
    got = np.full(db.count, -1, dtype=np.int32)
    with P.Scanner(0) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        for r in range(3):
            s.set_database(db, r, 3)
            idx = s.shard_indices()
            rep = s.scan(P.ScanOptions(alg=P.Algorithm.Msv))
            assert (got[idx] == -1).all()
            got[idx] = rep.raw
    np.testing.assert_array_equal(got, want)


def test_device_outputs_via_torch(ora):
    import torch
    rng = P.Rng(11)
    hmm = rng.random_profile(300)
    db = rng.random_records(1000, 10, 500)
    q = P.QuantParams()
    costs = P.quantize_emissions(hmm, q)
    raw = torch.zeros(db.count, dtype=torch.uint8, device="cuda:0")
    ps = torch.zeros(db.count, dtype=torch.uint8, device="cuda:0")
    with P.Scanner(0) as s:
        s.set_stream(torch.cuda.current_stream().cuda_stream)
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(db)
        st = s.scan_device(P.ScanOptions(alg=P.Algorithm.Ssv), raw.data_ptr(), ps.data_ptr())
    torch.cuda.synchronize()
    want = ora.scan_flat(1, costs.bytes, db.residues, db.offsets, oq(q))
    np.testing.assert_array_equal(raw.cpu().numpy(), want)
    assert st["launches"] == 1


def test_multiple_resident_profiles(ora):
    rng = P.Rng(12)
    db = rng.random_records(300, 10, 400)
    q = P.QuantParams(3.0, 120, 3, 20, 20)
    with P.Scanner(0) as s:
        s.set_database(db)
        ids, models = [], []
        for m in (48, 400, 1000):
            hmm = rng.random_profile(m)
            c = P.quantize_emissions(hmm, q)
            ids.append(s.add_profile(c, q, hmm.lambda_, hmm.tau))
            models.append(c)
        for pid, c in reversed(list(zip(ids, models))):
            s.select_profile(pid)
            rep = s.scan(P.ScanOptions(alg=P.Algorithm.Ssv))
            want = ora.scan_flat(1, c.bytes, db.residues, db.offsets, oq(q))
            np.testing.assert_array_equal(rep.raw, want)


@pytest.mark.parametrize("mem_ops", ["1", "0"], ids=["single_launch", "per_piece"])
def test_streamed_scan_matches_resident_scan(ora, mem_ops, monkeypatch):
    """lhmm_scan_streamed (H2D in pieces overlapped with the scan: one launch
    waiting on stream-written piece flags, or per-piece launches) returns
    exactly the resident scan's scores and pass bits, for every variant and
    the long-model kernel."""
    monkeypatch.setenv("LHMM_STREAM_MEM_OPS", mem_ops)
    rng = P.Rng(21)
    hmm = rng.random_profile(333)
    db = rng.lognormal_records(150000, 290, 0.65, 2)  # ~55 MB packed
    q = P.QuantParams(3.0, 120, 3, 20, 20)
    costs = P.quantize_emissions(hmm, q)
    want = ora.scan_flat(0, costs.bytes, db.residues, db.offsets, oq(q))
    with P.Scanner(0) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(db)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            # (explicit L=4, H=58/60: wide register rows, 12-warp CTAs)
            for variant, lanes, rows in ((P.Variant.Auto, 0, 0), (P.Variant.Fp16x, 0, 0),
                                         (P.Variant.Dpx16, 0, 0), (P.Variant.Fp16, 64, 0),
                                         (P.Variant.Fp16xMixed, 4, 58), (P.Variant.Fp16x, 4, 60)):
                o = P.ScanOptions(alg=alg, threshold=0.3, variant=variant, lanes=lanes, rows=rows)
                base = s.scan(o)
                for seg in (1, 3, 8, 64):
                    st = s.scan_streamed(o, seg)
                    np.testing.assert_array_equal(st.raw, base.raw)
                    np.testing.assert_array_equal(st.passed, base.passed)
                    # (+1 when a relaxed kernel's flagged sequences were rescored)
                    extra = 1 if st.stats["recomputed"] else 0
                    if mem_ops == "1":
                        assert st.stats["launches"] == 1 + extra
                    else:
                        assert 1 <= st.stats["launches"] <= seg + extra
        np.testing.assert_array_equal(s.scan(P.ScanOptions(alg=P.Algorithm.Msv)).raw, want)


@pytest.mark.parametrize("mem_ops", ["1", "0"], ids=["concurrent", "per_piece"])
def test_streamed_jobs_match_oracle_and_resident_scans(ora, mem_ops, monkeypatch):
    """lhmm_scan_streamed_jobs: several (profile, options) jobs over ONE
    streamed upload -- concurrent single launches on shares of the SMs
    waiting on piece flags, or per-piece launches -- each job's raw bytes and
    pass bits equal its resident lhmm_scan and the scalar oracle (MSV and SSV,
    default and non-saturating QuantParams, relaxed forms with rescoring, a
    long model, pageable and page-locked outputs)."""
    import torch
    monkeypatch.setenv("LHMM_STREAM_MEM_OPS", mem_ops)
    rng = P.Rng(0x10B5)
    db = rng.lognormal_records(150000, 290, 0.65, 2)  # ~55 MB packed: 3 pieces
    qd, qn = P.QuantParams(), P.QuantParams(3.0, 120, 3, 20, 20)
    spec = [(200, qd, P.Algorithm.Msv), (200, qd, P.Algorithm.Ssv), (400, qn, P.Algorithm.Msv),
            (1000, qd, P.Algorithm.Ssv), (5000, qn, P.Algorithm.Msv)]
    with P.Scanner(0) as s:
        s.set_database(db)
        jobs, want, lam = [], [], []
        for m, q, alg in spec:
            hmm = rng.random_profile(m)
            costs = P.quantize_emissions(hmm, q)
            pid = s.add_profile(costs, q, hmm.lambda_, hmm.tau)
            jobs.append((pid, P.ScanOptions(alg=alg, threshold=0.022)))
            want.append((costs, q, alg))
            lam.append((hmm.lambda_, hmm.tau))
        n = s.n_local
        pinned = [(torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy(),
                   torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()) for _ in jobs]
        for outs in (None, pinned):
            reps = s.scan_streamed_jobs(jobs, 64, outs=outs)
            for (pid, o), rep in zip(jobs, reps):
                s.select_profile(pid)
                base = s.scan(o)
                np.testing.assert_array_equal(rep.raw, base.raw)
                np.testing.assert_array_equal(rep.passed, base.passed)
                assert rep.stats["launches"] >= (1 if mem_ops == "1" else 3)
                assert rep.lanes == base.lanes and rep.rows == base.rows
        # oracle on a fixed-stride sample of every job
        idx = np.arange(0, db.count, 37)
        off = db.offsets
        res = np.concatenate([db.residues[off[i]:off[i + 1]] for i in idx])
        soff = np.concatenate([[0], np.cumsum(off[idx + 1] - off[idx])]).astype(np.uint64)
        for (costs, q, alg), rep in zip(want, reps):
            a = 0 if alg == P.Algorithm.Msv else 1
            np.testing.assert_array_equal(rep.raw[idx],
                                          ora.scan_flat(a, costs.bytes, res, soff, oq(q)))


def test_streamed_jobs_contract():
    """lhmm_scan_streamed_jobs: errors like the other scan entry points (no
    jobs, bad piece count, unknown profile id); the same profile may appear
    in several jobs."""
    rng = P.Rng(0x10B6)
    hmm = rng.random_profile(60)
    q = P.QuantParams()
    costs = P.quantize_emissions(hmm, q)
    with P.Scanner(0) as s:
        pid = s.add_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(rng.random_records(100, 20, 80))
        o = P.ScanOptions(alg=P.Algorithm.Msv)
        with pytest.raises(P.ContractError):
            s.scan_streamed_jobs([])
        with pytest.raises(P.ContractError):
            s.scan_streamed_jobs([(pid, o)], 0)
        with pytest.raises(P.ContractError):
            s.scan_streamed_jobs([(pid + 7, o)], 4)
        rep = s.scan_streamed_jobs([(pid, o), (pid, P.ScanOptions(alg=P.Algorithm.Ssv))], 4)
        assert [r.raw.size for r in rep] == [100, 100]
        s.select_profile(pid)
        np.testing.assert_array_equal(rep[0].raw, s.scan(o).raw)
        np.testing.assert_array_equal(rep[1].raw, s.scan(P.ScanOptions(alg=P.Algorithm.Ssv)).raw)


@pytest.mark.parametrize("threshold", [0.0, 0.022, 0.3, 1.0])
def test_device_filter_pipeline_matches_oracle(ora, threshold):
    """filter_pipeline semantics (test_engine.cpp:406-450, acceptance
    criterion 6): survivors are exactly {pValue <= t or overflow} of the SSV
    stage, and each survivor's MSV byte equals the scalar oracle's."""
    rng = P.Rng(0x5175)
    hmm = rng.random_profile(80)
    db = rng.random_records(3000, 20, 250, plant=(hmm, 0.2))
    q = P.QuantParams()
    costs = P.quantize_emissions(hmm, q)
    rep = P.filter_pipeline(hmm, costs, db, threshold, q)
    ssv = ora.scan_flat(1, costs.bytes, db.residues, db.offsets, oq(q))
    msv = ora.scan_flat(0, costs.bytes, db.residues, db.offsets, oq(q))
    lens = np.diff(db.offsets)
    expect = np.array([ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, oq(q), 1, threshold)
                       for r, n in zip(ssv, lens)])
    np.testing.assert_array_equal(rep.ssv_raw, ssv)
    np.testing.assert_array_equal(rep.passed, expect)
    assert rep.msv_rescored == int(expect.sum()) == rep.survivors.size
    np.testing.assert_array_equal(rep.msv_raw[expect], msv[expect])
    assert (rep.msv_raw[~expect] == 0).all()


def test_device_pipeline_matches_reference_library(ref):
    """Against the unmodified reference filter_pipeline (oracle/_ref)."""
    rng = P.Rng(42)
    hmm = rng.random_profile(48)
    db = rng.random_records(400, 30, 200, plant=(hmm, 0.15))
    q = P.QuantParams()
    costs = P.quantize_emissions(hmm, q)
    for t in (0.0, 0.02, 0.2, 1.0):
        ssv, msv, surv = ref.filter_pipeline(hmm.match_scores.reshape(-1), hmm.lambda_, hmm.tau,
                                             costs.bytes, oq(q), db.residues, db.offsets, t)
        rep = P.filter_pipeline(hmm, costs, db, t, q)
        np.testing.assert_array_equal(rep.ssv_raw, ssv)
        np.testing.assert_array_equal(rep.passed, surv)
        np.testing.assert_array_equal(rep.msv_raw, msv)


@pytest.mark.parametrize("alg", [P.Algorithm.Msv, P.Algorithm.Ssv], ids=lambda a: a.name)
def test_relaxed_variant_rescoring_is_exact(ora, alg):
    """FP16X SSV flags the sequences its relaxed arithmetic cannot certify
    (cells above 255-dbias) and rescores them exactly; FP16X MSV (two-mode)
    is exact without rescoring.  Force many SSV flags with planted motifs and
    check every byte against the oracle, including a flat profile."""
    rng = P.Rng(99)
    hmm = rng.random_profile(120)
    db = rng.random_records(4000, 20, 400, plant=(hmm, 0.5))
    flat = P.ProfileHMM("flat", 120, np.zeros((120, 20)), 0.7, 2.0)
    for prof, q in ((hmm, P.QuantParams()), (hmm, P.QuantParams(3.0, 120, 3, 20, 20)),
                    (flat, P.QuantParams()), (hmm, P.QuantParams(2.0, 240, 10, 1, 5))):
        costs = P.quantize_emissions(prof, q)
        want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
        rep = scan(costs, q, db, prof, alg=alg, variant=P.Variant.Fp16x, threshold=0.3)
        np.testing.assert_array_equal(rep.raw, want)
        # FP16X has several code forms (FP16X, FP16X_ALT for MSV, the
        # mixed-table FP16XM); the calibration picks one per geometry
        assert rep.variant in ((int(P.Variant.Fp16x), int(P.Variant.Fp16xAlt),
                                int(P.Variant.Fp16xMixed), int(P.Variant.Fp16xHybrid))
                               if alg == P.Algorithm.Msv else
                               (int(P.Variant.Fp16x), int(P.Variant.Fp16xMixed)))
        if alg == P.Algorithm.Msv:
            assert rep.stats["recomputed"] == 0
        elif prof is hmm and q == P.QuantParams():
            assert rep.stats["recomputed"] > 0


@pytest.mark.parametrize("L", [1, 2, 4, 8, 16, 32])
def test_mixed_table_ssv(ora, L):  # noqa: C901
    """FP16XM (SSV): subnormal-domain f16 words and signed-byte words in one
    16-byte slot per five rows; flagged sequences rescored exactly.  Every
    lane count, the four QuantParams sets (incl. dbias 10 and 0), planted
    motifs that force flags, a flat profile, full and partial top groups."""
    rng = P.Rng(0x3157 + L)
    for t, q in enumerate(QUANTS):
        for m in (10 * L * 7 - int(rng.next() % (2 * L)), 2 * L * 5, 37):
            m = max(1, min(m, 2 * L * 70))
            hmm = rng.random_profile(m)
            db = rng.random_records(300, 1, 300, plant=(hmm, 0.3))
            costs = P.quantize_emissions(hmm, q)
            H = next(h for h in rows_list(P.Variant.Fp16xMixed) if 2 * L * h >= m)
            rep = scan(costs, q, db, hmm, alg=P.Algorithm.Ssv, variant=P.Variant.Fp16xMixed,
                       lanes=L, rows=H, threshold=0.2)
            assert rep.variant == int(P.Variant.Fp16xMixed) and rep.rows == H
            want = ora.scan_flat(1, costs.bytes, db.residues, db.offsets, oq(q))
            np.testing.assert_array_equal(rep.raw, want, err_msg=f"L={L} m={m} q={q}")
    flat = P.ProfileHMM("flat", 2 * L * 5, np.zeros((2 * L * 5, 20)), 0.7, 2.0)
    costs = P.quantize_emissions(flat, P.QuantParams())
    rep = scan(costs, P.QuantParams(), db, flat, alg=P.Algorithm.Ssv,
               variant=P.Variant.Fp16xMixed, lanes=L, rows=5, threshold=0.2)
    want = ora.scan_flat(1, costs.bytes, db.residues, db.offsets, oq(P.QuantParams()))
    np.testing.assert_array_equal(rep.raw, want)


@pytest.mark.parametrize("variant", [P.Variant.Fp16x, P.Variant.Fp16xAlt, P.Variant.Fp16xMixed,
                                     P.Variant.Fp16xHybrid],
                         ids=lambda v: v.name)
@pytest.mark.parametrize("L", [1, 2, 4, 8, 16, 32])
def test_two_mode_msv_switch(ora, L, variant):
    """FP16X MSV switches a warp to the lazy-B form once all of its
    sequences reach E = 255.  Mix saturating (planted), slowly saturating and
    never-saturating sequences of varied lengths in the same warps, at
    default and non-saturating parameters, and compare with the oracle."""
    rng = P.Rng(0x5A7 + L)
    m = 2 * L * rows_for(variant, L, min(2 * L * 70, 700)) - L
    hmm = rng.random_profile(m)
    a = rng.random_records(300, 200, 900, plant=(hmm, 0.6))
    b = rng.random_records(300, 1, 900)
    db = P.SequenceDB.from_sequences([a.sequence(k) for k in range(a.count)] +
                                     [b.sequence(k) for k in range(b.count)])
    for q in (P.QuantParams(), P.QuantParams(3.0, 120, 3, 20, 20), P.QuantParams(2.0, 240, 10, 1, 5),
              P.QuantParams(3.0, 195, 3, 0, 0)):
        costs = P.quantize_emissions(hmm, q)
        want = ora.scan_flat(0, costs.bytes, db.residues, db.offsets, oq(q))
        rep = scan(costs, q, db, hmm, alg=P.Algorithm.Msv, variant=variant, lanes=L,
                   rows=rows_for(variant, L, m))
        assert rep.variant == int(variant)
        np.testing.assert_array_equal(rep.raw, want, err_msg=f"L={L} q={q}")


def wrap_model(alg, costs, m, seq, q, base):
    """The kernel's paper-wrap semantics (ReorderMode::PaperWrap analogue,
    src/vwarp.cpp:27-64) on a model whose striped capacity equals m: node 1
    takes node m's previous-row value instead of -inf."""
    c = costs.reshape(m, 21).astype(np.int32)
    floor = 0 if alg == P.Algorithm.Msv else 0x80
    M = np.full(m, floor, np.int32)
    E, B = floor, base
    for x in seq:
        prev = np.concatenate(([M[-1]], M[:-1]))
        if alg == P.Algorithm.Msv:
            v = np.minimum(np.maximum(prev, B) + q.dbias, 255) - c[:, x]
            M = np.maximum(v, 0)
            E = max(E, int(M.max()))
            B = max(base, E - q.tec - q.tjb)
        else:
            v = np.minimum(prev + q.dbias, 255) - c[:, x]
            M = np.maximum(v, 0x80)
            E = max(E, int(M.max()))
    return E


@pytest.mark.parametrize("variant", [P.Variant.Fp16, P.Variant.Dpx16, P.Variant.Swar8,
                                     P.Variant.Fp16x, P.Variant.Fp16xAlt, P.Variant.Fp16xMixed,
                                     P.Variant.Fp16xHybrid, P.Variant.Fp16xRelaxed,
                                     P.Variant.Fp16xRelaxedFixedB],
                         ids=lambda v: v.name)
@pytest.mark.parametrize("alg", [P.Algorithm.Msv, P.Algorithm.Ssv], ids=lambda a: a.name)
def test_paper_wrap_mode(ora, variant, alg):
    """The non-normative wrap study mode runs, matches its model, and differs
    from the normative (oracle-exact) -inf injection on a consensus-heavy
    instance (test_engine.cpp:265-278)."""
    if variant in (P.Variant.Fp16xHybrid, P.Variant.Fp16xRelaxed,
                   P.Variant.Fp16xRelaxedFixedB) and alg == P.Algorithm.Ssv:
        pytest.skip("an MSV form (SSV runs FP16XM / FP16X, tested above)")
    cpw = 4 if variant == P.Variant.Swar8 else 2
    differs = False
    geoms = {P.Variant.Fp16xMixed: ((1, 10), (2, 10), (8, 5), (32, 5)),
             P.Variant.Fp16xRelaxedFixedB: ((1, 10), (2, 10), (8, 5), (32, 5)),
             P.Variant.Fp16xHybrid: ((1, 8), (2, 10), (8, 8), (32, 10))}.get(
                 variant, ((1, 8), (2, 8), (8, 4), (32, 4)))
    # non-saturating parameters, and (two-mode MSV forms) default ones, whose
    # scores saturate so that the lazy rows run in the wrap mode too
    two_mode = alg == P.Algorithm.Msv and variant in (
        P.Variant.Fp16x, P.Variant.Fp16xAlt, P.Variant.Fp16xMixed, P.Variant.Fp16xHybrid)
    quants = [P.QuantParams(3.0, 120, 3, 20, 20)] + ([P.QuantParams()] if two_mode else [])
    for (L, H), q in [(g, q) for q in quants for g in geoms]:
        m = cpw * L * H
        rng = P.Rng(38 + L)
        hmm = rng.random_profile(m)
        hmm.match_scores[:] = np.where(np.arange(20)[None, :] == 0, 3.0, -3.0)
        db = rng.random_records(48, 30, 90, plant=(hmm, 0.5))
        costs = P.quantize_emissions(hmm, q)
        normative = scan(costs, q, db, hmm, alg=alg, variant=variant, lanes=L, rows=H)
        wrapped = scan(costs, q, db, hmm, alg=alg, variant=variant, lanes=L, rows=H,
                       paper_wrap=True)
        want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
        np.testing.assert_array_equal(normative.raw, want)
        lens = db.lengths()
        model = [wrap_model(alg, costs.bytes, m, db.sequence(k),
                            q, P.engine_sequence_base(int(lens[k]), q)) for k in range(db.count)]
        np.testing.assert_array_equal(wrapped.raw, np.array(model, np.uint8), err_msg=f"L={L}")
        differs = differs or bool((wrapped.raw != normative.raw).any())
    assert differs


@pytest.mark.parametrize("variant", [P.Variant.Fp16, P.Variant.Fp16x, P.Variant.Fp16xRelaxed],
                         ids=lambda v: v.name)
@pytest.mark.parametrize("alg", [P.Algorithm.Msv, P.Algorithm.Ssv], ids=lambda a: a.name)
def test_two_row_top_group(ora, variant, alg):
    """H = 2 (mod 4): the top row group is read with LDS.64 and folded as a
    pair; every lane count, models that fill the last rows exactly."""
    if variant == P.Variant.Fp16xRelaxed and alg == P.Algorithm.Ssv:
        pytest.skip("FP16XR is an MSV form")
    q = P.QuantParams(3.0, 120, 3, 20, 20)
    for L in (1, 2, 4, 8, 16, 32):
        for H in (34, 38, 70):
            m = 2 * L * H - (L * 7) % 5  # the top rows hold real nodes
            rng = P.Rng(5000 + L * 100 + H)
            hmm = rng.random_profile(m)
            db = rng.random_records(48, 1, max(8, min(300, 2_000_000 // (48 * m))),
                                    plant=(hmm, 0.25))
            costs = P.quantize_emissions(hmm, q)
            rep = scan(costs, q, db, hmm, alg=alg, variant=variant, lanes=L, rows=H)
            want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
            assert rep.rows == H
            np.testing.assert_array_equal(rep.raw, want, err_msg=f"L={L} H={H} m={m}")


def test_out_of_core_database_streams_through_the_ring(ora):
    """lhmm_context_set_db_budget: a database larger than the device budget
    stays in pinned host memory and is streamed through the device ring per
    scan; scores, pass bits and the pipeline equal the resident scan."""
    rng = P.Rng(0x00C)
    hmm = rng.random_profile(300)
    db = rng.lognormal_records(20000, 290, 0.65, 2, plant=(hmm, 0.05))
    q = P.QuantParams(3.0, 120, 3, 20, 20)
    costs = P.quantize_emissions(hmm, q)
    with P.Scanner(0) as res_s, P.Scanner(0) as ooc:
        res_s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        res_s.set_database(db)
        assert res_s.database_resident()
        ooc.set_db_budget(1 << 20)   # 1 MB: ~7 ring pieces for the 7 MB image
        ooc.set_profile(costs, q, hmm.lambda_, hmm.tau)
        ooc.set_database(db)
        assert not ooc.database_resident()
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            for variant, lanes, rows in ((P.Variant.Auto, 0, 0), (P.Variant.Fp16x, 0, 0),
                                         (P.Variant.Dpx16, 0, 0), (P.Variant.Fp16xMixed, 4, 58)):
                o = P.ScanOptions(alg=alg, variant=variant, threshold=0.05, lanes=lanes, rows=rows)
                a = res_s.scan(o)
                b = ooc.scan(o)
                np.testing.assert_array_equal(a.raw, b.raw)
                np.testing.assert_array_equal(a.passed, b.passed)
                assert b.stats["launches"] >= 4
            want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
            np.testing.assert_array_equal(b.raw, want)
        s1 = ooc.scan_streamed(P.ScanOptions(alg=P.Algorithm.Ssv), segments=4)
        np.testing.assert_array_equal(s1.raw, res_s.scan(P.ScanOptions(alg=P.Algorithm.Ssv)).raw)
        pa = res_s.filter_pipeline(0.05)
        pb = ooc.filter_pipeline(0.05)
        assert pa.msv_rescored == pb.msv_rescored > 0
        np.testing.assert_array_equal(pa.ssv_raw, pb.ssv_raw)
        np.testing.assert_array_equal(pa.msv_raw, pb.msv_raw)
    # FP16X SSV rescoring on a streamed database (flags gathered on the host)
    qd = P.QuantParams()
    dbp = rng.random_records(6000, 100, 600, plant=(hmm, 0.5))
    cd = P.quantize_emissions(hmm, qd)
    with P.Scanner(0) as ooc:
        ooc.set_db_budget(1 << 20)
        ooc.set_profile(cd, qd, hmm.lambda_, hmm.tau)
        ooc.set_database(dbp)
        assert not ooc.database_resident()
        rep = ooc.scan(P.ScanOptions(alg=P.Algorithm.Ssv, variant=P.Variant.Fp16x))
        assert rep.stats["recomputed"] > 0
        np.testing.assert_array_equal(
            rep.raw, ora.scan_flat(1, cd.bytes, dbp.residues, dbp.offsets, oq(qd)))
    with P.Scanner(0) as tiny:
        tiny.set_db_budget(4096)
        tiny.set_profile(costs, q, hmm.lambda_, hmm.tau)
        with pytest.raises(P.ContractError, match="largest tile"):
            tiny.set_database(db)


@pytest.mark.parametrize("alg", [P.Algorithm.Msv, P.Algorithm.Ssv], ids=lambda a: a.name)
def test_long_models_beyond_one_warp(ora, alg):
    """Models above one warp's capacity (M > 4352) run K warps per sequence
    (scan_kernel_long; the reference's S=1 path has no model-length bound,
    src/select.cpp:16-48).  Auto geometry and pinned group widths, saturating
    and non-saturating parameters, against the oracle."""
    for m, lanes in ((4353, 0), (6001, 0), (9000, 0), (17000, 0), (40000, 0), (700, 64),
                     (3000, 128), (5000, 256), (9000, 512)):
        rng = P.Rng(40000 + m + lanes)
        hmm = rng.random_profile(m)
        db = rng.random_records(40 if m > 10000 else 70, 1, 300, plant=(hmm, 0.3))
        for q in (P.QuantParams(), P.QuantParams(3.0, 120, 3, 20, 20)):
            costs = P.quantize_emissions(hmm, q)
            rep = scan(costs, q, db, hmm, alg=alg, lanes=lanes, threshold=0.1)
            want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
            assert rep.lanes > 32 and rep.lanes * rep.rows * 2 >= m
            np.testing.assert_array_equal(rep.raw, want, err_msg=f"m={m} lanes={rep.lanes}")
            lens = db.lengths()
            wp = np.array([ora.passes(int(r), int(n), hmm.lambda_, hmm.tau, oq(q), int(alg), 0.1)
                           for r, n in zip(rep.raw, lens)])
            np.testing.assert_array_equal(rep.passed, wp)


def test_long_model_pipeline_and_dropin_limits(ora):
    """The filter pipeline and the out-of-core ring also run long models."""
    rng = P.Rng(777)
    hmm = rng.random_profile(6000)
    db = rng.random_records(1500, 1, 200, plant=(hmm, 0.3))
    q = P.QuantParams()
    costs = P.quantize_emissions(hmm, q)
    with P.Scanner(0) as s:
        s.set_db_budget(1 << 15)
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(db)
        assert not s.database_resident()
        rep = s.filter_pipeline(0.05)
        np.testing.assert_array_equal(
            rep.ssv_raw, ora.scan_flat(1, costs.bytes, db.residues, db.offsets, oq(q)))
        want_msv = ora.scan_flat(0, costs.bytes, db.residues, db.offsets, oq(q))
        np.testing.assert_array_equal(rep.msv_raw[rep.passed], want_msv[rep.passed])


def test_policy_feedback_from_saturation_and_rescoring(ora):
    """The auto policy learns from the first scan of a profile/database pair:
    MSV keeps the one-body FP16 kernel when scores mostly do not saturate,
    SSV drops the relaxed FP16X kernel when it had to rescore > 20%; results
    stay exact either way."""
    rng = P.Rng(0xFEED)
    hmm = rng.random_profile(400)
    db = rng.lognormal_records(150000, 290, 0.65, 2)
    for q, msv_two_mode in ((P.QuantParams(), True), (P.QuantParams(3.0, 120, 3, 20, 20), False)):
        costs = P.quantize_emissions(hmm, q)
        with P.Scanner(0) as s:
            s.set_profile(costs, q, hmm.lambda_, hmm.tau)
            s.set_database(db)
            first = s.scan(P.ScanOptions(alg=P.Algorithm.Msv))
            second = s.scan(P.ScanOptions(alg=P.Algorithm.Msv))
            np.testing.assert_array_equal(first.raw, second.raw)
            two_mode = second.variant in (int(P.Variant.Fp16x), int(P.Variant.Fp16xAlt),
                                          int(P.Variant.Fp16xMixed), int(P.Variant.Fp16xHybrid))
            assert two_mode == msv_two_mode, (q, second.variant)
    planted = rng.lognormal_records(150000, 290, 0.65, 2, plant=(hmm, 0.9))
    q = P.QuantParams()
    costs = P.quantize_emissions(hmm, q)
    with P.Scanner(0) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(planted)
        first = s.scan(P.ScanOptions(alg=P.Algorithm.Ssv))
        second = s.scan(P.ScanOptions(alg=P.Algorithm.Ssv))
        np.testing.assert_array_equal(first.raw, second.raw)
        if (first.variant in (int(P.Variant.Fp16x), int(P.Variant.Fp16xMixed))
                and first.stats["recomputed"] > 0.2 * planted.count):
            assert second.variant == int(P.Variant.Fp16)


def test_global_outputs_two_shards_one_process(ora):
    """lhmm_scan_device_global from two shard contexts into one full-length
    buffer (what the fused gather does across processes), over the long-model
    kernel, an out-of-core shard and FP16X SSV rescoring."""
    rng = P.Rng(0x6B0)
    for m, budget, alg, variant in ((6000, 0, P.Algorithm.Msv, P.Variant.Auto),
                                    (700, 1 << 20, P.Algorithm.Msv, P.Variant.Auto),
                                    (300, 0, P.Algorithm.Ssv, P.Variant.Fp16x),
                                    (300, 1 << 20, P.Algorithm.Ssv, P.Variant.Fp16x)):
        hmm = rng.random_profile(m)
        db = rng.lognormal_records(8000 if m < 1000 else 1500, 250, 0.6, 2, plant=(hmm, 0.4))
        q = P.QuantParams()
        costs = P.quantize_emissions(hmm, q)
        a, b = P.Scanner(0), P.Scanner(0)
        try:
            base, _ = a.peer_buffer_create(2 * db.count)
            for rank, s in enumerate((a, b)):
                if budget:
                    s.set_db_budget(budget)
                s.set_profile(costs, q, hmm.lambda_, hmm.tau)
                s.set_database(db, rank, 2)
            a.device_fill(base, 2, 2 * db.count)
            for s in (a, b):
                s.scan_device_global(P.ScanOptions(alg=alg, variant=variant, threshold=0.05),
                                     base, base + db.count)
            buf = a.device_to_host(base, 2 * db.count)
            raw, ps = buf[:db.count], buf[db.count:]
            assert (ps <= 1).all()
            want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets, oq(q))
            np.testing.assert_array_equal(raw, want, err_msg=f"m={m} budget={budget}")
        finally:
            b.close()
            a.close()
