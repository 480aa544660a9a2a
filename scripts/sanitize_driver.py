#!/usr/bin/env python
"""Small workload touching every device code path, sized to run under
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every variant and algorithm at a few lane counts, the K-warp long-model
kernel, the relaxed-SSV rescoring, the device filter pipeline, the
single-launch streamed scan and the out-of-core ring.  Checks results
against the oracle as it goes (test infrastructure: scripts/ + oracle/).

    compute-sanitizer --tool memcheck python scripts/sanitize_driver.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1707_09683_b200 as P  # noqa: E402


def main():
    ora = oracle.Oracle()
    rng = P.Rng(0x5A17)
    checked = 0

    def check(rep, costs, q, db, alg):
        nonlocal checked
        want = ora.scan_flat(int(alg), costs.bytes, db.residues, db.offsets,
                             oracle.QuantParams(q.scale, q.base, q.dbias, q.tec, q.tjb))
        assert (rep.raw == want).all(), "mismatch"
        checked += 1

    q = P.QuantParams()
    hmm = rng.random_profile(120)
    db = rng.random_records(96, 1, 120, plant=(hmm, 0.3))
    costs = P.quantize_emissions(hmm, q)
    with P.Scanner(0) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_database(db)
        for v in (P.Variant.Fp16, P.Variant.Fp16x, P.Variant.Fp16xAlt, P.Variant.Fp16xMixed,
                  P.Variant.Fp16xHybrid, P.Variant.Fp16xRelaxed, P.Variant.Fp16xRelaxedFixedB,
                  P.Variant.Dpx16, P.Variant.Swar8):
            for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
                if v in (P.Variant.Fp16xAlt, P.Variant.Fp16xHybrid, P.Variant.Fp16xRelaxed,
                         P.Variant.Fp16xRelaxedFixedB) and alg == P.Algorithm.Ssv:
                    continue
                for L in (1, 4, 32):
                    rep = s.scan(P.ScanOptions(alg=alg, variant=v, lanes=L, threshold=0.2))
                    check(rep, costs, q, db, alg)
        # FP16XM five-row groups with a three-row top slot (H = 58, 12-warp CTAs)
        h3 = rng.random_profile(116)
        c3 = P.quantize_emissions(h3, q)
        s.set_profile(c3, q, h3.lambda_, h3.tau)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            rep = s.scan(P.ScanOptions(alg=alg, variant=P.Variant.Fp16xMixed, lanes=1, rows=58,
                                       threshold=0.2))
            assert rep.stats["threads"] == 384
            check(rep, c3, q, db, alg)
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        # paper wrap mode
        rep = s.scan(P.ScanOptions(alg=P.Algorithm.Msv, variant=P.Variant.Fp16, lanes=8,
                                   threshold=0.2, paper_wrap=True))
        # device pipeline
        s.filter_pipeline(0.3)
        # streamed (single launch, stream-written flags)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            rep = s.scan_streamed(P.ScanOptions(alg=alg, threshold=0.2), 4)
            check(rep, costs, q, db, alg)
    # long model (K warps per sequence)
    hl = rng.random_profile(5000)
    dl = rng.random_records(12, 1, 40)
    cl = P.quantize_emissions(hl, q)
    with P.Scanner(0) as s:
        s.set_profile(cl, q, hl.lambda_, hl.tau)
        s.set_database(dl)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            check(s.scan(P.ScanOptions(alg=alg, threshold=0.2)), cl, q, dl, alg)
    # out-of-core ring
    big = rng.random_records(3000, 20, 400)
    with P.Scanner(0) as s:
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        s.set_db_budget(1 << 20)
        s.set_database(big)
        for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
            check(s.scan(P.ScanOptions(alg=alg, threshold=0.2)), costs, q, big, alg)
    # relaxed MSV forms with rescoring (planted hits flag sequences) at
    # non-saturating parameters, and the block gather's scatter kernel
    qn = P.QuantParams(3.0, 120, 3, 20, 20)
    hits = rng.random_records(600, 1, 300, plant=(hmm, 0.5))
    cn = P.quantize_emissions(hmm, qn)
    with P.Scanner(0) as s:
        s.set_profile(cn, qn, hmm.lambda_, hmm.tau)
        s.set_database(hits)
        for v in (P.Variant.Fp16xRelaxed, P.Variant.Fp16xRelaxedFixedB):
            for L in (1, 8, 32):
                rep = s.scan(P.ScanOptions(alg=P.Algorithm.Msv, variant=v, lanes=L, threshold=0.2))
                check(rep, cn, qn, hits, P.Algorithm.Msv)
                assert rep.stats["recomputed"] > 0
        # several scans over one streamed upload (concurrent kernels on SM
        # shares waiting on piece flags, per-job counters and flags, rescoring)
        pd = s.add_profile(costs, q, hmm.lambda_, hmm.tau)
        pn = s.add_profile(cn, qn, hmm.lambda_, hmm.tau)
        jobs = [(pd, P.ScanOptions(alg=P.Algorithm.Msv, threshold=0.2)),
                (pd, P.ScanOptions(alg=P.Algorithm.Ssv, threshold=0.2)),
                (pn, P.ScanOptions(alg=P.Algorithm.Msv, variant=P.Variant.Fp16xRelaxedFixedB,
                                   lanes=8, threshold=0.2))]
        reps = s.scan_streamed_jobs(jobs, 4)
        check(reps[0], costs, q, hits, P.Algorithm.Msv)
        check(reps[1], costs, q, hits, P.Algorithm.Ssv)
        check(reps[2], cn, qn, hits, P.Algorithm.Msv)
        import torch
        n = hits.count
        perm = torch.randperm(n, device="cuda")
        src = torch.randint(0, 255, (2, n), dtype=torch.uint8, device="cuda")
        dst = torch.zeros((2, n), dtype=torch.uint8, device="cuda")
        s.scatter_results(dst[0].data_ptr(), dst[1].data_ptr(), src[0].data_ptr(),
                          src[1].data_ptr(), perm.data_ptr(), n)
        s.synchronize()
        # (compared on the host: .item() would draw on torch's pinned host
        # cache, which memcheck's leak check reports at exit)
        assert (dst[:, perm].cpu().numpy() == src.cpu().numpy()).all()
        del perm, src, dst
        torch.cuda.synchronize()
        torch.cuda.empty_cache()  # the caching allocator's blocks (memcheck leak check)
    print(f"sanitize driver ok: {checked} scans bit-exact")


if __name__ == "__main__":
    main()
