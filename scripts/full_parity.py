#!/usr/bin/env python
"""Full-database parity (test infrastructure): every sequence of the 1M
Swiss-Prot-like C2/C3 database (synth::lognormal_records(1e6, 290, 0.65, 2),
seed 0x5EED) scanned on the device with the auto policy -- SSV and MSV at the
default QuantParams, MSV at the non-saturating {3,120,3,20,20}, models
M = 48 / 400 / 1000 / 2405 (seed 7000+M) -- and compared raw byte and pass bit
for ALL sequences with the reference library's own scalar_msv / scalar_ssv
(src/oracle.cpp:41-91) and finalize_hit pass rule (oracle/_ref, OpenMP on the
host).  The bench's verify leg checks a 20k-sequence sample of every timed
scan; this is the exhaustive version for the BASELINE configs.  One JSON
line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_1707_09683_b200 as P  # noqa: E402

THRESHOLD = 0.022


def main():
    t0 = time.perf_counter()
    ref = oracle.Reference()
    db = P.Rng(0x5EED).lognormal_records(1_000_000, 290, 0.65, 2)
    res, off = db.residues, np.asarray(db.offsets, dtype=np.uint64)
    threads = os.cpu_count() or 1
    qd, qn = (3.0, 195, 3, 3, 3), (3.0, 120, 3, 20, 20)
    runs = [("ssv", qd, m) for m in (48, 400, 1000, 2405)] + \
           [("msv", qd, m) for m in (48, 400, 1000, 2405)] + \
           [("msv", qn, m) for m in (400, 2405)]
    out = {"what": __doc__.split("\n\n")[0].replace("\n", " "), "sequences": int(db.count),
           "residues": int(res.size), "checker": "oracle/_ref scalar_msv/scalar_ssv + "
           "finalize_hit (reference library built from its sources)", "scans": []}
    total_checked = total_bad = 0
    with P.Scanner(0) as s:
        s.set_database(db)
        for alg, q, m in runs:
            hmm = P.Rng(7000 + m).random_profile(m)
            qp = P.QuantParams(*q)
            costs = P.quantize_emissions(hmm, qp)
            s.set_profile(costs, qp, hmm.lambda_, hmm.tau)
            a = P.Algorithm.Msv if alg == "msv" else P.Algorithm.Ssv
            rep = s.scan(P.ScanOptions(alg=a, threshold=THRESHOLD))
            t1 = time.perf_counter()
            oq = oracle.QuantParams(*q)
            ai = 0 if alg == "msv" else 1
            want = ref.scalar_flat(ai, costs.bytes, res, off, oq, threads)
            wpass = ref.pass_flat(ai, want, off, hmm.lambda_, hmm.tau, oq, THRESHOLD)
            bad_raw = int(np.count_nonzero(rep.raw != want))
            bad_pass = int(np.count_nonzero(rep.passed.astype(np.uint8) != wpass))
            total_checked += 2 * int(db.count)
            total_bad += bad_raw + bad_pass
            e = {"alg": alg, "M": m, "quant": "QuantParams{%g,%d,%d,%d,%d}" % q,
                 "variant": rep.stats.get("variant"), "lanes": rep.lanes, "rows": rep.rows,
                 "device_gcups": round(rep.gcups, 1), "checked": 2 * int(db.count),
                 "raw_mismatches": bad_raw, "pass_mismatches": bad_pass,
                 "rescored_exactly": rep.stats.get("recomputed"),
                 "oracle_seconds": round(time.perf_counter() - t1, 1)}
            out["scans"].append(e)
            print(json.dumps(e), file=sys.stderr, flush=True)
    out["checked"], out["mismatches"] = total_checked, total_bad
    out["seconds"] = round(time.perf_counter() - t0, 1)
    out["host_threads"] = threads
    print(json.dumps(out))


if __name__ == "__main__":
    main()
