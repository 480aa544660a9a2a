#!/usr/bin/env python
"""Run-to-run spread of single scans: SSV M=800/1000 and MSV M=2405 over the
1M C2 database, N back-to-back scans each (device ms per scan), printed as
percentiles."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_09683_b200 as P  # noqa: E402

db = P.Rng(0x5EED).lognormal_records(1_000_000, 290, 0.65, 2)
with P.Scanner(0) as s:
    s.set_database(db)
    for alg, m in (("ssv", 800), ("ssv", 1000), ("msv", 2405)):
        hmm = P.Rng(7000 + m).random_profile(m)
        q = P.QuantParams()
        s.set_profile(P.quantize_emissions(hmm, q), q, hmm.lambda_, hmm.tau)
        o = P.ScanOptions(alg=P.Algorithm.Msv if alg == "msv" else P.Algorithm.Ssv)
        for _ in range(3):
            s.scan(o)
        t = np.array([s.scan(o).stats["device_ms"] for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60)])
        print(json.dumps({"alg": alg, "M": m, "n": int(t.size),
                          "pct": {p: round(float(np.percentile(t, p)), 4) for p in (0, 10, 50, 90, 100)},
                          "slow_gt_1pct": int((t > 1.01 * np.median(t)).sum())}), flush=True)
