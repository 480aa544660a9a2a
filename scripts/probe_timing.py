#!/usr/bin/env python
"""First-scan cost of the MSV saturation probe: for fresh profiles over the
1M C2 database (after a warm-up profile, so module loading is not counted),
the first and second auto MSV scans' device time and code form, with the
probe on and off (LHMM_SAT_PROBE).  JSON lines."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_09683_b200 as P  # noqa: E402

db = P.Rng(0x5EED).lognormal_records(1_000_000, 290, 0.65, 2)
for probe in ("1", "0"):
    os.environ["LHMM_SAT_PROBE"] = probe
    with P.Scanner(0) as s:
        s.set_database(db)
        for qn, q in (("default", P.QuantParams()), ("nonsat", P.QuantParams(3.0, 120, 3, 20, 20))):
            for m in (48, 400, 2405):
                for seed in (1, 2):  # seed 1 warms the kernels and the buffers
                    hmm = P.Rng(9000 + 10 * m + seed).random_profile(m)
                    c = P.quantize_emissions(hmm, q)
                    s.set_profile(c, q, hmm.lambda_, hmm.tau)
                    t0 = time.perf_counter()
                    r1 = s.scan(P.ScanOptions(alg=P.Algorithm.Msv))
                    w1 = time.perf_counter() - t0
                    r2 = s.scan(P.ScanOptions(alg=P.Algorithm.Msv))
                    if seed == 2:
                        print(json.dumps({"probe": probe, "q": qn, "M": m,
                                          "first_ms": round(r1.stats["device_ms"], 3),
                                          "first_wall_ms": round(w1 * 1e3, 3),
                                          "first_variant": P.Variant(r1.variant).name,
                                          "second_ms": round(r2.stats["device_ms"], 3),
                                          "second_variant": P.Variant(r2.variant).name}),
                              flush=True)
