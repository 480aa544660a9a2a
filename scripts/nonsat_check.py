import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1707_09683_b200 as P
db = P.Rng(0x5EED).lognormal_records(400000, 290, 0.65, 2)
for qs in ((3.0,195,3,3,3), (3.0,120,3,20,20)):
    q = P.QuantParams(*qs)
    for M in (400, 2405):
        hmm = P.Rng(7000 + M).random_profile(M)
        costs = P.quantize_emissions(hmm, q)
        with P.Scanner(0) as s:
            s.set_profile(costs, q, hmm.lambda_, hmm.tau)
            s.set_database(db)
            row = []
            for v in (P.Variant.Fp16, P.Variant.Fp16x, P.Variant.Fp16xAlt, P.Variant.Auto):
                o = P.ScanOptions(alg=P.Algorithm.Msv, variant=v)
                s.scan(o)
                r = min((s.scan(o) for _ in range(3)), key=lambda r: r.elapsed_seconds)
                row.append((v.name, round(r.gcups), r.lanes, r.rows, r.variant))
            print(qs, M, row, flush=True)
