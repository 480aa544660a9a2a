#!/usr/bin/env python
"""Two-mode MSV rates per mode: a profile that saturates on the first rows
(lazy mode throughout), one that never saturates (exact mode throughout)
and the default parameters, for FP16X and FP16XM at L=32, H=38/48."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1707_09683_b200 as P
db = P.Rng(0x5EED).lognormal_records(400000, 290, 0.65, 2)
s = P.Scanner(0); s.set_database(db); res = db.total_residues()
for qn, q in (("lazy", P.QuantParams(3.0, 252, 3, 0, 0)), ("exact", P.QuantParams(3.0, 120, 3, 20, 20)), ("default", P.QuantParams())):
    for v, H in ((P.Variant.Fp16x, 38), (P.Variant.Fp16xMixed, 38), (P.Variant.Fp16x, 48), (P.Variant.Fp16xMixed, 48)):
        m = 2 * 32 * H
        hmm = P.Rng(9000 + m).random_profile(m)
        s.set_profile(P.quantize_emissions(hmm, q), q, hmm.lambda_, hmm.tau)
        opt = P.ScanOptions(alg=P.Algorithm.Msv, variant=v, lanes=32, rows=H)
        s.scan(opt)
        t = min(s.scan(opt).stats["device_ms"] for _ in range(3))
        r = s.scan(opt)
        sat = (r.raw == 255).mean()
        print(qn, v.name, H, round(res * m / (t * 1e-3) / 1e9), "sat", round(float(sat), 3), flush=True)
