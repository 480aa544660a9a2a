#!/usr/bin/env python
"""One scan configuration repeated a few times (for ncu captures): the 1M
Swiss-Prot-like set (seed 0x5EED), model seed 7000+M."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_09683_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=400)
ap.add_argument("--alg", default="msv")
ap.add_argument("--quant", default="default", choices=["default", "nonsat"])
ap.add_argument("--variant", default="auto")
ap.add_argument("--lanes", type=int, default=0)
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--nseq", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
db = P.Rng(0x5EED).lognormal_records(a.nseq, 290, 0.65, 2)
hmm = P.Rng(7000 + a.m).random_profile(a.m)
q = P.QuantParams() if a.quant == "default" else P.QuantParams(3.0, 120, 3, 20, 20)
var = {"auto": P.Variant.Auto, "fp16": P.Variant.Fp16, "fp16x": P.Variant.Fp16x,
       "fp16xm": P.Variant.Fp16xMixed, "fp16xh": P.Variant.Fp16xHybrid,
       "fp16xr": P.Variant.Fp16xRelaxed, "fp16xrm": P.Variant.Fp16xRelaxedFixedB,
       "dpx16": P.Variant.Dpx16}[a.variant]
with P.Scanner(0) as s:
    s.set_profile(P.quantize_emissions(hmm, q), q, hmm.lambda_, hmm.tau)
    s.set_database(db)
    for _ in range(a.reps):
        r = s.scan(P.ScanOptions(alg=P.Algorithm.Msv if a.alg == "msv" else P.Algorithm.Ssv,
                                 variant=var, lanes=a.lanes, rows=a.rows))
        print(r.lanes, r.rows, r.variant, round(r.gcups, 1), flush=True)
