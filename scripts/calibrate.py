#!/usr/bin/env python
"""Calibration sweep for the B200 geometry policy (the analogue of the
reference's calibrate_hmax, src/select.cpp:80-105): for every instantiated
(variant, alg, L, H) measure device GCUPS on the 1M Swiss-Prot-like set with
a model that exactly fills the geometry (M = CPW*L*H, capped at 2405), and
report computed-cell efficiency = GCUPS * capacity / M.  Output: JSON lines."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "paper_1707_09683_b200", "csrc"))

import gen_instances  # noqa: E402
import paper_1707_09683_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nseq", type=int, default=1_000_000)
    ap.add_argument("--variants", default="fp16")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--algs", default="msv,ssv")
    ap.add_argument("--lanes", default="", help="subset of lane counts, e.g. 16,32")
    ap.add_argument("--quant", default="default", choices=["default", "nonsat"],
                    help="nonsat = QuantParams{3,120,3,20,20} (MSV scores that do not saturate: "
                         "the regime the relaxed FP16XR kernel is chosen for)")
    args = ap.parse_args()
    lanes = [int(x) for x in args.lanes.split(",")] if args.lanes else gen_instances.LANES
    db = P.Rng(0x5EED).lognormal_records(args.nseq, 290, 0.65, 2)
    q = P.QuantParams() if args.quant == "default" else P.QuantParams(3.0, 120, 3, 20, 20)
    s = P.Scanner(0)
    s.set_database(db)
    res = db.total_residues()
    vmap = {"dpx16": P.Variant.Dpx16, "fp16": P.Variant.Fp16, "swar8": P.Variant.Swar8,
            "fp16x": P.Variant.Fp16x, "fp16xalt": P.Variant.Fp16xAlt,
            "fp16xm": P.Variant.Fp16xMixed, "fp16xh": P.Variant.Fp16xHybrid,
            "fp16xr": P.Variant.Fp16xRelaxed, "fp16xrm": P.Variant.Fp16xRelaxedFixedB}
    for vn in args.variants.split(","):
        cpw = 4 if vn == "swar8" else 2
        for L in lanes:
            for H in gen_instances.ROWS[vn]:
                cap = cpw * L * H
                m = min(cap, 4096)
                hmm = P.Rng(9000 + m).random_profile(m)
                s.set_profile(P.quantize_emissions(hmm, q), q, hmm.lambda_, hmm.tau)
                for a in args.algs.split(","):
                    alg = P.Algorithm.Msv if a == "msv" else P.Algorithm.Ssv
                    opt = P.ScanOptions(alg=alg, variant=vmap[vn], lanes=L, rows=H)
                    try:
                        s.scan(opt)
                        t = min(s.scan(opt).stats["device_ms"] for _ in range(args.reps))
                    except Exception as e:  # noqa: BLE001  (e.g. table too large)
                        print(json.dumps({"variant": vn, "alg": a, "lanes": L, "rows": H,
                                          "error": str(e)}), flush=True)
                        continue
                    g = res * m / (t * 1e-3) / 1e9
                    print(json.dumps({"variant": vn, "alg": a, "lanes": L, "rows": H, "M": m,
                                      "quant": args.quant,
                                      "gcups": round(g, 1),
                                      "cell_gcups": round(g * cap / m, 1)}), flush=True)
    s.close()


if __name__ == "__main__":
    main()
