#!/usr/bin/env python
"""Geometry / variant sweep on one GPU: for each (alg, M, variant, lanes[, rows])
measure device GCUPS over the 1M Swiss-Prot-like database (the B200
analogue of the reference's calibrate_hmax, src/select.cpp:80-105).
Writes one JSON line per point to stdout."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1707_09683_b200 as P  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "paper_1707_09683_b200", "csrc"))
import gen_instances  # noqa: E402

ROWS = {P.Variant.Dpx16: gen_instances.ROWS["dpx16"], P.Variant.Fp16: gen_instances.ROWS["fp16"],
        P.Variant.Swar8: gen_instances.ROWS["swar8"], P.Variant.Fp16x: gen_instances.ROWS["fp16x"],
        P.Variant.Fp16xAlt: gen_instances.ROWS["fp16xalt"],
        P.Variant.Fp16xMixed: gen_instances.ROWS["fp16xm"],
        P.Variant.Fp16xHybrid: gen_instances.ROWS["fp16xh"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nseq", type=int, default=1_000_000)
    ap.add_argument("--models", default="48,100,200,400,800,1000,1500,2000,2405")
    ap.add_argument("--algs", default="msv,ssv")
    ap.add_argument("--variants", default="dpx16,fp16,swar8")
    ap.add_argument("--extra-rows", type=int, default=0, help="also try the next N larger H")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    db = P.Rng(0x5EED).lognormal_records(args.nseq, 290, 0.65, 2)
    q = P.QuantParams()
    s = P.Scanner(0)
    s.set_database(db)
    res = db.total_residues()
    vmap = {"dpx16": P.Variant.Dpx16, "fp16": P.Variant.Fp16, "swar8": P.Variant.Swar8,
            "fp16x": P.Variant.Fp16x, "fp16xalt": P.Variant.Fp16xAlt,
            "fp16xm": P.Variant.Fp16xMixed, "fp16xh": P.Variant.Fp16xHybrid}
    for m in [int(x) for x in args.models.split(",")]:
        hmm = P.Rng(7000 + m).random_profile(m)
        costs = P.quantize_emissions(hmm, q)
        s.set_profile(costs, q, hmm.lambda_, hmm.tau)
        ref_raw = {}
        for a in args.algs.split(","):
            alg = P.Algorithm.Msv if a == "msv" else P.Algorithm.Ssv
            for vn in args.variants.split(","):
                v = vmap[vn]
                cpw = 4 if v == P.Variant.Swar8 else 2
                auto = P.select_geometry(m, alg, v)
                for L in (1, 2, 4, 8, 16, 32):
                    hs = [h for h in ROWS[v] if cpw * L * h >= m]
                    for H in hs[:1 + args.extra_rows]:
                        try:
                            opt = P.ScanOptions(alg=alg, variant=v, lanes=L, rows=H)
                            rep = s.scan(opt)  # warm-up (and table staging)
                            ms = []
                            for _ in range(args.reps):
                                r = s.scan(opt)
                                ms.append(r.stats["device_ms"])
                            key = a
                            if key in ref_raw:
                                same = bool(np.array_equal(ref_raw[key], r.raw))
                            else:
                                ref_raw[key] = r.raw.copy()
                                same = True
                            t = min(ms)
                            print(json.dumps({"alg": a, "M": m, "variant": vn, "lanes": L,
                                              "rows": H, "auto": [L, H] == list(auto),
                                              "ms": round(t, 4),
                                              "gcups": round(res * m / (t * 1e-3) / 1e9, 1),
                                              "grid": r.stats["grid"],
                                              "smem": r.stats["smem_bytes"],
                                              "agree": same}), flush=True)
                        except Exception as e:  # noqa: BLE001
                            print(json.dumps({"alg": a, "M": m, "variant": vn, "lanes": L,
                                              "rows": H, "error": str(e)}), flush=True)
    s.close()


if __name__ == "__main__":
    main()
