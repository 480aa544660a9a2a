#!/usr/bin/env python
"""C1 geometry study (small database, latency-bound): BASELINE configs[0]
(MSV, M=200, 10k sequences, seed 0xC1) timed for every code form and lane
count at the smallest row count covering the model.  Each timed scan is
preceded by an L2 flush and a ~50 us device spin so the CUDA-event window
holds only the scan (the host enqueues while the GPU is busy).  JSON lines."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "paper_1707_09683_b200", "csrc"))

import gen_instances  # noqa: E402
import torch  # noqa: E402

import paper_1707_09683_b200 as P  # noqa: E402

torch.cuda.set_stream(torch.cuda.Stream())

VMAP = {"dpx16": P.Variant.Dpx16, "fp16": P.Variant.Fp16, "fp16x": P.Variant.Fp16x,
        "fp16xalt": P.Variant.Fp16xAlt, "fp16xm": P.Variant.Fp16xMixed,
        "fp16xh": P.Variant.Fp16xHybrid, "fp16xr": P.Variant.Fp16xRelaxed,
        "fp16xrm": P.Variant.Fp16xRelaxedFixedB,
        "auto": P.Variant.Auto}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=60)
    ap.add_argument("--variants", default="auto,fp16,fp16x,fp16xalt,fp16xm,fp16xh,fp16xr,dpx16")
    ap.add_argument("--algs", default="msv,ssv")
    ap.add_argument("--extra-rows", type=int, default=1, help="row counts beyond the smallest")
    ap.add_argument("--harness", action="store_true",
                    help="the reference acceptance harness's database instead (seed 0xBE5C+200, "
                         "3,000 records of 80..400 residues, acceptance_main.cpp:320-326)")
    args = ap.parse_args()
    if args.harness:
        rng = P.Rng(0xBE5C + 200)
        hmm = rng.random_profile(200)
        db = rng.random_records(3000, 80, 400)
    else:
        rng = P.Rng(0xC1)
        hmm = rng.random_profile(200)
        db = rng.random_records(10000, 50, 650, plant=(hmm, 0.05))
    cells = db.total_residues() * 200
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    raw = torch.empty(db.count, dtype=torch.uint8, device="cuda")
    ps = torch.empty(db.count, dtype=torch.uint8, device="cuda")
    s = P.Scanner(0)
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    s.set_database(db)
    for qn, q in (("default", P.QuantParams()), ("nonsat", P.QuantParams(3.0, 120, 3, 20, 20))):
        s.set_profile(P.quantize_emissions(hmm, q), q, hmm.lambda_, hmm.tau)
        for a in args.algs.split(","):
            alg = P.Algorithm.Msv if a == "msv" else P.Algorithm.Ssv
            for vn in args.variants.split(","):
                geos = [(0, 0)]
                if vn != "auto":
                    geos = []
                    for L in gen_instances.LANES:
                        hs = [h for h in gen_instances.ROWS[vn] if 2 * L * h >= 200]
                        geos += [(L, h) for h in hs[:1 + args.extra_rows]]
                for L, H in geos:
                    opt = P.ScanOptions(alg=alg, variant=VMAP[vn], lanes=L, rows=H)
                    try:
                        st = s.scan_device(opt, raw.data_ptr(), ps.data_ptr())
                        st = s.scan_device(opt, raw.data_ptr(), ps.data_ptr())
                    except Exception as e:  # noqa: BLE001
                        print(json.dumps({"q": qn, "alg": a, "variant": vn, "lanes": L,
                                          "rows": H, "error": str(e)}), flush=True)
                        continue
                    t = []
                    for _ in range(args.reps):
                        flush.fill_(1)
                        torch.cuda._sleep(100000)
                        t.append(s.scan_device(opt, raw.data_ptr(), ps.data_ptr())["device_ms"])
                    med = statistics.median(t)
                    print(json.dumps({"q": qn, "alg": a, "variant": vn,
                                      "lanes": st["lanes"], "rows": st["rows"],
                                      "form": int(st["variant"]), "grid": st["grid"],
                                      "ms_med": round(med, 4), "ms_min": round(min(t), 4),
                                      "gcups_med": round(cells / (med * 1e-3) / 1e9, 1)}),
                          flush=True)
    s.close()


if __name__ == "__main__":
    main()
