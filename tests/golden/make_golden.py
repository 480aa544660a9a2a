"""Generates tests/golden/oracle_golden.json from the UNMODIFIED reference
(oracle/_ref/liblanehmm_ref.so, built from /root/reference/proj/src):
inputs from the reference's own seeded generators (synth.cpp), raw scores
from its scalar oracle (oracle.cpp:41-91), pass bits from its finalize_hit
(engine.cpp:59-81) with the pipeline rule (engine.cpp:617).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

CASES = [
    # seed, m, generator, count, params, quant, plant fraction
    dict(seed=0xC1, m=200, gen="uniform", count=300, lo=50, hi=650,
         quant=[3.0, 195, 3, 3, 3], plant=0.05),
    dict(seed=0xC2, m=200, gen="uniform", count=300, lo=50, hi=650,
         quant=[3.0, 120, 3, 20, 20], plant=0.05),
    dict(seed=0xC3, m=48, gen="lognormal", count=300, median=290.0, sigma=0.65,
         quant=[3.0, 195, 3, 3, 3], plant=0.1),
    dict(seed=0xC4, m=400, gen="lognormal", count=200, median=290.0, sigma=0.65,
         quant=[2.0, 240, 10, 1, 5], plant=0.1),
    dict(seed=0xC5, m=1000, gen="uniform", count=120, lo=1, hi=400,
         quant=[3.0, 0, 0, 0, 0], plant=0.2),
    dict(seed=0xC6, m=2405, gen="uniform", count=60, lo=1, hi=300,
         quant=[3.0, 120, 3, 20, 20], plant=0.3),
    dict(seed=0xC7, m=7, gen="uniform", count=200, lo=1, hi=60,
         quant=[3.0, 195, 3, 3, 3], plant=0.0),
]
THRESHOLDS = ["0.0", "0.022", "0.103", "0.307", "0.458", "1.0"]


def main():
    ref = oracle.Reference()
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj",
           "cases": []}
    for c in CASES:
        g = ref.rng(c["seed"])
        s, lam, tau = g.random_profile(c["m"])
        plant = (s, c["plant"]) if c["plant"] else None
        if c["gen"] == "uniform":
            res, off = g.random_records(c["count"], c["lo"], c["hi"], plant=plant)
        else:
            res, off = g.lognormal_records(c["count"], c["median"], c["sigma"], 2, plant=plant)
        q = oracle.QuantParams(*c["quant"])
        costs = ref.quantize(s, q)
        case = dict(c)
        case["residue_sum"] = int(res.astype(np.uint64).sum())
        case["cost_sum"] = int(costs.astype(np.uint64).sum())
        lens = np.diff(off)
        for alg, key in ((0, "msv"), (1, "ssv")):
            raws = [ref.scalar(alg, costs, res[off[k]:off[k + 1]], q) for k in range(len(lens))]
            case[key] = raws
            case[f"pass_{key}"] = {}
            for t in THRESHOLDS:
                bits = []
                for r, n in zip(raws, lens):
                    _, p, ovf = ref.finalize(r, int(n), lam, tau, q, alg)
                    bits.append(bool(p <= float(t) or ovf))
                case[f"pass_{key}"][t] = bits
        out["cases"].append(case)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
