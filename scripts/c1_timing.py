#!/usr/bin/env python
"""Where does a small-database (C1) scan's device time go?  Times the same
auto-policy MSV scan three ways: the C ABI's own CUDA-event window
(device_ms), torch events around the whole ABI call on the same stream, and
(under `ncu --metrics gpu__time_duration.sum`) the kernel alone."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1707_09683_b200 as P  # noqa: E402

torch.cuda.set_stream(torch.cuda.Stream())


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = P.Rng(0xC1)
    hmm = rng.random_profile(200)
    db = rng.random_records(10000, 50, 650, plant=(hmm, 0.05))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    raw = torch.empty(db.count, dtype=torch.uint8, device="cuda")
    ps = torch.empty(db.count, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    s = P.Scanner(0)
    s.set_stream(st.cuda_stream)
    s.set_database(db)
    q = P.QuantParams()
    s.set_profile(P.quantize_emissions(hmm, q), q, hmm.lambda_, hmm.tau)
    for alg in (P.Algorithm.Msv, P.Algorithm.Ssv):
        opt = P.ScanOptions(alg=alg)
        for _ in range(5):
            s.scan_device(opt, raw.data_ptr(), ps.data_ptr())
        for mode in ("flush+sleep", "flush", "none"):
            abi, outer = [], []
            for _ in range(reps):
                if mode != "none":
                    flush.fill_(1)
                if mode == "flush+sleep":
                    torch.cuda._sleep(100000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                d = s.scan_device(opt, raw.data_ptr(), ps.data_ptr())
                e1.record(st)
                torch.cuda.synchronize()
                abi.append(d["device_ms"])
                outer.append(e0.elapsed_time(e1))
            print(json.dumps({"alg": alg.name, "mode": mode,
                              "abi_ms_med": round(statistics.median(abi), 4),
                              "abi_ms_min": round(min(abi), 4),
                              "outer_ms_med": round(statistics.median(outer), 4),
                              "outer_ms_min": round(min(outer), 4),
                              "lanes": d["lanes"], "rows": d["rows"], "variant": d["variant"]}),
                  flush=True)
    s.close()


if __name__ == "__main__":
    main()
