#!/usr/bin/env python
"""Where the end-to-end time of a C2 step goes: per model (SSV, M = 1000 /
400 / 48 over the 1M Swiss-Prot-like set), the resident scan into device
buffers, the resident scan with page-locked host outputs, and the streamed
scan (H2D of the packed image under the kernel), each as the library's
device time and a host clock around the synchronous call (median of 10)."""
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_09683_b200 as P  # noqa: E402


def timed(fn, reps=10):
    dev, wall = [], []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        wall.append((time.perf_counter() - t0) * 1e3)
        st = r if isinstance(r, dict) else r.stats  # (scan_device returns the stats dict)
        dev.append(st["device_ms"])
    return round(statistics.median(dev), 3), round(statistics.median(wall), 3)


def main():
    db = P.Rng(0x5EED).lognormal_records(1_000_000, 290, 0.65, 2)
    q = P.QuantParams()
    with P.Scanner(0) as s:
        s.set_database(db)
        n = s.n_local
        raw = torch.empty(n, dtype=torch.uint8, device="cuda")
        pas = torch.empty(n, dtype=torch.uint8, device="cuda")
        host = (torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy(),
                torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy())
        o = P.ScanOptions(alg=P.Algorithm.Ssv, threshold=0.022)
        for m in (1000, 400, 48):
            hmm = P.Rng(7000 + m).random_profile(m)
            s.set_profile(P.quantize_emissions(hmm, q), q, hmm.lambda_, hmm.tau)
            for _ in range(2):
                s.scan(o)
            row = {"M": m,
                   "device_outputs": timed(lambda: s.scan_device(o, raw.data_ptr(), pas.data_ptr())),
                   "host_outputs": timed(lambda: s.scan(o, out=host)),
                   "streamed": timed(lambda: s.scan_streamed(o, 64, out=host))}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
