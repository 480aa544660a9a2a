#!/usr/bin/env python
"""Where the end-to-end time of a bench step goes (C2 by default): per model,
the resident device scan (device outputs), the resident scan with host
outputs, and the streamed scan (H2D under the kernel), each timed with a
host clock around a synchronised call and with the library's device time."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1707_09683_b200 as P  # noqa: E402


def main():
    wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    alg, models_m, gen = wl[1], wl[2], wl[4]
    q = P.QuantParams()
    db = bench.make_db(P, gen, 1_000_000)
    models = bench.make_models(P, models_m, q)
    s = P.Scanner(0)
    s.set_stream(torch.cuda.current_stream().cuda_stream)
    s.set_database(db)
    pids = [s.add_profile(c, q, h.lambda_, h.tau) for h, c in models]
    n = db.count
    raw = torch.empty(n, dtype=torch.uint8, device="cuda")
    pas = torch.empty(n, dtype=torch.uint8, device="cuda")
    pinned = (torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy(),
              torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy())
    a = P.Algorithm.Msv if alg == "msv" else P.Algorithm.Ssv
    opt = P.ScanOptions(alg=a, threshold=0.022)

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev = 0.0
        for _ in range(reps):
            st = fn()
            dev += st if isinstance(st, float) else 0.0
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3, dev / reps

    for pid, (h, _) in zip(pids, models):
        s.select_profile(pid)
        w1, d1 = timed(lambda: s.scan_device(opt, raw.data_ptr(), pas.data_ptr())["device_ms"])
        w2, d2 = timed(lambda: s.scan(opt).elapsed_seconds * 1e3)
        w3, d3 = timed(lambda: s.scan_streamed(opt, 64).elapsed_seconds * 1e3)
        w4, d4 = timed(lambda: s.scan(opt, out=pinned).elapsed_seconds * 1e3)
        w5, d5 = timed(lambda: s.scan_streamed(opt, 64, out=pinned).elapsed_seconds * 1e3)
        print(f"M={h.length}: device-out wall {w1:.3f} ms (dev {d1:.3f}); host-out wall {w2:.3f} "
              f"(dev {d2:.3f}); streamed wall {w3:.3f} (dev {d3:.3f}); pinned host-out wall "
              f"{w4:.3f}; pinned streamed wall {w5:.3f}", flush=True)


if __name__ == "__main__":
    main()
