"""NEXT-2 bench: the paper's own benchmark: 2D diffusion, 1000 time
steps, 2500^2 and 10000^2 grids, space order swept, fp32.  One JSON line per case.

    python tools/bench_diffusion.py [--sizes 2500,10000] [--orders 2,4,8,12] [--nt 1000] [--reps 3]

Metric: grid-point updates/s; roofline: 8 algorithmic B per point update (read u^n,
write u^{n+1}) over the kernel's per-launch CUDA-event time vs MEASURED_PEAKS.json.
Paper context (GTX 1080, 320 GB/s): "peak utilisation" 62% (lowest so) to 28%
(highest so) with divisions hoisted, 20%/7% without.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2500,10000")
    ap.add_argument("--orders", default="2,4,8,12")
    ap.add_argument("--nt", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    from paper_1906_10811_b200.diffusion import Diffusion
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for n in [int(s) for s in args.sizes.split(",")]:
        shape = (n, n)
        extent = (1.0, 1.0)  # Devito's default Grid extent (PAPER.md:739 passes only shape)
        x = torch.linspace(0, 1, n, device="cuda")
        u0 = torch.exp(-((x[:, None] - 0.5) ** 2 + (x[None, :] - 0.5) ** 2) / 0.02).float().contiguous()
        for k in [int(s) for s in args.orders.split(",")]:
            c = np.array([float(v) for v in _weights(k)])
            S = abs(c[0]) + 2 * np.abs(c[1:]).sum()
            h = 1.0 / (n - 1)
            nu = 0.5
            dt = 0.9 * 2 / (nu * 2 * S / h ** 2)
            d = Diffusion(shape, extent, k, nu, stream=torch.cuda.current_stream())
            d.set_option(aw.AW_OPT_TIMING, 1)
            d.set(u0)
            d.run(20, dt)  # warm-up (+ event pool)
            best = None
            for _ in range(args.reps):
                d.set(u0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                d.run(args.nt, dt)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                st = d.stats()
                if best is None or ms < best[0]:
                    best = (ms, st)
            ms, st = best
            kern = st["ms_stencil"] / max(1, st["n_stencil"])
            pts = n * n
            ach = 8 * pts / (kern * 1e-3) / 1e9
            print(json.dumps({"workload": f"diffusion {n}x{n}", "space_order": k, "time_steps": args.nt,
                              "value": round(pts * args.nt / (ms * 1e-3) / 1e9, 2), "unit": "Gpts/s",
                              "kernel_ms_avg": round(kern, 4),
                              "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                                           "frac": round(ach / peak, 4), "bytes_per_point": 8}}), flush=True)
            d.close()


def _weights(k):
    from fractions import Fraction
    from math import factorial
    m = k // 2
    cs = [Fraction(2 * factorial(m) ** 2 * (1 if j % 2 else -1), j * j * factorial(m - j) * factorial(m + j))
          for j in range(1, m + 1)]
    return [-2 * sum(cs)] + cs


if __name__ == "__main__":
    main()
