"""Developer check: streaming kernel vs v1 kernel (value-identical) for every R.

    python tools/kernel_check.py [--shapes small|all] [--R 1,2,...]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--shapes", default="small")
    ap.add_argument("--nt", type=int, default=20)
    args = ap.parse_args()
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    shapes = [(40, 36, 72), (33, 70, 130), (21, 19, 23)]
    if args.shapes == "big":
        shapes = [(40, 36, 72), (33, 70, 130)]
    if args.shapes == "all":
        shapes += [(64, 64, 64), (130, 129, 131)]
    for R in [int(r) for r in args.R.split(",")]:
        k = 2 * R
        for shape in shapes:
            if min(shape) < R + 1:
                continue
            w = workloads.small_case(shape, k, args.nt, nbl=max(3, R), ns=2, nr=5)
            outs = []
            for kern in (aw.AW_KERNEL_V1, aw.AW_KERNEL_STREAM):
                g = aw.Grid(w.shape, w.extent, k)
                g.set_option(aw.AW_OPT_KERNEL, kern)
                g.set_model(w.m, w.damp)
                g.add_sources(w.src_coords, w.wavelet)
                g.add_receivers(w.rec_coords, w.nt)
                t = time.time()
                try:
                    g.run(w.nt, w.dt)
                    outs.append((g.read_wavefield(0), g.read_receivers()))
                except Exception as e:  # noqa: BLE001
                    print(f"R={R} shape={shape} kernel={kern}: ERROR {e}", flush=True)
                    outs.append(None)
                g.close()
            if outs[0] is None or outs[1] is None:
                continue
            du = np.argwhere(outs[0][0] != outs[1][0])
            dr = np.argwhere(outs[0][1] != outs[1][1])
            status = "OK" if du.size == 0 and dr.size == 0 else f"MISMATCH u:{len(du)} rec:{len(dr)} first {du[:3].tolist()}"
            print(f"R={R} shape={shape}: {status}", flush=True)


if __name__ == "__main__":
    main()
