#!/usr/bin/env python
"""NEXT-1 tuning sweep: ms per two-step pass of the temporal-blocking kernel on C3 for chunk
sizes Z (AW_TB_Z) and B lags (AW_TB_LEAD), next to the one-step kernel (CUDA events per launch).

    python tools/tb_sweep.py [--nt 40] [--z 16,24,32] [--lead 1,2]
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
    ap.add_argument("--nt", type=int, default=40)
    ap.add_argument("--z", default="16,24,32,48")
    ap.add_argument("--lead", default="1,2")
    ap.add_argument("--so", type=int, default=8)
    ap.add_argument("--shape", default="512,512,512")
    args = ap.parse_args()
    import torch
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    import workloads as W
    base = W.c3(with_arrays=False)
    shape = tuple(int(v) for v in args.shape.split(","))
    m = W.random_smooth_m(shape, device="cuda")
    damp = torch.from_numpy(W.damping_profile(shape, 32)).cuda()
    wav = torch.from_numpy(W.ricker(args.nt, base.dt, base.f0)).cuda()
    extent = [10.0 * (n - 1) for n in shape]
    N = float(np.prod(shape))
    h = 10.0
    src = np.array([[h * (shape[0] - 1) / 2 + 0.3, h * (shape[1] - 1) / 2 + 0.7, h * (shape[2] - 1) / 2 + 0.1]])
    rec = np.array([[400.5, h * (shape[1] - 1) / 2, h * r] for r in range(shape[2])])

    def measure(temporal, env):
        for k in ("AW_TB_Z", "AW_TB_LEAD"):
            os.environ.pop(k, None)
        os.environ.update(env)
        g = aw.Grid(shape, extent, args.so, device=0)
        g.set_option(aw.AW_OPT_TEMPORAL, temporal)
        g.set_option(aw.AW_OPT_TIMING, 1)
        g.set_model(m, damp)
        g.add_sources(src, wav)
        g.add_receivers(rec, args.nt)
        g.run(args.nt, base.dt)  # warm-up (plan, maps)
        g.reset()
        g.run(args.nt, base.dt)
        st = g.stats()
        g.close()
        per_step = st["ms_stencil"] / st["n_stencil"]
        return {"shape": list(shape), "temporal": temporal, **env, "ms_per_step": round(per_step, 4),
                "gpts": round(N / (per_step * 1e-3) / 1e9, 1), "run_ms": round(st["ms_total"], 2)}

    print(json.dumps(measure(0, {})), flush=True)
    for z in args.z.split(","):
        for lead in args.lead.split(","):
            print(json.dumps(measure(1, {"AW_TB_Z": z, "AW_TB_LEAD": lead})), flush=True)


if __name__ == "__main__":
    main()
