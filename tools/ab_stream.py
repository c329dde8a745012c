#!/usr/bin/env python
"""Same-box A/B of two libaw builds: ms per launch of the one-step 3D streaming kernel on a
512^3 grid (random smooth model, nbl 32, one source, a receiver line) for each space order.

    python tools/ab_stream.py --libs new=paper_1906_10811_b200/libaw.so,old=/path/libaw_old.so \
        [--so 2,4,8,12,16] [--nt 40] [--rounds 2]
    (a library entry name=path@V also sets AW_STREAM_VARIANT=V for that arm)

Each (library, so) measurement runs in its own process (AW_LIBRARY selects the build), and the
libraries alternate within every round so clock/power drift hits both alike.  Prints one JSON
line per measurement; the per-launch time is the library's own CUDA-event timing of the
stencil launches (AW_OPT_TIMING).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(so, nt, shape):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_1906_10811_b200 as aw
    import workloads as W
    base = W.c3(with_arrays=False)
    m = W.random_smooth_m(shape, device="cuda")
    damp = torch.from_numpy(W.damping_profile(shape, 32)).cuda()
    wav = torch.from_numpy(W.ricker(nt, base.dt, base.f0)).cuda()
    extent = [10.0 * (n - 1) for n in shape]
    h = 10.0
    src = np.array([[h * (shape[0] - 1) / 2 + 0.3, h * (shape[1] - 1) / 2 + 0.7, h * (shape[2] - 1) / 2 + 0.1]])
    rec = np.array([[min(400.5, h * (shape[0] - 1)), h * (shape[1] - 1) / 2, h * r] for r in range(shape[2])])
    g = aw.Grid(shape, extent, so, device=0)
    g.set_model(m, damp)
    g.add_sources(src, wav)
    g.add_receivers(rec, nt)
    n = float(np.prod(shape))
    res = {"so": so}
    # events: per-launch CUDA events (direct launches); graph: whole-run time / nt on the production
    # path (CUDA graphs of 16 steps), i.e. launch gaps included
    for mode, opt in (("events", 1), ("graph", 0)):
        g.set_option(aw.AW_OPT_TIMING, opt)
        g.reset()
        g.run(nt, base.dt)  # warm-up (plan, maps, graphs)
        best = None
        for _ in range(3):
            g.reset()
            g.run(nt, base.dt)
            st = g.stats()
            ms = st["ms_stencil"] / st["n_stencil"] if opt else st["ms_total"] / nt
            best = ms if best is None else min(best, ms)
        res[f"ms_{mode}"] = round(best, 4)
        res[f"gpts_{mode}"] = round(n / (best * 1e-3) / 1e9, 1)
    g.close()
    res["hbm_frac_16B_6537"] = round(n / (res["ms_events"] * 1e-3) * 16 / 6537e9, 3)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default="new=" + os.path.join(ROOT, "paper_1906_10811_b200", "libaw.so"))
    ap.add_argument("--so", default="2,4,8,12,16")
    ap.add_argument("--nt", type=int, default=40)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--shape", default="512,512,512")
    ap.add_argument("--child", type=int, default=0)
    args = ap.parse_args()
    shape = tuple(int(v) for v in args.shape.split(","))
    if args.child:
        print(json.dumps(child(args.child, args.nt, shape)), flush=True)
        return
    libs = [kv.split("=", 1) for kv in args.libs.split(",")]
    for rnd in range(args.rounds):
        for so in (int(s) for s in args.so.split(",")):
            for name, path in libs:
                path, _, var = path.partition("@")  # name=path@V: with AW_STREAM_VARIANT=V
                env = dict(os.environ, AW_LIBRARY=os.path.abspath(path))
                if var:
                    env["AW_STREAM_VARIANT"] = var
                out = subprocess.run([sys.executable, __file__, "--child", str(so), "--nt", str(args.nt),
                                      "--shape", args.shape], env=env, capture_output=True, text=True)
                line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else ""
                try:
                    rec = json.loads(line)
                except ValueError:
                    rec = {"so": so, "error": (out.stderr or out.stdout)[-400:]}
                print(json.dumps({"lib": name, "round": rnd, **rec}), flush=True)


if __name__ == "__main__":
    main()
