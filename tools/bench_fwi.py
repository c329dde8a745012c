#!/usr/bin/env python
"""NEXT-3 measurement: the adjoint-state FWI gradient (aw_fwi_gradient) on B200.

    python tools/bench_fwi.py [--workload C3|C2] [--nt N] [--steps K] [--warmup W] [--ckpt K]

One "step" = one whole gradient: forward run with checkpoints, residual and
misfit, checkpoint replays, time-reversed adjoint run with the imaging
condition, gradient finalisation.  Inputs are resident in HBM (model, observed
traces); the observed traces are the GPU forward traces of a model 2 % faster
in a central sphere (synthetic).  value = grid points x time steps / s of the
gradient.  The algorithmic HBM bytes of one gradient are summed per kernel
(DESIGN.md §4): 16 B/pt per stencil step (forward, replay, adjoint), 24 B/pt
per imaging launch, 8 B/pt per checkpoint level copy (read + write) -- their
sum over the CUDA-event time of the gradient gives the composite roofline
fraction against MEASURED_PEAKS.json (else the profiling guide's fallback).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3", choices=["C3", "C2"])
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--ckpt", type=int, default=0)
    args = ap.parse_args()

    import torch
    from paper_1906_10811_b200 import build
    build.build()
    import paper_1906_10811_b200 as aw
    import workloads as W
    import bench

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if args.workload == "C3":
        base = W.c3(with_arrays=False)
        shape, so, nbl = base.shape, 8, 32
        m = W.random_smooth_m(shape, device="cuda")
    else:
        base = W.c2()
        shape, so, nbl = base.shape, 4, 16
        m = torch.from_numpy(base.m).to(dev)
    nt = args.nt or base.nt
    damp = torch.from_numpy(W.damping_profile(shape, nbl)).to(dev)
    zz, yy, xx = torch.meshgrid(*[torch.arange(n, device=dev, dtype=torch.float32) for n in shape], indexing="ij")
    r2 = sum((c - (n - 1) / 2) ** 2 for c, n in zip((zz, yy, xx), shape))
    sphere = r2 < (0.2 * shape[0]) ** 2
    m_true = torch.where(sphere, m / 1.0404, m).contiguous()  # v * 1.02 inside the sphere
    del zz, yy, xx, r2, sphere
    wav = torch.from_numpy(W.ricker(nt, base.dt, base.f0, ns=len(base.src_coords))).to(dev)
    extent = [10.0 * (n - 1) for n in shape]
    stream = torch.cuda.current_stream()
    g = aw.Grid(shape, extent, so, device=0, stream=stream)
    if args.ckpt:
        g.set_option(aw.AW_OPT_CHECKPOINT_STEPS, args.ckpt)
    nr = len(base.rec_coords)
    g.add_sources(base.src_coords, wav)
    g.add_receivers(base.rec_coords, nt)
    g.set_model(m_true, damp)
    g.run(nt, base.dt)
    dobs = torch.zeros((nt, nr), dtype=torch.float32, device=dev)
    g.read_receivers(out=dobs)
    g.set_model(m, damp)
    grad = torch.zeros(shape, dtype=torch.float32, device=dev)
    res = torch.zeros((nt, nr), dtype=torch.float32, device=dev)
    J = None
    for _ in range(args.warmup):
        _, _, J = g.fwi_gradient(nt, base.dt, dobs, grad=grad, residual=res)
    torch.cuda.synchronize()
    clocks = bench.Clocks(0)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        _, _, J = g.fwi_gradient(nt, base.dt, dobs, grad=grad, residual=res)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    st = g.stats()
    K = st["fwi_checkpoint"]
    nseg = (nt + K - 1) // K
    N = float(np.prod(shape))
    stencil_steps = st["fwi_steps"]
    alg_bytes = N * (16.0 * stencil_steps + 24.0 * nt + 8.0 * 4 * (nseg - 1))  # 4 level copies per boundary
    peak, peak_src = bench.load_peaks()
    achieved = alg_bytes / (ms * 1e-3) / 1e9
    line = {
        "metric": "FWI gradient throughput (grid points x time steps / s)", "value": round(N * nt / (ms * 1e-3) / 1e9, 3),
        "unit": "Gpts/s", "ms_per_gradient": round(ms, 2), "steps": args.steps, "warmup": args.warmup,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.workload, "shape": list(shape), "space_order": so, "time_steps": nt,
                   "checkpoint_steps": K, "segments": nseg, "history_buffers": K + 2 + 2 * (nseg - 1),
                   "stencil_steps": stencil_steps, "receivers": nr,
                   "observed": "GPU forward traces of m with v x 1.02 in a central sphere"},
        "stencil_step_rate_gpts": round(N * stencil_steps / (ms * 1e-3) / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_src,
                     "bytes": "16 B/pt per stencil step + 24 B/pt per imaging + 8 B/pt per checkpoint level copy"},
        "J": J, "grad_absmax": float(grad.abs().max().item()), "gpu_launches_per_gradient": st["launches"],
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    g.close()


if __name__ == "__main__":
    main()
