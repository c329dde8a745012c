"""Parity at the benchmark configurations, at full size, with data everywhere (test infrastructure).

SURVEY.md:539 asks for parity at C3-C5 "with the full nt whenever the oracle finished; otherwise
nt=100".  A run from rest with one point source leaves almost the whole production grid at 0 for
the first hundreds of steps, so here both sides start from the SAME seeded random levels u^0, u^-1
(uniform in [-1, 1], every tile, z chunk and damping tile-plane carries data) plus the config's
Ricker source, its receivers and two receiver lines through the source.  The CUDA path runs in the
bench's launch configuration (default options: streaming kernel, CUDA graphs of 16 steps, fused
sparse work); the oracle is oracle.run(FP32CANON).  Contract: relL2 <= 1e-5
for the wavefield and the traces (BASELINE.json:5), and the design claim is value identity.

    python -m tests.parity_full [--cases C3,C5,C4g] [--out profiles/r2/parity_full.jsonl]

This module imports the oracle, so it lives under tests/ (only tests/, smoke() and bench.py's CPU
legs may run the oracle).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402

# (config, shape override, steps): C3 and C5 at their full 512^3 size; "C4g" = the C4 plane
# geometry (1024 x 1024, so 12) with 96 planes of axis 0 so the oracle fits the host's time budget
CASES = {
    "C3": dict(make=lambda: workloads.c3(nt=100, with_arrays=False), shape=(512, 512, 512), nt=100),
    "C5": dict(make=lambda: workloads.c5(1, nt=50, with_arrays=False), shape=(512, 512, 512), nt=50),
    "C4g": dict(make=lambda: workloads.c4(nt=12, with_arrays=False), shape=(96, 1024, 1024), nt=12),
}


def max_ulp(a, b) -> int:
    """Largest distance in units in the last place between two fp32 arrays (+0 == -0)."""
    ia = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    ib = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    # map the sign-magnitude ordering onto a monotone integer line
    ia = np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)
    ib = np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    return int(np.max(np.abs(ia - ib))) if ia.size else 0


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def build_case(name: str, seed: int = 539):
    spec = CASES[name]
    w = spec["make"]()
    shape, nt = spec["shape"], spec["nt"]
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    m = workloads.random_smooth_m(shape, device=dev)  # the config's recipe at this shape (one array, both sides)
    w.m = m.cpu().numpy() if hasattr(m, "cpu") else m
    w.damp = workloads.damping_profile(shape, w.nbl)
    w.shape = shape
    w.extent = tuple(workloads.H * (n - 1) for n in shape)
    w.nt = nt
    w.wavelet = np.ascontiguousarray(w.wavelet[:nt])
    ext = w.extent
    # a source outside the reduced grid (C4g) moves to the middle of axis 0, off-node
    w.src_coords = np.array([[c if 0.0 <= c <= ext[d] else 0.5 * ext[d] + 0.3 for d, c in enumerate(s)]
                             for s in w.src_coords])
    # receivers: the config's lines that fit, plus two lines through the source (axis 2 and axis 0)
    src = w.src_coords[0]
    keep = [r for r in w.rec_coords if all(0.0 <= r[d] <= ext[d] for d in range(3))]
    through = [[src[0], src[1], 10.0 * r + 0.37] for r in range(shape[2] - 1)]
    through += [[10.0 * r + 0.61, src[1], src[2]] for r in range(shape[0] - 1)]
    w.rec_coords = np.array(keep + through, np.float64)
    rng = np.random.default_rng(seed)
    u0 = rng.uniform(-1.0, 1.0, size=shape).astype(np.float32)
    u1 = rng.uniform(-1.0, 1.0, size=shape).astype(np.float32)
    return w, u0, u1


def run_gpu(w, u0, u1):
    import paper_1906_10811_b200 as aw
    g = aw.Grid(w.shape, w.extent, w.space_order, w.origin)
    g.set_model(w.m, w.damp)
    g.add_sources(w.src_coords, w.wavelet)
    g.add_receivers(w.rec_coords, w.nt)
    g.set_wavefield(u0, u1)
    t = time.perf_counter()
    g.run(w.nt, w.dt)
    gpu_s = time.perf_counter() - t
    st = g.stats()
    out = g.read_wavefield(0), g.read_wavefield(1), g.read_receivers()
    g.close()
    return out, gpu_s, st


def run_oracle(w, u0, u1):
    t = time.perf_counter()
    u, up, rec = oracle.run(oracle.FP32CANON, w.shape, w.extent, w.space_order, w.m, w.dt, w.nt, damp=w.damp,
                            origin=w.origin, src_coords=w.src_coords, wavelet=w.wavelet, rec_coords=w.rec_coords,
                            u_cur=u0, u_prev=u1)
    return (u, up, rec), time.perf_counter() - t


def compare(name: str) -> dict:
    w, u0, u1 = build_case(name)
    (gu, gup, grec), gpu_s, st = run_gpu(w, u0, u1)
    (ou, oup, orec), oracle_s = run_oracle(w, u0, u1)
    return {
        "workload": name, "shape": list(w.shape), "space_order": w.space_order, "nt": w.nt,
        "init": "seeded uniform[-1,1] u^0, u^-1 (seed 539) + the config's source", "nr": int(len(w.rec_coords)),
        "kernel": int(st["kernel"]), "launches": int(st["launches"]),
        "relL2_wave": rel_l2(gu, ou), "relL2_wave_prev": rel_l2(gup, oup), "relL2_rec": rel_l2(grec, orec),
        "maxulp_wave": max_ulp(gu, ou), "maxulp_rec": max_ulp(grec, orec),
        "n_diff_wave": int(np.count_nonzero(gu != ou)), "n_diff_rec": int(np.count_nonzero(grec != orec)),
        "nonzero_frac_wave": float(np.count_nonzero(ou)) / ou.size,
        "nonzero_frac_rec": float(np.count_nonzero(orec)) / max(orec.size, 1),
        "gpu_run_s": round(gpu_s, 3), "oracle_s": round(oracle_s, 1),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="C3,C5,C4g")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    for name in args.cases.split(","):
        rec = compare(name)
        line = json.dumps(rec)
        print(line, flush=True)
        if args.out:
            os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
            with open(args.out, "a") as f:
                f.write(line + "\n")


if __name__ == "__main__":
    main()
