"""BASELINE config 3: degree sweep N = 1..7 in fp64 and fp32 on the warped
32^3 x 6 = 196,608-tet cube (one GPU), Gaussian pulse, fused LSRK stage.

Reports per (dtype, N): GDOF/s per RK stage, the fused kernel's HBM fraction
(algorithmic fused lower-bound bytes / time vs MEASURED_PEAKS hbm_gbs) and FP
fraction (algorithmic flops / time vs the measured FMA-pipe peak of
scripts/fma_peak.py), and the per-element storage of the WADG weights versus
dense per-element M_J^{-1} (solver.py:153-154 vs 166-167).

    python scripts/sweep.py [--n 32] [--steps 10] [--orders 1 2 ...] > sweep.json
"""

import argparse
import gc
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import bench  # noqa: E402
from paper_1608_03836_b200 import _native, meshgen, solver  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "scripts"))
import fma_peak  # noqa: E402


def run_point(mesh, N, dtype, steps, warmup=2):
    cfg = solver.SolverConfig(N=N, formulation=solver.Formulation.StrongWeak, dtype=dtype)
    disc = solver.Discretization(mesh, cfg)
    d = disc.dev
    Q = solver.project_initial_condition_device(disc, bench.gaussian_ic)
    stepper = solver.DeviceStepper(disc)
    dt = 0.5 * mesh.h / (N + 1) ** 2
    for _ in range(warmup):
        Q = stepper.step(Q, dt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        Q = stepper.step(Q, dt)
    e1.record()
    torch.cuda.synchronize()
    ms_stage = e0.elapsed_time(e1) / (5 * steps)
    ref = disc.ref
    K, Np, Nq = d.K, ref.Np, ref.Nq
    w = 4 if dtype == "float32" else 8
    F = ref.n_faces * ref.nfq
    B_F = K * (w * (16 * Np + 9 * Nq + Nq + 4 * F) + 16)
    _, FL = bench.algorithmic_model(3, K, Np, Nq, disc.ref_upd.Nq, F, w, 1)
    flops = sum(FL.values())
    e = solver.device_energy(disc, Q)
    return {
        "N": N, "dtype": dtype, "K": K, "Np": Np, "Nq": Nq,
        "fused_kernel": {0: "cuda-core", 2: "tcgen05 split-tf32", 3: "dmma f64", 4: "mma.sync split-tf32", 5: "register"}[getattr(d, "fused_kind", 0)],
        "ms_per_stage": ms_stage, "GDOF_s": 4 * K * Np / (ms_stage * 1e-3) / 1e9,
        "hbm_GBs": B_F / (ms_stage * 1e-3) / 1e9, "fp_TFLOPs": flops / (ms_stage * 1e-3) / 1e12,
        "energy_finite": bool(np.isfinite(e)),
        "storage_words_per_element": {"wadg": 2 * disc.ref_upd.Nq, "dense_MJinv": 2 * Np * Np,
                                      "ratio": Np * Np / disc.ref_upd.Nq},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--orders", type=int, nargs="+", default=list(range(1, 8)))
    ap.add_argument("--dtypes", nargs="+", default=["float32", "float64"])
    args = ap.parse_args()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        hbm = float(json.load(f)["hbm_gbs"])
    peaks = {"float32": fma_peak.measure(_native.WADG_F32, torch.float32),
             "float64": fma_peak.measure(_native.WADG_F64, torch.float64)}
    rows = []
    for N in args.orders:
        mesh = meshgen.warped_cube_tet_mesh(args.n, N)
        for dtype in args.dtypes:
            r = run_point(mesh, N, dtype, args.steps)
            r["hbm_frac"] = r["hbm_GBs"] / hbm
            r["fp_frac"] = r["fp_TFLOPs"] / peaks[dtype]
            rows.append(r)
            print(json.dumps(r), flush=True)
            gc.collect()                 # Discretization <-> disc.rhs is a reference cycle
            torch.cuda.empty_cache()
    print(json.dumps({"summary": "config3", "hbm_peak_GBs": hbm, "fma_peak_TFLOPs": peaks,
                      "n": args.n, "steps": args.steps}))


if __name__ == "__main__":
    main()
