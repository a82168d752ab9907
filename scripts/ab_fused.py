"""A/B timing of the fused-stage tiling variants (debug tool).

    python scripts/ab_fused.py --n 24 --orders 3 4 5 --dtypes float32 float64
"""

import argparse
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1608_03836_b200 import _native, meshgen, solver  # noqa: E402


def time_variant(mesh, N, dtype, var, stages=15):
    if var >= 0 and hasattr(_native.load(), "wadg_debug_set_fused_variant"):
        _native.call("wadg_debug_set_fused_variant", var)
    cfg = solver.SolverConfig(N=N, formulation=solver.Formulation.StrongWeak, dtype=dtype)
    disc = solver.Discretization(mesh, cfg)
    d = disc.dev
    Q = d.empty_fields().normal_()
    Q2, res = d.empty_fields(), d.empty_fields()
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())

    def stage(a, b):
        nonlocal Q, Q2
        _native.call("wadg_stage_fused", ctypes.byref(d.struct), vp(Q), vp(Q2), vp(res), 1.0, 1.0,
                     a, b, 1e-4, 0, -1, sp)
        Q, Q2 = Q2, Q

    for _ in range(3):
        stage(0.0, 0.1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(stages):
        stage(-0.5 if i else 0.0, 0.1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / stages
    return ms, 4 * mesh.K * disc.ref.Np / (ms * 1e-3) / 1e9, d.fused


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=24)
    ap.add_argument("--orders", type=int, nargs="+", default=[3, 4, 5])
    ap.add_argument("--dtypes", nargs="+", default=["float32", "float64"])
    ap.add_argument("--variants", type=int, nargs="+", default=[-1])
    args = ap.parse_args()
    for N in args.orders:
        mesh = meshgen.warped_cube_tet_mesh(args.n, N)
        for dtype in args.dtypes:
            row = {"N": N, "dtype": dtype, "K": mesh.K}
            for v in args.variants:
                ms, g, kb = time_variant(mesh, N, dtype, v)
                row[f"v{v}"] = {"ms": round(ms, 3), "GDOF/s": round(g, 2), "KB": kb}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
