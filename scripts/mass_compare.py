"""WADG versus the ExactCurvedMass comparator on the device (the paper's
storage / runtime claim, R/PAPER.md: WADG needs pointwise weights instead of
dense per-element inverses).  Times wadg_mass_inverse for both modes on the
warped cube (config 3 mesh, heterogeneous c^2) and reports per-element
storage and the achieved bandwidth of the dense path.

    python scripts/mass_compare.py [--n 32] [--orders 2 3 4 5] > mass_compare.jsonl
"""
import argparse, ctypes, json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402
__graft_entry__.build()
import bench  # noqa: E402
from paper_1608_03836_b200 import _native, meshgen, solver  # noqa: E402


def time_minv(disc, reps=20):
    d = disc.dev
    R = d.empty_fields().normal_()
    out = d.empty_fields()
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    for _ in range(3):
        _native.call("wadg_mass_inverse", ctypes.byref(d.struct), vp(R), vp(out), sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        _native.call("wadg_mass_inverse", ctypes.byref(d.struct), vp(R), vp(out), sp)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--orders", type=int, nargs="+", default=[2, 3, 4, 5])
    ap.add_argument("--dtypes", nargs="+", default=["float32", "float64"])
    args = ap.parse_args()
    for N in args.orders:
        mesh = meshgen.warped_cube_tet_mesh(args.n, N)
        for dtype in args.dtypes:
            row = {"N": N, "dtype": dtype, "K": mesh.K}
            for mode in (solver.MassMode.WADG, solver.MassMode.ExactCurvedMass):
                cfg = solver.SolverConfig(N=N, formulation=solver.Formulation.StrongWeak, mass_mode=mode, dtype=dtype)
                disc = solver.Discretization(mesh, cfg, solver.MediumField(bench.c2_het))
                ms = time_minv(disc)
                Np, Nqu, w = disc.ref.Np, disc.ref_upd.Nq, (4 if dtype == "float32" else 8)
                words = 2 * Nqu if mode is solver.MassMode.WADG else 2 * Np * Np
                moved = mesh.K * w * (words + 2 * 4 * Np)         # per-element operator data + 4 fields in/out
                row[mode.value] = {"ms": ms, "storage_words_per_element": words,
                                   "storage_GB": mesh.K * w * words / 1e9, "GB_s": moved / (ms * 1e-3) / 1e9}
                del disc
                torch.cuda.empty_cache()
            row["dense_over_wadg_time"] = row["exact"]["ms"] / row["wadg"]["ms"]
            row["dense_over_wadg_storage"] = row["exact"]["storage_words_per_element"] / row["wadg"]["storage_words_per_element"]
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
