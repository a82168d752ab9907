"""Strong form vs strong-weak, fused stage vs the three-kernel path, per order
(debug tool): ms per RK stage through DeviceStepper on the warped cube.

    python scripts/strong_time.py --n 32 --orders 2 3 4 --dtype float32
"""
import argparse, gc, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_1608_03836_b200 import meshgen, solver  # noqa: E402
from paper_1608_03836_b200.solver import Formulation, SolverConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--orders", type=int, nargs="+", default=[2, 3, 4])
ap.add_argument("--dtype", default="float32")
ap.add_argument("--steps", type=int, default=4)
args = ap.parse_args()
for N in args.orders:
    mesh = meshgen.warped_cube_tet_mesh(args.n, N)
    for form, name in ((Formulation.Strong, "strong"), (Formulation.StrongWeak, "strong-weak")):
        disc = solver.Discretization(mesh, SolverConfig(N=N, formulation=form, dtype=args.dtype))
        for fused in (True, False):
            if fused and disc.dev.fused is None:      # no fused stage for this (form, N, dtype)
                continue
            st = solver.DeviceStepper(disc, fused=fused)
            Q = disc.dev.empty_fields().normal_()
            Q[:, :, mesh.K:] = 0
            for _ in range(2):
                Q = st.step(Q, 1e-5)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                Q = st.step(Q, 1e-5)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / (5 * args.steps)
            print(json.dumps({"N": N, "dtype": args.dtype, "form": name, "fused": fused,
                              "kind": disc.dev.fused_kind if fused else -1, "K": mesh.K, "ms_stage": ms,
                              "GDOF/s": 4 * mesh.K * disc.ref.Np / (ms * 1e-3) / 1e9}), flush=True)
            del st, Q
        del disc
        gc.collect()
        torch.cuda.empty_cache()
