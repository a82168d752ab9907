"""Time one full-mesh fused stage (a != 0) per order on a warped cube (debug tool).

    python scripts/stage_time.py --n 48 --orders 2 3 4
"""
import argparse, ctypes, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_1608_03836_b200 import _native, meshgen, solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=48)
ap.add_argument("--orders", type=int, nargs="+", default=[2, 3, 4])
ap.add_argument("--dtype", default="float32")
ap.add_argument("--variant", type=int, default=-1, help="fused kernel: 0 CUDA cores, 2 tcgen05, 3 DMMA")
args = ap.parse_args()
if args.variant >= 0:
    _native.call("wadg_debug_set_fused_variant", args.variant)
for N in args.orders:
    mesh = meshgen.warped_cube_tet_mesh(args.n, N)
    disc = solver.Discretization(mesh, solver.SolverConfig(N=N, formulation=solver.Formulation.StrongWeak,
                                                           dtype=args.dtype))
    d = disc.dev
    A, B, res = d.empty_fields().normal_(), d.empty_fields(), d.empty_fields()
    s = ctypes.byref(d.struct)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    run = lambda: _native.call("wadg_stage_fused", s, vp(A), vp(B), vp(res), disc.flux.tau_p, disc.flux.tau_u,
                               0.5, 0.5, 1e-5, 0, -1, sp)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"N": N, "dtype": args.dtype, "kind": d.fused_kind, "K": mesh.K, "ms": ms, "GDOF/s": 4 * mesh.K * disc.ref.Np / (ms * 1e-3) / 1e9}),
          flush=True)
    del disc, d, A, B, res
    torch.cuda.empty_cache()
