"""Debug: the tcgen05 fused stage (variant 2) against the CUDA-core one
(variant 0) and the oracle on a small warped cube, per order."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
from paper_1608_03836_b200 import _native, meshgen, solver
from paper_1608_03836_b200.solver import FieldState, SolverConfig, Formulation

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))

for N in [int(x) for x in (sys.argv[1:] or ["2", "3", "4"])]:
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    Np = (N + 1) * (N + 2) * (N + 3) // 6
    rng = np.random.default_rng(1234)
    fl = [rng.standard_normal((mesh.K, Np)) for _ in range(4)]
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype="float32")
    outs = {}
    for v in (0, 2):
        _native.call("wadg_debug_set_fused_variant", v)
        disc = solver.Discretization(mesh, cfg)
        st = FieldState.from_fields(fl)
        for _ in range(1):
            st = solver.lsrk_step(st, 2e-3, disc.rhs)
        torch.cuda.synchronize()
        outs[v] = [np.asarray(x) for x in st.fields()]
        print(N, v, disc.dev.fused_kind, flush=True)
    per = [rel(a, b) for a, b in zip(outs[2], outs[0])]
    print(json.dumps({"N": N, "rel_all": rel(np.concatenate(outs[2]), np.concatenate(outs[0])), "per_field": per}), flush=True)
