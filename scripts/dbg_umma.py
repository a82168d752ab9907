import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import __graft_entry__; __graft_entry__.build()
from paper_1608_03836_b200 import _native, meshgen, solver
from paper_1608_03836_b200.solver import FieldState, SolverConfig, Formulation
N = int(sys.argv[1]); n = int(sys.argv[2])
_native.call("wadg_debug_set_fused_variant", 2)
mesh = meshgen.warped_cube_tet_mesh(n, N)
Np = (N+1)*(N+2)*(N+3)//6
rng = np.random.default_rng(0)
fl = [rng.standard_normal((mesh.K, Np)) for _ in range(4)]
disc = solver.Discretization(mesh, SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype="float32"))
st = solver.lsrk_step(FieldState.from_fields(fl), 1e-3, disc.rhs)
torch.cuda.synchronize(); print("ok", N, n)
