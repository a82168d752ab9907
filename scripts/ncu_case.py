"""One workload per invocation for ncu captures (debug tool): a few stages of
the chosen case after warm-up, so `ncu -k regex:... -s W -c 1` lands on a
steady-state launch.

    python scripts/ncu_case.py c5_f32 | split_c4 | strong_f64_N4    (WADG_VARIANT=4: kernel kind)
"""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_1608_03836_b200 import meshgen, solver  # noqa: E402
from paper_1608_03836_b200.solver import Formulation, SolverConfig  # noqa: E402

case = sys.argv[1]
if os.environ.get("WADG_VARIANT"):          # force a fused kernel (wadg_debug_set_fused_variant)
    from paper_1608_03836_b200 import _native  # noqa: E402
    _native.call("wadg_debug_set_fused_variant", int(os.environ["WADG_VARIANT"]))
het = lambda x, y, z: 1.0 + 0.5 * torch.sin(2 * np.pi * x) * torch.sin(2 * np.pi * y) * torch.sin(2 * np.pi * z)
if case == "c5_f32":
    mesh, cfg, med, fused = meshgen.warped_cube_tet_mesh(48, 5), SolverConfig(N=5, formulation=Formulation.StrongWeak, dtype="float32"), 1.0, True
elif case == "split_c4":
    mesh, cfg, med, fused = meshgen.warped_cube_tet_mesh(64, 4), SolverConfig(N=4, formulation=Formulation.StrongWeak, dtype="float32"), het, False
elif case.startswith("c3_f64_N") or case.startswith("c3_f32_N"):   # config-3 mesh, strong-weak at order N
    Nc = int(case[len("c3_f64_N"):])
    dt = "float64" if case.startswith("c3_f64") else "float32"
    mesh, cfg, med, fused = (meshgen.warped_cube_tet_mesh(32, Nc),
                             SolverConfig(N=Nc, formulation=Formulation.StrongWeak, dtype=dt), 1.0, True)
elif case.startswith("big_f64_N") or case.startswith("big_f32_N"):  # K = 1.57M mesh, strong-weak at order N
    Nc = int(case[len("big_f64_N"):])
    dt = "float64" if case.startswith("big_f64") else "float32"
    mesh, cfg, med, fused = (meshgen.warped_cube_tet_mesh(64, Nc),
                             SolverConfig(N=Nc, formulation=Formulation.StrongWeak, dtype=dt), 1.0, True)
elif case == "strong_f32_N4":
    mesh, cfg, med, fused = meshgen.warped_cube_tet_mesh(32, 4), SolverConfig(N=4, formulation=Formulation.Strong, dtype="float32"), 1.0, True
elif case == "strong_f64_N4":
    mesh, cfg, med, fused = meshgen.warped_cube_tet_mesh(32, 4), SolverConfig(N=4, formulation=Formulation.Strong), 1.0, True
elif case == "c1_2d_big":                    # config-1 physics (2D triangles, fp64 N = 4) on 256^2 x 2 triangles
    mesh, cfg, med, fused = (meshgen.warped_triangle_mesh(256, 4),
                             SolverConfig(N=4, formulation=Formulation.StrongWeak), 1.0, False)
elif case == "exact_c3_N4":                 # ExactCurvedMass comparator (dense M_J^-1), config-3 mesh, fp64 N = 4
    mesh, cfg, med, fused = (meshgen.warped_cube_tet_mesh(32, 4),
                             SolverConfig(N=4, formulation=Formulation.StrongWeak,
                                          mass_mode=solver.MassMode.ExactCurvedMass), 1.0, False)
else:
    raise SystemExit(f"unknown case {case}")
disc = solver.Discretization(mesh, cfg, solver.MediumField(med))
st = solver.DeviceStepper(disc, fused=fused)
Q = disc.dev.empty_fields().normal_()
Q[:, :, mesh.K:] = 0
for _ in range(2):
    Q = st.step(Q, 1e-4)
torch.cuda.synchronize()
print(case, "K", mesh.K, "kind", disc.dev.fused_kind if fused else "split", flush=True)
