"""Step time of DeviceStepper.step vs step_graphed on BASELINE configs 1 and 2
(launch-bound small meshes)."""
import json, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_1608_03836_b200 import meshgen, solver  # noqa: E402

for name, mesh, N in (("config 1 (2D tri, K=512, N=4, fp64)", meshgen.warped_triangle_mesh(16, 4), 4),
                      ("config 2 (3D tet, K=3072, N=3, fp64)", meshgen.warped_cube_tet_mesh(8, 3), 3)):
    disc = solver.Discretization(mesh, solver.SolverConfig(N=N, formulation=solver.Formulation.StrongWeak))
    Q = disc.dev.empty_fields().normal_()
    st = solver.DeviceStepper(disc)
    out = {"case": name}
    for mode in ("eager", "graph"):
        fn = st.step if mode == "eager" else st.step_graphed
        for _ in range(5):
            Q = fn(Q, 1e-4)
        torch.cuda.synchronize()
        n = 200
        t0 = time.perf_counter()
        for _ in range(n):
            Q = fn(Q, 1e-4)
        torch.cuda.synchronize()
        out[f"{mode}_us_per_step"] = (time.perf_counter() - t0) / n * 1e6
    print(json.dumps(out), flush=True)
