"""MMA-warp timeline of the tcgen05 stage (debug build with -DWADG_MMA_TRACE):
median SM-clock intervals between marks for volume chunks 2, 3 and surface
steps 3, 4 on the config-4 mesh.  Run with WADG_LIB pointing at the trace build."""
import ctypes, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1608_03836_b200 import _native, meshgen, solver

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
mesh = meshgen.warped_cube_tet_mesh(n, 4)
disc = solver.Discretization(mesh, solver.SolverConfig(N=4, formulation=solver.Formulation.StrongWeak, dtype="float32"))
d = disc.dev
nblk = d.Kpad // d.fused
buf = torch.zeros(nblk * 32, dtype=torch.int64, device="cuda")
Q = d.empty_fields().normal_()
Q2, res = d.empty_fields(), d.empty_fields()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
for it in range(3):
    if it == 2:
        _native.call("wadg_debug_set_phase_clock_buffer", vp(buf))
    _native.call("wadg_stage_fused", ctypes.byref(d.struct), vp(Q), vp(Q2), vp(res), 1.0, 1.0, 0.0, 0.1, 1e-3, 0, -1, sp)
_native.call("wadg_debug_set_phase_clock_buffer", ctypes.c_void_p(0))
torch.cuda.synchronize()
t = buf.view(nblk, 32).cpu().numpy().astype(np.float64)
med = lambda a, b: float(np.median(t[:, b] - t[:, a]))
out = {"phases": {k: med(a, a + 1) for k, a in (("stageQ", 0), ("volume", 1), ("surface", 2), ("update", 3), ("write", 4))}}
for ch, base in ((2, 6), (3, 14)):
    names = ["wait_epi_p", "op_wait_Pq", "issue_V2p_V1p", "wait_epi_u", "op_wait_DTW", "issue_V2u_V1u+wait_V2p",
             "wait_V2u"]
    r = {nm: med(base + i, base + i + 1) for i, nm in enumerate(names)}
    r["total"] = med(base, base + 7)
    out[f"volume_chunk{ch}"] = r
out["surface_step3"] = {"wait_traces_read(B_S2)": med(22, 23), "issue_traces": med(23, 24),
                        "wait_lift(step-2)+Pf_load": med(24, 25), "wait_flux(B_S1)": med(25, 26),
                        "issue_lift": med(26, 27), "to_step4_top": med(27, 28), "step4_wait_nodes(B_S0)": med(28, 29),
                        "step3_total": med(22, 28)}
print(json.dumps(out, indent=1))
