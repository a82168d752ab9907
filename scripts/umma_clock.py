"""Fine-grained clocks of the tcgen05 fused stage (debug): phase marks 0..5
and chunk-3 volume marks (thread 0 = MMA issuer: 8..15, thread 511: 16..20)."""
import ctypes, json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
from paper_1608_03836_b200 import _native, meshgen, solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
_native.call("wadg_debug_set_fused_variant", 2)
mesh = meshgen.warped_cube_tet_mesh(n, N)
disc = solver.Discretization(mesh, solver.SolverConfig(N=N, formulation=solver.Formulation.StrongWeak, dtype="float32"))
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
def med(a, b):
    return float(np.median(t[:, b] - t[:, a]))
out = {"phases": {nm: med(i, i + 1) for i, nm in enumerate(["stageQ", "volume", "surface", "update", "write"])},
       "surface_face1_t511": {"store_nodes": med(8, 9), "gather_issue+sync": med(9, 10)},
       "surface_step2_t511": {"wait_traces": med(11, 12), "flux_epilogue": med(12, 13), "sync": med(13, 14),
                              "lift+wait": med(14, 15)},
       "volume_chunk3": {"t511_wait_p": med(20, 21), "t511_epi_p": med(21, 22), "t511_sync_p": med(22, 23),
                         "t511_wait_u": med(23, 24), "t511_epi_u": med(24, 25), "t511_sync_u": med(25, 26),
                         "issuer_p_opwait_to_commit": med(28, 29), "issuer_p_commit_to_u_opwait": med(29, 30),
                         "issuer_u_opwait_to_commit": med(30, 31),
                         "sync_p_to_issuer_p_opwait_done": med(23, 28)},
       "update_step1_t511": {"wait_U1": med(16, 17), "epilogue": med(17, 18), "sync+U2+wait": med(18, 19)}}
print(json.dumps(out, indent=1))
