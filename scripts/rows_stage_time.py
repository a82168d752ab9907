"""Time one full-mesh fused stage on config 4 with the field layout and with the
row layout on Q_in (layout 1) or Q_out (layout 2)."""
import ctypes, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
import bench
from paper_1608_03836_b200 import _native

mesh, cfg, medium, disc, desc = bench.build_problem("c4")
d = disc.dev
K, Np = d.K, disc.ref.Np
A, B, res = d.empty_fields().normal_(), d.empty_fields(), d.empty_fields()
rows = torch.randn((4, K, Np), dtype=torch.float32, device="cuda")
s = ctypes.byref(d.struct)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
fl = disc.flux
out = {}
for lay, qi, qo in ((0, A, B), (1, rows, B), (2, A, rows)):
    def run():
        _native.call("wadg_stage_fused_rows", s, vp(qi), vp(qo), vp(res), fl.tau_p, fl.tau_u, 0.5, 0.5, 1e-5,
                     0, -1, lay, sp)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record(); torch.cuda.synchronize()
    out[f"layout{lay}_ms"] = e0.elapsed_time(e1) / 10
print(json.dumps(out))
