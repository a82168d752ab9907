"""Break down the end-to-end step (host state -> device -> 5 stages -> host) on config 4."""
import json, os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__
__graft_entry__.build()
import bench
from paper_1608_03836_b200 import solver

mesh, cfg, medium, disc, desc = bench.build_problem("c4")
d = disc.dev
K, Np = d.K, disc.ref.Np
host = [torch.randn((K, Np), dtype=torch.float32).pin_memory() for _ in range(4)]
st = solver.FieldState.from_fields(host)
dt = 1e-4
ev = lambda: torch.cuda.Event(enable_timing=True)
out = {}
# H2D only
Q = disc.to_device(st); torch.cuda.synchronize()
e0, e1 = ev(), ev(); e0.record()
for _ in range(3): Q = disc.to_device(st)
e1.record(); torch.cuda.synchronize(); out["to_device_ms"] = e0.elapsed_time(e1) / 3
# raw H2D of one pinned field
e0, e1 = ev(), ev(); e0.record()
for _ in range(3): g = host[0].to("cuda", non_blocking=True)
e1.record(); torch.cuda.synchronize(); out["raw_h2d_one_field_ms"] = e0.elapsed_time(e1) / 3
out["raw_h2d_GBs"] = host[0].numel() * 4 / (out["raw_h2d_one_field_ms"] * 1e-3) / 1e9
# D2H
r = disc.from_device(Q, st, 0.0); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3): r = disc.from_device(Q, st, 0.0)
torch.cuda.synchronize(); out["from_device_ms"] = (time.perf_counter() - t0) / 3 * 1e3
# full step
s2 = solver.lsrk_step(st, dt, disc.rhs); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3): s2 = solver.lsrk_step(st, dt, disc.rhs)
torch.cuda.synchronize(); out["lsrk_step_e2e_ms"] = (time.perf_counter() - t0) / 3 * 1e3
print(json.dumps(out))
