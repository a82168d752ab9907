"""Per-phase SM-clock breakdown of the fused stage kernel (debug tool).

    python scripts/phase_clock.py --n 32 --order 4 --dtype float32
"""

import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1608_03836_b200 import _native, meshgen, solver  # noqa: E402

PHASES = ["stage Q", "volume", "gather", "flux+lift", "update", "write"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--variant", type=int, default=-1)
    args = ap.parse_args()
    if args.variant >= 0:
        _native.call("wadg_debug_set_fused_variant", args.variant)
    mesh = meshgen.warped_cube_tet_mesh(args.n, args.order)
    cfg = solver.SolverConfig(N=args.order, formulation=solver.Formulation.StrongWeak, dtype=args.dtype)
    disc = solver.Discretization(mesh, cfg)
    d = disc.dev
    kb = d.fused
    nblk = d.Kpad // kb
    stride = 32 if d.fused_kind == 2 else 8      # the tcgen05 kernel keeps 32 slots per CTA
    buf = torch.zeros(nblk * stride, dtype=torch.int64, device="cuda")
    Q = d.empty_fields().normal_()
    Q2, res = d.empty_fields(), d.empty_fields()
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    for it in range(3):
        if it == 2:
            _native.call("wadg_debug_set_phase_clock_buffer", vp(buf))
        _native.call("wadg_stage_fused", ctypes.byref(d.struct), vp(Q), vp(Q2), vp(res), 1.0, 1.0,
                     0.0, 0.1, 1e-3, 0, -1, sp)
    _native.call("wadg_debug_set_phase_clock_buffer", ctypes.c_void_p(0))
    torch.cuda.synchronize()
    t = buf.view(nblk, stride).cpu().numpy().astype(np.float64)[:, :8]
    nm = int(np.max(np.nonzero(t[0])[0])) + 1          # marks written by this kernel
    t = t[:, :nm]
    dur = np.diff(t, axis=1)
    phases = PHASES if d.fused_kind == 0 else ["stage Q", "volume", "surface", "update", "write"]
    med = np.median(dur, axis=0)
    tot = med.sum()
    out = {"K": mesh.K, "N": args.order, "dtype": args.dtype, "elems_per_block": kb,
           "cycles_per_cta_median": float(tot),
           "phases": {p: {"cycles": float(c), "share": float(c / tot)} for p, c in zip(phases, med)}}
    if d.fused_kind == 2:          # per-SM occupancy: gaps between consecutive CTAs on one SM
        raw = buf.view(nblk, stride).cpu().numpy()
        t0, t1, sm = raw[:, 0].astype(np.float64), raw[:, 5].astype(np.float64), raw[:, 30]
        gaps, busy, span = [], 0.0, 0.0
        for s_ in np.unique(sm):
            i = np.where(sm == s_)[0]
            i = i[np.argsort(t0[i])]
            gaps += list(t0[i][1:] - t1[i][:-1])
            busy += float(np.sum(t1[i] - t0[i]))
            span += float(t1[i][-1] - t0[i][0])
        out["inter_cta_gap_cycles_median"] = float(np.median(gaps)) if gaps else None
        out["inter_cta_gap_cycles_p90"] = float(np.percentile(gaps, 90)) if gaps else None
        out["sm_busy_fraction"] = busy / span
        out["ctas_per_sm"] = nblk / len(np.unique(sm))
        out["cta_cycles_mean"] = float(np.mean(t1 - t0))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
