"""fp32 accuracy probe of the fused stage kernels (debug tool).

Config-4 physics (N = 4, heterogeneous c^2, Gaussian pulse) on the 8^3 x 6
warped cube: for each fused variant, the relative L2 error after 100 steps
against a precomputed fp64 oracle trajectory, and one stage's right-hand side
against the oracle with its signed bias (mean of err * sign(R) / mean |R|),
which separates rounding noise from a systematic shrink.

    python scripts/precision_probe.py make     # CPU: write scratch/oracle_c4phys_8.npz
    python scripts/precision_probe.py run 0 2  # GPU: variants (0 CUDA cores, 2 tcgen05)
"""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import wadg_oracle as O  # noqa: E402
from paper_1608_03836_b200 import meshgen  # noqa: E402

FN = os.path.join(ROOT, "scratch", "oracle_c4phys_8.npz")
n, N, STEPS = 8, 4, 100


def c2_het(x, y, z):
    return 1.0 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)


def gaussian(x, y, z):
    p = np.exp(-25.0 * (x * x + y * y + z * z))
    return p, 0 * p, 0 * p, 0 * p


mesh = meshgen.warped_cube_tet_mesh(n, N)
dt = 0.5 * (2.0 / n) / (N + 1) ** 2
if sys.argv[1] == "make":
    od = O.OracleDiscretization(mesh, N, True, c2=c2_het)
    st0 = O.project_initial_condition(mesh, N, gaussian)
    rng = np.random.default_rng(3)
    Qr = [rng.standard_normal(st0.p.shape) for _ in range(4)]
    R = O.rhs_full(O.State(Qr[0], Qr[1:]), od).fields()
    st = st0
    for _ in range(STEPS):
        st = O.lsrk_step(st, dt, lambda y: O.rhs_full(y, od))
    Rs = O.rhs_full(st, od).fields()
    np.savez(FN, st0=np.stack(st0.fields()), end=np.stack(st.fields()), Qr=np.stack(Qr), R=np.stack(R),
             Rs=np.stack(Rs))
    sys.exit(0)

import torch  # noqa: E402
import __graft_entry__  # noqa: E402
__graft_entry__.build()
from paper_1608_03836_b200 import _native, solver  # noqa: E402
from paper_1608_03836_b200.solver import FieldState, Formulation, SolverConfig  # noqa: E402

z = np.load(FN)
for v in map(int, sys.argv[2:]):
    _native.call("wadg_debug_set_fused_variant", v)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype="float32")
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2_het))
    st = solver.DeviceStepper(disc)
    Q = disc.to_device(FieldState.from_fields(list(z["Qr"])))
    out = st.stage(Q, 0.0, 1.0, 1.0)          # res = R, Q' = Q + R
    R = st.res[:, :, :mesh.K].transpose(1, 2).double().cpu().numpy()
    W = z["R"]
    err = R - W
    rel = float(np.sqrt((err ** 2).sum() / (W ** 2).sum()))
    bias = float((err * np.sign(W)).mean() / np.abs(W).mean())
    Q = disc.to_device(FieldState.from_fields(list(z["end"])))
    st.stage(Q, 0.0, 1.0, 1.0)
    R = st.res[:, :, :mesh.K].transpose(1, 2).double().cpu().numpy()
    W = z["Rs"]
    smooth = {}
    for name, sl in (("p", slice(0, 1)), ("u", slice(1, 4))):
        e = R[sl] - W[sl]
        smooth[name + "_rel"] = float(np.sqrt((e ** 2).sum() / (W[sl] ** 2).sum()))
        smooth[name + "_bias"] = float((e * np.sign(W[sl])).mean() / np.abs(W[sl]).mean())
    Q = disc.to_device(FieldState.from_fields(list(z["st0"])))
    errs = {}
    for k in range(1, STEPS + 1):
        Q = st.step(Q, dt)
        if k in (10, 50, 100):
            got = Q[:, :, :mesh.K].transpose(1, 2).double().cpu().numpy()
            if k == STEPS:
                e = got - z["end"]
                errs[k] = float(np.sqrt((e ** 2).sum() / (z["end"] ** 2).sum()))
    print(json.dumps({"variant": v, "kind": disc.dev.fused_kind, "lib": os.environ.get("WADG_LIB", "default"),
                      "split": os.environ.get("WADG_TF32_SPLIT", "trunc"), "stage_rhs_rel": rel,
                      "stage_rhs_bias": bias, "smooth_rhs": smooth, "steps100_rel": errs[STEPS]}), flush=True)
