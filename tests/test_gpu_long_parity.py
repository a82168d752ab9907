"""Parity at the BASELINE step counts (north_star: relative L2 of (p, u)
after the stated number of steps <= 1e-11 in fp64 and <= 1e-5 in fp32),
the default kernels (fp32: tcgen05 stage at N = 2..4, split-TF32 mma.sync
stage at N = 5..7, CUDA cores at N = 1; fp64: DMMA stage at N = 2..7, CUDA
cores at N = 1) against the fp64 oracle (oracle/wadg_oracle.py) on meshes of
several 128-element tiles, so cross-tile neighbour gathers are checked
against the oracle and not against the product.

* config-4 physics: N = 4, heterogeneous c^2 = 1 + 0.5 sin 2 pi x sin 2 pi y
  sin 2 pi z, Gaussian pulse, 100 steps, 8^3 x 6 tets (24 tiles), fp32 and fp64;
* config-5 physics: N = 5, c^2 = 1, Gaussian pulse, 100 steps, 6^3 x 6 tets;
* config-3 physics: N = 1..7, Gaussian pulse, 50 steps, 4^3 x 6 tets (3
  tiles), fp32 and fp64;
* the strong form (the reference default) with the heterogeneous medium at
  N = 2..5, 50 steps, fp32 and fp64 (fused stages with the sufficiency rules);
* the full config-4 mesh (K = 1,572,864): one LSRK stage (a != 0) of the
  tcgen05 kernel checked element by element against the oracle on a sample
  of tets, each with its face neighbours (a stage is local to that patch).

dt = 0.5 h / (N+1)^2, h = 2/n.  Both sides start from the
same projected state (the oracle's projection), so the comparison covers
exactly the time stepping; the projection itself is compared separately.
The measured errors are printed in pytest's terminal summary.
"""

import functools

import numpy as np
import pytest
import torch

import wadg_oracle as O
from conftest import record_parity, submesh
from paper_1608_03836_b200 import meshgen, solver
from paper_1608_03836_b200.solver import FieldState, Formulation, SolverConfig

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-11, "float32": 1e-5}


def c2_het(x, y, z):
    return 1.0 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)


def gaussian(x, y, z):
    p = np.exp(-25.0 * (x * x + y * y + z * z))
    return p, 0 * p, 0 * p, 0 * p


def rel(got, want):
    num = sum(float(np.sum((np.asarray(a, dtype=np.float64) - b) ** 2)) for a, b in zip(got, want))
    den = sum(float(np.sum(b ** 2)) for b in want)
    return np.sqrt(num / den)


@functools.lru_cache(maxsize=None)
def oracle_run(n, N, het, steps, strong=False):
    """(mesh, initial oracle state, final oracle state, dt); cached so the
    fp32 and fp64 cases share one oracle trajectory."""
    mesh = meshgen.warped_cube_tet_mesh(n, N)
    c2 = c2_het if het else 1.0
    od = O.OracleDiscretization(mesh, N, not strong, c2=c2)
    st0 = O.project_initial_condition(mesh, N, gaussian)
    dt = 0.5 * (2.0 / n) / (N + 1) ** 2
    st = st0
    for _ in range(steps):
        st = O.lsrk_step(st, dt, lambda y: O.rhs_full(y, od))
    return mesh, st0, st, dt


def device_run(mesh, N, het, dtype, st0, dt, steps, strong=False):
    cfg = SolverConfig(N=N, formulation=Formulation.Strong if strong else Formulation.StrongWeak, dtype=dtype)
    medium = solver.MediumField(c2_het if het else 1.0)
    disc = solver.Discretization(mesh, cfg, medium)
    Q = disc.to_device(FieldState.from_fields(st0.fields()))
    stepper = solver.DeviceStepper(disc)
    for _ in range(steps):
        Q = stepper.step(Q, dt)
    out = disc.from_device(Q, FieldState.from_fields(st0.fields()), steps * dt)
    return disc, [np.asarray(a) for a in out.fields()]


def _check(name, n, N, het, dtype, steps, strong=False):
    mesh, st0, want, dt = oracle_run(n, N, het, steps, strong)
    disc, got = device_run(mesh, N, het, dtype, st0, dt, steps, strong)
    err = rel(got, want.fields())
    change = rel(st0.fields(), want.fields())
    record_parity(f"{name} K={mesh.K} N={N} {dtype} {steps} steps kernel={disc.dev.fused_kind}", err, TOL[dtype])
    assert change > 1e-2, "the state should evolve over the run"
    assert err < TOL[dtype], (name, N, dtype, err)
    return disc


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_config4_physics_100_steps(dtype):
    disc = _check("config-4 physics", 8, 4, True, dtype, 100)
    if dtype == "float32":
        assert disc.dev.fused_kind == 2          # the tcgen05 stage of the headline


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_config5_physics_100_steps(dtype):
    disc = _check("config-5 physics", 6, 5, False, dtype, 100)
    if dtype == "float32":
        assert disc.dev.fused_kind == 4          # the split-TF32 mma.sync stage


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7])
def test_config3_physics_50_steps(N, dtype):
    _check("config-3 physics", 4, N, False, dtype, 50)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_strong_form_50_steps(N, dtype):
    """The reference's default formulation through its fused stages (N = 1:
    the register stage; fp32 split-TF32 mma.sync, fp64 DMMA), heterogeneous
    medium."""
    disc = _check("strong form, config-3 physics + het c2", 4, N, True, dtype, 50, strong=True)
    assert disc.dev.fused_kind == (5 if N == 1 else 4 if dtype == "float32" else 3)


def test_projection_matches_oracle():
    mesh = meshgen.warped_cube_tet_mesh(4, 4)
    cfg = SolverConfig(N=4, formulation=Formulation.StrongWeak)
    got = solver.project_initial_condition(mesh, cfg, gaussian)
    want = O.project_initial_condition(mesh, 4, gaussian)
    err = rel(got.fields()[:1], want.fields()[:1])
    record_parity("Gaussian projection K=384 N=4", err, 1e-12)
    assert err < 1e-12
    assert all(np.max(np.abs(a)) == 0 for a in got.fields()[1:])


# ---------------------------------------------------------------------------
# full config-4 size: sampled element-local parity of one tcgen05 stage

def _sampled_stage_check(n, N, dtype, label, n_blocks=64, per_block=8):
    """One LSRK stage res' = a res + dt M^-1 rhs(Q), Q' = Q + b res' (a != 0) of
    the default fused kernel on random Q and res over the whole mesh, compared
    with the oracle for sampled elements (every tile position, boundary and
    interior), each evaluated on its one-neighbour patch."""
    mesh = meshgen.warped_cube_tet_mesh(n, N)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype=dtype)
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2_het))
    d = disc.dev
    tdt = torch.float32 if dtype == "float32" else torch.float64
    g = torch.Generator(device="cuda").manual_seed(77)
    Q = torch.randn(d.empty_fields().shape, generator=g, device="cuda", dtype=tdt)
    res = torch.randn(Q.shape, generator=g, device="cuda", dtype=tdt)
    Q[:, :, mesh.K:] = 0
    res[:, :, mesh.K:] = 0
    stepper = solver.DeviceStepper(disc)
    assert stepper.fused
    stepper.res.copy_(res)
    a, b, dt = solver.LSRK4A[2], solver.LSRK4B[2], 0.5 * mesh.h / (N + 1) ** 2
    Qout = stepper.stage(Q, a, b, dt)
    rng = np.random.default_rng(5)
    blocks = rng.choice(mesh.K // 128, n_blocks, replace=False)
    elems = np.unique(np.concatenate([(blocks[:, None] * 128 + rng.choice(128, per_block, replace=False)[None, :]).ravel(),
                                      [0, 127, 128, mesh.K - 1]]))
    sub, patch, loc = submesh(mesh, elems)
    host = lambda X: [X[i, :, :mesh.K][:, torch.as_tensor(patch, device="cuda")].T.double().cpu().numpy()
                      for i in range(4)]
    Qp, Rp = host(Q), host(res)
    od = O.OracleDiscretization(sub, N, True, c2=c2_het)
    r = O.rhs_full(O.State(Qp[0], Qp[1:]), od).fields()
    want_res = [a * x + dt * y for x, y in zip(Rp, r)]
    want_Q = [q + b * x for q, x in zip(Qp, want_res)]
    got_res, got_Q = host(stepper.res), host(Qout)
    e_res = rel([x[loc] for x in got_res], [x[loc] for x in want_res])
    e_Q = rel([x[loc] for x in got_Q], [x[loc] for x in want_Q])
    # the rhs part alone (res' - a res = dt rhs), the quantity most exposed to rounding
    e_rhs = rel([(x - a * y)[loc] for x, y in zip(got_res, Rp)], [dt * y[loc] for y in r])
    tag = f"{label} K={mesh.K} N={N} {dtype} kernel={d.fused_kind}, one stage, {len(elems)} sampled tets"
    record_parity(tag + ": res", e_res, TOL[dtype])
    record_parity(tag + ": Q", e_Q, TOL[dtype])
    record_parity(tag + ": dt*rhs", e_rhs, TOL[dtype])
    kind = d.fused_kind
    del disc, d, Q, res, Qout, stepper
    torch.cuda.empty_cache()
    assert e_res < TOL[dtype] and e_Q < TOL[dtype] and e_rhs < TOL[dtype]
    return mesh.K, kind


def test_full_size_stage_sampled_against_oracle():
    """BASELINE config 4 at full size: K = 1,572,864, N = 4, fp32,
    heterogeneous c^2, the tcgen05 stage."""
    K, kind = _sampled_stage_check(64, 4, "float32", "config-4 full size")
    assert K == 1572864 and kind == 2


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7])
def test_million_tet_stage_sampled_against_oracle(N, dtype):
    """north_star: fp64 and fp32 on a >= 1M-tet curvilinear mesh at N = 1..7
    matching the oracle: 56^3 x 6 = 1,053,696 warped tets, heterogeneous c^2."""
    K, _ = _sampled_stage_check(56, N, dtype, ">=1M tets", n_blocks=32, per_block=4)
    assert K >= 1_000_000
