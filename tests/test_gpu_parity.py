"""Parity of the CUDA path (through the C ABI via the drop-in solver API)
against the reference's golden vectors (2D) and the CPU oracle (2D + 3D).

Bars (BASELINE.json north_star): relative L2 of (p, u) after the stated
steps <= 1e-11 in fp64 and <= 1e-5 in fp32.
"""

import numpy as np
import pytest
import torch

import wadg_oracle as O
from conftest import GOLDEN_CASES, golden_mesh, load_golden, record_parity
from paper_1608_03836_b200 import meshgen, solver
from paper_1608_03836_b200.solver import FieldState, FluxParams, Formulation, SolverConfig

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-11, "float32": 1e-5}


def rel(got, want):
    """max over fields of ||got - want|| / ||want|| (coefficient 2-norm)."""
    num = sum(float(np.sum((np.asarray(a) - np.asarray(b)) ** 2)) for a, b in zip(got, want))
    den = sum(float(np.sum(np.asarray(b) ** 2)) for b in want)
    return np.sqrt(num / den)


def golden_disc(name, dtype="float64"):
    g = load_golden(name)
    mesh = golden_mesh(g)
    form = Formulation.StrongWeak if int(g["strong_weak"]) else Formulation.Strong
    mode = solver.MassMode.ExactCurvedMass if int(g["exact_mass"]) else solver.MassMode.WADG
    cfg = SolverConfig(N=int(g["N"]), formulation=form, mass_mode=mode,
                       flux=FluxParams(float(g["tau_p"]), float(g["tau_u"])), dtype=dtype)
    disc = solver.Discretization(mesh, cfg, solver.MediumField(GOLDEN_CASES[name]))
    return g, mesh, disc


def gfields(g, pfx):
    return [g[f"{pfx}_p"], g[f"{pfx}_u1"], g[f"{pfx}_u2"]]


@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_rhs_phases_match_reference(name):
    g, mesh, disc = golden_disc(name)
    st = FieldState(*gfields(g, "rand"))
    sw = bool(g["strong_weak"])
    assert rel(solver._volume_terms(st, disc, sw), gfields(g, "vol")) < 1e-13
    assert rel(solver._surface_terms(st, disc, sw), gfields(g, "sur")) < 1e-13
    assert rel(solver.rhs_pre_mass(st, disc).fields(), gfields(g, "pre")) < 1e-13
    assert rel(solver.apply_mass_inverse(st, disc).fields(), gfields(g, "minv")) < 1e-13
    assert rel(solver.rhs_full(st, disc).fields(), gfields(g, "full")) < 1e-13


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_lsrk_steps_match_reference(name, dtype):
    g, mesh, disc = golden_disc(name, dtype)
    st = FieldState(*gfields(g, "ic"))
    for _ in range(int(g["steps"])):
        st = solver.lsrk_step(st, float(g["dt"]), disc.rhs)
    assert st.t == pytest.approx(float(g["end_t"]), abs=1e-15)
    assert rel(st.fields(), gfields(g, "end")) < TOL[dtype]


def test_config1_device_resident_20_steps_and_energy():
    """Config 1 exactly as BASELINE.json states it: 20 steps of dt =
    0.5 h/(N+1)^2 from the projected cos-mode, fields resident on device."""
    g, mesh, disc = golden_disc("config1_tri")
    Q = disc.to_device(FieldState(*gfields(g, "ic")))
    stepper = solver.DeviceStepper(disc)
    for _ in range(20):
        Q = stepper.step(Q, float(g["dt"]))
    out = disc.from_device(Q, FieldState(*gfields(g, "ic")), 0.0)
    assert rel(out.fields(), gfields(g, "end")) < 1e-11
    e = solver.device_energy(disc, Q)
    assert e == pytest.approx(float(g["energy_end"]), rel=1e-12)


def test_run_matches_reference_diagnostics():
    g, mesh, disc = golden_disc("config1_tri")
    cfg = disc.config

    def ic(x, y):
        p = np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2)
        return p, 0 * p, 0 * p

    def exact(x, y, t):
        return np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2) * np.cos(np.pi * np.sqrt(2) / 2 * t)

    state, diag = solver.run(mesh, cfg, ic, float(g["run_T"]), exact_p=exact, n_outputs=2,
                             dt=float(g["dt"]))
    np.testing.assert_allclose(diag["t"], g["run_t"], atol=1e-15)
    np.testing.assert_allclose(diag["energy"], g["run_energy"], rtol=1e-11)
    np.testing.assert_allclose(diag["l2_error_p"], g["run_l2"], rtol=1e-6)


def test_generic_rhs_fn_and_scalar_lsrk():
    """lsrk_step with an arbitrary callable goes through wadg_lsrk_axpy."""
    lam, dt = -0.37, 0.21
    st = FieldState(np.array([[1.0]]), np.zeros((1, 1)), np.zeros((1, 1)))
    out = solver.lsrk_step(st, dt, lambda s: FieldState(lam * s.p, 0 * s.u1, 0 * s.u2))
    want = O.lsrk_step(O.State(np.array([[1.0]]), [np.zeros((1, 1))] * 2), dt,
                       lambda s: O.State(lam * s.p, [0 * a for a in s.u]))
    assert out.p[0, 0] == pytest.approx(want.p[0, 0], abs=1e-15)
    # a numpy-only callable (np.sin, ndarray @) gets a numpy FieldState, as in the reference
    A = np.array([[0.3, -0.1], [0.2, 0.5]])
    st2 = FieldState(np.array([[0.4, -0.2]]), np.array([[0.1, 0.3]]), np.zeros((1, 2)))
    f = lambda s: FieldState(np.sin(s.p) @ A, s.u1 @ A.T, 0 * s.u2)
    got = solver.lsrk_step(st2, 0.1, f)
    want = O.lsrk_step(O.State(st2.p.copy(), [st2.u1.copy(), st2.u2.copy()]), 0.1,
                       lambda s: O.State(np.sin(s.p) @ A, [s.u[0] @ A.T, 0 * s.u[1]]))
    assert isinstance(got.p, np.ndarray)
    assert rel(got.fields(), want.fields()) < 1e-14
    g, mesh, disc = golden_disc("tri_strong_het")
    st = FieldState(*gfields(g, "ic"))
    a = solver.lsrk_step(st, 1e-3, lambda s: solver.rhs_full(s, disc))
    b = solver.lsrk_step(st, 1e-3, disc.rhs)
    assert rel(a.fields(), b.fields()) < 1e-14


# ---------------------------------------------------------------------------
# 3D: device vs oracle (no reference implementation exists)

def _state3(K, Np, rng):
    return [rng.standard_normal((K, Np)) for _ in range(4)]


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7])
def test_3d_rhs_full_vs_oracle_degree_sweep(N, rng):
    mesh = meshgen.warped_cube_tet_mesh(2, N)
    for form, sw in ((Formulation.StrongWeak, True), (Formulation.Strong, False)):
        disc = solver.Discretization(mesh, SolverConfig(N=N, formulation=form,
                                                        flux=FluxParams(0.8, 1.1)))
        od = O.OracleDiscretization(mesh, N, sw, 0.8, 1.1)
        fl = _state3(mesh.K, disc.ref.Np, rng)
        got = solver.rhs_full(FieldState.from_fields(fl), disc).fields()
        want = O.rhs_full(O.State(fl[0], fl[1:]), od).fields()
        assert rel(got, want) < 1e-12, (N, form)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_config2_10_steps_vs_oracle(dtype):
    """Config 2: 8^3 x 6 warped tets (K=3072), N=3, cos-mode IC, 10 steps."""
    mesh = meshgen.warped_cube_tet_mesh(8, 3)
    N = 3
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype=dtype)
    disc = solver.Discretization(mesh, cfg)

    def ic(x, y, z):
        p = np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2) * np.cos(np.pi * z / 2)
        return p, 0 * p, 0 * p, 0 * p

    st = solver.project_initial_condition(mesh, cfg, ic)
    od = O.OracleDiscretization(mesh, N, True)
    ost = O.State(st.p, st.fields()[1:])
    dt = 0.5 * (2.0 / 8) / (N + 1) ** 2
    for _ in range(10):
        st = solver.lsrk_step(st, dt, disc.rhs)
        ost = O.lsrk_step(ost, dt, lambda y: O.rhs_full(y, od))
    assert rel(st.fields(), ost.fields()) < TOL[dtype]


def test_3d_heterogeneous_medium_vs_oracle(rng):
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    mesh = meshgen.warped_cube_tet_mesh(3, 3)
    disc = solver.Discretization(mesh, SolverConfig(N=3, formulation=Formulation.StrongWeak),
                                 solver.MediumField(c2))
    od = O.OracleDiscretization(mesh, 3, True, c2=c2)
    fl = _state3(mesh.K, disc.ref.Np, rng)
    got = solver.rhs_full(FieldState.from_fields(fl), disc).fields()
    want = O.rhs_full(O.State(fl[0], fl[1:]), od).fields()
    assert rel(got, want) < 1e-12
    e = solver.energy(FieldState.from_fields(fl), disc)
    assert e == pytest.approx(O.energy(O.State(fl[0], fl[1:]), od), rel=1e-12)


def test_device_tensor_states_stay_on_device(rng):
    mesh = meshgen.warped_cube_tet_mesh(2, 2)
    disc = solver.Discretization(mesh, SolverConfig(N=2, formulation=Formulation.StrongWeak))
    fl = _state3(mesh.K, disc.ref.Np, rng)
    dst = FieldState.from_fields([torch.as_tensor(a, device="cuda") for a in fl])
    out = solver.rhs_full(dst, disc)
    assert isinstance(out.p, torch.Tensor) and out.p.is_cuda
    host = solver.rhs_full(FieldState.from_fields(fl), disc)
    assert rel([a.cpu().numpy() for a in out.fields()], host.fields()) < 1e-15


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7])
def test_fused_stage_matches_split_kernels_and_oracle(N, dtype, rng):
    """wadg_stage_fused (one kernel per stage, ping-pong Q) against the
    three-kernel stage and the oracle, heterogeneous medium, 2 steps."""
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, flux=FluxParams(0.9, 1.2), dtype=dtype)
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2))
    assert disc.dev.fused is not None
    fl = _state3(mesh.K, disc.ref.Np, rng)
    st = FieldState.from_fields(fl)
    Qf = disc.to_device(st)
    Qs = Qf.clone()
    sf, ss = solver.DeviceStepper(disc, fused=True), solver.DeviceStepper(disc, fused=False)
    assert sf.fused and not ss.fused
    dt = 2e-3
    for _ in range(2):
        Qf = sf.step(Qf, dt)
        Qs = ss.step(Qs, dt)
    a = disc.from_device(Qf, st, 0.0).fields()
    b = disc.from_device(Qs, st, 0.0).fields()
    assert rel(a, b) < (1e-13 if dtype == "float64" else 2e-6)
    od = O.OracleDiscretization(mesh, N, True, 0.9, 1.2, c2=c2)
    ost = O.State(fl[0], fl[1:])
    for _ in range(2):
        ost = O.lsrk_step(ost, dt, lambda y: O.rhs_full(y, od))
    assert rel(a, ost.fields()) < TOL[dtype]


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("fused", [True, False])
def test_two_slab_halo_path_is_bitwise_single_domain(dtype, fused, rng):
    """Slab decomposition on one device: each slab packs its interface face
    traces with wadg_pack_halo, the buffers are exchanged by device copies
    (what NCCL does between ranks), and 3 LSRK steps reproduce the single
    domain bit for bit (same per-element arithmetic, exact halo copies)."""
    import ctypes
    from paper_1608_03836_b200 import _native, parallel
    N = 3
    mesh = meshgen.warped_cube_tet_mesh(4, N, nz=4)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype=dtype)
    whole = solver.Discretization(mesh, cfg)
    ranges = parallel.slab_ranges(mesh.K, 2, 4)
    plans = parallel.halo_plans(mesh, ranges)
    parts = [solver.Discretization(mesh, cfg, k_range=ranges[r], halo=plans[r]) for r in range(2)]
    fl = _state3(mesh.K, whole.ref.Np, rng)
    Qw = whole.to_device(FieldState.from_fields(fl))
    Qp = [p.to_device(FieldState.from_fields([a[lo:hi] for a in fl])) for p, (lo, hi) in zip(parts, ranges)]
    sw = solver.DeviceStepper(whole, fused=fused)
    sp = [solver.DeviceStepper(p, fused=fused) for p in parts]
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    dt = 2e-3
    for _ in range(3):
        for a, b in zip(solver.LSRK4A, solver.LSRK4B):
            Qw = sw.stage(Qw, a, b, dt)
            for p, pl, Q in zip(parts, plans, Qp):
                d = p.dev
                _native.call("wadg_pack_halo", ctypes.byref(d.struct), vp(Q), vp(d.send_k), vp(d.send_f),
                             len(pl.send_k), vp(d.send_buf), st)
            parts[0].dev.halo_buf.copy_(parts[1].dev.send_buf)
            parts[1].dev.halo_buf.copy_(parts[0].dev.send_buf)
            Qp = [s.stage(Q, a, b, dt) for s, Q in zip(sp, Qp)]
    whole_out = Qw[:, :, :mesh.K]
    split_out = torch.cat([Q[:, :, :hi - lo] for Q, (lo, hi) in zip(Qp, ranges)], dim=2)
    assert torch.equal(whole_out, split_out)


@pytest.mark.parametrize("N", [2, 3, 4])
def test_tensor_core_and_cuda_core_fused_kernels_agree(N, rng):
    """fp32: the split-TF32 tcgen05 fused stage and the CUDA-core FMA one give
    the same 2 steps to fp32 rounding, and both match the oracle.  The packing
    choice is a debug switch; the launch follows what the operators were packed
    for (wadg_problem.fused_kind), so flipping the switch after a
    Discretization exists does not change which kernel it runs."""
    from paper_1608_03836_b200 import _native
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype="float32")
    fl = _state3(mesh.K, refelem_np(N), rng)
    outs = {}
    try:
        for v in (0, 2):
            _native.call("wadg_debug_set_fused_variant", v)
            disc = solver.Discretization(mesh, cfg)
            assert disc.dev.fused_kind == v and disc.dev.struct.fused_kind == v
            _native.call("wadg_debug_set_fused_variant", 2 - v)     # must not affect this disc
            st = FieldState.from_fields(fl)
            for _ in range(2):
                st = solver.lsrk_step(st, 2e-3, disc.rhs)
            outs[v] = st.fields()
    finally:
        _native.call("wadg_debug_set_fused_variant", -1)
    assert rel(outs[0], outs[2]) < 2e-6
    od = O.OracleDiscretization(mesh, N, True)
    ost = O.State(fl[0], fl[1:])
    for _ in range(2):
        ost = O.lsrk_step(ost, 2e-3, lambda y: O.rhs_full(y, od))
    assert rel(outs[0], ost.fields()) < 1e-5
    assert rel(outs[2], ost.fields()) < 1e-5


@pytest.mark.parametrize("N", [1, 2])
@pytest.mark.parametrize("dtype,tol", [("float32", 1e-5), ("float64", 1e-12)])
def test_register_and_cuda_core_fused_kernels_agree(N, dtype, tol, rng):
    """N = 1, 2: the thread-per-element register stage (kind 5; the default at
    N = 1) and the CUDA-core tiled one give the same 2 steps to rounding (wall
    faces, heterogeneous c^2, nonzero penalties), and both match the oracle."""
    from paper_1608_03836_b200 import _native
    mesh = meshgen.warped_cube_tet_mesh(5, N)
    c2 = lambda x, y, z: 1.0 + 0.5 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, flux=FluxParams(0.7, 1.3), dtype=dtype)
    fl = _state3(mesh.K, refelem_np(N), rng)
    outs = {}
    try:
        for v in (0, 5):
            _native.call("wadg_debug_set_fused_variant", v)
            disc = solver.Discretization(mesh, cfg, solver.MediumField(c2))
            assert disc.dev.fused_kind == v and disc.dev.struct.fused_kind == v
            st = FieldState.from_fields(fl)
            for _ in range(2):
                st = solver.lsrk_step(st, 2e-3, disc.rhs)
            outs[v] = st.fields()
    finally:
        _native.call("wadg_debug_set_fused_variant", -1)
    if N == 1:
        assert solver.Discretization(mesh, cfg, solver.MediumField(c2)).dev.fused_kind == 5   # the default
    assert rel(outs[0], outs[5]) < (2e-6 if dtype == "float32" else 1e-13)
    od = O.OracleDiscretization(mesh, N, True, tau_p=0.7, tau_u=1.3, c2=c2)
    ost = O.State(fl[0], fl[1:])
    for _ in range(2):
        ost = O.lsrk_step(ost, 2e-3, lambda y: O.rhs_full(y, od))
    record_parity(f"register stage vs oracle N={N} {dtype} 2 steps", rel(outs[5], ost.fields()), tol)
    assert rel(outs[5], ost.fields()) < tol


@pytest.mark.parametrize("N", [5, 6, 7])
def test_tmma_and_cuda_core_fused_kernels_agree(N, rng):
    """fp32 N >= 5: the split-TF32 mma.sync fused stage (kind 4) and the
    CUDA-core FMA one give the same 2 steps to fp32 rounding, and both match
    the oracle."""
    from paper_1608_03836_b200 import _native
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, flux=FluxParams(0.7, 1.3), dtype="float32")
    fl = _state3(mesh.K, refelem_np(N), rng)
    outs = {}
    try:
        for v in (0, 4):
            _native.call("wadg_debug_set_fused_variant", v)
            disc = solver.Discretization(mesh, cfg)
            assert disc.dev.fused_kind == v and disc.dev.struct.fused_kind == v
            st = FieldState.from_fields(fl)
            for _ in range(2):
                st = solver.lsrk_step(st, 2e-3, disc.rhs)
            outs[v] = st.fields()
    finally:
        _native.call("wadg_debug_set_fused_variant", -1)
    assert rel(outs[0], outs[4]) < 2e-6
    od = O.OracleDiscretization(mesh, N, True, tau_p=0.7, tau_u=1.3)
    ost = O.State(fl[0], fl[1:])
    for _ in range(2):
        ost = O.lsrk_step(ost, 2e-3, lambda y: O.rhs_full(y, od))
    record_parity(f"tmma vs oracle N={N} fp32 2 steps", rel(outs[4], ost.fields()), 1e-5)
    assert rel(outs[4], ost.fields()) < 1e-5


def refelem_np(N):
    return (N + 1) * (N + 2) * (N + 3) // 6


def _cube_mode_ic(x, y, z):
    p = np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2) * np.cos(np.pi * z / 2)
    return p, 0 * p, 0 * p, 0 * p


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_exact_mass_comparator_matches_oracle_3d(dtype, rng):
    """ExactCurvedMass on curved tets with a heterogeneous medium: the device
    dense-inverse path (wadg_mass_inverse / wadg_stage with minv_p) against the
    oracle's restatement of R/.../solver.py:156-167, 302-306."""
    N = 3
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    c2 = lambda x, y, z: 1.0 + 0.5 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, mass_mode=solver.MassMode.ExactCurvedMass,
                       dtype=dtype)
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2))
    od = O.OracleDiscretization(mesh, N, True, c2=c2, exact_mass=True)
    fl = [rng.standard_normal((mesh.K, refelem_np(N))) for _ in range(4)]
    got = solver.rhs_full(FieldState.from_fields(fl), disc).fields()
    want = O.rhs_full(O.State(fl[0], fl[1:]), od).fields()
    assert rel(got, want) < (1e-12 if dtype == "float64" else 1e-5)
    # stored dense inverses equal the oracle's (host view of the device data)
    assert np.max(np.abs(disc.mass_inv_p - od.mass_inv_p)) < (1e-10 if dtype == "float64" else 1e-4) * np.abs(
        od.mass_inv_p).max()
    # two LSRK steps through the three-kernel stage (the fused stage is WADG-only)
    st, ost = FieldState.from_fields(fl), O.State(fl[0], fl[1:])
    for _ in range(2):
        st = solver.lsrk_step(st, 2e-3, disc.rhs)
        ost = O.lsrk_step(ost, 2e-3, lambda y: O.rhs_full(y, od))
    assert rel(st.fields(), ost.fields()) < TOL[dtype]


def test_exact_mass_equals_wadg_on_affine_unit_speed(rng):
    """R/pkg/tests/test_solver.py:118-126 on affine tetrahedra with c = 1."""
    N = 3
    mesh = meshgen.warped_cube_tet_mesh(2, N, amp=0.0)
    fl = [rng.standard_normal((mesh.K, refelem_np(N))) for _ in range(4)]
    outs = []
    for mode in (solver.MassMode.WADG, solver.MassMode.ExactCurvedMass):
        disc = solver.Discretization(mesh, SolverConfig(N=N, formulation=Formulation.StrongWeak, mass_mode=mode))
        outs.append(solver.rhs_full(FieldState.from_fields(fl), disc).fields())
    for x, y in zip(*outs):
        assert np.max(np.abs(np.asarray(x) - np.asarray(y))) < 1e-10 * max(1.0, np.abs(np.asarray(y)).max())


def test_wadg_vs_exact_mass_error_ratio_3d():
    """The paper's accuracy claim, the 3D analogue of R/pkg/tests/test_solver.py:
    143-152: on curved tetrahedra the WADG solution error against the exact
    Dirichlet eigenmode equals the exact-mass solution error to within 1 %."""
    N, T, steps = 3, 0.25, 25
    mesh = meshgen.warped_cube_tet_mesh(4, N)
    w = np.pi * np.sqrt(3) / 2
    od = O.OracleDiscretization(mesh, N, True)
    xq = od.geo.xyzq
    pex = np.cos(np.pi * xq[0] / 2) * np.cos(np.pi * xq[1] / 2) * np.cos(np.pi * xq[2] / 2) * np.cos(w * T)
    W = od.ref.wq[None, :] * od.geo.Jq
    errs = {}
    for mode in (solver.MassMode.WADG, solver.MassMode.ExactCurvedMass):
        disc = solver.Discretization(mesh, SolverConfig(N=N, formulation=Formulation.StrongWeak, mass_mode=mode))
        st = solver.project_initial_condition(mesh, disc.config, _cube_mode_ic)
        for _ in range(steps):
            st = solver.lsrk_step(st, T / steps, disc.rhs)
        errs[mode] = np.sqrt(np.sum(W * (od.interp(np.asarray(st.p)) - pex) ** 2))
    ratio = errs[solver.MassMode.WADG] / errs[solver.MassMode.ExactCurvedMass]
    assert 0.99 <= ratio <= 1.01


@pytest.mark.parametrize("N", [2, 3, 4, 5])
def test_fused_strong_form_stage_fp64(N, rng):
    """The reference's default formulation (Strong, R/pkg/src/wadg/solver.py:70)
    as one fused DMMA stage (fp64, the 4N-3 / 4N-2 sufficiency rules): against
    the three-kernel stage and the oracle, heterogeneous medium, 2 steps; and
    strong = strong-weak under sufficient quadrature on the same state."""
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    cfg = SolverConfig(N=N, formulation=Formulation.Strong, flux=FluxParams(0.9, 1.2))
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2))
    assert disc.dev.fused is not None and disc.dev.fused_kind == 3
    fl = _state3(mesh.K, disc.ref.Np, rng)
    st = FieldState.from_fields(fl)
    Qf = disc.to_device(st)
    Qs = Qf.clone()
    sf, ss = solver.DeviceStepper(disc, fused=True), solver.DeviceStepper(disc, fused=False)
    dt = 2e-3
    for _ in range(2):
        Qf = sf.step(Qf, dt)
        Qs = ss.step(Qs, dt)
    a = disc.from_device(Qf, st, 0.0).fields()
    b = disc.from_device(Qs, st, 0.0).fields()
    assert rel(a, b) < 1e-13
    od = O.OracleDiscretization(mesh, N, False, 0.9, 1.2, c2=c2)
    ost = O.State(fl[0], fl[1:])
    for _ in range(2):
        ost = O.lsrk_step(ost, dt, lambda y: O.rhs_full(y, od))
    assert rel(a, ost.fields()) < 1e-11
    # lsrk_step(state, dt, disc.rhs) runs the fused stage for the strong form too
    got = solver.lsrk_step(st, dt, disc.rhs)
    want = O.lsrk_step(O.State(fl[0], fl[1:]), dt, lambda y: O.rhs_full(y, od))
    assert rel(got.fields(), want.fields()) < 1e-11


@pytest.mark.parametrize("N", [2, 3, 4])
def test_tcgen05_stage_more_tiles_than_sms(N):
    """More 128-element tiles than SMs (K = 16^3 x 6 = 24,576: 192 tiles), so the
    persistent tcgen05 CTAs (N = 2, 3) loop over several tiles each: one fused
    stage against the three-kernel stage, heterogeneous medium."""
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    mesh = meshgen.warped_cube_tet_mesh(16, N)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype="float32")
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2))
    assert disc.dev.fused_kind == 2 and disc.dev.Kpad // 128 > torch.cuda.get_device_properties(0).multi_processor_count
    g = torch.Generator(device="cuda").manual_seed(3)
    Q = torch.randn(disc.dev.empty_fields().shape, generator=g, device="cuda")
    Q[:, :, mesh.K:] = 0
    sf, ss = solver.DeviceStepper(disc, fused=True), solver.DeviceStepper(disc, fused=False)
    res = torch.randn(Q.shape, generator=g, device="cuda")
    res[:, :, mesh.K:] = 0
    sf.res.copy_(res)
    ss.res.copy_(res)
    a, b, dt = solver.LSRK4A[1], solver.LSRK4B[1], 1e-3
    Qf, Qs = sf.stage(Q, a, b, dt), ss.stage(Q, a, b, dt)
    K = mesh.K
    err = (torch.linalg.norm((Qf - Qs)[:, :, :K]) / torch.linalg.norm(Qs[:, :, :K])).item()
    err_r = (torch.linalg.norm((sf.res - ss.res)[:, :, :K]) / torch.linalg.norm(ss.res[:, :, :K])).item()
    assert err < 2e-6 and err_r < 2e-6, (err, err_r)


@pytest.mark.parametrize("N", [2, 3, 4, 5])
def test_fused_strong_form_stage_fp32(N, rng):
    """The strong form in fp32 as one fused split-TF32 mma.sync stage (kind 4):
    against the fp32 three-kernel strong stage and the fp64 oracle,
    heterogeneous medium, 2 steps."""
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    cfg = SolverConfig(N=N, formulation=Formulation.Strong, flux=FluxParams(0.9, 1.2), dtype="float32")
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2))
    assert disc.dev.fused is not None and disc.dev.fused_kind == 4
    fl = _state3(mesh.K, disc.ref.Np, rng)
    st = FieldState.from_fields(fl)
    Qf = disc.to_device(st)
    Qs = Qf.clone()
    sf, ss = solver.DeviceStepper(disc, fused=True), solver.DeviceStepper(disc, fused=False)
    dt = 2e-3
    for _ in range(2):
        Qf = sf.step(Qf, dt)
        Qs = ss.step(Qs, dt)
    a = disc.from_device(Qf, st, 0.0).fields()
    b = disc.from_device(Qs, st, 0.0).fields()
    assert rel(a, b) < 2e-6
    od = O.OracleDiscretization(mesh, N, False, 0.9, 1.2, c2=c2)
    ost = O.State(fl[0], fl[1:])
    for _ in range(2):
        ost = O.lsrk_step(ost, dt, lambda y: O.rhs_full(y, od))
    err = rel(a, ost.fields())
    record_parity(f"strong form fused fp32 (tmma) N={N} 2 steps", err, 1e-5)
    assert err < 1e-5


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("N", [2, 3, 4])
def test_single_curved_tet_fused_stage(N, dtype, rng):
    """Edge case: one curved tetrahedron (K = 1, every face a mirror boundary,
    a block that is almost all padding) through the default fused stage
    (tcgen05 / DMMA) against the oracle, 3 steps."""
    from test_oracle_3d import single_curved_tet
    mesh = single_curved_tet(N)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, flux=FluxParams(0.6, 1.4), dtype=dtype)
    disc = solver.Discretization(mesh, cfg)
    assert disc.dev.fused is not None
    fl = _state3(1, disc.ref.Np, rng)
    st = FieldState.from_fields(fl)
    od = O.OracleDiscretization(mesh, N, True, 0.6, 1.4)
    ost = O.State(fl[0], fl[1:])
    for _ in range(3):
        st = solver.lsrk_step(st, 1e-2, disc.rhs)
        ost = O.lsrk_step(ost, 1e-2, lambda y: O.rhs_full(y, od))
    assert rel(st.fields(), ost.fields()) < TOL[dtype]
