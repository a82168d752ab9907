"""Pin the CPU oracle (and the host setup it shares with the product) to the
REAL reference: golden vectors produced by tests/golden/make_golden.py with
the reference package (R/pkg/src/wadg) importable."""

import numpy as np
import pytest

import wadg_oracle as O
from conftest import GOLDEN_CASES, golden_mesh, load_golden
from paper_1608_03836_b200 import geometry, refelem


def rel(got, want):
    num = sum(float(np.sum((np.asarray(a) - np.asarray(b)) ** 2)) for a, b in zip(got, want))
    den = sum(float(np.sum(np.asarray(b) ** 2)) for b in want)
    return np.sqrt(num / max(den, 1e-300))


def setup(name, exterior):
    g = load_golden(name)
    mesh = golden_mesh(g)
    od = O.OracleDiscretization(mesh, int(g["N"]), bool(g["strong_weak"]), float(g["tau_p"]),
                                float(g["tau_u"]), GOLDEN_CASES[name], exterior=exterior,
                                exact_mass=bool(g["exact_mass"]))
    return g, mesh, od


def test_exact_mass_inverses_match_reference():
    """ExactCurvedMass comparator: the dense inverses of the J/c^2- and
    J-weighted mass matrices (R/.../solver.py:156-167) equal the reference's."""
    g, mesh, od = setup("tri_exact", "gather")
    for mine, ref in ((od.mass_inv_p, g["mass_inv_p"]), (od.mass_inv_u, g["mass_inv_u"])):
        assert np.max(np.abs(mine - ref)) < 1e-11 * np.abs(ref).max()


def fields(g, pfx):
    return [g[f"{pfx}_p"], g[f"{pfx}_u1"], g[f"{pfx}_u2"]]


@pytest.mark.parametrize("exterior", ["gather", "evaluate"])
@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_rhs_phases(name, exterior):
    g, mesh, od = setup(name, exterior)
    st = O.State(g["rand_p"], [g["rand_u1"], g["rand_u2"]])
    vp, vu = O.volume_terms(st, od)
    sp, su = O.surface_terms(st, od)
    assert rel([vp] + vu, fields(g, "vol")) < 1e-13
    assert rel([sp] + su, fields(g, "sur")) < 1e-13
    assert rel(O.rhs_pre_mass(st, od).fields(), fields(g, "pre")) < 1e-13
    assert rel(O.apply_mass_inverse(st, od).fields(), fields(g, "minv")) < 1e-13
    assert rel(O.rhs_full(st, od).fields(), fields(g, "full")) < 1e-13


@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_lsrk_steps_and_energy(name):
    g, mesh, od = setup(name, "gather")
    st = O.State(g["ic_p"], [g["ic_u1"], g["ic_u2"]])
    for _ in range(int(g["steps"])):
        st = O.lsrk_step(st, float(g["dt"]), lambda y: O.rhs_full(y, od))
    assert st.t == pytest.approx(float(g["end_t"]), abs=1e-15)
    assert rel(st.fields(), fields(g, "end")) < 1e-13
    assert O.energy(st, od) == pytest.approx(float(g["energy_end"]), rel=1e-13)
    rnd = O.State(g["rand_p"], [g["rand_u1"], g["rand_u2"]])
    assert O.energy(rnd, od) == pytest.approx(float(g["energy_rand"]), rel=1e-13)


@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_initial_condition_projection(name):
    g, mesh, od = setup(name, "gather")

    def ic(x, y):
        p = np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2)
        return p, 0 * p, 0 * p

    st = O.project_initial_condition(mesh, int(g["N"]), ic)
    assert np.max(np.abs(st.p - g["ic_p"])) < 1e-13
    assert np.max(np.abs(st.u[0])) == 0.0


@pytest.mark.parametrize("name", sorted(GOLDEN_CASES))
def test_reference_element_and_geometry_match_reference(name):
    """The product's host setup reproduces the reference's operator matrices
    and metric data (the data both the oracle and the kernels consume)."""
    g = load_golden(name)
    mesh = golden_mesh(g)
    N = int(g["N"])
    sw = bool(g["strong_weak"])
    vdeg, fdeg = O.quadrature_degrees(N, mesh.N_geo, mesh.shape, sw)
    ref = refelem.build_reference_element(N, mesh.shape, vdeg, fdeg)
    for k in ("nodes", "Vq", "Pq", "Drq", "Dsq", "Mhat_inv", "Vfq", "Pfq", "wq", "wfq"):
        assert np.max(np.abs(getattr(ref, k) - g[k])) < 1e-12, k
    assert np.array_equal(np.array(ref.face_nodes), g["face_nodes"])
    ru = refelem.build_reference_element(N, mesh.shape, 2 * N + 1, 1)
    assert np.max(np.abs(ru.Vq - g["upd_Vq"])) < 1e-13
    assert np.max(np.abs(ru.Pq - g["upd_Pq"])) < 1e-12
    geo = geometry.compute_geometric_data(mesh, ref)
    for k in ("Jq", "rxq", "ryq", "sxq", "syq", "Jfq", "nxq", "nyq"):
        assert np.max(np.abs(getattr(geo, k) - g[k])) < 1e-12 * max(1.0, np.abs(g[k]).max()), k


def test_config1_golden_is_the_baseline_config():
    """config1_tri is BASELINE config 1: 16x16x2 warped triangles, N=4, dt =
    0.5 h/(N+1)^2 with h = 2/16, 20 steps, strong-weak, tau = 1."""
    g = load_golden("config1_tri")
    assert g["elem_map_nodes"].shape == (512, 15, 2)
    assert int(g["N"]) == 4 and int(g["steps"]) == 20 and int(g["strong_weak"]) == 1
    assert float(g["dt"]) == pytest.approx(0.5 * (2 / 16) / 25)
    # the exact standing mode is tracked: energy nearly conserved over 20 steps
    assert float(g["energy_end"]) == pytest.approx(float(g["energy_ic"]), rel=1e-3)
