"""Generate golden vectors from the REAL reference package (run in the build
container, where /root/reference exists; the outputs are committed so the
GPU box never needs the reference).

    PYTHONPATH=/root/reference/pkg/src:/root/repo PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Each case stores the mesh, the reference's operator / geometry arrays, a
seeded random state (np.random.default_rng(1234), the reference tests' rng
fixture, R/pkg/tests/conftest.py:40-42) and the reference's outputs of
_volume_terms, _surface_terms, rhs_pre_mass, apply_mass_inverse, rhs_full,
project_initial_condition, repeated lsrk_step and run().
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from wadg import meshgen as rmg          # noqa: E402  (the reference)
from wadg import refelem as rrf          # noqa: E402
from wadg import solver as rsv           # noqa: E402

from paper_1608_03836_b200 import meshgen as mg   # noqa: E402  (only the triangle generator)


def to_ref_mesh(m):
    return rmg.CurvedMesh2D(shape=rrf.ElementShape(m.shape.value), N_geo=m.N_geo,
                            elem_map_nodes=m.elem_map_nodes,
                            face_connectivity=m.face_connectivity,
                            boundary_tags=m.boundary_tags, h=m.h, provenance={})


def cos_mode(x, y):
    p = np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2)
    return p, np.zeros_like(p), np.zeros_like(p)


def cos_mode_exact(x, y, t):
    return np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2) * np.cos(np.pi * np.sqrt(2) / 2 * t)


def het_c2(x, y):
    return 1.0 + 0.5 * np.sin(np.pi * np.hypot(x, y))


def dump_case(name, rmesh, cfg, medium, steps, dt, ic=cos_mode, run_T=None, exact=None):
    disc = rsv.Discretization(rmesh, cfg, medium)
    ref, ru, geo = disc.ref, disc.ref_upd, disc.geo
    rng = np.random.default_rng(1234)
    K, Np = rmesh.K, ref.Np
    st = rsv.FieldState(*(rng.standard_normal((K, Np)) for _ in range(3)))
    sw = cfg.formulation is rsv.Formulation.StrongWeak
    vol = rsv._volume_terms(st, disc, sw)
    sur = rsv._surface_terms(st, disc, sw)
    pre = rsv.rhs_pre_mass(st, disc)
    minv = rsv.apply_mass_inverse(st, disc)
    full = rsv.rhs_full(st, disc)
    s0 = rsv.project_initial_condition(rmesh, cfg, ic, medium)
    s = s0
    for _ in range(steps):
        s = rsv.lsrk_step(s, dt, lambda y: rsv.rhs_full(y, disc))
    out = dict(
        shape=rmesh.shape.value, N=cfg.N, N_geo=rmesh.N_geo, strong_weak=int(sw),
        tau_p=cfg.flux.tau_p, tau_u=cfg.flux.tau_u, steps=steps, dt=dt,
        elem_map_nodes=rmesh.elem_map_nodes, face_connectivity=rmesh.face_connectivity,
        boundary_tags=rmesh.boundary_tags, h=rmesh.h,
        nodes=ref.nodes, Vq=ref.Vq, Pq=ref.Pq, Drq=ref.Drq, Dsq=ref.Dsq, Mhat_inv=ref.Mhat_inv,
        Vfq=ref.Vfq, Pfq=ref.Pfq, wq=ref.wq, wfq=ref.wfq,
        face_nodes=np.array(ref.face_nodes), upd_Vq=ru.Vq, upd_Pq=ru.Pq,
        Jq=geo.Jq, rxq=geo.rxq, ryq=geo.ryq, sxq=geo.sxq, syq=geo.syq,
        Jfq=geo.Jfq, nxq=geo.nxq, nyq=geo.nyq, w_upd_p=disc.w_upd_p, w_upd_u=disc.w_upd_u,
        rand_p=st.p, rand_u1=st.u1, rand_u2=st.u2,
        vol_p=vol[0], vol_u1=vol[1], vol_u2=vol[2],
        sur_p=sur[0], sur_u1=sur[1], sur_u2=sur[2],
        pre_p=pre.p, pre_u1=pre.u1, pre_u2=pre.u2,
        minv_p=minv.p, minv_u1=minv.u1, minv_u2=minv.u2,
        full_p=full.p, full_u1=full.u1, full_u2=full.u2,
        ic_p=s0.p, ic_u1=s0.u1, ic_u2=s0.u2,
        end_p=s.p, end_u1=s.u1, end_u2=s.u2, end_t=s.t,
        energy_ic=rsv.energy(s0, disc), energy_end=rsv.energy(s, disc),
        energy_rand=rsv.energy(st, disc),
        exact_mass=int(cfg.mass_mode is rsv.MassMode.ExactCurvedMass),
    )
    if disc.mass_inv_p is not None:
        out.update(mass_inv_p=disc.mass_inv_p, mass_inv_u=disc.mass_inv_u)
    if run_T is not None:
        _, diag = rsv.run(rmesh, cfg, ic, run_T, medium, exact_p=exact, n_outputs=2, dt=dt)
        out.update(run_T=run_T, run_t=diag["t"], run_energy=diag["energy"],
                   run_l2=diag["l2_error_p"] if exact is not None else np.zeros(0))
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(name, K, Np, os.path.getsize(path))


def main():
    SC, FP, F = rsv.SolverConfig, rsv.FluxParams, rsv.Formulation
    # config 1: K=512 warped triangles, N=4, strong-weak, c^2 = 1, 20 steps dt = 2.5e-3
    m1 = to_ref_mesh(mg.warped_triangle_mesh(16, 4, 0.125))
    dump_case("config1_tri", m1, SC(N=4, formulation=F.StrongWeak), rsv.MediumField(1.0),
              20, 0.5 * (2 / 16) / 25, run_T=0.05, exact=cos_mode_exact)
    # strong form + penalties + heterogeneous medium on a coarse warped triangle mesh
    m2 = to_ref_mesh(mg.warped_triangle_mesh(4, 3, 0.125))
    dump_case("tri_strong_het", m2, SC(N=3, formulation=F.Strong, flux=FP(0.7, 1.3)),
              rsv.MediumField(het_c2), 3, 1e-3)
    # quadrilaterals, the reference's own warped family (strong-weak and strong)
    mq = rmg.warped_arnold_mesh(rmg.WarpParams(1.0, 4), 3)
    dump_case("quad_sw", mq, SC(N=3, formulation=F.StrongWeak), rsv.MediumField(1.0), 3, 2e-3)
    dump_case("quad_strong", mq, SC(N=2, formulation=F.Strong, flux=FP(0.0, 0.5)),
              rsv.MediumField(het_c2), 2, 2e-3)
    # ExactCurvedMass comparator: dense per-element inverses (solver.py:156-167, 302-306)
    dump_case("tri_exact", m2, SC(N=3, formulation=F.StrongWeak, mass_mode=rsv.MassMode.ExactCurvedMass),
              rsv.MediumField(het_c2), 3, 1e-3)


if __name__ == "__main__":
    main()
