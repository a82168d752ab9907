"""Benchmark of the WADG RHS + LSRK45 path (BASELINE.json metric: DOF-updates
per second per RK stage, GDOF/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
                    [--impl wadg|reference]

A "step" is one full LSRK45 time step (5 RK stages, each = volume + surface
+ fused WADG-update/axpy kernel) over the whole mesh.  value = (d+1) K Np x 5
x steps / device time, summed over ranks (max-over-ranks time).

Default workload (N=1): BASELINE config 4 — warped Kuhn cube 64^3 x 6 =
1,572,864 tets, N = 4, fp32, c^2 = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z)
folded into the WADG update weights, Gaussian pulse, strong-weak form.
Inputs (fields 0.9 GB, geometry 9.9 GB) are far larger than the 126 MB L2, so
no explicit L2 flush is needed between timed steps.

--impl reference times the reference algorithm on the host: the reference
package is pure Python/numpy and cannot travel to the GPU box, so its
restatement in oracle/wadg_oracle.py (pinned to the reference's golden
vectors) is timed on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (description, n, N, dtype, heterogeneous c2, steps in BASELINE)
    "c2": ("config 2: warped cube 8^3x6 tets, N=3, fp64", 8, 3, "float64", False, 10),
    "c3": ("config 3: warped cube 32^3x6 tets, fp64/fp32 sweep", 32, 4, "float64", False, 50),
    "c4": ("config 4: warped cube 64^3x6 tets, N=4, fp32, heterogeneous c^2", 64, 4, "float32", True, 100),
    "c5": ("config 5: warped cube 48x48x(48G)x6 tets per GPU, N=5, fp32", 48, 5, "float32", False, 100),
}


def c2_het(x, y, z):
    """Config 4's wavespeed; a torch expression on device points (setup stays on the GPU)."""
    import torch
    sin = torch.sin if isinstance(x, torch.Tensor) else np.sin
    return 1.0 + 0.5 * sin(2 * np.pi * x) * sin(2 * np.pi * y) * sin(2 * np.pi * z)


def gaussian_ic(*xyz):
    r2 = sum(a * a for a in xyz)
    try:
        import torch
        if isinstance(r2, torch.Tensor):
            p = torch.exp(-25.0 * r2)
            return (p,) + tuple(torch.zeros_like(p) for _ in xyz)
    except ImportError:
        pass
    p = np.exp(-25.0 * r2)
    return (p,) + tuple(np.zeros_like(p) for _ in xyz)


def algorithmic_model(d, K, Np, Nq, Nqu, F, w, n_omega):
    """SURVEY.md §8(d) per-element bytes / flops per RK stage, times K."""
    fld = d + 1
    B = {
        "volume": w * (2 * fld * Np + d * d * Nq),
        "surface": w * (3 * fld * Np + fld * F + (d + 1) * F) + 4 * F,
        "update": w * (5 * fld * Np + n_omega * Nqu),
    }
    FL = {
        "volume": 8 * d * Np * Nq + (2 * d * (2 * d - 1) + d) * Nq,
        "surface": 4 * fld * Np * F + 30 * F,
        "update": fld * (4 * Np * Nqu + Nqu) + 4 * fld * Np,
    }
    return {k: v * K for k, v in B.items()}, {k: v * K for k, v in FL.items()}


class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_problem(cfg_name, N_override=None, dtype_override=None, rank=0, world=1):
    from paper_1608_03836_b200 import meshgen, parallel, solver
    desc, n, N, dtype, het, _ = CONFIGS[cfg_name]
    N = N_override or N
    dtype = dtype_override or dtype
    nz, z_range = (48 * world, (-1.0, -1.0 + 2.0 * 48 * world / n)) if cfg_name == "c5" else (n, None)
    cfg = solver.SolverConfig(N=N, formulation=solver.Formulation.StrongWeak, dtype=dtype)
    medium = solver.MediumField(c2_het if het else 1.0)
    if world > 1:
        # each rank generates only its z-slab plus one ghost layer per neighbour
        # (parallel.ghosted_slab_mesh): no global mesh on any rank
        disc = parallel.local_slab_discretization(n, N, cfg, medium, rank, world, nz=nz, z_range=z_range)
        mesh = disc.mesh
        mesh.K_total = 6 * n * n * nz
    else:
        mesh = meshgen.warped_cube_tet_mesh(n, N, nz=nz, z_range=z_range)
        disc = solver.Discretization(mesh, cfg, medium)
    return mesh, cfg, medium, disc, desc


def cpu_oracle_rate(cfg_name, n_sample, steps, N_override=None):
    """Time the reference algorithm (numpy oracle, fp64, all host threads) on
    a bounded sample mesh: GDOF-updates per RK stage per second."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import wadg_oracle as O
    from paper_1608_03836_b200 import meshgen
    _, _, N, _, het, _ = CONFIGS[cfg_name]
    N = N_override or N
    mesh = meshgen.warped_cube_tet_mesh(n_sample, N)
    od = O.OracleDiscretization(mesh, N, True, c2=(c2_het if het else 1.0))
    st = O.project_initial_condition(mesh, N, gaussian_ic)
    dt = 0.5 * (2.0 / n_sample) / (N + 1) ** 2
    fn = lambda y: O.rhs_full(y, od)
    st = O.lsrk_step(st, dt, fn)                      # warm-up
    t0 = time.perf_counter()
    for _ in range(steps):
        st = O.lsrk_step(st, dt, fn)
    el = time.perf_counter() - t0
    dof = 4 * mesh.K * od.ref.Np
    return dof * 5 * steps / el / 1e9, mesh.K, el


def reference_2d_calibration(K1D=64, N=4, steps=2):
    """Time the UNMODIFIED reference package (baseline/_ref, 2D only) and the
    numpy oracle port on the same warped-triangle mesh, so the port timing
    used for the 3D workload is calibrated against the real reference."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "wadg")):
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, ref_dir)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        from wadg import meshgen as rmg, refelem as rrf, solver as rsv
    except Exception as exc:                     # pragma: no cover
        return {"unavailable": f"reference import failed: {exc}"}
    import wadg_oracle as O
    from paper_1608_03836_b200 import meshgen
    m = meshgen.warped_triangle_mesh(K1D, N)
    rm = rmg.CurvedMesh2D(shape=rrf.ElementShape.Triangle, N_geo=m.N_geo, elem_map_nodes=m.elem_map_nodes,
                          face_connectivity=m.face_connectivity, boundary_tags=m.boundary_tags, h=m.h)
    cfg = rsv.SolverConfig(N=N, formulation=rsv.Formulation.StrongWeak)
    rd = rsv.Discretization(rm, cfg)
    rng = np.random.default_rng(0)
    st = rsv.FieldState(*(rng.standard_normal((m.K, rd.ref.Np)) for _ in range(3)))
    dt = 1e-4
    st = rsv.lsrk_step(st, dt, lambda y: rsv.rhs_full(y, rd))
    t0 = time.perf_counter()
    for _ in range(steps):
        st = rsv.lsrk_step(st, dt, lambda y: rsv.rhs_full(y, rd))
    t_ref = (time.perf_counter() - t0) / steps
    od = O.OracleDiscretization(m, N, True)
    ost = O.State(st.p, [st.u1, st.u2])
    ost = O.lsrk_step(ost, dt, lambda y: O.rhs_full(y, od))
    t0 = time.perf_counter()
    for _ in range(steps):
        ost = O.lsrk_step(ost, dt, lambda y: O.rhs_full(y, od))
    t_port = (time.perf_counter() - t0) / steps
    dof = 3 * m.K * rd.ref.Np * 5
    return {"mesh": f"warped triangles {K1D}x{K1D}x2 = {m.K}, N={N}, strong-weak",
            "reference_gdofs": dof / t_ref / 1e9, "port_gdofs": dof / t_port / 1e9,
            "port_over_reference_speed": t_ref / t_port}


def umma_issued_flops(N, Kpad):
    """Tensor-core flops the tcgen05 stage issues per launch: every MMA of
    csrc/wadg_fused_umma.cuh (M = 128, K = 8, split-TF32: 3 MMAs per product,
    padded extents) times 2 * 128 * N_mma * 8."""
    rup = lambda a, b: -(-a // b) * b
    NP = (N + 1) * (N + 2) * (N + 3) // 6
    NPK = NPN = rup(NP, 8)
    NQ = (N + 1) ** 3
    NCH = -(-NQ // 16)
    NFPK = rup((N + 1) * (N + 2) // 2, 8)
    NFH = -(-((N + 1) ** 2) // 16)
    mac = lambda n: 128 * n * 8
    per_chunk = (NPK // 8 * 3 * mac(48) + NPK // 8 * 9 * mac(16)      # D_a p, Vq u_i
                 + 2 * 9 * mac(NPN) + 2 * 9 * mac(NPN))               # -Pq gp_i, DTW_a F_a
    per_step = NFPK // 8 * 3 * 8 * mac(16) + 2 * 3 * 4 * mac(NPN)     # traces (own + ext), lifts
    per_uchunk = NPK // 8 * 3 * 4 * mac(16) + 2 * 3 * 4 * mac(NPN)    # z = Vu R, R (+)= Pu omega z
    per_tile = NCH * per_chunk + 4 * NFH * per_step + NCH * per_uchunk
    return 2.0 * per_tile * (Kpad // 128)


def dmma_issued_flops(N, Kpad):
    """FP64 tensor-core flops the DMMA stage issues per launch (csrc/wadg_fused_dmma.cuh:
    8 x 8 x 4 MMAs over padded extents)."""
    rup = lambda a, b: -(-a // b) * b
    NP = (N + 1) * (N + 2) * (N + 3) // 6
    NPP, NQ = rup(NP, 8), (N + 1) ** 3
    QC = 16
    NCH = -(-NQ // QC)
    NFPK, NFQP = rup((N + 1) * (N + 2) // 2, 4), rup((N + 1) ** 2, 8)
    fma = (NCH * QC * NPP * (6 + 6)          # volume: 6 products each way
           + 4 * (NFQP * NFPK * 8 + NFQP * NPP * 4)   # traces (own + ext, 4 fields), lifts
           + NCH * QC * NPP * (4 + 4))       # update z, R'
    return 2.0 * fma * Kpad


def tmma_issued_flops(N, Kpad):
    """Tensor-core flops the split-TF32 mma.sync stage issues per launch
    (csrc/wadg_fused_tmma.cuh: m16n8k8 tf32 MMAs over padded extents, three per
    product)."""
    rup = lambda a, b: -(-a // b) * b
    NP = (N + 1) * (N + 2) * (N + 3) // 6
    NPP, NQ = rup(NP, 8), (N + 1) ** 3
    QC = 16
    NCH = -(-NQ // QC)
    NFPK, NFQP = rup((N + 1) * (N + 2) // 2, 8), rup((N + 1) ** 2, 8)
    fma = (NCH * QC * NPP * (6 + 6)
           + 4 * (NFQP * NFPK * 8 + NFQP * NPP * 4)
           + NCH * QC * NPP * (4 + 4))
    return 2.0 * 3 * fma * Kpad


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_benchmark_rhs():
    """The reference's own per-phase timer (R/pkg/src/wadg/analysis.py:238-266,
    baseline/_ref, 2D only) on the warped triangles of config 1 at N = 4:
    ns per DOF of volume / surface / update, median of 10."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "wadg")):
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, ref_dir)
    try:
        from wadg import analysis as ran, meshgen as rmg, refelem as rrf, solver as rsv
        from paper_1608_03836_b200 import meshgen
        m = meshgen.warped_triangle_mesh(64, 4)
        rm = rmg.CurvedMesh2D(shape=rrf.ElementShape.Triangle, N_geo=m.N_geo, elem_map_nodes=m.elem_map_nodes,
                              face_connectivity=m.face_connectivity, boundary_tags=m.boundary_tags, h=m.h)
        rep = ran.benchmark_rhs(rm, rsv.SolverConfig(N=4, formulation=rsv.Formulation.StrongWeak), repetitions=10)
        return {"mesh": f"warped triangles 64x64x2 = {m.K}, N=4, strong-weak", "ns_per_dof": rep}
    except Exception as exc:                     # pragma: no cover
        return {"unavailable": f"{type(exc).__name__}: {exc}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_sample = 16
    t_all = []
    K = None
    for _ in range(args.warmup):
        cpu_oracle_rate(args.config, n_sample, 1, args.order)
    for _ in range(args.steps):
        v, K, el = cpu_oracle_rate(args.config, n_sample, 1, args.order)
        t_all.append(el)
    _, _, N, _, het, _ = CONFIGS[args.config]
    N = args.order or N
    from paper_1608_03836_b200 import refelem
    Np = refelem.basis_dimension(refelem.ElementShape.Tetrahedron, N)
    dof = 4 * K * Np
    t = float(np.median(t_all))
    value = dof * 5 / t / 1e9
    cores = os.cpu_count()
    sample = f"warped cube {n_sample}^3x6 = {K} tets, N={N}, fp64 numpy oracle, 1 LSRK step per timed step"
    line = {
        "impl": "reference", "metric": "GDOF/s per RK stage", "value": value, "unit": "GDOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.config == "c5" else "strong",   # as the GPU arm's line for this config
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config][0], "sample": sample},
        "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_2d_calibration": reference_2d_calibration(),
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--order", type=int, default=None, help="override N (config 3 sweep)")
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--impl", default="wadg", choices=["wadg", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--split", action="store_true", help="three kernels per stage instead of the fused one")
    ap.add_argument("--variant", type=int, default=-1,
                    help="fused kernel: 0 CUDA-core, 2 tcgen05 (default: per-order choice)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1608_03836_b200 import _native, solver

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.variant >= 0:
        _native.call("wadg_debug_set_fused_variant", args.variant)
    t_setup = time.perf_counter()
    mesh, cfg, medium, disc, desc = build_problem(args.config, args.order, args.dtype, rank, world)
    d = disc.dev
    state = solver.project_initial_condition_device(disc, gaussian_ic)
    setup_s = time.perf_counter() - t_setup
    N = cfg.N
    dt = 0.5 * mesh.h / (N + 1) ** 2
    Q = state
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    res, rhs = d.empty_fields(), d.empty_fields()
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    fl = disc.flux
    exch = getattr(disc, "exchange", None)

    fused = d.fused is not None and not args.split
    other = d.empty_fields() if fused else None
    bufs = {"Q": Q, "other": other}

    def stage(a, b, ev=None):
        Qc = bufs["Q"]
        if exch is not None:
            exch.start(Qc)
        if ev is not None:
            ev[0].record(stream)
        if fused:
            out = bufs["other"]
            if exch is not None:
                exch.fused_stage(Qc, out, res, fl.tau_p, fl.tau_u, a, b, dt, sp)
            else:
                _native.call("wadg_stage_fused", ctypes.byref(d.struct), vp(Qc), vp(out), vp(res),
                             fl.tau_p, fl.tau_u, a, b, dt, 0, -1, sp)
            bufs["Q"], bufs["other"] = out, Qc
            if ev is not None:
                ev[1].record(stream)
            return
        _native.call("wadg_volume", ctypes.byref(d.struct), vp(Qc), vp(rhs), sp)
        if ev is not None:
            ev[1].record(stream)
        if exch is not None:
            exch.surface(Qc, rhs, fl.tau_p, fl.tau_u, sp)
        else:
            _native.call("wadg_surface", ctypes.byref(d.struct), vp(Qc), vp(rhs), fl.tau_p, fl.tau_u,
                         1, 0, -1, sp)
        if ev is not None:
            ev[2].record(stream)
        _native.call("wadg_update_lsrk", ctypes.byref(d.struct), vp(rhs), vp(res), vp(Qc), a, b, dt, sp)
        if ev is not None:
            ev[3].record(stream)

    def step(evs=None):
        for s, (a, b) in enumerate(zip(solver.LSRK4A, solver.LSRK4B)):
            stage(a, b, None if evs is None else evs[s])

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()

    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(5)]
           for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t1.record(stream)
    torch.cuda.synchronize()
    ms_total = t0.elapsed_time(t1)
    clk = clocks.stop()
    names = ["stage_fused"] if fused else ["volume", "surface", "update"]
    kern = {k: [] for k in names}
    for i in range(args.steps):
        for s in range(5):
            e = evs[i][s]
            for m, k in enumerate(names):
                kern[k].append(e[m].elapsed_time(e[m + 1]))
    if world > 1:
        tt = torch.tensor([ms_total], device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms_total = float(tt.item())
    ms_step = ms_total / args.steps

    ref = disc.ref
    K_local = d.K
    Np = ref.Np
    dof_stage = (mesh.dim + 1) * K_local * Np
    dof_all = dof_stage * world
    value = dof_all * 5 * args.steps / (ms_total * 1e-3) / 1e9

    # roofline of the dominant kernel
    w = 4 if cfg.dtype == "float32" else 8
    B, FL = algorithmic_model(mesh.dim, K_local, Np, ref.Nq, disc.ref_upd.Nq,
                              ref.n_faces * ref.nfq, w, 2 if callable(medium.c2) else 1)
    if fused:
        fldn = mesh.dim + 1
        n_om = 2 if callable(medium.c2) else 1
        F = ref.n_faces * ref.nfq
        B = {"stage_fused": K_local * (w * (4 * fldn * Np + mesh.dim ** 2 * ref.Nq + n_om * disc.ref_upd.Nq
                                            + (mesh.dim + 1) * F) + 4 * ref.n_faces)}
        FL = {"stage_fused": sum(FL.values())}
    avg = {k: float(np.mean(v)) for k, v in kern.items()}
    top = max(avg, key=avg.get)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm_peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        with open(peaks_path) as f:
            hbm_peak = float(json.load(f)["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    achieved = B[top] / (avg[top] * 1e-3) / 1e9
    # compute side of the dominant kernel: flops the tensor / FP pipes are issued
    # (padded MMA extents, the 3 split-TF32 MMAs per product counted) against the
    # measured peaks (profiles/r02_measured_peaks.json), and the binding roof =
    # the larger of the two lower-bound times
    kind = getattr(d, "fused_kind", -1) if fused else -1
    peaks_r02 = {"tcgen05_tf32": 1105.2, "dmma_f64": 37.1, "ffma": 71.8, "dfma": 34.1, "mma_sync_tf32": 278.8}
    pk_path = os.path.join(ROOT, "profiles", "r02_measured_peaks.json")
    if os.path.exists(pk_path):
        with open(pk_path) as f:
            tf = json.load(f)["tflops"]
        peaks_r02 = {"tcgen05_tf32": tf["tcgen05_tf32_tflops_TS_N256"], "dmma_f64": tf["dmma_f64_tflops"],
                     "ffma": tf["fp32_fma_tflops"], "dfma": tf["fp64_fma_tflops"],
                     "mma_sync_tf32": tf["mma_sync_tf32_tflops"]}
    if kind == 2:
        issued, cpeak, cname = umma_issued_flops(N, d.Kpad), peaks_r02["tcgen05_tf32"], "tcgen05 kind::tf32"
    elif kind == 3:
        issued, cpeak, cname = dmma_issued_flops(N, d.Kpad), peaks_r02["dmma_f64"], "DMMA f64"
    elif kind == 4:
        issued, cpeak, cname = tmma_issued_flops(N, d.Kpad), peaks_r02["mma_sync_tf32"], "mma.sync tf32"
    else:
        issued = FL[top]
        cpeak, cname = (peaks_r02["ffma"], "FFMA") if cfg.dtype == "float32" else (peaks_r02["dfma"], "DFMA")
    t_hbm = B[top] / (hbm_peak * 1e9)
    t_cmp = issued / (cpeak * 1e12)
    compute = {"pipe": cname, "issued_tflop_per_launch": issued / 1e12,
               "achieved_tflops": issued / (avg[top] * 1e-3) / 1e12, "peak_tflops": cpeak,
               "frac": issued / (avg[top] * 1e-3) / 1e12 / cpeak,
               "lower_bound_ms": {"hbm": t_hbm * 1e3, "compute": t_cmp * 1e3}}
    # measured DRAM traffic per launch from the committed ncu --set full capture
    traffic = None
    kname = {2: "umma", 3: "dmma", 4: "tmma", 5: "reg"}.get(getattr(d, "fused_kind", 0), "fused")
    tname = f"ncu_stage_{kname}_{'f32' if cfg.dtype == 'float32' else 'f64'}_N{N}_{args.config}.json"
    tpath = os.path.join(ROOT, "profiles", "r02_" + tname)
    if not os.path.exists(tpath):
        tpath = os.path.join(ROOT, "profiles", "r01_" + tname)
    if fused and world == 1 and os.path.exists(tpath):
        with open(tpath) as f:
            nd = json.load(f)
        unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        traffic = sum(float(nd[k][0]) * unit.get(nd[k][1], 1e9)
                      for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    kernels = {k: {"ms": avg[k], "GB/s": B[k] / (avg[k] * 1e-3) / 1e9,
                   "hbm_frac": B[k] / (avg[k] * 1e-3) / 1e9 / hbm_peak,
                   "TFLOP/s": FL[k] / (avg[k] * 1e-3) / 1e12,
                   "share": avg[k] / sum(avg.values())} for k in avg}

    # end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e and world == 1:
        import torch as _t
        host = [_t.empty((K_local, Np), dtype=d.dtype).pin_memory() for _ in range(mesh.dim + 1)]
        for i in range(mesh.dim + 1):
            host[i].copy_(bufs["Q"][i, :, :K_local].T.cpu())
        hstate = solver.FieldState.from_fields(host)
        n_e2e = max(2, min(args.steps, 5))
        # two untimed calls: the first fills torch's pinned-host block cache with the
        # output buffer, the second with the one the next call writes while its input
        # (the previous output) is still alive; later calls reuse the two blocks
        for _ in range(2):
            hstate = solver.lsrk_step(hstate, dt, disc.rhs)
        torch.cuda.synchronize()
        e0, e1 = _t.cuda.Event(enable_timing=True), _t.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n_e2e):
            hstate = solver.lsrk_step(hstate, dt, disc.rhs)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / n_e2e
        nb = sum(h.numel() * h.element_size() for h in host)
        e2e = {"value": dof_stage * 5 / (e_ms * 1e-3) / 1e9, "unit": "GDOF/s",
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "ms_per_step": e_ms,
               "api": "solver.lsrk_step(FieldState(pinned host tensors), dt, disc.rhs) -> HostPipeline (chunked H2D / stages / D2H overlap)"}

    # multi-rank: each rank steps its slab's pinned host state through the same
    # public call (copy in, 5 stages with the per-stage halo exchange, copy out)
    if not args.no_e2e and world > 1:
        try:
            import torch as _t
            host = [_t.empty((K_local, Np), dtype=d.dtype).pin_memory() for _ in range(mesh.dim + 1)]
            for i in range(mesh.dim + 1):
                host[i].copy_(bufs["Q"][i, :, :K_local].T.cpu())
            hstate = solver.FieldState.from_fields(host)
            n_e2e = max(2, min(args.steps, 5))
            for _ in range(2):
                hstate = solver.lsrk_step(hstate, dt, disc.rhs)
            torch.cuda.synchronize()
            torch.distributed.barrier()
            e0, e1 = _t.cuda.Event(enable_timing=True), _t.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(n_e2e):
                hstate = solver.lsrk_step(hstate, dt, disc.rhs)
            e1.record(stream)
            torch.cuda.synchronize()
            tt = _t.tensor([e0.elapsed_time(e1) / n_e2e], device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(tt.item())
            nb = sum(h.numel() * h.element_size() for h in host)
            e2e = {"value": dof_all * 5 / (e_ms * 1e-3) / 1e9, "unit": "GDOF/s",
                   "h2d_bytes_per_step": nb * world, "d2h_bytes_per_step": nb * world, "ms_per_step": e_ms,
                   "api": "solver.lsrk_step(FieldState(pinned host slab), dt, disc.rhs) per rank, "
                          "halo exchange per stage; max over ranks"}
        except Exception as exc:                   # never lose the device-timed line
            e2e = {"error": f"{type(exc).__name__}: {exc}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, Ks, el = cpu_oracle_rate(args.config, 16, 3, args.order)
        try:
            from threadpoolctl import threadpool_limits
            with threadpool_limits(1):
                v1, _, el1 = cpu_oracle_rate(args.config, 12, 1, args.order)
            one = {"value": v1, "sample": f"warped cube 12^3x6, 1 LSRK step, {el1:.1f} s, 1 BLAS thread"}
        except Exception as exc:                  # pragma: no cover
            one = {"unavailable": f"{type(exc).__name__}: {exc}"}
        cpu = {"value": v, "unit": "GDOF/s", "cores": os.cpu_count(), "kind": "port",
               "cpu_model": cpu_model(),
               "sample": f"numpy oracle (fp64) on warped cube 16^3x6 = {Ks} tets, N={N}, "
                         f"3 LSRK steps, {el:.1f} s",
               "one_thread": one,
               "reference_benchmark_rhs_2d": reference_benchmark_rhs()}

    if rank == 0:
        Np2, Nqu = Np * Np, disc.ref_upd.Nq
        line = {
            "metric": "GDOF/s per RK stage", "value": value, "unit": "GDOF/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if args.config == "c5" else "strong",
            "vs_baseline": None,
            "dtype": "f32" if cfg.dtype == "float32" else "f64", "data": "synthetic",
            "config": {"workload": desc, "K": getattr(mesh, "K_total", mesh.K), "N": N, "Np": Np,
                       "formulation": "strong-weak",
                       "dt": dt, "l2": "inputs > L2 (fields+geometry ~GBs); no flush needed",
                       "parallelism": f"z-slabs x{world}", "setup_s": round(setup_s, 1)},
            "roofline": ({"bound": "hbm", "kernel": top, "achieved": achieved, "peak": hbm_peak,
                          "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                          "peak_source": peak_src, "algorithmic_bytes_per_launch": B[top],
                          "algorithmic_tflop_per_launch": FL[top] / 1e12,
                          "bound_from": "larger lower-bound time of HBM bytes vs issued compute",
                          "compute": compute}
                         if t_hbm >= t_cmp else
                         {"bound": "tensor" if kind in (2, 3) else "fp", "kernel": top,
                          "achieved": compute["achieved_tflops"], "peak": cpeak, "unit": "TFLOP/s",
                          "frac": compute["frac"], "traffic": traffic,
                          "peak_source": "measured (profiles/r02_measured_peaks.json)",
                          "hbm": {"achieved_gbs": achieved, "peak_gbs": hbm_peak, "frac": achieved / hbm_peak,
                                  "algorithmic_bytes_per_launch": B[top]},
                          "bound_from": "larger lower-bound time of HBM bytes vs issued compute",
                          "compute": compute}),
            "kernels": kernels,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": (5 if fused else 15) * args.steps,
            "stage_kernel": "wadg_stage_fused" if fused else "wadg_volume+wadg_surface+wadg_update_lsrk",
            "fused_kernel": ({0: "k_stage_fused (CUDA-core FMA)", 2: "k_stage_umma (tcgen05 split-TF32, TMEM)",
                              3: "k_stage_dmma (FP64 tensor cores, mma.sync m8n8k4)",
                              4: "k_stage_tmma (split-TF32 mma.sync m16n8k8)",
                              5: "k_stage_reg (one element per thread, registers)"}.get(getattr(d, "fused_kind", -1))
                             if fused else None),
            "clocks": clk,
            "storage_words_per_element": {"wadg_weights": 2 * Nqu, "dense_inverse": 2 * Np2,
                                          "ratio": Np2 / Nqu},
        }
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
