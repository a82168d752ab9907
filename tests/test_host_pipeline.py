"""Pipelined host-state LSRK step (solver.HostPipeline): the wavefront launch
order on CPU, and on the GPU bitwise agreement with the device-resident
stepper (the same per-element arithmetic on block ranges)."""

import numpy as np
import pytest
import torch

from paper_1608_03836_b200 import meshgen, solver
from paper_1608_03836_b200.solver import (FieldState, Formulation, SolverConfig, chunk_neighbour_ranges,
                                          pipeline_chunks, wavefront_schedule)


def _simulate(order, lo, hi, n_stages=5):
    """Replay an in-order launch list and check every read-after-write and
    write-after-read dependency of the ping-pong sweep."""
    nc = len(lo)
    done = {}                                   # (stage, chunk) -> launch position
    for pos, (s, c) in enumerate(order):
        assert (s, c) not in done
        if s > 1:
            for c2 in range(lo[c], hi[c] + 1):  # inputs: stage s-1 of the chunks c reads
                assert done.get((s - 1, c2), 10**9) < pos
            for c2 in range(nc):                # overwritten input: readers of c at stage s-1
                if lo[c2] <= c <= hi[c2]:
                    assert done.get((s - 1, c2), 10**9) < pos
        if s > 1:
            assert done[(s - 1, c)] < pos
        done[(s, c)] = pos
    assert len(done) == n_stages * nc


@pytest.mark.parametrize("nc,span", [(1, 0), (2, 1), (7, 1), (16, 1), (12, 2), (9, 3)])
def test_wavefront_schedule_respects_dependencies(nc, span):
    lo = [max(0, c - span) for c in range(nc)]
    hi = [min(nc - 1, c + span) for c in range(nc)]
    order = wavefront_schedule(lo, hi)
    _simulate(order, lo, hi)
    # stage 5 of chunk 0 finishes well before the sweep ends when there is room
    if nc >= 8 and span == 1:
        first5 = order.index((5, 0))
        assert first5 < len(order) // 2


def test_wavefront_schedule_irregular_ranges():
    rng = np.random.default_rng(3)
    nc = 10
    lo = [max(0, c - int(rng.integers(0, 3))) for c in range(nc)]
    hi = [min(nc - 1, c + int(rng.integers(0, 3))) for c in range(nc)]
    _simulate(wavefront_schedule(lo, hi), lo, hi)


@pytest.mark.parametrize("n,nblk_chunk", [(8, 2), (8, 5), (12, 7)])
def test_schedule_on_type_ordered_warped_cube(n, nblk_chunk):
    """The pipeline's chunk neighbour ranges on a real z-ordered tet mesh:
    neighbours reach at most one z layer, and the wavefront order over the
    chunks respects every dependency of the ping-pong sweep."""
    from paper_1608_03836_b200 import device, refelem
    mesh = meshgen.warped_cube_tet_mesh(n, 1)
    n_or = len(refelem.orientation_permutations(mesh.shape))
    nbr, _ = device.neighbour_tables(mesh, n_or)
    eb = 128
    nblk = -(-mesh.K // eb)
    blocks = [(b, min(b + nblk_chunk, nblk)) for b in range(0, nblk, nblk_chunk)]
    lo, hi = chunk_neighbour_ranges(nbr, blocks, eb)
    layer_blocks = 6 * n * n / eb                        # one z layer of the type-ordered mesh
    span = int(np.ceil(layer_blocks / nblk_chunk)) + 1
    assert all(0 <= c - lo[c] <= span and 0 <= hi[c] - c <= span for c in range(len(blocks)))
    # a neighbour outside [lo, hi] would break the schedule: check against the table
    owner = np.minimum(np.arange(mesh.K) // (eb * nblk_chunk), len(blocks) - 1)
    for f in range(4):
        m = nbr[f] >= 0
        oc, ok = owner[nbr[f][m]], owner[np.arange(mesh.K)[m]]
        assert np.all(lo[ok] <= oc) and np.all(oc <= hi[ok])
    _simulate(wavefront_schedule(lo, hi), lo, hi)


def test_pipeline_chunks_cover_whole_waves():
    for nblk, sms in [(12288, 148), (1536, 148), (100, 148), (5000, 132)]:
        c = pipeline_chunks(nblk, sms)
        assert sum(c) == nblk and min(c) > 0
        # whole waves everywhere except one chunk that takes the remainder
        assert sum(1 for x in c if x % sms) <= 1


@pytest.mark.gpu
@pytest.mark.parametrize("direct", [True, False])
@pytest.mark.parametrize("dtype,N", [("float32", 4), ("float32", 2), ("float64", 3), ("float32", 5), ("float32", 1)])
def test_host_pipeline_bitwise_device_stepper(dtype, N, direct):
    mesh = meshgen.warped_cube_tet_mesh(6, N)
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * z)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype=dtype)
    disc = solver.Discretization(mesh, cfg, solver.MediumField(c2))
    d = disc.dev
    assert d.fused is not None
    g = torch.Generator().manual_seed(11)
    tdt = d.dtype
    host = [torch.randn((mesh.K, disc.ref.Np), generator=g, dtype=torch.float64).to(tdt).pin_memory()
            for _ in range(4)]
    st = FieldState.from_fields(host)
    pipe = solver.HostPipeline(disc, chunk_blocks=2, direct=direct)
    assert len(pipe.blocks) > 3
    assert pipe.direct == (direct and d.fused_kind == 2)      # only the tcgen05 stage writes rows
    assert solver.HostPipeline.accepts(disc, st)
    ref = solver.DeviceStepper(disc, fused=True)
    Q = disc.to_device(st)
    dt = 1e-3
    a = st
    for _ in range(3):
        a = pipe.step(a, dt)
        Q = ref.step(Q, dt)
    b = disc.from_device(Q, st, 0.0)
    for x, y in zip(a.fields(), b.fields()):
        assert x.is_pinned()
        assert torch.equal(x, y)
    assert abs(a.t - 3 * dt) < 1e-15
    # the public entry point routes pinned host states through the pipeline
    c = solver.lsrk_step(st, dt, disc.rhs)
    assert disc._pipeline is not pipe
    assert getattr(disc, "_pipeline", None) is not None
    Q1 = solver.DeviceStepper(disc, fused=True).step(disc.to_device(st), dt)
    for x, y in zip(c.fields(), disc.from_device(Q1, st, 0.0).fields()):
        assert torch.equal(x, y)


@pytest.mark.gpu
def test_host_pipeline_chunks_of_more_tiles_than_sms():
    """Chunks larger than the SM count: the persistent tcgen05 CTAs (N = 3) loop
    over several tiles of a block range [b0, b1) with b0 > 0; bitwise equal to
    the device stepper."""
    mesh = meshgen.warped_cube_tet_mesh(16, 3)
    disc = solver.Discretization(mesh, SolverConfig(N=3, formulation=Formulation.StrongWeak, dtype="float32"))
    d = disc.dev
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nblk = d.Kpad // d.fused
    assert d.fused_kind == 2 and nblk > sms + 8
    g = torch.Generator().manual_seed(5)
    host = [torch.randn((mesh.K, disc.ref.Np), generator=g).pin_memory() for _ in range(4)]
    st = FieldState.from_fields(host)
    pipe = solver.HostPipeline(disc, chunk_blocks=[8, sms + 8, nblk - sms - 16])
    Q = disc.to_device(st)
    a = pipe.step(st, 1e-3)
    Q = solver.DeviceStepper(disc, fused=True).step(Q, 1e-3)
    for x, y in zip(a.fields(), disc.from_device(Q, st, 0.0).fields()):
        assert torch.equal(x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", [1, 2])
def test_stage_fused_rows_matches_field_layout(layout):
    """wadg_stage_fused_rows with Q_in (1) or Q_out (2) in the FieldState row
    layout is bitwise the field-layout stage; K is not a multiple of the
    128-element tile, so the last tile is partly padding."""
    import ctypes
    from paper_1608_03836_b200 import _native
    mesh = meshgen.warped_cube_tet_mesh(5, 3)
    assert mesh.K % 128
    disc = solver.Discretization(mesh, SolverConfig(N=3, formulation=Formulation.StrongWeak, dtype="float32"))
    d = disc.dev
    if getattr(d, "fused_kind", -1) != 2:
        pytest.skip("row layouts need the tcgen05 stage")
    K, Np = d.K, disc.ref.Np
    g = torch.Generator(device="cuda").manual_seed(5)
    rows = torch.randn((4, K, Np), generator=g, device="cuda")
    Q = d.empty_fields()
    Q[:, :, :K] = rows.transpose(1, 2)
    res0 = torch.randn(d.empty_fields().shape, generator=g, device="cuda")
    res0[:, :, K:] = 0
    s = ctypes.byref(d.struct)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    fl = disc.flux
    ra, rb = res0.clone(), res0.clone()
    out_a = d.empty_fields()
    _native.call("wadg_stage_fused", s, vp(Q), vp(out_a), vp(ra), fl.tau_p, fl.tau_u, 0.3, 0.7, 1e-3, 0, -1, sp)
    if layout == 1:
        out_b = d.empty_fields()
        _native.call("wadg_stage_fused_rows", s, vp(rows), vp(out_b), vp(rb), fl.tau_p, fl.tau_u, 0.3, 0.7, 1e-3,
                     0, -1, 1, sp)
        assert torch.equal(out_a[:, :, :K], out_b[:, :, :K])
    else:
        out_b = torch.full((4, K, Np), float("nan"), device="cuda")
        _native.call("wadg_stage_fused_rows", s, vp(Q), vp(out_b), vp(rb), fl.tau_p, fl.tau_u, 0.3, 0.7, 1e-3,
                     0, -1, 2, sp)
        assert torch.equal(out_a[:, :, :K].transpose(1, 2), out_b)
    assert torch.equal(ra[:, :, :K], rb[:, :, :K])
    with pytest.raises(_native.NativeError):
        _native.call("wadg_stage_fused_rows", s, vp(Q), vp(out_a), vp(rb), fl.tau_p, fl.tau_u, 0.3, 0.7, 1e-3,
                     0, -1, 3, sp)


class _RecordingExchange:
    """Stands in for parallel.HaloExchange on a single domain (no halo
    slots): records the calls DeviceStepper makes and runs the full range."""

    def __init__(self, disc):
        self.disc, self.calls = disc, []

    def start(self, Q):
        self.calls.append("start")

    def fused_stage(self, Qin, Qout, res, tau_p, tau_u, a, b, dt, sp):
        import ctypes
        from paper_1608_03836_b200 import _native
        self.calls.append("fused")
        vp = lambda t: ctypes.c_void_p(t.data_ptr())
        _native.call("wadg_stage_fused", ctypes.byref(self.disc.dev.struct), vp(Qin), vp(Qout), vp(res),
                     tau_p, tau_u, a, b, dt, 0, -1, sp)

    def surface(self, Q, rhs, tau_p, tau_u, sp):
        import ctypes
        from paper_1608_03836_b200 import _native
        self.calls.append("surface")
        vp = lambda t: ctypes.c_void_p(t.data_ptr())
        _native.call("wadg_surface", ctypes.byref(self.disc.dev.struct), vp(Q), vp(rhs), tau_p, tau_u,
                     1, 0, -1, sp)


@pytest.mark.gpu
@pytest.mark.parametrize("fused", [True, False])
def test_device_stepper_routes_stages_through_the_slab_exchange(fused):
    """A slab discretization (disc.exchange set by parallel.slab_discretization)
    must post its halo every stage: DeviceStepper, and so lsrk_step on a slab,
    goes through exchange.start + exchange.fused_stage / surface, with results
    identical to the single-domain stage."""
    mesh = meshgen.warped_cube_tet_mesh(4, 3)
    cfg = SolverConfig(N=3, formulation=Formulation.StrongWeak, dtype="float32")
    disc = solver.Discretization(mesh, cfg)
    g = torch.Generator().manual_seed(2)
    st = FieldState.from_fields([torch.randn((mesh.K, disc.ref.Np), generator=g) for _ in range(4)])
    Q0 = disc.to_device(st)
    want = solver.DeviceStepper(disc, fused=fused).step(Q0.clone(), 1e-3)
    disc.exchange = _RecordingExchange(disc)
    got = solver.DeviceStepper(disc, fused=fused).step(Q0.clone(), 1e-3)
    assert torch.equal(got[:, :, :mesh.K], want[:, :, :mesh.K])
    assert disc.exchange.calls == ["start", "fused" if fused else "surface"] * 5
    pinned = FieldState.from_fields([a.pin_memory() for a in st.fields()])
    assert not solver.HostPipeline.accepts(disc, pinned)      # slabs step through the exchange


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["tet_fused_f64", "tet_fused_f32", "tet5_fused_f32", "tet1_fused_f64", "tri_split_f64"])
def test_graphed_steps_bitwise_eager(case):
    """DeviceStepper.step_graphed (captured CUDA graph, replayed) gives the
    eager step's result bit for bit, across the ping-pong buffer alternation
    (tcgen05, DMMA, mma.sync tf32 (N = 5), the N = 1 register stage and
    per-phase kernels)."""
    if case.startswith("tet5"):
        mesh, N = meshgen.warped_cube_tet_mesh(3, 5), 5
    elif case.startswith("tet1"):
        mesh, N = meshgen.warped_cube_tet_mesh(3, 1), 1
    elif case.startswith("tet"):
        mesh, N = meshgen.warped_cube_tet_mesh(3, 3), 3
    else:
        mesh, N = meshgen.warped_triangle_mesh(4, 3), 3
    dtype = "float32" if case.endswith("f32") else "float64"
    disc = solver.Discretization(mesh, SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype=dtype))
    g = torch.Generator().manual_seed(4)
    st = FieldState.from_fields([torch.randn((mesh.K, disc.ref.Np), generator=g, dtype=torch.float64)
                                 for _ in range(mesh.dim + 1)])
    a, b = solver.DeviceStepper(disc), solver.DeviceStepper(disc)
    Qa, Qb = disc.to_device(st), disc.to_device(st)
    Qa = a.step(Qa, 1e-3)                  # warm the kernels before any capture
    Qb = b.step(Qb, 1e-3)
    for _ in range(4):
        Qa = a.step(Qa, 1e-3)
        Qb = b.step_graphed(Qb, 1e-3)
    torch.cuda.synchronize()
    assert torch.equal(Qa[:, :, :mesh.K], Qb[:, :, :mesh.K])
