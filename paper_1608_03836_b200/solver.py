"""Drop-in replacement for the reference's ``wadg.solver`` right-hand-side
and time-step path (R/pkg/src/wadg/solver.py), executed by the sm_100a
kernels of libwadg_b200.so.

Same names, signatures, error types and semantics as the reference:
``Discretization(mesh, config, medium)``, ``_volume_terms``,
``_surface_terms``, ``rhs_strong``, ``rhs_strong_weak``, ``rhs_pre_mass``,
``apply_mass_inverse``, ``rhs_full``, ``lsrk_step``, ``energy``,
``stable_dt``, ``project_initial_condition``, ``run``.

FieldState arrays may be host numpy arrays (copied to the GPU and back per
call, like a drop-in replacement must) or CUDA torch tensors (stay
resident).  ``Discretization.rhs`` is the bound RHS that ``lsrk_step``
recognises to run each stage as one fused device pass; any other callable
goes through the generic device stage axpy.  There is no CPU fallback: every
RHS / update / step evaluation runs in the CUDA library.

Extensions over the reference: tetrahedral meshes (fields p, u1, u2, u3),
``SolverConfig.dtype`` ("float64" / "float32").
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native, geometry, refelem
from .device import DeviceProblem, medium_on_device
from .errors import BlowUp, ConfigError  # noqa: F401  (reference names)
from .refelem import ElementShape


class Formulation(enum.Enum):
    Strong = "strong"
    StrongWeak = "strong-weak"


class MassMode(enum.Enum):
    WADG = "wadg"
    ExactCurvedMass = "exact"


@dataclass(frozen=True)
class FluxParams:
    tau_p: float = 1.0
    tau_u: float = 1.0

    def __post_init__(self):
        if self.tau_p < 0 or self.tau_u < 0:
            raise ConfigError("penalty parameters must be nonnegative")


@dataclass(frozen=True)
class MediumField:
    """Squared wavespeed, constant or a callable c2(x, y[, z]); density 1."""

    c2: object = 1.0

    def values(self, *xyz):
        x = xyz[0]
        if callable(self.c2):
            v = np.broadcast_to(np.asarray(self.c2(*xyz), dtype=float), x.shape).copy()
        else:
            v = np.full_like(x, float(self.c2))
        if np.any(v <= 0):
            raise ConfigError("wavespeed squared must be positive")
        return v

    def spec(self):
        """Constant float or the callable (validated lazily on the device)."""
        if callable(self.c2):
            return self.c2
        if float(self.c2) <= 0:
            raise ConfigError("wavespeed squared must be positive")
        return float(self.c2)


@dataclass(frozen=True)
class SolverConfig:
    N: int
    formulation: Formulation = Formulation.Strong
    mass_mode: MassMode = MassMode.WADG
    flux: FluxParams = field(default_factory=FluxParams)
    cfl: float = 0.5
    volume_quad_degree: int | None = None
    face_quad_degree: int | None = None
    update_quad_degree: int | None = None
    unsafe_quadrature: bool = False
    dtype: str = "float64"


def sufficient_quadrature_degrees(N, N_geo, shape):
    """R/.../solver.py:80-90; tetrahedra: cofactors are degree 2(N_geo-1),
    giving the paper's 4N-3 / 4N-2 at N_geo = N (R/PAPER.md:288,294)."""
    if shape is ElementShape.Triangle:
        return 2 * N + N_geo - 2, 2 * N + N_geo - 1
    if shape is ElementShape.Tetrahedron:
        return 2 * N + 2 * N_geo - 3, 2 * N + 2 * N_geo - 2
    return 2 * N + N_geo - 1, 2 * N + N_geo - 1


@dataclass
class FieldState:
    """Pressure and velocity coefficients, (K, Np) each, at time t."""

    p: object
    u1: object
    u2: object
    u3: object = None
    t: float = 0.0

    def __post_init__(self):
        # reference positional form FieldState(p, u1, u2, t)
        if self.u3 is not None and np.isscalar(self.u3):
            self.t, self.u3 = float(self.u3), None

    def fields(self):
        return [self.p, self.u1, self.u2] + ([self.u3] if self.u3 is not None else [])

    @classmethod
    def from_fields(cls, fs, t=0.0):
        return cls(fs[0], fs[1], fs[2], fs[3] if len(fs) > 3 else None, t)

    def copy(self):
        c = (lambda a: a.clone()) if isinstance(self.p, torch.Tensor) else (lambda a: a.copy())
        return FieldState.from_fields([c(a) for a in self.fields()], self.t)

    def check_finite(self):
        for a in self.fields():
            ok = bool(torch.isfinite(a).all()) if isinstance(a, torch.Tensor) else bool(np.all(np.isfinite(a)))
            if not ok:
                raise FloatingPointError("non-finite field values")


def _degrees(mesh, config):
    N = config.N
    vol_deg, face_deg = sufficient_quadrature_degrees(N, mesh.N_geo, mesh.shape)
    if config.formulation is Formulation.StrongWeak:
        vol_deg, face_deg = 2 * N + 1, 2 * N + 1
    if config.volume_quad_degree is not None:
        vol_deg = config.volume_quad_degree
    if config.face_quad_degree is not None:
        face_deg = config.face_quad_degree
    if config.formulation is Formulation.Strong and not config.unsafe_quadrature:
        need = sufficient_quadrature_degrees(N, mesh.N_geo, mesh.shape)
        if vol_deg < need[0] or face_deg < need[1]:
            raise ConfigError(
                f"strong form needs volume/face quadrature degrees {need}; "
                f"got ({vol_deg}, {face_deg}); set unsafe_quadrature to override")
    return vol_deg, face_deg


class Discretization:
    """Prepared operator data for one (mesh, config, medium) triple, resident
    on the GPU (R/.../solver.py:111-204).  Host-side reference attributes
    (geo, w_upd_p, w_upd_u, c2q, bc_mask) are computed on first access."""

    def __init__(self, mesh, config, medium=MediumField(), device="cuda", k_range=None, halo=None):
        vol_deg, face_deg = _degrees(mesh, config)
        if config.dtype not in ("float64", "float32"):
            raise ConfigError(f"dtype must be float64 or float32, got {config.dtype!r}")
        self.mesh, self.config, self.medium = mesh, config, medium
        self.flux = config.flux
        self.c2_spec = medium.spec()
        self.ref = refelem.build_reference_element(
            config.N, mesh.shape, volume_quad_degree=vol_deg, face_quad_degree=face_deg)
        upd_deg = config.update_quad_degree or (2 * config.N + 1)
        self.ref_upd = refelem.build_reference_element(
            config.N, mesh.shape, volume_quad_degree=upd_deg, face_quad_degree=1)
        self.exact_mass = config.mass_mode is MassMode.ExactCurvedMass
        self.strong_weak = config.formulation is Formulation.StrongWeak
        self.dim = mesh.shape.dim
        self._device = device
        self._k_range = k_range
        self._halo = halo
        self._dev = None
        self._host = {}

    @property
    def rhs(self):
        """rhs_full bound to this discretization (a fresh small object per access,
        so the discretization holds no reference cycle through it)."""
        return _BoundRHS(self)

    # -- device ------------------------------------------------------------------
    @property
    def dev(self):
        if self._dev is None:
            k0, k1 = self._k_range if self._k_range is not None else (0, self.mesh.K)
            self._dev = DeviceProblem(self.mesh, self.ref, self.ref_upd, self.c2_spec,
                                      self.strong_weak, self.config.dtype, self._device,
                                      k0, k1, self._halo, exact_mass=self.exact_mass)
        return self._dev

    # -- ExactCurvedMass comparator: dense per-element inverses (solver.py:156-167);
    # None in WADG mode, which stores only pointwise weights
    @property
    def mass_inv_p(self):
        if not self.exact_mass:
            return None
        if "mass_inv" not in self._host:
            self._host["mass_inv"] = self.dev.host_mass_inverses()
        return self._host["mass_inv"][0]

    @property
    def mass_inv_u(self):
        if not self.exact_mass:
            return None
        self.mass_inv_p
        return self._host["mass_inv"][1]

    # -- host reference attributes (diagnostics / compatibility) -------------
    def _host_geo(self):
        if "geo" not in self._host:
            self._host["geo"] = geometry.compute_geometric_data(self.mesh, self.ref)
        return self._host["geo"]

    @property
    def geo(self):
        return self._host_geo()

    @property
    def w_upd_p(self):
        if "w_upd_p" not in self._host:
            gu = geometry.compute_geometric_data(self.mesh, self.ref_upd)
            self._host["w_upd_p"] = self.medium.values(*gu.xyzq) / gu.Jq
            self._host["w_upd_u"] = 1.0 / gu.Jq
        return self._host["w_upd_p"]

    @property
    def w_upd_u(self):
        self.w_upd_p
        return self._host["w_upd_u"]

    @property
    def c2q(self):
        if "c2q" not in self._host:
            self._host["c2q"] = self.medium.values(*self.geo.xyzq)
        return self._host["c2q"]

    @property
    def c_max(self):
        return np.sqrt(self.c2q.max(axis=1))

    @property
    def bc_mask(self):
        return np.repeat(self.mesh.boundary_tags > 0, self.ref.nfq, axis=1)

    def interp(self, u):
        return u @ self.ref.Vq.T

    def face_traces(self, u):
        """Interior / exterior traces at face quadrature points (host numpy,
        a diagnostic helper kept for reference-API compatibility; the device
        surface kernel builds these from nodal face values)."""
        ref, mesh = self.ref, self.mesh
        perms = ref.face_perms
        fm = np.array(ref.face_nodes)
        uf = u @ ref.Vfq.T
        up = uf.copy()
        conn, ori = mesh.face_connectivity, mesh.face_orientation
        for f in range(mesh.n_faces):
            inner = conn[:, f, 0] >= 0
            k2, f2, o = conn[inner, f, 0], conn[inner, f, 1], ori[inner, f]
            nodes = fm[f2[:, None], perms[o]]
            vals = np.take_along_axis(u[k2], nodes, axis=1)
            up[inner, f * ref.nfq:(f + 1) * ref.nfq] = vals @ ref.face_interp.T
        return uf, up

    # -- packing -----------------------------------------------------------------
    def to_device(self, state):
        """(K, Np) host numpy / host torch (pinned) / CUDA tensors -> the
        (dim+1, Np, Kpad) device layout in the working dtype."""
        d = self.dev
        Q = d.empty_fields()
        for i, a in enumerate(state.fields()):
            if not isinstance(a, torch.Tensor):
                a = torch.from_numpy(np.ascontiguousarray(a))
            a = a.to(d.device, non_blocking=True)
            Q[i, :, :d.K].copy_(a.T)
        return Q

    def from_device(self, Q, like, t):
        """Inverse of to_device, returning the container type of ``like``.
        The (dim+1, Np, K) -> (dim+1, K, Np) transpose happens on the device so
        the device-to-host copy is one contiguous transfer."""
        d = self.dev
        Qt = Q[:, :, :d.K].transpose(1, 2)
        if isinstance(like.p, torch.Tensor) and like.p.is_cuda:
            return FieldState.from_fields([a.contiguous() for a in Qt], t)
        if isinstance(like.p, torch.Tensor):
            dev = Qt.to(like.p.dtype).contiguous()
            h = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=like.p.is_pinned())
            h.copy_(dev)
            return FieldState.from_fields(list(h.unbind(0)), t)
        h = Qt.to(torch.float64).contiguous().cpu().numpy()
        return FieldState.from_fields([h[i] for i in range(d.fld)], t)


def _stream():
    return ctypes_ptr(torch.cuda.current_stream().cuda_stream)


def _on_disc_device(fn):
    """Run a compute entry point with the Discretization's device current, so
    the launches, their stream (_stream) and the per-device kernel attributes
    all refer to that device even when another device is current."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kw):
        disc = next((a for a in args if isinstance(a, Discretization)), None)
        if disc is None and args:
            disc = getattr(args[0], "disc", None)
        if disc is None or not torch.cuda.is_available():
            return fn(*args, **kw)      # no device: the call itself raises (no CPU fallback)
        with torch.cuda.device(disc.dev.device):
            return fn(*args, **kw)
    return wrapper


def ctypes_ptr(v):
    import ctypes
    return ctypes.c_void_p(v)


def _vp(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def _check_state(state, disc):
    if len(state.fields()) != disc.dim + 1:
        raise ValueError(f"state has {len(state.fields())} fields, mesh needs {disc.dim + 1}")


@_on_disc_device
def _volume_terms(state, disc, strong_weak):
    _check_state(state, disc)
    d = disc.dev
    Q = disc.to_device(state)
    out = d.empty_fields()
    s = d.with_formulation(strong_weak)
    import ctypes
    _native.call("wadg_volume", ctypes.byref(s), _vp(Q), _vp(out), _stream())
    return tuple(disc.from_device(out, state, state.t).fields())


@_on_disc_device
def _surface_terms(state, disc, strong_weak):
    _check_state(state, disc)
    d = disc.dev
    Q = disc.to_device(state)
    out = d.empty_fields()
    s = d.with_formulation(strong_weak)
    import ctypes
    _native.call("wadg_surface", ctypes.byref(s), _vp(Q), _vp(out), disc.flux.tau_p,
                 disc.flux.tau_u, 0, 0, -1, _stream())
    return tuple(disc.from_device(out, state, state.t).fields())


@_on_disc_device
def _rhs_pre(state, disc, strong_weak):
    import ctypes
    _check_state(state, disc)
    d = disc.dev
    Q = disc.to_device(state)
    out = d.empty_fields()
    s = d.with_formulation(strong_weak)
    _native.call("wadg_volume", ctypes.byref(s), _vp(Q), _vp(out), _stream())
    _native.call("wadg_surface", ctypes.byref(s), _vp(Q), _vp(out), disc.flux.tau_p,
                 disc.flux.tau_u, 1, 0, -1, _stream())
    return disc.from_device(out, state, state.t)


def rhs_strong(state, disc):
    """Strong-form RHS, Mhat^-1-premultiplied (R/.../solver.py:268-273)."""
    return _rhs_pre(state, disc, False)


def rhs_strong_weak(state, disc):
    """Strong-weak RHS, Mhat^-1-premultiplied (R/.../solver.py:276-281)."""
    return _rhs_pre(state, disc, True)


def rhs_pre_mass(state, disc):
    return _rhs_pre(state, disc, disc.strong_weak)


@_on_disc_device
def apply_mass_inverse(rhs_pre, disc):
    """Mass inverse on a premultiplied RHS (R/.../solver.py:290-306): matrix-free
    WADG, or the stored dense inverses of the ExactCurvedMass comparator."""
    import ctypes
    _check_state(rhs_pre, disc)
    d = disc.dev
    R = disc.to_device(rhs_pre)
    out = d.empty_fields()
    _native.call("wadg_mass_inverse", ctypes.byref(d.struct), _vp(R), _vp(out), _stream())
    return disc.from_device(out, rhs_pre, rhs_pre.t)


@_on_disc_device
def rhs_full(state, disc):
    """apply_mass_inverse(rhs_pre_mass(state)) in one device pass.  Where the
    fused tetrahedral stage applies (one domain, WADG mass inverse), this is one
    fused-stage launch with a = b = 0 and dt = 1, whose LSRK register output is
    exactly M^-1 rhs; otherwise the per-phase volume, surface and mass-inverse
    kernels."""
    import ctypes
    _check_state(state, disc)
    d = disc.dev
    Q = disc.to_device(state)
    out = d.empty_fields()
    s = d.struct
    if d.fused is not None and getattr(disc, "exchange", None) is None and (d.halo is None or not d.halo.n_recv):
        scratch = d.empty_fields()
        _native.call("wadg_stage_fused", ctypes.byref(s), _vp(Q), _vp(scratch), _vp(out), disc.flux.tau_p,
                     disc.flux.tau_u, 0.0, 0.0, 1.0, 0, -1, _stream())
        return disc.from_device(out, state, state.t)
    pre = d.empty_fields()
    _native.call("wadg_volume", ctypes.byref(s), _vp(Q), _vp(pre), _stream())
    _native.call("wadg_surface", ctypes.byref(s), _vp(Q), _vp(pre), disc.flux.tau_p,
                 disc.flux.tau_u, 1, 0, -1, _stream())
    _native.call("wadg_mass_inverse", ctypes.byref(s), _vp(pre), _vp(out), _stream())
    return disc.from_device(out, state, state.t)


class _BoundRHS:
    """disc.rhs: rhs_full bound to a discretization; lsrk_step runs it as
    fused device stages."""

    def __init__(self, disc):
        self.disc = disc

    def __call__(self, state):
        return rhs_full(state, self.disc)


@_on_disc_device
def energy(state, disc):
    """1/2 int (p^2/c^2 + |u|^2) by volume quadrature (R/.../solver.py:314-321)."""
    d = disc.dev
    Q = state if isinstance(state, torch.Tensor) else disc.to_device(state)
    return device_energy(disc, Q)


@_on_disc_device
def device_energy(disc, Q):
    import ctypes
    d = disc.dev
    d.prepare_energy(disc.c2_spec)
    _native.call("wadg_energy", ctypes.byref(d.struct), _vp(Q), _vp(d.energy_partials),
                 _vp(d.energy_out), _stream())
    return float(d.energy_out.item())


# Carpenter-Kennedy low-storage five-stage fourth-order coefficients
LSRK4A = (
    0.0,
    -567301805773.0 / 1357537059087.0,
    -2404267990393.0 / 2016746695238.0,
    -3550918686646.0 / 2091501179385.0,
    -1275806237668.0 / 842570457699.0,
)
LSRK4B = (
    1432997174477.0 / 9575080441755.0,
    5161836677717.0 / 13612068292357.0,
    1720146321549.0 / 2090206949498.0,
    3134564353537.0 / 4481467310338.0,
    2277821191437.0 / 14882151754819.0,
)
LSRK4C = (
    0.0,
    1432997174477.0 / 9575080441755.0,
    2526269341429.0 / 6820363962896.0,
    2006345519317.0 / 3224310063776.0,
    2802321613138.0 / 2924317926251.0,
)


class DeviceStepper:
    """Device-resident LSRK45 driver.  For 3D strong-weak problems each stage
    is one fused kernel (wadg_stage_fused) reading Q from one buffer and
    writing the other; otherwise a stage is the volume, surface and
    update+axpy kernels in place.  ``step`` returns the buffer that holds the
    new state."""

    def __init__(self, disc, fused=None):
        self.disc = disc
        d = disc.dev
        self.fused = (d.fused is not None) if fused is None else (fused and d.fused is not None)
        self.res = d.empty_fields()
        self.rhs = None if self.fused else d.empty_fields()
        self.other = d.empty_fields() if self.fused else None

    @_on_disc_device
    def stage(self, Q, a, b, dt, started=False):
        """One LSRK stage; for a slab (disc.exchange) the halo of Q is packed and
        posted first, unless the caller did that already (started=True, e.g. a
        driver of several slabs in one process posts every slab's halo before
        running any stage)."""
        import ctypes
        d = self.disc.dev
        fl = self.disc.flux
        exch = getattr(self.disc, "exchange", None)      # slab of a multi-rank run (parallel.py)
        if exch is not None and not started:
            exch.start(Q)                                # pack + post this stage's halo traces
        if self.fused:
            out = self.other
            if exch is not None:
                exch.fused_stage(Q, out, self.res, fl.tau_p, fl.tau_u, a, b, dt, _stream())
            else:
                _native.call("wadg_stage_fused", ctypes.byref(d.struct), _vp(Q), _vp(out), _vp(self.res),
                             fl.tau_p, fl.tau_u, a, b, dt, 0, -1, _stream())
            self.other = Q
            return out
        if exch is not None:
            _native.call("wadg_volume", ctypes.byref(d.struct), _vp(Q), _vp(self.rhs), _stream())
            exch.surface(Q, self.rhs, fl.tau_p, fl.tau_u, _stream())
            _native.call("wadg_update_lsrk", ctypes.byref(d.struct), _vp(self.rhs), _vp(self.res), _vp(Q),
                         a, b, dt, _stream())
            return Q
        _native.call("wadg_stage", ctypes.byref(d.struct), _vp(Q), _vp(self.res), _vp(self.rhs),
                     fl.tau_p, fl.tau_u, a, b, dt, _stream())
        return Q

    def step(self, Q, dt):
        for a, b in zip(LSRK4A, LSRK4B):
            Q = self.stage(Q, a, b, dt)
        return Q

    @_on_disc_device
    def step_graphed(self, Q, dt):
        """``step`` replayed from a CUDA graph.  The launches of one step are
        captured once per (input buffer, dt) and replayed, which removes the
        host launch overhead that dominates small meshes.  The kernels and
        results are the same.  Slab steps with a halo exchange (NCCL) stay
        eager."""
        if getattr(self.disc, "exchange", None) is not None:
            return self.step(Q, dt)
        graphs = self.__dict__.setdefault("_graphs", {})
        key = (Q.data_ptr(), float(dt))
        if key not in graphs:
            if len(graphs) >= 4:
                graphs.clear()
            torch.cuda.current_stream().synchronize()
            other_before = self.other
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                out = self.step(Q, dt)
            graphs[key] = (graph, out, self.other)
            self.other = other_before            # capture did not run anything
        graph, out, other_after = graphs[key]
        graph.replay()
        self.other = other_after
        return out


def pipeline_chunks(nblk, sms, wave_chunk=3):
    """Chunk sizes (in fused blocks) for the host pipeline: whole waves of
    ``sms`` blocks, ``wave_chunk`` waves in the middle and one wave at both
    ends.  Small first chunks shorten the fill (stage 1 waits for the first
    chunks to arrive) and small last chunks the drain (the last chunk's copy
    back)."""
    big = sms * wave_chunk
    if nblk <= 4 * big:
        cb = max(1, min(nblk, sms))
        return [min(cb, nblk - b) for b in range(0, nblk, cb)]
    head = [sms] * wave_chunk
    tail = [sms] * wave_chunk
    mid = nblk - sum(head) - sum(tail)
    body = [big] * (mid // big)
    rest = mid - sum(body)
    if rest:
        body.append(rest)
    return head + body + tail


def chunk_neighbour_ranges(nbr, blocks, eb):
    """For element chunks given as fused-block ranges ``blocks`` (eb elements
    per block), the lowest and highest chunk holding a face neighbour of each
    chunk, itself included.  ``nbr`` is the (Nf, K) neighbour table (< 0 =
    boundary or halo)."""
    K = nbr.shape[1]
    edges = np.array([b0 for b0, _ in blocks] + [blocks[-1][1]])
    owner = np.searchsorted(edges, np.arange(K) // eb, side="right") - 1
    nc = len(blocks)
    lo, hi = np.arange(nc), np.arange(nc)
    for c, (b0, b1) in enumerate(blocks):
        nb = nbr[:, min(b0 * eb, K):min(b1 * eb, K)]
        nb = nb[nb >= 0]
        if nb.size:
            oc = owner[nb]
            lo[c], hi[c] = min(c, int(oc.min())), max(c, int(oc.max()))
    return lo, hi


def wavefront_schedule(lo, hi, n_stages=5):
    """Launch order of (stage, chunk) pairs for a chunked multi-stage sweep on
    one in-order stream.  Chunk c reads the chunks lo[c]..hi[c] of the
    previous stage.  Stage s on c runs once stage s-1 has finished every chunk
    c reads (read after write).  It must also wait for every chunk that reads
    c, because it overwrites that stage's input buffer (write after read).
    Among the ready pairs the highest stage goes first, so finished chunks
    leave early."""
    nc = len(lo)
    reach = [max([hi[c]] + [c2 for c2 in range(nc) if lo[c2] <= c <= hi[c2]]) for c in range(nc)]
    done = [nc] + [0] * n_stages              # chunks finished per stage (stage 0 = input)
    order = []
    while done[n_stages] < nc:
        for s in range(n_stages, 0, -1):
            c = done[s]
            if c < nc and done[s - 1] > (reach[c] if s > 1 else -1):
                order.append((s, c))
                done[s] += 1
                break
    return order


class HostPipeline:
    """LSRK45 step on a host-resident state, pipelined over element chunks.

    The state is split into chunks of whole fused-stage blocks (a multiple of
    the SM count by default).  Three streams overlap the work:
      * a copy stream moves chunk c host -> device, and a conversion stream
        turns it into the field layout (wadg_rows_to_fields) once it lands, so
        the copy engine never waits behind a kernel;
      * the current stream runs the five stage kernels on block ranges in a
        wavefront order;
      * a second copy stream converts each chunk back (wadg_fields_to_rows) and
        copies it device -> host as soon as stage 5 has finished it.
    Stage s of chunk c needs stage s-1 on every chunk that holds a face
    neighbour of c.  The ping-pong buffer it writes is also read by stage s-1
    of those chunks, so one in-order stream and that dependency suffice; the
    neighbour chunk range comes from the nbr table.  Needs the fused stage,
    one rank and pinned host tensors of the device dtype (FieldState layout,
    (K, Np) per field).  The input is converted by wadg_rows_to_fields on the
    copy stream.  With the tcgen05 stage the last stage writes the row layout
    itself (wadg_stage_fused_rows); other kernels convert back with
    wadg_fields_to_rows on the second copy stream."""

    def __init__(self, disc, chunk_blocks=None, direct=True):
        d = disc.dev
        if d.fused is None:
            raise ConfigError("host pipeline needs the fused stage kernel")
        if d.halo is not None and d.halo.n_recv:
            raise ConfigError("host pipeline is single-rank")
        self.disc = disc
        self.stepper = DeviceStepper(disc, fused=True)
        eb = d.fused
        assert d.Kpad % eb == 0
        nblk = d.Kpad // eb
        sms = torch.cuda.get_device_properties(d.device).multi_processor_count
        if chunk_blocks is None:
            chunk_blocks = pipeline_chunks(nblk, sms)
        elif isinstance(chunk_blocks, int):
            cb = max(1, min(chunk_blocks, nblk))
            chunk_blocks = [min(cb, nblk - b) for b in range(0, nblk, cb)]
        assert sum(chunk_blocks) == nblk and min(chunk_blocks) > 0
        edges = np.concatenate([[0], np.cumsum(chunk_blocks)])
        self.blocks = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]
        K = d.K
        self.elems = [(min(b0 * eb, K), min(b1 * eb, K)) for b0, b1 in self.blocks]
        nc = len(self.blocks)
        self.lo, self.hi = chunk_neighbour_ranges(d.nbr[:, :K].cpu().numpy(), self.blocks, eb)
        self.schedule = wavefront_schedule(self.lo, self.hi)
        fld = d.fld
        self.rows_in = torch.empty((fld, K, d.ref.Np), dtype=d.dtype, device=d.device)
        self.rows_out = torch.empty_like(self.rows_in)
        self.bufs = [d.empty_fields(), self.stepper.other]
        # the tcgen05 stage writes the row layout itself in the last stage.  Reading
        # it in the first stage works too (layout 1) but the neighbour gather from
        # rows of Np values costs more than the conversion kernel
        # (scripts/rows_stage_time.py), so the input is converted on the copy stream
        self.direct = bool(direct) and getattr(d, "fused_kind", -1) == 2
        self.trace = None                     # debug: list -> per-launch timing events
        self.lookahead = 8                    # chunks of copy-in queued beyond the next stage-1 needs
        self.h2d, self.d2h = torch.cuda.Stream(d.device), torch.cuda.Stream(d.device)
        self.pack = torch.cuda.Stream(d.device)
        self.ev_copied = [torch.cuda.Event() for _ in range(nc)]
        self.ev_in = [torch.cuda.Event() for _ in range(nc)]
        self.ev_out = [torch.cuda.Event() for _ in range(nc)]

    @staticmethod
    def accepts(disc, state):
        """Pinned host torch tensors of the device dtype, (K, Np) each, on a
        single-rank fused discretization."""
        d = disc.dev
        if d.fused is None or d.halo is not None or getattr(disc, "exchange", None) is not None:
            return False
        return all(isinstance(a, torch.Tensor) and not a.is_cuda and a.is_pinned() and a.dtype == d.dtype
                   and a.is_contiguous() and tuple(a.shape) == (d.K, d.ref.Np) for a in state.fields())

    @_on_disc_device
    def step(self, state, dt):
        import ctypes
        disc, d = self.disc, self.disc.dev
        fl = disc.flux
        s = ctypes.byref(d.struct)
        cur = torch.cuda.current_stream(d.device)
        sp = lambda st: ctypes.c_void_p(st.cuda_stream)
        host_in = state.fields()
        out = torch.empty((d.fld, d.K, d.ref.Np), dtype=d.dtype, pin_memory=True)
        self.h2d.wait_stream(cur)
        self.d2h.wait_stream(cur)
        direct = self.direct
        self.pack.wait_stream(cur)
        nc = len(self.elems)
        queued = [-1]                        # last chunk whose copy-in is enqueued

        def enqueue_input(upto):             # copy engine first, conversion on its own stream
            while queued[0] < upto:
                c = queued[0] + 1
                k0, k1 = self.elems[c]
                with torch.cuda.stream(self.h2d):
                    for f in range(d.fld):
                        self.rows_in[f, k0:k1].copy_(host_in[f][k0:k1], non_blocking=True)
                    self.ev_copied[c].record(self.h2d)
                with torch.cuda.stream(self.pack):
                    self.pack.wait_event(self.ev_copied[c])
                    _native.call("wadg_rows_to_fields", s, _vp(self.rows_in), k0, k1, _vp(self.bufs[0]),
                                 sp(self.pack))
                    self.ev_in[c].record(self.pack)
                queued[0] = c

        # Host enqueue order follows the device order: a chunk's copy-in goes out
        # just ahead of the first stage that needs it, and its copy-out right behind
        # its last stage, so the first stage launch is queued after a few chunks of
        # copies rather than after all of them
        waited = -1
        res = self.stepper.res
        for st, c in self.schedule:
            if st == 1:
                enqueue_input(min(nc - 1, int(self.hi[c]) + self.lookahead))
                if self.hi[c] > waited:
                    waited = int(self.hi[c])
                    cur.wait_event(self.ev_in[waited])
            b0, b1 = self.blocks[c]
            qi, qo = self.bufs[(st - 1) % 2], self.bufs[st % 2]
            if self.trace is not None:       # debug: per-launch start times
                ev0 = torch.cuda.Event(enable_timing=True)
                ev0.record(cur)
            if direct and st == 5:           # the last stage writes the row layout
                _native.call("wadg_stage_fused_rows", s, _vp(qi), _vp(self.rows_out), _vp(res), fl.tau_p,
                             fl.tau_u, LSRK4A[st - 1], LSRK4B[st - 1], dt, b0, b1, 2, sp(cur))
            else:
                _native.call("wadg_stage_fused", s, _vp(qi), _vp(qo), _vp(res), fl.tau_p, fl.tau_u,
                             LSRK4A[st - 1], LSRK4B[st - 1], dt, b0, b1, sp(cur))
            if self.trace is not None:       # debug: per-launch end times on the compute stream
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(cur)
                self.trace.append((st, c, ev0, ev))
            if st == 5:
                self.ev_out[c].record(cur)
                k0, k1 = self.elems[c]
                with torch.cuda.stream(self.d2h):
                    self.d2h.wait_event(self.ev_out[c])
                    if not direct:
                        _native.call("wadg_fields_to_rows", s, _vp(self.bufs[1]), k0, k1, _vp(self.rows_out),
                                     sp(self.d2h))
                    for f in range(d.fld):
                        out[f, k0:k1].copy_(self.rows_out[f, k0:k1], non_blocking=True)
        enqueue_input(nc - 1)
        cur.wait_stream(self.h2d)
        cur.wait_stream(self.pack)
        cur.wait_stream(self.d2h)
        self.d2h.synchronize()
        return FieldState.from_fields(list(out.unbind(0)), state.t + dt)


def lsrk_step(state, dt, rhs_fn):
    """One five-stage low-storage RK4 step (R/.../solver.py:348-363)."""
    if isinstance(rhs_fn, _BoundRHS):
        disc = rhs_fn.disc
        _check_state(state, disc)
        if HostPipeline.accepts(disc, state):
            if getattr(disc, "_pipeline", None) is None:
                disc._pipeline = HostPipeline(disc)
            return disc._pipeline.step(state, dt)
        Q = disc.to_device(state)
        Q = DeviceStepper(disc).step(Q, dt)
        return disc.from_device(Q, state, state.t + dt)
    return _generic_lsrk_step(state, dt, rhs_fn)


def _as_cuda(a, dtype=None):
    if isinstance(a, torch.Tensor):
        return a.to("cuda", dtype or a.dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype or torch.float64, device="cuda")


def _generic_lsrk_step(state, dt, rhs_fn):
    """Arbitrary rhs_fn: the state and the LSRK register live on the GPU and
    every stage axpy runs in wadg_lsrk_axpy.  rhs_fn sees the state in the
    caller's container type: a numpy FieldState for a host numpy state (as the
    reference's lsrk_step, R/.../solver.py:348-363, passes it), device tensors
    for CUDA tensors."""
    import ctypes
    host = not isinstance(state.p, torch.Tensor)
    ys = [_as_cuda(a).clone() for a in state.fields()]
    res = [torch.zeros_like(a) for a in ys]
    t0 = state.t
    y = FieldState.from_fields(ys, t0)
    for a, b, c in zip(LSRK4A, LSRK4B, LSRK4C):
        y.t = t0 + c * dt
        arg = FieldState.from_fields([x.cpu().numpy() for x in ys], y.t) if host else y
        dfs = rhs_fn(arg).fields()
        for m, dm in enumerate(dfs):
            dm = _as_cuda(dm, ys[m].dtype)
            code = _native.WADG_F64 if ys[m].dtype == torch.float64 else _native.WADG_F32
            _native.call("wadg_lsrk_axpy", code, ys[m].numel(), _vp(dm), _vp(res[m]), _vp(ys[m]),
                         a, b, dt, _stream())
    if host:
        ys = [a.cpu().numpy() for a in ys]
    return FieldState.from_fields(ys, t0 + dt)


def stable_dt(mesh, ref, medium, cfl):
    """dt = cfl min_k h_k / (c_max,k (N+1)^2), h_k = dim |K| / |dK|
    (R/.../solver.py:366-376; dim = 2 reproduces the reference)."""
    if cfl <= 0:
        raise ConfigError("cfl must be positive")
    geo = geometry.compute_geometric_data(mesh, ref)
    area = geometry.element_areas(geo)
    perim = geometry.element_perimeters(geo)
    c2 = medium.values(*geo.xyzq)
    c_max = np.sqrt(c2.max(axis=1))
    hmin = mesh.shape.dim * area / perim
    return float(cfl * np.min(hmin / (c_max * (ref.N + 1) ** 2)))


def _projection_chunks(mesh, N, initial_fn, dev, k0=0, k1=None, chunk=None):
    """Yield (c0, c1, [coefficients (Kc, Np) per field]) of the J-weighted L2
    projection at the mass-exact degree 2N + 2 N_geo (R/.../solver.py:379-389,
    operators.py:64-73).  initial_fn gets torch tensors first (so a torch
    expression runs on the device) and numpy arrays if that fails."""
    k1 = mesh.K if k1 is None else k1
    ref_m = refelem.build_reference_element(
        N, mesh.shape, volume_quad_degree=2 * N + 2 * mesh.N_geo, face_quad_degree=1)
    mops = geometry.map_operators(mesh.shape, mesh.N_geo, ref_m).to(dev)
    Vq = torch.as_tensor(ref_m.Vq, device=dev)
    wq = torch.as_tensor(ref_m.wq, device=dev)
    if chunk is None:       # bound the (chunk, Np, Nq) float64 temporaries to ~1 GB
        chunk = int(max(256, min(1 << 15, 2 ** 30 // (8 * ref_m.Np * ref_m.Nq))))
    for c0 in range(k0, k1, chunk):
        c1 = min(k1, c0 + chunk)
        X = torch.as_tensor(np.asarray(mesh.elem_map_nodes[c0:c1], dtype=np.float64), device=dev)
        g = geometry.geometric_factors(X, mops, check=False)
        try:
            vals = [torch.as_tensor(v, dtype=torch.float64, device=dev).expand_as(g["J"])
                    for v in initial_fn(*g["xq"])]
        except (TypeError, RuntimeError, AttributeError):
            xyz = [a.cpu().numpy() for a in g["xq"]]
            vals = [torch.as_tensor(np.broadcast_to(np.asarray(v, dtype=float), g["J"].shape).copy(),
                                    device=dev) for v in initial_fn(*xyz)]
        W = wq[None, :] * g["J"]
        M = (Vq.T[None, :, :] * W[:, None, :]) @ Vq
        M = 0.5 * (M + M.transpose(1, 2))
        L = torch.linalg.cholesky(M)
        out = []
        for v in vals:
            rhs = (W * v) @ Vq
            out.append(torch.cholesky_solve(rhs[:, :, None], L)[:, :, 0])
        yield c0, c1, out


def project_initial_condition(mesh, config, initial_fn, medium=MediumField()):
    """L2-project the initial fields with a mass-exact quadrature
    (R/.../solver.py:379-389).  Setup step: dense per-element solves in
    element chunks on the GPU; returns host arrays.  Needs CUDA like every
    other compute entry point (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError("project_initial_condition needs a CUDA device (no CPU fallback)")
    dev = "cuda"
    nf = mesh.shape.dim + 1
    out = [np.empty((mesh.K, refelem.basis_dimension(mesh.shape, config.N))) for _ in range(nf)]
    for c0, c1, cs in _projection_chunks(mesh, config.N, initial_fn, dev):
        for i, c in enumerate(cs):
            out[i][c0:c1] = c.cpu().numpy()
    return FieldState.from_fields(out, 0.0)


def project_initial_condition_device(disc, initial_fn):
    """Projection straight into the device field layout (dim+1, Np, Kpad) of
    ``disc`` (its element range), for meshes too large for host arrays."""
    d = disc.dev
    Q = d.empty_fields()
    for c0, c1, cs in _projection_chunks(disc.mesh, disc.config.N, initial_fn, d.device,
                                         d.k0, d.k1):
        for i, c in enumerate(cs):
            Q[i, :, c0 - d.k0:c1 - d.k0] = c.T.to(d.dtype)
    return Q


def global_l2_error(ref, geo, coeffs, exact_fn):
    """sqrt(sum w J (u_h - u)^2) (R/.../operators.py:103-107), host arrays."""
    uq = np.atleast_2d(coeffs) @ ref.Vq.T
    fq = exact_fn(*geo.xyzq)
    return float(np.sqrt(np.sum(ref.wq[None, :] * geo.Jq * (uq - fq) ** 2)))


def _field_values(fn, xq, shape, dev):
    """fn(*xq) as a float64 device tensor: torch expressions run on the device,
    a numpy-only callable is evaluated on a host copy of the points."""
    try:
        v = fn(*xq)
        if not isinstance(v, torch.Tensor):
            raise TypeError("numpy result")
        return v.to(device=dev, dtype=torch.float64).expand(shape)
    except (TypeError, RuntimeError, AttributeError):
        xyz = [a.cpu().numpy() for a in xq]
        return torch.as_tensor(np.array(np.broadcast_to(np.asarray(fn(*xyz), dtype=float), shape)), device=dev)


@_on_disc_device
def device_l2_error(disc, Q, exact_fn, ref_err=None, chunk=1 << 15):
    """global_l2_error of the pressure field resident on the device (field
    layout Q[0], (Np, Kpad)): the error quadrature's geometry is rebuilt on
    the device in element chunks and the sum reduced there; only the scalar
    comes back to the host."""
    d = disc.dev
    mesh, N = disc.mesh, disc.config.N
    if ref_err is None:
        ref_err = refelem.build_reference_element(N, mesh.shape, volume_quad_degree=2 * N + 4,
                                                  face_quad_degree=1)
    mops = geometry.map_operators(mesh.shape, mesh.N_geo, ref_err).to(d.device)
    Vq = torch.as_tensor(ref_err.Vq, dtype=torch.float64, device=d.device)
    wq = torch.as_tensor(ref_err.wq, dtype=torch.float64, device=d.device)
    total = torch.zeros((), dtype=torch.float64, device=d.device)
    for c0 in range(0, d.K, chunk):
        c1 = min(d.K, c0 + chunk)
        X = torch.as_tensor(np.asarray(mesh.elem_map_nodes[d.k0 + c0:d.k0 + c1], dtype=np.float64),
                            device=d.device)
        g = geometry.geometric_factors(X, mops, check=False)
        uq = Q[0, :, c0:c1].to(torch.float64).T @ Vq.T
        f = _field_values(exact_fn, g["xq"], g["J"].shape, d.device)
        total += torch.sum(wq[None, :] * g["J"] * (uq - f) ** 2)
    return float(torch.sqrt(total))


def run(mesh, config, initial_fn, T, medium=MediumField(), exact_p=None, n_outputs=10, dt=None):
    """Advance the projected initial condition to time T on the GPU
    (R/.../solver.py:392-439): the state stays resident; energy (device
    reduction) and the optional pressure L2 error are recorded at
    n_outputs+1 sample times; the last step of each interval lands exactly
    on the sample time; BlowUp when the energy exceeds 1e6 x initial."""
    disc = Discretization(mesh, config, medium)
    state = project_initial_condition(mesh, config, initial_fn, medium)
    if dt is None:
        dt = stable_dt(mesh, disc.ref, medium, config.cfl)
    Q = disc.to_device(state)
    stepper = DeviceStepper(disc)
    sample_ts = np.linspace(0.0, T, n_outputs + 1)
    diag = {"t": [], "energy": [], "l2_error_p": []}
    ref_err = None
    if exact_p is not None:
        ref_err = refelem.build_reference_element(
            config.N, mesh.shape, volume_quad_degree=2 * config.N + 4, face_quad_degree=1)
    t = 0.0

    def record(t):
        # energy and pressure error are device reductions; only scalars reach the host
        e = device_energy(disc, Q)
        diag["t"].append(t)
        diag["energy"].append(e)
        if exact_p is not None:
            diag["l2_error_p"].append(device_l2_error(disc, Q, lambda *xyz: exact_p(*xyz, t), ref_err))
        return e

    e0 = record(t)
    for target in sample_ts[1:]:
        while t < target - 1e-12:
            step = min(dt, target - t)
            # full steps replay a captured CUDA graph; the shortened last step of an
            # interval runs eagerly
            Q = stepper.step_graphed(Q, step) if step == dt else stepper.step(Q, step)
            t = t + step
        t = float(target)
        e = record(t)
        if not np.isfinite(e) or (e0 > 0 and e > 1e6 * e0):
            raise BlowUp(f"energy {e:.3e} at t = {t:.4f} (initial {e0:.3e})")
    state = disc.from_device(Q, state, t)
    diag = {k: np.asarray(v) for k, v in diag.items()}
    return state, diag


# ---------------------------------------------------------------------------
# Exact disk solution (R/pkg/src/wadg/solver.py:445-466): the standing pressure
# mode of the unit disk with the Dirichlet mirror BC.  Host diagnostics for
# run(..., exact_p=bessel_pressure); J0 / J1 from scipy.special (the reference
# restates them as series / Hankel expansions, R/pkg/src/wadg/bessel.py).

DISK_LAMBDA = 5.52007811028631     # second zero of J0 (R/pkg/src/wadg/bessel.py:18)


def bessel_pressure(x, y, t, lam=DISK_LAMBDA):
    """p = J0(lam r) cos(lam t)."""
    from scipy.special import j0
    return j0(lam * np.hypot(x, y)) * np.cos(lam * t)


def bessel_velocity(x, y, t, lam=DISK_LAMBDA):
    """u = J1(lam r) sin(lam t) r_hat."""
    from scipy.special import j1
    r = np.hypot(x, y)
    mag = j1(lam * r) * np.sin(lam * t)
    with np.errstate(invalid="ignore", divide="ignore"):
        cx = np.where(r > 0, x / np.where(r > 0, r, 1.0), 0.0)
        cy = np.where(r > 0, y / np.where(r > 0, r, 1.0), 0.0)
    return mag * cx, mag * cy


def bessel_initial_condition(x, y):
    p = bessel_pressure(x, y, 0.0)
    return p, np.zeros_like(p), np.zeros_like(p)
