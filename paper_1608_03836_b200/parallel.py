"""Element-slab domain decomposition with a face-trace halo exchanged every
RK stage (north_star item 4).  The reference is single
process (R/SPEC.md:559); this module has no reference counterpart.

* Elements of the warped-cube meshes are z-major, so a z-slab is one
  contiguous element range per rank.
* Each rank packs the nodal face traces of its faces on a slab interface
  (``wadg_pack_halo``; (dim+1) x Nfp values per face, in the sender's face-node
  order) and exchanges them with its neighbours using NCCL point-to-point
  (``torch.distributed.batch_isend_irecv``) on NCCL's stream, while the volume
  kernel and the surface kernel of interface-free element blocks run.  The
  surface kernel reads a halo slot through the receiver's orientation
  permutation, exactly as it reads a local neighbour.
* Results are independent of the number of ranks (same per-element
  arithmetic, halo values are exact copies).
"""

from __future__ import annotations

import ctypes

import numpy as np

from .device import HaloPlan


def slab_ranges(K, world, n_layers):
    """Contiguous element ranges of ``world`` z-slabs over ``n_layers``
    equal element layers."""
    if K % n_layers:
        raise ValueError("K is not a whole number of layers")
    per = K // n_layers
    bounds = [(r * n_layers) // world for r in range(world + 1)]
    return [(bounds[r] * per, bounds[r + 1] * per) for r in range(world)]


def halo_plans(mesh, ranges):
    """One HaloPlan per rank; local element indices relative to each range.

    Interface face pairs between ranks r < s are put in a canonical order
    (sorted by the (element, face) of the lower rank's side) that both sides
    derive independently; rank r's message to s is its side of those pairs
    in that order and its receive slots from s follow the same order."""
    owner = np.empty(mesh.K, dtype=np.int64)
    for r, (a, b) in enumerate(ranges):
        owner[a:b] = r
    conn = mesh.face_connectivity
    kk, ff = np.nonzero(conn[:, :, 0] >= 0)
    k2, f2 = conn[kk, ff, 0], conn[kk, ff, 1]
    cross = owner[kk] != owner[k2]
    kk, ff, k2, f2 = kk[cross], ff[cross], k2[cross], f2[cross]
    plans = []
    for r, (a, b) in enumerate(ranges):
        recv_slot, send_k, send_f, peers = {}, [], [], []
        mine = owner[kk] == r
        for s in sorted(set(owner[k2[mine]].tolist())):
            sel = mine & (owner[k2] == s)
            mk, mf, ok, of = kk[sel], ff[sel], k2[sel], f2[sel]
            if r < s:
                order = np.lexsort((mf, mk))
            else:
                order = np.lexsort((of, ok))
            mk, mf = mk[order], mf[order]
            base = len(recv_slot)
            for i, (k, f) in enumerate(zip(mk.tolist(), mf.tolist())):
                recv_slot[(k - a, f)] = base + i
            send_k.extend((mk - a).tolist())
            send_f.extend(mf.tolist())
            peers.append((s, len(mk), len(mk)))
        plans.append(HaloPlan(recv_slot, send_k, send_f, peers))
    return plans


def halo_blocks(disc_dev, block):
    """Element blocks whose surface work reads halo slots."""
    nbr = disc_dev.nbr[:, :disc_dev.K].cpu().numpy()
    dep = np.any(nbr <= -2, axis=0)
    nb = disc_dev.n_blocks
    blk = np.zeros(nb, dtype=bool)
    idx = np.nonzero(dep)[0] // block
    blk[idx] = True
    return blk


def _runs(mask, value):
    runs, start = [], None
    for i, v in enumerate(list(mask) + [not value]):
        if v == value and start is None:
            start = i
        elif v != value and start is not None:
            runs.append((start, i))
            start = None
    return runs


class HaloExchange:
    """Per-stage halo exchange for one rank; ``start`` packs and posts the
    NCCL send/recv, ``surface`` / ``fused_stage`` run the halo-free element
    blocks on the current stream and the blocks that read halo slots on a
    high-priority side stream that waits for the transfer, so those blocks
    start as soon as their traces arrive and SMs free up, instead of after
    the whole interior wave.  The current stream waits for the side stream
    before the next kernel.

    ``dist`` is torch.distributed, or any object with the same P2POp /
    isend / irecv / batch_isend_irecv interface (tests use a loopback one)."""

    def __init__(self, disc, plan, group=None, dist=None):
        import torch
        if dist is None:
            import torch.distributed as dist
        from . import _native
        self.dist, self.native = dist, _native
        self.disc, self.plan, self.group = disc, plan, group
        d = disc.dev
        blk = halo_blocks(d, _native.ELEMS_PER_BLOCK)
        self.free_runs = _runs(blk, False)
        self.halo_runs = _runs(blk, True)
        if d.fused is not None:
            fblk = halo_blocks(d, d.fused)
            self.free_runs_f = _runs(fblk, False)
            self.halo_runs_f = _runs(fblk, True)
        with torch.cuda.device(d.device):
            lo, hi = torch.cuda.Stream.priority_range()
            self.side = torch.cuda.Stream(device=d.device, priority=min(lo, hi))
        self.reqs = []

    def start(self, Q):
        import torch
        d, plan = self.disc.dev, self.plan
        sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        if len(plan.send_k):
            self.native.call("wadg_pack_halo", ctypes.byref(d.struct), ctypes.c_void_p(Q.data_ptr()),
                             ctypes.c_void_p(d.send_k.data_ptr()), ctypes.c_void_p(d.send_f.data_ptr()),
                             len(plan.send_k), ctypes.c_void_p(d.send_buf.data_ptr()), sp)
        ops, so, ro = [], 0, 0
        for peer, ns, nr in plan.peers:
            ops.append(self.dist.P2POp(self.dist.isend, d.send_buf[so:so + ns], peer, self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, d.halo_buf[ro:ro + nr], peer, self.group))
            so += ns
            ro += nr
        self.reqs = self.dist.batch_isend_irecv(ops) if ops else []

    def _split_launch(self, free, halo, launch):
        """launch(b0, b1, stream_ptr) over the free runs on the current stream,
        then over the halo runs on the side stream after the transfer."""
        import torch
        main = torch.cuda.current_stream()
        ready = torch.cuda.Event()
        ready.record(main)                       # previous stage and this stage's pack are ordered
        for b0, b1 in free:
            launch(b0, b1, ctypes.c_void_p(main.cuda_stream))
        with torch.cuda.stream(self.side):
            self.side.wait_event(ready)
            for r in self.reqs:                  # NCCL: the side stream waits for the transfer
                r.wait()
            for b0, b1 in halo:
                launch(b0, b1, ctypes.c_void_p(self.side.cuda_stream))
            done = torch.cuda.Event()
            done.record(self.side)
        main.wait_event(done)
        self.reqs = []

    def surface(self, Q, rhs, tau_p, tau_u, sp):
        d = self.disc.dev
        vp = lambda t: ctypes.c_void_p(t.data_ptr())
        self._split_launch(self.free_runs, self.halo_runs, lambda b0, b1, st: self.native.call(
            "wadg_surface", ctypes.byref(d.struct), vp(Q), vp(rhs), tau_p, tau_u, 1, b0, b1, st))

    def fused_stage(self, Qin, Qout, res, tau_p, tau_u, a, b, dt, sp):
        """Fused stage: interface-free element blocks while the halo is in
        flight, the blocks that read halo slots on the side stream."""
        d = self.disc.dev
        vp = lambda t: ctypes.c_void_p(t.data_ptr())
        args = (ctypes.byref(d.struct), vp(Qin), vp(Qout), vp(res), tau_p, tau_u, a, b, dt)
        self._split_launch(self.free_runs_f, self.halo_runs_f,
                           lambda b0, b1, st: self.native.call("wadg_stage_fused", *args, b0, b1, st))


def ghosted_slab_mesh(n, N_geo, rank, world, nz=None, z_range=None, amp=0.1, domain=(-1.0, 1.0)):
    """Rank's z-slab of the warped cube (meshgen.warped_cube_tet_mesh) with one
    ghost layer of cubes towards each neighbour rank, generated directly: no
    global mesh.  Node coordinates are bitwise those of the global mesh (the
    global layer planes are passed through), and element numbering is the
    global one shifted by a constant, so canonical halo orders agree.
    Returns (mesh, owned element range in it, [(local range, global rank)] of
    all parts)."""
    from . import meshgen
    nz = n if nz is None else nz
    zlo, zhi = domain if z_range is None else z_range
    gz = np.linspace(zlo, zhi, nz + 1)
    bounds = [(r * nz) // world for r in range(world + 1)]
    l0, l1 = bounds[rank], bounds[rank + 1]
    g0, g1 = max(0, l0 - 1), min(nz, l1 + 1)
    mesh = meshgen.warped_cube_tet_mesh(n, N_geo, amp=amp, domain=domain, z_grid=gz[g0:g1 + 1])
    per = mesh.K // (g1 - g0)
    parts = []
    if l0 > g0:
        parts.append(((0, (l0 - g0) * per), rank - 1))
    owned = ((l0 - g0) * per, (l1 - g0) * per)
    parts.append((owned, rank))
    if g1 > l1:
        parts.append((((l1 - g0) * per, (g1 - g0) * per), rank + 1))
    return mesh, owned, parts


def local_halo_plan(mesh, parts, rank):
    """The rank's HaloPlan from its ghosted slab mesh (same message orders and
    slots as halo_plans on the global mesh; peers are global ranks)."""
    ranges = [r for r, _ in parts]
    ranks = [g for _, g in parts]
    me = ranks.index(rank)
    plan = halo_plans(mesh, ranges)[me]
    plan.peers = [(ranks[s], ns, nr) for s, ns, nr in plan.peers]
    return plan


def local_slab_discretization(n, N_geo, config, medium, rank, world, nz=None, z_range=None, amp=0.1,
                              group=None, dist=None):
    """slab_discretization without the global mesh: the rank builds only its
    ghosted slab (ghosted_slab_mesh) and its own halo plan."""
    from .solver import Discretization
    mesh, owned, parts = ghosted_slab_mesh(n, N_geo, rank, world, nz, z_range, amp)
    plan = local_halo_plan(mesh, parts, rank)
    disc = Discretization(mesh, config, medium, k_range=owned, halo=plan)
    disc.dev
    disc.exchange = HaloExchange(disc, plan, group, dist)
    return disc


def slab_discretization(mesh, config, medium, rank, world, n_layers, group=None, dist=None):
    """Discretization of rank's z-slab with its halo exchange attached as
    ``disc.exchange``."""
    from .solver import Discretization
    ranges = slab_ranges(mesh.K, world, n_layers)
    plans = halo_plans(mesh, ranges)
    disc = Discretization(mesh, config, medium, k_range=ranges[rank], halo=plans[rank])
    disc.dev
    disc.exchange = HaloExchange(disc, plans[rank], group, dist)
    return disc
