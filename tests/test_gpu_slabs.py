"""The production multi-rank path on one device: real ``parallel.slab_discretization``
and ``parallel.HaloExchange`` objects for 3 z-slabs, with their NCCL calls
answered by a loopback stand-in of torch.distributed that copies each send
buffer into the matching receive buffer on the device.  Every stage packs
(wadg_pack_halo), posts, runs the halo-free blocks on the current stream and
the halo blocks on the exchange's high-priority side stream, exactly as on 8
GPUs; only the transport differs.  Required: bitwise equality with the single
domain, fused and three-kernel stages, fp32 (tcgen05) and fp64.
(there is no reference multi-GPU code, R/SPEC.md:559.)"""

import numpy as np
import pytest
import torch

from paper_1608_03836_b200 import meshgen, parallel, solver
from paper_1608_03836_b200.solver import FieldState, Formulation, SolverConfig

pytestmark = pytest.mark.gpu


class LoopbackNet:
    """Mailboxes shared by the ranks of one process."""

    def __init__(self):
        self.sent = {}


class LoopbackDist:
    """torch.distributed P2P interface of one rank: isend stores the buffer
    in the mailbox (src, dst); the irecv request's wait() copies it on the
    current stream (as NCCL's wait orders the current stream after the
    transfer)."""

    class P2POp:
        def __init__(self, op, tensor, peer, group=None):
            self.op, self.tensor, self.peer = op, tensor, peer

    class _Req:
        def __init__(self, fn=None):
            self.fn = fn

        def wait(self):
            if self.fn is not None:
                self.fn()

    def __init__(self, net, rank):
        self.net, self.rank = net, rank
        self.isend, self.irecv = "isend", "irecv"
        self.posted = 0

    def batch_isend_irecv(self, ops):
        reqs = []
        for o in ops:
            if o.op == "isend":
                self.net.sent[(self.rank, o.peer)] = o.tensor
                reqs.append(self._Req())
            else:
                src, dst, buf = o.peer, self.rank, o.tensor
                reqs.append(self._Req(lambda src=src, dst=dst, buf=buf: buf.copy_(self.net.sent[(src, dst)])))
        self.posted += 1
        return reqs


@pytest.mark.parametrize("local", [False, True])
@pytest.mark.parametrize("dtype,N", [("float32", 3), ("float64", 3), ("float32", 5), ("float32", 1), ("float64", 1)])
@pytest.mark.parametrize("fused", [True, False])
def test_slab_exchange_loopback_is_bitwise_single_domain(dtype, N, fused, local, rng):
    """N = 3: the tcgen05 (fp32) and DMMA (fp64) stages; N = 5 fp32: the
    split-TF32 mma.sync stage of config 5 (the weak-scaling configuration);
    N = 1: the one-element-per-thread register stage (halo slots read directly)."""
    world, nz = 3, 6
    mesh = meshgen.warped_cube_tet_mesh(4, N, nz=nz, z_range=(-1.0, 2.0))
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, dtype=dtype)
    c2 = lambda x, y, z: 1.0 + 0.5 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    medium = solver.MediumField(c2)
    whole = solver.Discretization(mesh, cfg, medium)
    net = LoopbackNet()
    dists = [LoopbackDist(net, r) for r in range(world)]
    if local:       # each rank builds only its ghosted slab (no global mesh)
        slabs = [parallel.local_slab_discretization(4, N, cfg, medium, r, world, nz=nz, z_range=(-1.0, 2.0),
                                                    dist=dists[r]) for r in range(world)]
    else:
        slabs = [parallel.slab_discretization(mesh, cfg, medium, r, world, nz, dist=dists[r]) for r in range(world)]
    ranges = parallel.slab_ranges(mesh.K, world, nz)
    assert all(len(s.exchange.halo_runs_f if fused else s.exchange.halo_runs) > 0 for s in slabs)
    if dtype == "float32" or N == 1:
        kind = 5 if N == 1 else (2 if N <= 4 else 4)
        assert whole.dev.fused_kind == kind and all(s.dev.fused_kind == kind for s in slabs)
    fl = [rng.standard_normal((mesh.K, whole.ref.Np)) for _ in range(4)]
    Qw = whole.to_device(FieldState.from_fields(fl))
    Qs = [s.to_device(FieldState.from_fields([a[lo:hi] for a in fl])) for s, (lo, hi) in zip(slabs, ranges)]
    sw = solver.DeviceStepper(whole, fused=fused)
    ss = [solver.DeviceStepper(s, fused=fused) for s in slabs]
    dt = 2e-3
    for _ in range(3):
        for a, b in zip(solver.LSRK4A, solver.LSRK4B):
            Qw = sw.stage(Qw, a, b, dt)
            for s, Q in zip(slabs, Qs):          # every rank posts its halo first ...
                s.exchange.start(Q)
            Qs = [st.stage(Q, a, b, dt, started=True) for st, Q in zip(ss, Qs)]   # ... then runs
    torch.cuda.synchronize()
    assert all(d.posted == 15 for d in dists)
    whole_out = Qw[:, :, :mesh.K]
    split_out = torch.cat([Q[:, :, :hi - lo] for Q, (lo, hi) in zip(Qs, ranges)], dim=2)
    assert torch.equal(whole_out, split_out)
    assert float(torch.linalg.vector_norm(whole_out.double())) > 0
