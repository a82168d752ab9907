"""Element-slab decomposition and the per-stage face-trace halo, exercised on
CPU with the gloo backend at world_size 2 (the GPU path uses the same plans
with NCCL; only one GPU is available to this build)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1608_03836_b200 import device, meshgen, parallel, refelem


def test_slab_ranges_are_contiguous_layers():
    r = parallel.slab_ranges(4 * 4 * 6 * 5, 3, 5)
    assert r[0][0] == 0 and r[-1][1] == 4 * 4 * 6 * 5
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    assert all((hi - lo) % 96 == 0 for lo, hi in r)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_halo_plans_are_symmetric(world):
    mesh = meshgen.warped_cube_tet_mesh(3, 1, nz=4, z_range=(-1.0, 1.0 + 2.0 / 3.0))
    ranges = parallel.slab_ranges(mesh.K, world, 4)
    plans = parallel.halo_plans(mesh, ranges)
    for r, pl in enumerate(plans):
        for s, ns, nr in pl.peers:
            back = [p for p in plans[s].peers if p[0] == r][0]
            assert back[1] == nr and back[2] == ns
        assert pl.n_recv == len(pl.send_k)
    # z-slabs: only neighbouring ranks exchange, n*n*2 faces per interface
    assert all(abs(s - r) == 1 for r, pl in enumerate(plans) for s, _, _ in pl.peers)
    assert plans[0].peers[0][1] == 3 * 3 * 2


def test_neighbour_tables_use_halo_slots():
    mesh = meshgen.warped_cube_tet_mesh(2, 1)
    ranges = parallel.slab_ranges(mesh.K, 2, 2)
    plans = parallel.halo_plans(mesh, ranges)
    nbr, code = device.neighbour_tables(mesh, 6, *ranges[1], plans[1])
    slots = -nbr[nbr <= -2] - 2
    assert sorted(slots.tolist()) == list(range(plans[1].n_recv))
    with pytest.raises(ValueError):
        device.neighbour_tables(mesh, 6, *ranges[1], None)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 2
        mesh = meshgen.warped_cube_tet_mesh(2, N, nz=4, z_range=(-1.0, 3.0))
        ref = refelem.build_reference_element(N, refelem.ElementShape.Tetrahedron)
        fm = np.array(ref.face_nodes)
        ranges = parallel.slab_ranges(mesh.K, world, 4)
        plans = parallel.halo_plans(mesh, ranges)
        k0, k1 = ranges[rank]
        plan = plans[rank]
        # "fields" = physical node coordinates + a field id, so a received
        # value identifies the exact physical point it belongs to
        X = mesh.elem_map_nodes[k0:k1]                         # (K, Np, 3)
        Q = np.concatenate([X.transpose(2, 1, 0), np.ones((1, ref.Np, k1 - k0))], 0)
        # pack exactly as wadg_pack_halo: buf[s][fld][i] = Q[fld][fmask[f][i]][k]
        send = np.stack([Q[:, fm[f], k] for k, f in zip(plan.send_k, plan.send_f)])
        send = torch.as_tensor(send) if len(send) else torch.zeros((0, 4, ref.nfp), dtype=torch.float64)
        recv = torch.zeros((plan.n_recv, 4, ref.nfp), dtype=torch.float64)
        ops, so, ro = [], 0, 0
        for peer, ns, nr in plan.peers:
            ops.append(dist.P2POp(dist.isend, send[so:so + ns].contiguous(), peer))
            ops.append(dist.P2POp(dist.irecv, recv[ro:ro + nr], peer))
            so += ns
            ro += nr
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        # read halo slots as the surface kernel does: value at my face node i
        # = halo[slot][fld][perm[o][i]], which must be my own physical point
        nbr, code = device.neighbour_tables(mesh, 6, k0, k1, plan)
        err = 0.0
        for f in range(4):
            for k in np.nonzero(nbr[f] <= -2)[0]:
                slot = -nbr[f, k] - 2
                o = code[f, k] % 6
                got = recv[slot].numpy()[:3, ref.face_perms[o]]
                mine = X[k, fm[f]].T
                err = max(err, float(np.abs(got - mine).max()))
        out[rank] = (err, plan.n_recv)
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_halo_exchange():
    world = 2
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        err, n = out[r]
        assert n == 2 * 2 * 2
        assert err < 1e-14


@pytest.mark.parametrize("world", [2, 3, 4])
def test_ghosted_slab_mesh_matches_global_partition(world):
    """Per-rank slab generation (no global mesh): the owned elements' nodes,
    the halo plan (message orders, receive slots, peers) and the device
    neighbour tables equal those derived from the global mesh."""
    n, N, nz = 3, 2, 8
    mesh = meshgen.warped_cube_tet_mesh(n, N, nz=nz, z_range=(-1.0, 1.5))
    ranges = parallel.slab_ranges(mesh.K, world, nz)
    plans = parallel.halo_plans(mesh, ranges)
    for r in range(world):
        lm, owned, parts = parallel.ghosted_slab_mesh(n, N, r, world, nz=nz, z_range=(-1.0, 1.5))
        lp = parallel.local_halo_plan(lm, parts, r)
        a, b = ranges[r]
        assert owned[1] - owned[0] == b - a
        assert np.array_equal(lm.elem_map_nodes[owned[0]:owned[1]], mesh.elem_map_nodes[a:b])
        gp = plans[r]
        assert lp.peers == gp.peers
        assert np.array_equal(lp.send_k, gp.send_k) and np.array_equal(lp.send_f, gp.send_f)
        assert lp.recv_slot == gp.recv_slot
        ln, lc = device.neighbour_tables(lm, 6, owned[0], owned[1], lp)
        gn, gc = device.neighbour_tables(mesh, 6, a, b, gp)
        assert np.array_equal(ln, gn) and np.array_equal(lc, gc)
