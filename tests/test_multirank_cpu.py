"""N > 1 host logic on CPU (world_size 2..4, gloo, 127.0.0.1).

The library's exchange plan (lb_exchange_plan: ring neighbours, the four
contiguous 3-column messages in the internal layout, their posting order) is
exercised with real point-to-point messages between processes; each rank steps
its X-slab with the oracle, its halo columns filled ONLY by those messages.
After several steps the concatenated slabs must equal the 1-slab oracle run
bit for bit (SPEC S:240 ring consistency; SURVEY §8e "N == 1 bit-exact")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lbgen
import oracle
import paper_1703_00186_b200 as lb

Q = 37


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def canon_to_internal(buf, L):
    """Full canonical slab buffer [37][NX][NY] -> internal layout (include/lb.h)."""
    out = np.zeros(L.elems)
    v = out.reshape(L.nx, Q, L.nyp)
    v[:, :, L.y0 - 3:L.y0 + L.ly + 3] = buf.transpose(1, 0, 2)
    return out


def internal_halos_to_canon(arr, L, buf):
    """Copy the 3+3 halo columns of an internal-layout array into a canonical buffer."""
    v = arr.reshape(L.nx, Q, L.nyp)[:, :, L.y0 - 3:L.y0 + L.ly + 3].transpose(1, 0, 2)
    buf[:, 0:3, :] = v[:, 0:3, :]
    buf[:, L.lx + 3:L.lx + 6, :] = v[:, L.lx + 3:L.lx + 6, :]


def _worker(rank, world, port, lx_total, ly, bc, nsteps, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bcn = {"thermal": oracle.WALL_THERMAL, "adiabatic": oracle.WALL_ADIABATIC}[bc]
        p = lb.make_params(lx_total, ly, bc_y=bc)
        L = lb.query_layout(p, rank, world)
        X = lb.exchange_plan(p, rank, world)
        lx = L.lx
        assert L.x0_global == rank * lx
        o = oracle.Lattice(lx, ly, bc_y=bcn)
        o.init_macro(*lbgen.rt_macro(lx_total, ly, oracle.t0(), x0=rank * lx, lx=lx))
        for _ in range(nsteps):
            A = o.buffer(0)
            arr = torch.from_numpy(canon_to_internal(A, L))
            n = int(X.count)
            recv_l = torch.empty(n, dtype=torch.float64)
            recv_r = torch.empty(n, dtype=torch.float64)
            # the plan's posting order: recv left, recv right, send right, send left
            reqs = [dist.irecv(recv_l, src=X.left), dist.irecv(recv_r, src=X.right),
                    dist.isend(arr[X.send_right_off:X.send_right_off + n].clone(), dst=X.right),
                    dist.isend(arr[X.send_left_off:X.send_left_off + n].clone(), dst=X.left)]
            for r in reqs:
                r.wait()
            arr[X.recv_left_off:X.recv_left_off + n] = recv_l
            arr[X.recv_right_off:X.recv_right_off + n] = recv_r
            internal_halos_to_canon(arr.numpy(), L, A)
            o.propagate()
            o.bc()
            o.collide()
            o.swap()
        st = torch.from_numpy(np.ascontiguousarray(o.get_state(0)))
        parts = [torch.empty_like(st) for _ in range(world)] if rank == 0 else None
        dist.gather(st, parts, dst=0)
        if rank == 0:
            np.save(out_path, np.concatenate([t.numpy() for t in parts], axis=1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,lx_total,ly,bc", [(2, 24, 16, "thermal"), (3, 36, 12, "adiabatic"),
                                                  (4, 48, 10, "thermal")])
def test_ring_exchange_plan_n_equals_1(world, lx_total, ly, bc, tmp_path):
    nsteps = 4
    out = str(tmp_path / "state.npy")
    mp.start_processes(_worker, args=(world, free_port(), lx_total, ly, bc, nsteps, out), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    ref = oracle.Lattice(lx_total, ly, bc_y={"thermal": oracle.WALL_THERMAL,
                                               "adiabatic": oracle.WALL_ADIABATIC}[bc])
    ref.init_macro(*lbgen.rt_macro(lx_total, ly, oracle.t0()))
    ref.step(nsteps)
    assert np.array_equal(got, ref.get_state(0))


@pytest.mark.parametrize("lx_total,world", [(64, 1), (64, 2), (48, 8), (6, 1), (12, 2)])
def test_bulk_border_columns(lx_total, world):
    """Bulk + border = all physical columns, disjoint; the bulk never reads a halo column."""
    p = lb.make_params(lx_total, 32)
    for rank in range(world):
        X = lb.exchange_plan(p, rank, world)
        L = lb.query_layout(p, rank, world)
        cols = list(range(X.bulk_x0, X.bulk_x1)) + list(range(X.border_x0, X.border_x1)) + \
            list(range(X.border_x2, X.border_x3))
        assert sorted(cols) == list(range(3, 3 + L.lx))
        if X.bulk_x1 > X.bulk_x0:
            assert X.bulk_x0 - 3 >= 3 and X.bulk_x1 - 1 + 3 <= L.lx + 2
        assert X.left == (rank - 1) % world and X.right == (rank + 1) % world
        assert X.count == 3 * 37 * L.nyp
        assert X.recv_left_off == 0 and X.send_left_off == 3 * 37 * L.nyp
        assert X.send_right_off == L.lx * 37 * L.nyp and X.recv_right_off == (L.lx + 3) * 37 * L.nyp
