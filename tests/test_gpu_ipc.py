"""Peer-store exchange across PROCESSES through CUDA IPC (the N > 1 production
mapping), run as 2 ranks sharing cuda:0 (this pool gives one GPU per job):
each rank maps its neighbour's buffers and step counter via
torch.multiprocessing's tensor reduction and steps its X-slab with
lb_set_peers; the gathered slabs must equal the single-lattice run bit for bit."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, lx, ly, nsteps, out):
    import torch.distributed as dist

    import lbgen
    import paper_1703_00186_b200 as lb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        lx_total = lx * world
        g = lb.Lattice(lx_total, ly, rank=rank, nranks=world)
        g.init_macro(*lbgen.rt_macro(lx_total, ly, lb.t0(), x0=rank * lx, lx=lx))
        g.set_peers_ipc()
        g.step(nsteps)
        g.sync()
        dist.barrier()
        np.save(out + f".{rank}.npy", g.peek(0))
        dist.barrier()
        g.close()
    finally:
        dist.destroy_process_group()


def test_ipc_peer_exchange_two_processes(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import lbgen
    import paper_1703_00186_b200 as lb
    world, lx, ly, nsteps = 2, 16, 48, 6
    out = str(tmp_path / "slab")
    mp.start_processes(_rank, args=(world, _free_port(), lx, ly, nsteps, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.concatenate([np.load(out + f".{r}.npy") for r in range(world)], axis=1)
    ref = lb.Lattice(lx * world, ly)
    ref.init_macro(*lbgen.rt_macro(lx * world, ly, lb.t0()))
    ref.step(nsteps)
    assert np.array_equal(got, ref.gather())
