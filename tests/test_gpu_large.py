"""Full BASELINE sizes beyond config #2, in the launch configuration bench.py
times, checked on SAMPLED columns: for a column x the step result depends only
on columns x-3..x+3 of the previous state, so the oracle steps that 7-column
window (any halo) and its centre column must match the GPU's column x.
Also the peer-exchange watchdog."""
import numpy as np
import pytest

import lbgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1703_00186_b200 as m
    return m


def window(g, x, lx):
    cols = [(x + d) % lx for d in range(-3, 4)]
    return np.concatenate([g.peek_cols(c, 1) for c in cols], axis=1)


@pytest.mark.parametrize("lx,ly,coll", [(8192, 8192, "bgk"), (4096, 8192, "regularized")])
def test_sampled_columns_full_size(lb, lx, ly, coll):
    """BASELINE configs #3 (8192x8192, N=1) and #4 (4096x8192 per GPU)."""
    g = lb.Lattice(lx, ly, collision=coll)
    g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
    g.step(2)
    samples = [0, 1, 2, 3, lx // 2 + 1, lx - 4, lx - 3, lx - 2, lx - 1]
    wins = {x: window(g, x, lx) for x in samples}
    g.step(1)
    for x in samples:
        got = g.peek_cols(x, 1)[:, 0, :]
        o = oracle.Lattice(7, ly, collision=oracle.REGULARIZED if coll == "regularized" else oracle.BGK)
        o.set_state(wins[x])
        o.step(1)
        ref = o.get_state(0)[:, 3, :]
        err = float(np.max(np.abs(got - ref) / np.abs(ref)))
        assert err < 1e-12, (x, err)
    g.close()


@pytest.mark.parametrize("temporal", [False, True])
def test_peer_watchdog_reports_dead_neighbour(lb, monkeypatch, temporal):
    """A rank whose neighbour never steps must not hang: the waiting blocks
    (one-step: the border blocks; two-step: k_tb_pull) give up after
    LB_PEER_TIMEOUT_MS and lb_sync returns LB_EPEER."""
    monkeypatch.setenv("LB_PEER_TIMEOUT_MS", "200")
    lx, ly = 16, 40
    r = [lb.Lattice(2 * lx, ly, rank=k, nranks=2, temporal=temporal) for k in range(2)]
    for k, x in enumerate(r):
        x.init_macro(*lbgen.rt_macro(2 * lx, ly, lb.t0(), x0=k * lx, lx=lx))
    r[0].set_peers(r[1], r[1])
    r[1].set_peers(r[0], r[0])
    # the second launch needs r[1]'s first, which never comes
    r[0].step(4 if temporal else 2)
    with pytest.raises(lb.LBError) as ei:
        r[0].sync()
    assert ei.value.status == 7
    for x in r:
        x.close()


def window13(g, x, lx):
    cols = [(x + d) % lx for d in range(-6, 7)]
    return np.concatenate([g.peek_cols(c, 1) for c in cols], axis=1)


@pytest.mark.parametrize("lx,ly,coll", [(1920, 2048, "bgk"), (8192, 8192, "bgk"), (4096, 8192, "regularized")])
def test_sampled_columns_full_size_two_step(lb, lx, ly, coll):
    """The two-step kernel (the default bench path) at BASELINE configs #2, #3
    (8192x8192, N=1) and #4 (4096x8192 per GPU): after one two-step launch,
    column x depends only on columns x-6..x+6 of the previous state; the oracle
    steps that 13-column window twice and its centre must match (edge columns
    of the periodic wrap, strip boundaries and the middle)."""
    g = lb.Lattice(lx, ly, collision=coll, temporal=True)
    g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
    g.step(2)
    samples = [0, 1, 2, 5, 6, lx // 2 + 1, lx - 7, lx - 6, lx - 3, lx - 1]
    wins = {x: window13(g, x, lx) for x in samples}
    g.step(2)
    for x in samples:
        got = g.peek_cols(x, 1)[:, 0, :]
        o = oracle.Lattice(13, ly, collision=oracle.REGULARIZED if coll == "regularized" else oracle.BGK)
        o.set_state(wins[x])
        o.step(2)
        ref = o.get_state(0)[:, 6, :]
        err = float(np.max(np.abs(got - ref) / np.abs(ref)))
        assert err < 1e-12, (x, err)
    g.close()


def test_two_step_equals_one_step_full_size(lb):
    """At 1920x2048 (config #2) two two-step launches == four one-step launches, bit for bit."""
    lx, ly = 1920, 2048
    outs = []
    for temporal in (False, True):
        g = lb.Lattice(lx, ly, temporal=temporal)
        g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
        g.step(4)
        outs.append(g.gather())
        g.close()
        torch.cuda.empty_cache()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("l2", [1, 2, 3])
def test_two_step_refill_ordered_after_the_gather(lb, l2):
    """The phase-1 gather of the two-step kernel reads a state-n buffer with
    generic-proxy shared-memory loads, then the TMA (async proxy) refills that
    buffer: without a proxy fence between them a load still in flight at the
    barrier can read the refill.  A refill that hits L2 is fast enough to land
    in that window: with the L2 prefetch of the windows on, 4 of 8 such
    1000-step runs at 1920x2048 differed from the one-step kernel before the
    fence (profiles/r02_tb_experiments.json, round 2), 0 of 15 after.  Here:
    600 steps, the current state compared bit for bit on the device."""
    lx, ly, nsteps = 1920, 2048, 600
    T0 = oracle.t0()
    runs = []
    for tb in (False, True):
        s = torch.cuda.Stream()
        g = lb.Lattice(lx, ly, stream=s, temporal=False)
        if tb:
            g.temporal(True, l2_prefetch=l2)
        g.init_macro(*lbgen.rt_macro(lx, ly, T0))
        g.step(nsteps)
        g.sync()
        nyp, y0 = int(g.layout.nyp), int(g.layout.y0)
        c0 = torch.from_numpy(g.peek_cols(0, 1)[:, 0, :]).cuda()
        phys = [b.view(-1, 37, nyp)[3:3 + lx, :, y0:y0 + ly] for b in g.bufs]
        cur = 0 if torch.equal(phys[0][0], c0) else 1
        assert torch.equal(phys[cur][0], c0)
        runs.append((g, phys[cur]))
    assert torch.equal(runs[0][1], runs[1][1])
    for g, _ in runs:
        g.close()
