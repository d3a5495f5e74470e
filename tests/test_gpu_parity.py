"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bars (BASELINE.json north_star): pbc / propagate / bc bit-exact; collide and
full steps within 1e-12 max relative error in fp64 (G17: max over physical
(l, x, y) of |f - f_ref| / |f_ref|, with f_ref > 1e-12 asserted).

Inputs: lbgen macro fields (no LB arithmetic) fed to each side's own
equilibrium (``init_macro``), or lbgen random population fields for the pure
data-movement kernels.  For the isolated collide test the input state is built
by the oracle on the host and uploaded to both sides (oracle -> GPU only;
nothing flows from the GPU to the oracle).
"""
import numpy as np
import pytest

import lbgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

Q = 37
TOL = 1e-12
BCN = {"thermal": oracle.WALL_THERMAL, "adiabatic": oracle.WALL_ADIABATIC, "periodic": oracle.PERIODIC}


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1703_00186_b200 as m
    m.lib()
    return m


def pair(lb, lx, ly, bc="thermal", mode="fused", overlap=False, tau=0.8, tb=None, tt=None):
    """(library lattice, oracle lattice).  overlap=True runs the library through
    an NCCL 1-rank self-ring: the only N = 1 configuration in which the
    bulk || exchange, then borders schedule (§8a6) exists — lb_init rejects
    overlap where it would have no effect."""
    T0 = oracle.t0()
    tb = 1.05 * T0 if tb is None else tb
    tt = 0.95 * T0 if tt is None else tt
    g = lb.Lattice(lx, ly, tau=tau, t_bottom=tb, t_top=tt, bc_y=bc, mode=mode, overlap=overlap,
                   nccl_id=lb.nccl_unique_id() if overlap else None)
    o = oracle.Lattice(lx, ly, tau=tau, t_bottom=tb, t_top=tt, bc_y=BCN[bc])
    return g, o


def max_rel(a, ref):
    assert a.shape == ref.shape
    assert np.all(np.abs(ref) > 1e-12), "G17: reference values must stay away from 0"
    return float(np.max(np.abs(a - ref) / np.abs(ref)))


def oracle_state(lx, ly, seed=3, noise=0.01):
    """A realistic post-collision-like state built by the oracle: f_eq of random
    near-equilibrium macro fields times (1 + noise) (test infrastructure)."""
    o = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC)
    o.init_macro(*lbgen.perturbed_macro(lx, ly, oracle.t0(), seed=seed))
    st = o.get_state(0)
    return st * (1.0 + noise * lbgen.uniform_noise(st.shape, seed=seed + 1))


# ------------------------------------------------------------------ state I/O

def test_set_state_gather_peek_roundtrip(lb):
    g = lb.Lattice(37, 45)
    st = lbgen.random_field(Q, 37, 45, seed=1)
    g.set_state(st)
    assert np.array_equal(g.gather(), st)
    assert np.array_equal(g.peek(0), st)
    dev = torch.from_numpy(st).cuda()
    g.set_state(dev)
    assert np.array_equal(g.gather(), st)


@pytest.mark.parametrize("macro", ["rt", "perturbed"])
def test_init_macro_equilibrium_parity(lb, macro):
    lx, ly = 64, 32
    fields = lbgen.rt_macro(lx, ly, oracle.t0()) if macro == "rt" else lbgen.perturbed_macro(lx, ly, oracle.t0())
    g, o = pair(lb, lx, ly)
    g.init_macro(*fields)
    o.init_macro(*fields)
    assert max_rel(g.gather(), o.get_state(0)) < 1e-13
    # device-resident macro input path
    g.init_macro(*[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in fields])
    assert max_rel(g.gather(), o.get_state(0)) < 1e-13


# ------------------------------------------------------------------ per-kernel, identical inputs

@pytest.mark.parametrize("bc", ["thermal", "adiabatic", "periodic"])
@pytest.mark.parametrize("shape", [(64, 32), (3, 6), (7, 131), (130, 37)])
def test_pbc_propagate_bc_bit_exact(lb, bc, shape):
    lx, ly = shape
    if bc != "periodic" and ly < 6:
        pytest.skip()
    g, o = pair(lb, lx, ly, bc=bc, mode="split")
    st = lbgen.random_field(Q, lx, ly, seed=lx + ly)
    g.set_state(st)
    o.set_state(st)
    g.exchange()
    g.propagate()
    o.pbc()
    o.propagate()
    assert np.array_equal(g.peek(1), o.get_state(1)), "propagate (raw pull) not bit-exact"
    g.bc()
    o.bc()
    assert np.array_equal(g.peek(1), o.get_state(1)), "bc not bit-exact"


@pytest.mark.parametrize("tau", [0.8, 1.0, 0.5, 2.0])
def test_collide_parity(lb, tau):
    lx, ly = 40, 33
    st = oracle_state(lx, ly, seed=int(tau * 10))
    g, o = pair(lb, lx, ly, bc="periodic", mode="split", tau=tau)
    g.set_state(st)
    o.set_state(st)
    # periodic: exchange + propagate are bit-exact (tested above), bc is a no-op
    g.exchange(); g.propagate(); g.bc(); g.collide()
    o.step(1)
    assert max_rel(g.gather(), o.get_state(0)) < TOL


# ------------------------------------------------------------------ trajectories (config #1)

@pytest.mark.parametrize("mode,overlap,stride", [("split", False, 1), ("fused", False, 1), ("fused", True, 1),
                                                 ("fused", False, 2)])
@pytest.mark.parametrize("bc", ["thermal", "adiabatic", "periodic"])
def test_trajectory_64x32_10_steps(lb, mode, overlap, stride, bc):
    """Config #1: 64x32, RT init on each side, 10 steps, compared after every step
    (stride 1: the one-step kernels) or every second step (stride 2, fused: the
    two-step kernel, the default for walls at N = 1).  overlap: the NCCL
    self-ring's overlapped schedule (walls only: periodic Y has no overlap)."""
    if overlap and bc == "periodic":
        pytest.skip("periodic Y: the y-halo wrap rewrites rows the bulk reads; overlap is rejected")
    lx, ly = 64, 32
    g, o = pair(lb, lx, ly, bc=bc, mode=mode, overlap=overlap)
    fields = lbgen.rt_macro(lx, ly, oracle.t0())
    g.init_macro(*fields)
    o.init_macro(*fields)
    for k in range(10 // stride):
        g.step(stride)
        o.step(stride)
        err = max_rel(g.gather(), o.get_state(0))
        assert err < TOL, (k, err)
    inv_g = g.invariants()
    inv_o = o.invariants(0)
    assert abs(inv_g[0] - inv_o[0]) / inv_o[0] < 1e-13
    assert np.allclose(inv_g[1:4], inv_o[1:4], rtol=1e-12, atol=1e-13 * inv_o[0])


@pytest.mark.parametrize("shape,tau,bc", [((3, 6), 0.8, "thermal"), ((7, 131), 0.5, "thermal"),
                                          ((130, 37), 1.0, "adiabatic"), ((12, 3), 0.6, "periodic"),
                                          ((33, 200), 2.0, "thermal")])
def test_trajectory_edge_shapes(lb, shape, tau, bc):
    lx, ly = shape
    g, o = pair(lb, lx, ly, bc=bc, tau=tau)
    fields = lbgen.perturbed_macro(lx, ly, oracle.t0(), seed=lx * ly)
    g.init_macro(*fields)
    o.init_macro(*fields)
    g.step(5)
    o.step(5)
    assert max_rel(g.gather(), o.get_state(0)) < TOL


# ------------------------------------------------------------------ internal consistency (bitwise)

@pytest.mark.parametrize("bc", ["thermal", "periodic"])
def test_split_fused_overlap_bit_identical(lb, bc):
    lx, ly = 70, 129
    st = oracle_state(lx, ly, seed=9)
    outs = []
    arms = [("split", False), ("fused", False)] + ([("fused", True)] if bc != "periodic" else [])
    for mode, ov in arms:
        # overlap: the NCCL self-ring (bulk || exchange on the comm stream, then borders)
        g = lb.Lattice(lx, ly, bc_y=bc, mode=mode, overlap=ov, nccl_id=lb.nccl_unique_id() if ov else None)
        g.set_state(st)
        g.step(7)
        outs.append(g.gather())
        g.close()
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


def test_overlap_without_effect_is_rejected(lb):
    """lb_init returns LB_EINVAL for overlap=1 where the overlapped schedule
    cannot run (N = 1 without a communicator, split mode, periodic Y), so no
    configuration can claim an overlap it does not perform."""
    for kw in ({}, {"mode": "split", "nccl": True}, {"bc_y": "periodic", "nccl": True}):
        nccl = kw.pop("nccl", False)
        with pytest.raises(lb.LBError) as ei:
            lb.Lattice(40, 32, overlap=True, nccl_id=lb.nccl_unique_id() if nccl else None, **kw)
        assert ei.value.status == 1, kw


def test_uniform_wall_equilibrium_fixed_point(lb):
    Tw = 0.98 * oracle.t0()
    lx, ly = 32, 64
    g = lb.Lattice(lx, ly, t_bottom=Tw, t_top=Tw)
    ones = np.ones((lx, ly))
    g.init_macro(1.02 * ones, 0 * ones, 0 * ones, Tw * ones)
    st0 = g.gather()
    g.step(100)
    assert np.abs(g.gather() - st0).max() / st0.max() < 1e-12


# ------------------------------------------------------------------ invariants / errors

def test_invariants_and_nonphysical_detection(lb):
    lx, ly = 48, 40
    g, o = pair(lb, lx, ly)
    fields = lbgen.perturbed_macro(lx, ly, oracle.t0(), seed=4)
    g.init_macro(*fields)
    o.init_macro(*fields)
    inv = g.invariants()
    ref = o.invariants(0)
    assert abs(inv[0] - ref[0]) / ref[0] < 1e-13
    assert np.allclose(inv[1:4], ref[1:4], rtol=1e-12, atol=1e-13 * ref[0])
    assert 0.9 < inv[4] < 1.1
    st = g.gather()
    st[5, 3, 7] = np.nan
    g.set_state(st)
    with pytest.raises(lb.LBError) as ei:
        g.invariants()
    assert ei.value.status == 5
    st[5, 3, 7] = -20.0
    g.set_state(st)
    with pytest.raises(lb.LBError) as ei:
        g.invariants()
    assert ei.value.status == 5


def test_call_order_errors(lb):
    g = lb.Lattice(16, 16, mode="split")
    with pytest.raises(lb.LBError) as ei:
        g.bc()
    assert ei.value.status == 2
    g.propagate()
    with pytest.raises(lb.LBError) as ei:
        g.gather()
    assert ei.value.status == 2
    g.bc()
    g.collide()
    g.gather()


def test_api_error_paths(lb):
    """Documented LB_EINVAL / LB_ESTATE cases of include/lb.h."""
    def status(fn):
        with pytest.raises(lb.LBError) as ei:
            fn()
        return ei.value.status
    g = lb.Lattice(16, 16)                      # default (legacy) stream
    assert status(lambda: g.use_graphs(True)) == 1
    assert status(lambda: lb.lib().lb_set_option(g._ctx, 99, 1) and lb.lb._check(
        lb.lib().lb_set_option(g._ctx, 99, 1))) == 1
    s = lb.Lattice(16, 16, mode="split")
    assert status(lambda: s.set_peers(s, s)) == 1        # peers need fused mode
    p = lb.Lattice(16, 16, bc_y="periodic")
    assert status(lambda: p.set_peers(p, p)) == 1        # and walls
    a, b = (lb.Lattice(32, 16, rank=r, nranks=2) for r in range(2))
    assert status(lambda: a.step(1)) == 2                # N > 1 without NCCL or peers
    assert status(lambda: a.gather()) == 2               # gather needs the communicator
    assert status(lambda: a.peek_cols(10, 10)) == 1      # column range out of bounds
    for x in (g, s, p, a, b):
        x.close()


# ------------------------------------------------------------------ full size (config #2)

@pytest.mark.parametrize("overlap", [False, True])
def test_full_size_1920x2048_one_step(lb, overlap):
    """Config #2 lattice in the launch configuration bench.py times (fused)."""
    lx, ly = 1920, 2048
    fields = lbgen.rt_macro(lx, ly, oracle.t0())
    g = lb.Lattice(lx, ly, mode="fused", overlap=overlap, nccl_id=lb.nccl_unique_id() if overlap else None)
    g.init_macro(*fields)
    g.step(2)
    got = g.gather()
    del g
    o = oracle.Lattice(lx, ly)
    o.init_macro(*fields)
    o.step(2)
    ref = o.get_state(0)
    assert max_rel(got, ref) < TOL


def test_full_size_1920x2048_regularized_gravity_split():
    """Full config #2 size with the NEXT rows switched on (regularised collide,
    gravity) in split mode — every per-kernel launch at full size."""
    import paper_1703_00186_b200 as lbm
    lx, ly = 1920, 2048
    grav = (0.0, -1e-5)
    fields = lbgen.rt_macro(lx, ly, oracle.t0())
    g = lbm.Lattice(lx, ly, mode="split", collision="regularized", gravity=grav)
    g.init_macro(*fields)
    g.step(1)
    got = g.gather()
    del g
    o = oracle.Lattice(lx, ly, collision=oracle.REGULARIZED, gravity=grav)
    o.init_macro(*fields)
    o.step(1)
    assert max_rel(got, o.get_state(0)) < TOL


# ------------------------------------------------------------------ NCCL transport on one GPU

@pytest.mark.parametrize("bc,mode,overlap", [("thermal", "fused", True), ("thermal", "fused", False),
                                             ("thermal", "split", False), ("periodic", "fused", False),
                                             ("adiabatic", "fused", True)])
def test_nccl_self_ring_equals_local_wrap(lb, bc, mode, overlap):
    """N = 1 with an NCCL communicator: the exchange runs the N > 1 code path
    (grouped ncclSend/ncclRecv of the contiguous 3-column blocks on the comm
    stream; with overlap the bulk columns run while it is in flight and the
    3+3 border columns after its event) as a 1-rank ring.  It must equal the
    oracle (<= 1e-12) and the local wrap bit for bit, and invariants go
    through ncclAllReduce."""
    lx, ly = 40, 70
    st = oracle_state(lx, ly, seed=31)
    ref = lb.Lattice(lx, ly, bc_y=bc, mode=mode, temporal=False)
    ref.set_state(st)
    ref.step(6)
    want = ref.gather()
    g = lb.Lattice(lx, ly, bc_y=bc, mode=mode, overlap=overlap, nccl_id=lb.nccl_unique_id())
    g.profile(True)
    g.set_state(st)
    g.step(6)
    got = g.gather()
    names = g.profile_read()
    if overlap:   # the schedule really ran: bulk and border launches, every step
        assert names["k_step_fused_bulk"]["launches"] == 6 and names["k_step_fused_border"]["launches"] == 6, names
    assert np.array_equal(got, want)
    o = oracle.Lattice(lx, ly, bc_y=BCN[bc])
    o.set_state(st)
    o.step(6)
    assert max_rel(got, o.get_state(0)) < TOL
    assert np.allclose(g.invariants(), ref.invariants(), rtol=1e-15, atol=0)
    g.close()


# ------------------------------------------------------------------ regularised collide (NEXT 1)

def reg_pair(lb, lx, ly, bc="thermal", mode="fused", tau=0.8):
    T0 = oracle.t0()
    g = lb.Lattice(lx, ly, tau=tau, bc_y=bc, mode=mode, collision="regularized")
    o = oracle.Lattice(lx, ly, tau=tau, bc_y=BCN[bc], collision=oracle.REGULARIZED)
    return g, o


@pytest.mark.parametrize("tau", [0.8, 1.0, 0.55, 2.0])
def test_regularized_collide_parity(lb, tau):
    lx, ly = 40, 33
    st = oracle_state(lx, ly, seed=int(tau * 100), noise=0.03)
    g, o = reg_pair(lb, lx, ly, bc="periodic", mode="split", tau=tau)
    g.set_state(st)
    o.set_state(st)
    g.exchange(); g.propagate(); g.bc(); g.collide()
    o.step(1)
    assert max_rel(g.gather(), o.get_state(0)) < TOL


@pytest.mark.parametrize("mode", ["fused", "split"])
@pytest.mark.parametrize("bc", ["thermal", "adiabatic"])
def test_regularized_trajectory_64x32(lb, mode, bc):
    lx, ly = 64, 32
    g, o = reg_pair(lb, lx, ly, bc=bc, mode=mode)
    fields = lbgen.rt_macro(lx, ly, oracle.t0())
    g.init_macro(*fields)
    o.init_macro(*fields)
    for k in range(10):
        g.step(1)
        o.step(1)
        assert max_rel(g.gather(), o.get_state(0)) < TOL, k


def test_regularized_split_fused_bit_identical_and_256(lb):
    lx, ly = 256, 256
    fields = lbgen.perturbed_macro(lx, ly, oracle.t0(), seed=17)
    outs = []
    for mode in ("split", "fused"):
        g = lb.Lattice(lx, ly, mode=mode, collision="regularized")
        g.init_macro(*fields)
        g.step(3)
        outs.append(g.gather())
    assert np.array_equal(outs[0], outs[1])
    o = oracle.Lattice(lx, ly, collision=oracle.REGULARIZED)
    o.init_macro(*fields)
    o.step(3)
    assert max_rel(outs[1], o.get_state(0)) < TOL


# ------------------------------------------------------------------ peer-store exchange (NEXT 3)

@pytest.mark.parametrize("nranks,streams,coll", [(2, "separate", "bgk"), (3, "separate", "regularized"),
                                                 (4, "shared", "bgk"), (1, "separate", "bgk")])
def test_peer_exchange_ring_equals_single_lattice(lb, nranks, streams, coll):
    """N X-slabs in one process on one GPU, exchanging halos only through the
    fused kernel's peer stores + step counters (lb_set_peers): after several
    steps the slabs equal the 1-slab run bit for bit, and the oracle."""
    lx, ly, nsteps = 24, 70, 9
    lx_total = lx * nranks
    T0 = oracle.t0()
    ref = lb.Lattice(lx_total, ly, collision=coll)
    ref.init_macro(*lbgen.rt_macro(lx_total, ly, T0))
    ref.step(nsteps)
    want = ref.gather()
    ranks = []
    for r in range(nranks):
        st = torch.cuda.Stream() if streams == "separate" else None
        g = lb.Lattice(lx_total, ly, rank=r, nranks=nranks, stream=st, collision=coll)
        g.init_macro(*lbgen.rt_macro(lx_total, ly, T0, x0=r * lx, lx=lx))
        ranks.append(g)
    for r, g in enumerate(ranks):
        g.set_peers(ranks[(r - 1) % nranks], ranks[(r + 1) % nranks])
    torch.cuda.synchronize()
    for _ in range(nsteps):
        for g in ranks:
            g.step(1)
    for g in ranks:
        g.sync()
    got = np.concatenate([g.peek(0) for g in ranks], axis=1)
    assert np.array_equal(got, want)
    o = oracle.Lattice(lx_total, ly, collision=oracle.REGULARIZED if coll == "regularized" else oracle.BGK)
    o.init_macro(*lbgen.rt_macro(lx_total, ly, T0))
    o.step(nsteps)
    assert max_rel(got, o.get_state(0)) < TOL
    for g in ranks:
        g.close()


@pytest.mark.parametrize("nranks,ly,stride,nsteps,lx", [(2, 70, 2, 9, 24), (3, 150, 2, 6, 24), (4, 230, 2, 7, 24),
                                                        (2, 40, 3, 9, 24), (3, 300, 2, 8, 200)])
@pytest.mark.parametrize("coll", ["bgk", "regularized"])
@pytest.mark.parametrize("edge_pull", [True, False])
def test_peer_ring_two_step_kernel(lb, nranks, ly, stride, nsteps, lx, coll, edge_pull):
    """Two-step kernel at N > 1 (peer mode).  edge_pull (the default): only the
    CTAs whose sweep comes within 6 columns of a slab edge wait for that
    neighbour's launch counter and stage their strip's rows of its 6 edge
    columns inside the kernel (interior CTAs start at once; with lx = 24 many
    CTAs share an edge, with lx = 200 one per strip and side); else a k_tb_pull
    launch stages whole columns first.  Steps in pairs (odd remainders:
    one-step peer launches, whose halo pull follows a two-step launch) on
    separate streams == the 1-slab run (one-step kernel) bit for bit."""
    lx_total = lx * nranks
    T0 = oracle.t0()
    ref = lb.Lattice(lx_total, ly, collision=coll, gravity=(1e-6, -1e-5), temporal=False)   # one-step kernel
    ref.init_macro(*lbgen.rt_macro(lx_total, ly, T0))
    ref.step(nsteps)
    want = ref.gather()
    ranks = []
    for r in range(nranks):
        g = lb.Lattice(lx_total, ly, rank=r, nranks=nranks, stream=torch.cuda.Stream(), collision=coll,
                       gravity=(1e-6, -1e-5))
        g.init_macro(*lbgen.rt_macro(lx_total, ly, T0, x0=r * lx, lx=lx))
        g.edge_pull(edge_pull)
        g.profile(True)
        ranks.append(g)
    for r, g in enumerate(ranks):
        g.set_peers(ranks[(r - 1) % nranks], ranks[(r + 1) % nranks])
    torch.cuda.synchronize()
    done = 0
    while done < nsteps:
        k = min(stride, nsteps - done)
        for g in ranks:
            g.step(k)
        done += k
    for g in ranks:
        g.sync()
    got = np.concatenate([g.peek(0) for g in ranks], axis=1)
    assert np.array_equal(got, want)
    for g in ranks:
        names = g.profile_read()
        assert names.get("k_step2_tb" + ("_reg" if coll == "regularized" else ""), {}).get("launches", 0) > 0
        assert ("k_tb_pull" in names) == (not edge_pull), names
        g.close()


@pytest.mark.parametrize("edge_pull", [True, False])
def test_peer_ring_two_step_injected_delay(lb, edge_pull):
    """Two-step kernel at N = 4 with an injected ~1 ms delay in front of one
    rank's every launch: the edge CTAs' counter waits order the exchange, the
    result is the 1-slab run bit for bit."""
    lx, ly, n, nsteps = 60, 230, 4, 8
    T0 = oracle.t0()
    ref = lb.Lattice(lx * n, ly, temporal=False)
    ref.init_macro(*lbgen.rt_macro(lx * n, ly, T0))
    ref.step(nsteps)
    streams = [torch.cuda.Stream() for _ in range(n)]
    ranks = [lb.Lattice(lx * n, ly, rank=r, nranks=n, stream=streams[r]) for r in range(n)]
    for r, g in enumerate(ranks):
        g.init_macro(*lbgen.rt_macro(lx * n, ly, T0, x0=r * lx, lx=lx))
        g.edge_pull(edge_pull)
    for r, g in enumerate(ranks):
        g.set_peers(ranks[(r - 1) % n], ranks[(r + 1) % n])
    torch.cuda.synchronize()
    for _ in range(nsteps // 2):
        for r, g in enumerate(ranks):
            if r == 1:
                with torch.cuda.stream(streams[r]):
                    torch.cuda._sleep(2_000_000)
            g.step(2)
    for g in ranks:
        g.sync()
    got = np.concatenate([g.peek(0) for g in ranks], axis=1)
    assert np.array_equal(got, ref.gather())
    for g in ranks:
        g.close()


# ------------------------------------------------------------------ body force (NEXT 2)

@pytest.mark.parametrize("mode,coll", [("fused", "bgk"), ("split", "bgk"), ("fused", "regularized")])
def test_gravity_trajectory_parity(lb, mode, coll):
    """Rayleigh-Taylor with gravity (shifted equilibrium, reading G7b), 64x32, 10 steps."""
    lx, ly = 64, 32
    grav = (0.0, -2e-4)
    g = lb.Lattice(lx, ly, mode=mode, collision=coll, gravity=grav)
    o = oracle.Lattice(lx, ly, collision=oracle.REGULARIZED if coll == "regularized" else oracle.BGK,
                       gravity=grav)
    fields = lbgen.rt_macro(lx, ly, oracle.t0())
    g.init_macro(*fields)
    o.init_macro(*fields)
    for k in range(10):
        g.step(1)
        o.step(1)
        assert max_rel(g.gather(), o.get_state(0)) < TOL, k


def test_gravity_zero_is_bit_identical_to_unforced(lb):
    lx, ly = 40, 50
    st = oracle_state(lx, ly, seed=5)
    a = lb.Lattice(lx, ly)
    b = lb.Lattice(lx, ly, gravity=(0.0, 0.0))
    for x in (a, b):
        x.set_state(st)
        x.step(4)
    assert np.array_equal(a.gather(), b.gather())


def test_gravity_free_fall_periodic(lb):
    """Uniform fluid at rest, periodic box: momentum grows as n rho g (closed form)."""
    lx, ly, n, gy = 16, 24, 30, -1e-4
    g = lb.Lattice(lx, ly, bc_y="periodic", gravity=(0.0, gy))
    ones = np.ones((lx, ly))
    g.init_macro(ones, 0 * ones, 0 * ones, oracle.t0() * ones)
    g.step(n)
    inv = g.invariants()
    assert abs(inv[2] - n * lx * ly * gy) < 1e-10 * abs(n * lx * ly * gy)


# ------------------------------------------------------------------ fused monitors

def test_invariants_async_matches_sync(lb):
    lx, ly = 40, 64
    g = lb.Lattice(lx, ly)
    g.init_macro(*lbgen.rt_macro(lx, ly, oracle.t0()))
    g.monitor(True)
    out = torch.zeros((6, 5), dtype=torch.float64).pin_memory()
    sync_vals = []
    for k in range(3):
        g.step(1)
        g.invariants_async(out[k])
    g.sync()
    ref = lb.Lattice(lx, ly)
    ref.init_macro(*lbgen.rt_macro(lx, ly, oracle.t0()))
    ref.monitor(True)
    for k in range(3):
        ref.step(1)
        sync_vals.append(ref.invariants())
    assert np.array_equal(out[:3].numpy(), np.array(sync_vals))


# ------------------------------------------------------------------ device RT init

@pytest.mark.parametrize("lx,ly", [(64, 32), (96, 200)])
def test_init_rt_matches_host_fields(lb, lx, ly):
    """lb_init_rt (recipe evaluated on the device) = f_eq of lbgen.rt_macro's
    host fields (oracle init) up to device cos/tanh rounding, and its X slabs
    are the columns of the 1-slab state bit for bit (global column index)."""
    g = lb.Lattice(lx, ly)
    g.init_rt(lbgen.rt_eps(lx), oracle.t0())
    o = oracle.Lattice(lx, ly)
    o.init_macro(*lbgen.rt_macro(lx, ly, oracle.t0()))
    full = g.peek(0)
    assert max_rel(full, o.get_state(0)) < 1e-13
    h = lx // 2
    s1 = lb.Lattice(lx, ly, rank=1, nranks=2)
    s1.init_rt(lbgen.rt_eps(lx), oracle.t0())
    assert np.array_equal(s1.peek(0), full[:, h:, :])
    with pytest.raises(lb.LBError):
        g.init_rt(lbgen.rt_eps(lx), -1.0)
    for x in (g, s1):
        x.close()


@pytest.mark.parametrize("lx,ly", [(7, 6), (300, 2048), (2400, 2048)])
def test_monitor_reduce_multiblock(lb, lx, ly):
    """The one-launch slot reduction (1, 19 and the capped 148 blocks): equal to
    the full pass to rounding, deterministic across calls (ticket reset), and
    the same whether delivered into pinned memory (written by the kernel) or
    into a pageable array (D2H copy)."""
    g = lb.Lattice(lx, ly)
    g.init_macro(*lbgen.rt_macro(lx, ly, oracle.t0()))
    g.monitor(True)
    g.step(1)
    pinned = torch.zeros((3, 5), dtype=torch.float64).pin_memory()
    pageable = np.zeros((2, 5))
    for k in range(3):
        g.invariants_async(pinned[k])
    for k in range(2):
        g.invariants_async(pageable[k])
    g.sync()
    p = pinned.numpy()
    assert np.array_equal(p[0], p[1]) and np.array_equal(p[0], p[2])
    assert np.array_equal(pageable[0], p[0]) and np.array_equal(pageable[1], p[0])
    g.monitor(False)
    full = g.invariants()
    assert np.allclose(p[0, :4], full[:4], rtol=1e-13, atol=1e-13 * full[0])
    assert p[0, 4] == full[4]
    g.close()


@pytest.mark.parametrize("overlap,nccl", [(False, False), (True, True)])
def test_fused_monitors(lb, overlap, nccl):
    """Monitored fused steps leave the state bit-identical, and the in-kernel
    invariants equal the full-pass invariants and the oracle's to rounding."""
    lx, ly = 50, 131
    st = oracle_state(lx, ly, seed=12)
    # one fresh NCCL unique id per communicator
    a = lb.Lattice(lx, ly, overlap=overlap, nccl_id=lb.nccl_unique_id() if nccl else None)
    b = lb.Lattice(lx, ly, overlap=overlap, nccl_id=lb.nccl_unique_id() if nccl else None)
    for x in (a, b):
        x.set_state(st)
    b.monitor(True)
    a.step(3)
    b.step(3)
    inv_mon = b.invariants()          # from the per-block partials
    assert np.array_equal(a.gather(), b.gather())
    b.monitor(False)
    inv_full = b.invariants()         # full pass over the lattice
    assert np.allclose(inv_mon[:4], inv_full[:4], rtol=1e-13, atol=1e-13 * inv_full[0])
    assert inv_mon[4] == inv_full[4]
    o = oracle.Lattice(lx, ly)
    o.set_state(st)
    o.step(3)
    ref = o.invariants(0)
    assert abs(inv_mon[0] - ref[0]) < 1e-13 * ref[0]


# ------------------------------------------------------------------ TMA-staged propagate

@pytest.mark.parametrize("bc", ["thermal", "periodic"])
@pytest.mark.parametrize("shape", [(64, 32), (3, 6), (7, 131), (130, 37), (20, 600)])
def test_tma_propagate_bit_exact(lb, bc, shape):
    """LB_OPT_PROPAGATE_IMPL = 1 (TMA loads of the +-3-row windows into shared
    memory, 16-byte vector stores) is bit-exact with the oracle's pull, incl.
    ragged tails and odd Ly, and with the default gather over several steps
    (so from both buffers, i.e. both tensor maps)."""
    lx, ly = shape
    g, o = pair(lb, lx, ly, bc=bc, mode="split")
    g.set_propagate_impl("tma")
    st = lbgen.random_field(Q, lx, ly, seed=lx * 7 + ly)
    g.set_state(st)
    o.set_state(st)
    g.exchange()
    g.propagate()
    o.pbc()
    o.propagate()
    assert np.array_equal(g.peek(1), o.get_state(1))
    g.bc(); g.collide()
    ref = lb.Lattice(lx, ly, bc_y=bc, mode="split")
    ref.set_state(st)
    ref.step(1)
    for _ in range(3):
        g.exchange(); ref.exchange()
        g.propagate(); ref.propagate()
        assert np.array_equal(g.peek(1), ref.peek(1))
        g.bc(); ref.bc()
        g.collide(); ref.collide()
    assert np.array_equal(g.gather(), ref.gather())


@pytest.mark.parametrize("coll", ["bgk", "regularized"])
@pytest.mark.parametrize("bc", ["thermal", "adiabatic"])
@pytest.mark.parametrize("shape", [(24, 6), (17, 131), (9, 300), (40, 509)])
def test_tma_fused_step_bit_identical(lb, coll, bc, shape):
    """LB_OPT_FUSED_IMPL = 1 (TMA-staged windows) == the register-gather fused
    step bit for bit (multi-tile columns, ragged last tile, wall bands)."""
    lx, ly = shape
    st = oracle_state(lx, ly, seed=lx + ly)
    outs = []
    for impl in ("ldg", "tma"):
        g = lb.Lattice(lx, ly, bc_y=bc, collision=coll, gravity=(0.0, -1e-5), temporal=False)
        g.set_fused_impl(impl)
        g.set_state(st)
        g.step(5)
        outs.append(g.gather())
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------------------------ two steps per pass (temporal blocking)

TB_HT = 104   # strip height of the shipped two-step kernel (lb_tb.cu LB_TB_HT; test_lib_host pins it)


@pytest.mark.parametrize("coll", ["bgk", "regularized"])
@pytest.mark.parametrize("bc", ["thermal", "adiabatic"])
@pytest.mark.parametrize("shape", [(6, 6), (24, 40), (17, 131), (64, 32), (9, 300), (131, 200), (12, 60),
                                   # the strip-layout edges of HT (strip_ya / tb_layout_ok):
                                   (10, TB_HT), (9, TB_HT + 1), (8, TB_HT + 3), (7, TB_HT + 5),
                                   (11, TB_HT + 6), (9, TB_HT + 7), (9, 2 * TB_HT), (13, 2 * TB_HT + 6),
                                   (9, 2 * TB_HT + 7), (8, 3 * TB_HT), (7, 3 * TB_HT + 6)])
def test_two_step_kernel_bit_identical(lb, coll, bc, shape):
    """LB_OPT_TEMPORAL (k_step2_tb: states n+1 and n+2 in one pass, n+1 kept in
    shared memory) == two one-step fused launches bit for bit, and both == the
    oracle (<= 1e-12).  Shapes around the shipped strip height HT: exactly one
    strip (HT), the band HT+1..HT+5 where no strip layout keeps the wall bands
    inside wall strips (lb_step must fall back to the one-step kernel —
    asserted from the launch names), the moved second strip (HT+6, HT+7), two
    exact strips (2 HT) plus 6 / 7 rows, three strips (3 HT, 3 HT + 6); sweeps
    that wrap periodically in x, CTA ranges that cross strip boundaries; odd
    step counts end with one fused step."""
    lx, ly = shape
    st = oracle_state(lx, ly, seed=lx * 7 + ly)
    grav = (1e-6, -1e-5)
    outs = []
    for tb in (False, True):
        g = lb.Lattice(lx, ly, bc_y=bc, collision=coll, gravity=grav, temporal=tb)
        g.profile(True)
        g.set_state(st)
        g.step(4)
        g.step(3)
        names = g.profile_read()
        outs.append(g.gather())
        two = sum(v["launches"] for k, v in names.items() if k.startswith("k_step2_tb"))
        if not tb:
            assert two == 0, names
        elif lb.tb_strip_height() < ly < lb.tb_strip_height() + 6:   # (variant builds: their own HT)
            assert two == 0 and names["k_step_fused_reg" if coll == "regularized" else "k_step_fused"][
                "launches"] == 7, names
        else:
            assert two == 3, names   # 4 = 2 + 2, 3 = 2 + one fused step
        g.close()
    assert np.array_equal(outs[0], outs[1])
    o = oracle.Lattice(lx, ly, bc_y=BCN[bc], collision=oracle.REGULARIZED if coll == "regularized" else oracle.BGK,
                       gravity=grav)
    o.set_state(st)
    o.step(7)
    assert max_rel(outs[1], o.get_state(0)) < TOL


def test_two_step_kernel_l2_promotion(lb):
    """LB_OPT_TB_L2_PROMOTION only changes how the window loads fill L2: every
    legal value gives the same bits (also switched mid-run, which re-encodes
    the tensor maps); other values are rejected."""
    lx, ly = 24, 230
    st = oracle_state(lx, ly, seed=11)
    ref = lb.Lattice(lx, ly, temporal=False)   # one-step kernel reference
    ref.set_state(st)
    ref.step(4)
    for promo in (0, 64, 128, 256):
        g = lb.Lattice(lx, ly)
        g.temporal(True, l2_promotion=promo)
        g.set_state(st)
        g.step(2)
        g.temporal(True, l2_promotion=256 if promo != 256 else 0)
        g.step(2)
        assert np.array_equal(g.gather(), ref.gather()), promo
        with pytest.raises(lb.LBError):
            g.temporal(True, l2_promotion=32)
        g.close()


@pytest.mark.parametrize("coll", ["bgk", "regularized"])
@pytest.mark.parametrize("lx,ly,grid", [(240, 520, 0), (96, 1040, 0), (48, 7800, 0), (200, 214, 37), (64, 104, 0)])
def test_two_step_work_split_and_pdl(lb, coll, lx, ly, grid):
    """The time-aligned work split (default), its tail / wall weights, the
    contiguous split (LB_OPT_TB_TAIL_WEIGHT = 1) and programmatic dependent
    launch on / off only change which CTA sweeps which columns and when a
    launch may start: every combination gives the one-step kernel's bits, with
    monitors on the per-step invariants agree to rounding, and illegal values
    are rejected.  Shapes (148 CTAs unless given): R = 29 / 14 main ranges per
    strip and a tail of 3 / 8 CTAs, R = 1 (75 strips, 73 tail CTAs), an odd CTA
    count (37 CTAs on 3 strips), one strip (no aligned split)."""
    st = oracle_state(lx, ly, seed=lx + ly)
    ref = lb.Lattice(lx, ly, collision=coll, temporal=False)
    ref.set_state(st)
    ref.step(6)
    want = ref.gather()
    ref.close()
    invs = []
    for tail, wall, pdl in ((0, 0, True), (1, 0, True), (16, 24, False), (40, 17, True), (17, 21, False)):
        g = lb.Lattice(lx, ly, collision=coll)
        g.temporal(True, grid=grid, tail_weight16=tail, wall_weight16=wall, pdl=pdl)
        g.monitor(True)
        g.set_state(st)
        out = np.zeros(10)
        for _ in range(3):
            g.step(2)
            g.invariants_pair_async(out)
        g.sync()
        invs.append(out.copy())
        assert np.array_equal(g.gather(), want), (tail, wall, pdl)
        for bad in ((lambda: g.temporal(True, tail_weight16=8)), (lambda: g.temporal(True, tail_weight16=65)),
                    (lambda: lb.lib().lb_set_option(g._ctx, 10, 2))):
            r = None
            try:
                r = bad()
            except lb.LBError:
                r = "raised"
            assert r == "raised" or r != 0
        g.close()
    for v in invs[1:]:
        assert np.allclose(v, invs[0], rtol=1e-13, atol=1e-13 * abs(invs[0][0]))


@pytest.mark.parametrize("coll", ["bgk", "regularized"])
@pytest.mark.parametrize("grid,l2", [(1, 0), (7, 4), (300, 8)])
def test_two_step_kernel_grid_and_prefetch(lb, grid, l2, coll):
    """Any CTA count (one CTA sweeping everything, uneven ranges, more CTAs than
    SMs) and any L2 prefetch distance give the same bits — for the regularised
    kernel this also runs its mbarrier hand-over across many sweeps per CTA."""
    lx, ly = 40, 150
    st = oracle_state(lx, ly, seed=5)
    ref = lb.Lattice(lx, ly, collision=coll, temporal=False)   # one-step kernel reference
    ref.set_state(st)
    ref.step(6)
    g = lb.Lattice(lx, ly, collision=coll)
    g.temporal(True, grid=grid, l2_prefetch=l2)
    g.set_state(st)
    g.step(6)
    assert np.array_equal(g.gather(), ref.gather())


def test_two_step_kernel_oracle_parity(lb):
    """The two-step path against the oracle directly (RT state, 10 steps)."""
    lx, ly = 64, 96
    fields = lbgen.rt_macro(lx, ly, oracle.t0())
    g, o = pair(lb, lx, ly)
    g.temporal(True)
    g.init_macro(*fields)
    o.init_macro(*fields)
    g.step(10)
    o.step(10)
    assert max_rel(g.gather(), o.get_state(0)) < TOL


@pytest.mark.parametrize("coll", ["bgk", "regularized"])
@pytest.mark.parametrize("shape", [(64, 32), (40, 150), (9, 211), (17, 131)])
def test_two_step_kernel_monitors(lb, coll, shape):
    """Monitors inside the two-step kernel: both states' invariants (owned rows
    and columns, each site once) equal full-pass invariants to 1e-13, the state
    is bit-identical to monitors off, and grids of 1..300 CTAs agree."""
    lx, ly = shape
    st = oracle_state(lx, ly, seed=lx + 3 * ly)
    ref = lb.Lattice(lx, ly, collision=coll)
    ref.set_state(st)
    full = []
    for _ in range(2):
        ref.step(1)
        full.append(ref.invariants())
    for grid in (0, 1, 7, 300):
        g = lb.Lattice(lx, ly, collision=coll)
        g.temporal(True, grid=grid)
        g.monitor(True)
        g.set_state(st)
        g.step(2)
        pair_out = np.zeros(10)
        g.invariants_pair_async(pair_out)
        g.sync()
        latest = g.invariants()
        for k in range(2):
            got, want = pair_out[5 * k:5 * k + 5], full[k]
            assert abs(got[0] - want[0]) <= 1e-13 * want[0], (grid, k)
            assert np.allclose(got[1:4], want[1:4], rtol=1e-12, atol=1e-13 * want[0]), (grid, k)
            assert abs(got[4] - want[4]) <= 1e-14 * want[4], (grid, k)
        assert np.array_equal(latest, pair_out[5:])
        assert np.array_equal(g.gather(), ref.gather())
        g.close()


def test_two_step_pair_invariants_state_errors(lb):
    g = lb.Lattice(40, 60)
    g.monitor(True)
    g.init_macro(*lbgen.rt_macro(40, 60, oracle.t0()))
    with pytest.raises(lb.LBError):
        g.invariants_pair_async(np.zeros(10))   # no two-step launch yet
    g.step(1)
    with pytest.raises(lb.LBError):
        g.invariants_pair_async(np.zeros(10))   # last step was a one-step launch
    g.step(2)
    g.invariants_pair_async(np.zeros(10))


# ------------------------------------------------------------------ CUDA-graph stepping

@pytest.mark.parametrize("coll,monitor", [("bgk", False), ("regularized", True)])
def test_graph_steps_bit_identical(lb, coll, monitor):
    lx, ly = 64, 32
    st = oracle_state(lx, ly, seed=77)
    outs, invs = [], []
    for graphs in (False, True):
        g = lb.Lattice(lx, ly, collision=coll, stream=torch.cuda.Stream(), temporal=False)
        if graphs:
            g.use_graphs(True)
        if monitor:
            g.monitor(True)
        g.set_state(st)
        g.step(7)
        g.step(4)
        invs.append(g.invariants())
        outs.append(g.gather())
        g.close()
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(invs[0], invs[1])


def test_graph_steps_peer_ring(lb):
    """Peer path replayed from graphs (device-side step counters) == 1 lattice."""
    lx, ly, n, nsteps = 24, 70, 3, 9
    T0 = oracle.t0()
    ref = lb.Lattice(lx * n, ly)
    ref.init_macro(*lbgen.rt_macro(lx * n, ly, T0))
    ref.step(nsteps)
    ranks = [lb.Lattice(lx * n, ly, rank=r, nranks=n, stream=torch.cuda.Stream()) for r in range(n)]
    for r, g in enumerate(ranks):
        g.init_macro(*lbgen.rt_macro(lx * n, ly, T0, x0=r * lx, lx=lx))
    for r, g in enumerate(ranks):
        g.set_peers(ranks[(r - 1) % n], ranks[(r + 1) % n])
        g.use_graphs(True)
    torch.cuda.synchronize()
    for _ in range(3):          # 1 + 2 + 2 + ... mixes plain steps and graph replays
        for g in ranks:
            g.step(3)
    for g in ranks:
        g.sync()
    got = np.concatenate([g.peek(0) for g in ranks], axis=1)
    assert np.array_equal(got, ref.gather())


@pytest.mark.parametrize("lx_total,ly,n", [(64, 32, 2), (48, 64, 4), (96, 32, 8), (48, 64, 8)])
def test_peer_ring_survey_geometries_with_injected_delay(lb, lx_total, ly, n):
    """SURVEY §4 multi-GPU tier geometries (64x32, 48x64, 96x32 at N = 2..8) as
    in-process peer rings, with an injected delay (a sleep kernel) in front of
    every step of one rank (SPEC S:292 'injected-delay regime'): the step
    counters must order everything, the result is the 1-slab run bit for bit."""
    nsteps = 6
    T0 = oracle.t0()
    ref = lb.Lattice(lx_total, ly)
    ref.init_macro(*lbgen.rt_macro(lx_total, ly, T0))
    ref.step(nsteps)
    lx = lx_total // n
    streams = [torch.cuda.Stream() for _ in range(n)]
    ranks = [lb.Lattice(lx_total, ly, rank=r, nranks=n, stream=streams[r]) for r in range(n)]
    for r, g in enumerate(ranks):
        g.init_macro(*lbgen.rt_macro(lx_total, ly, T0, x0=r * lx, lx=lx))
    for r, g in enumerate(ranks):
        g.set_peers(ranks[(r - 1) % n], ranks[(r + 1) % n])
    torch.cuda.synchronize()
    slow = n // 2
    for _ in range(nsteps):
        for r, g in enumerate(ranks):
            if r == slow:
                with torch.cuda.stream(streams[r]):
                    torch.cuda._sleep(2_000_000)   # ~1 ms of spinning before this rank's step
            g.step(1)
    for g in ranks:
        g.sync()
    got = np.concatenate([g.peek(0) for g in ranks], axis=1)
    assert np.array_equal(got, ref.gather())
    for g in ranks:
        g.close()


# ------------------------------------------------------------------ failure detection

def _inject_nan(g, x, y, l=11):
    """A blow-up mid-run: NaN written straight into BOTH device buffers at one
    physical site (whichever holds the current state), bypassing the API."""
    L = g.layout
    idx = ((3 + x) * 37 + l) * L.nyp + L.y0 + y
    for b in g.bufs:
        b[idx] = float("nan")
    torch.cuda.synchronize()


@pytest.mark.parametrize("temporal", [False, True])
def test_nan_mid_run_raises_enonphys_at_sync(lb, temporal):
    """SPEC S:298 / S:469: a NaN appearing mid-run on the monitored asynchronous
    path (one-step kernel + lb_invariants_async, or the two-step kernel +
    lb_invariants_pair_async) sets the device non-physical flag, and the next
    lb_sync returns LB_ENONPHYS; the flag is sticky until the state is
    replaced, and a clean state clears it."""
    lx, ly = 48, 150
    g = lb.Lattice(lx, ly, temporal=temporal, stream=torch.cuda.Stream())
    fields = lbgen.rt_macro(lx, ly, oracle.t0())
    g.init_macro(*fields)
    g.monitor(True)
    out = torch.zeros(10, dtype=torch.float64).pin_memory()
    for _ in range(2):                                  # healthy steps: no error
        g.step(2)
        (g.invariants_pair_async if temporal else g.invariants_async)(out)
        g.sync()
    assert out[4] > 0.5
    _inject_nan(g, 17, 60)
    g.step(2)
    (g.invariants_pair_async if temporal else g.invariants_async)(out)
    with pytest.raises(lb.LBError) as ei:
        g.sync()
    assert ei.value.status == 5
    if temporal:   # caught in the first state of the pair: the step where it spread
        assert out[4] == -np.inf
    with pytest.raises(lb.LBError) as ei:               # sticky
        g.sync()
    assert ei.value.status == 5
    g.init_macro(*fields)                               # a clean state clears it
    g.step(2)
    (g.invariants_pair_async if temporal else g.invariants_async)(out)
    g.sync()
    assert out[4] > 0.5
    g.close()


def test_nonphysical_flag_from_collision_output(lb):
    """A blow-up created by a collision is flagged by the launch that performs
    it: the state is finite everywhere, but after propagate one site holds
    rho = 0 with momentum (its pulled populations: +0.25 along (1,0), -0.25
    along (-1,0), all others 0) — the collision then produces non-finite
    values (u = j/rho), and the two-step launch's own monitors set the flag."""
    lx, ly = 40, 64
    st = oracle_state(lx, ly, seed=8)
    c = oracle.velocities()
    x, y = 20, 30
    for l in range(Q):            # the pull sources of site (x, y): x - c_l
        st[l, x - c[l, 0], y - c[l, 1]] = 0.0
    st[11, x - 1, y], st[25, x + 1, y] = 0.25, -0.25
    assert tuple(c[11]) == (1, 0) and tuple(c[25]) == (-1, 0)
    assert np.all(np.isfinite(st))
    g = lb.Lattice(lx, ly, bc_y="adiabatic")
    g.set_state(st)
    g.monitor(True)
    g.step(2)
    out = np.zeros(10)
    g.invariants_pair_async(out)
    with pytest.raises(lb.LBError) as ei:
        g.sync()
    assert ei.value.status == 5
    assert not out[4] > 0.0       # state n+1's minimum: the collision at (x, y)
