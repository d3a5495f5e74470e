"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these re-types the oracle's formulas: each compares it with an
independent fact — the two propagate offsets printed in the paper,
Gaussian (Maxwellian) moments in closed form, conservation laws, hand-stepped
deltas, brute force on tiny lattices.  CPU only (marker: not gpu).
"""
import math
import os

import numpy as np
import pytest

import lbgen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
Q = 37


def gauss_moment(k: int) -> float:
    """E[Z^k] for Z ~ N(0,1): (k-1)!! for even k, 0 for odd k."""
    if k % 2:
        return 0.0
    r = 1.0
    for j in range(k - 1, 0, -2):
        r *= j
    return r


def shifted_gauss_moment(p: int, mean: float, var: float) -> float:
    """E[(mean + sqrt(var) Z)^p], binomial expansion."""
    s = math.sqrt(var)
    return sum(math.comb(p, k) * mean ** (p - k) * s ** k * gauss_moment(k) for k in range(p + 1))


# ---------------------------------------------------------------- velocity set

def test_velocity_set_basic():
    """G1/G2: 37 distinct vectors, reach 3, one zero, symmetric, sum |c|^2 = 216."""
    c = oracle.velocities()
    assert c.shape == (Q, 2)
    assert len({tuple(v) for v in c}) == Q
    assert np.abs(c).max() == 3
    assert sum(1 for v in c if v[0] == 0 and v[1] == 0) == 1
    assert (c.sum(axis=0) == 0).all()
    assert int((c ** 2).sum()) == 216
    shells = {}
    for v in c:
        shells[int(v @ v)] = shells.get(int(v @ v), 0) + 1
    assert shells == {0: 1, 1: 4, 2: 4, 4: 4, 5: 8, 8: 4, 9: 4, 10: 8}


def test_velocity_labels_match_paper_offsets():
    """nxt[site] = prv[site-3*NY+1] (l=0), nxt[NX*NY+site] = prv[NX*NY+site-3*NY] (l=1)."""
    c = oracle.velocities()
    rows = [l.split() for l in open(os.path.join(GOLDEN, "paper_offsets.txt")) if not l.startswith("#")]
    for lab, plane, dx, dy in (map(int, r) for r in rows if r):
        assert plane == lab
        # pull: source = x - c_l
        assert (-c[lab][0], -c[lab][1]) == (dx, dy)


def test_refl_opp():
    c = oracle.velocities()
    for l in range(Q):
        r, o = oracle.refl(l), oracle.opp(l)
        assert tuple(c[r]) == (c[l][0], -c[l][1])
        assert tuple(c[o]) == (-c[l][0], -c[l][1])
        assert oracle.refl(r) == l and oracle.opp(o) == l
        assert o == Q - 1 - l          # consequence of the G2 label order
    assert tuple(c[18]) == (0, 0)


# ---------------------------------------------------------------- weights / a

def test_quadrature_is_gaussian_to_degree_9():
    """G4: sum_l w_l xi_x^p xi_y^q = E[Z^p] E[Z^q] for p+q <= 9, xi = a c."""
    c = oracle.velocities().astype(float)
    w = oracle.weights()
    a = oracle.scale_a()
    xi = a * c
    for p in range(10):
        for q in range(10 - p):
            terms = w * xi[:, 0] ** p * xi[:, 1] ** q
            m = float(np.sum(terms))
            exact = gauss_moment(p) * gauss_moment(q)
            # rounding bound: a few ulps of the sum of |terms|
            assert abs(m - exact) <= 1e-15 * float(np.abs(terms).sum()) * 8, (p, q, m, exact)
    # and the degree is exactly 9: the 10th moment misses 945
    m10 = float(np.sum(w * xi[:, 0] ** 10))
    assert abs(m10 - 945.0) > 1.0
    assert abs(oracle.t0() - 1.0 / (a * a)) < 1e-16


def test_weights_positive_and_by_shell():
    c = oracle.velocities()
    w = oracle.weights()
    assert (w > 0).all()
    c2 = (c ** 2).sum(axis=1)
    for s in set(c2.tolist()):
        assert len(set(w[c2 == s].tolist())) == 1


# ---------------------------------------------------------------- Eq. 2 moments

def test_macro_special_cases():
    """all ones -> (37, 0, 216/74); rest population alone -> T = 0."""
    m = oracle.macro(np.ones(Q))
    assert m[0] == 37.0 and abs(m[1]) < 1e-15 and abs(m[2]) < 1e-15
    assert abs(m[3] - 216.0 / 74.0) < 1e-14
    f = np.zeros(Q)
    f[18] = 5.0
    assert np.allclose(oracle.macro(f), [5.0, 0.0, 0.0, 0.0], atol=0, rtol=0)
    # a single moving population: rho = v, u = c_l, T = 0
    c = oracle.velocities()
    for l in (0, 7, 22):
        f = np.zeros(Q)
        f[l] = 0.3
        m = oracle.macro(f)
        assert abs(m[0] - 0.3) < 1e-16 and abs(m[1] - c[l][0]) < 1e-15 and abs(m[2] - c[l][1]) < 1e-15
        assert abs(m[3]) < 1e-14


def test_macro_temperature_second_form():
    """G8: D rho T = sum |c-u|^2 f  equals  (sum |c|^2 f - rho |u|^2)/(D rho)."""
    c = oracle.velocities().astype(float)
    f = lbgen.random_field(Q, 1, 1, seed=3).reshape(Q)
    m = oracle.macro(f)
    rho = f.sum()
    j = c.T @ f
    T2 = ((c ** 2).sum(axis=1) @ f / rho - (j @ j) / rho ** 2) / 2.0
    assert abs(m[3] - T2) < 1e-14 * abs(T2)


# ---------------------------------------------------------------- App. B f_eq

@pytest.mark.parametrize("rho,ux,uy,T", [
    (1.3, 0.05, -0.02, 1.1),
    (0.9, -0.1, 0.07, 0.6),
    (1.0, 0.0, 0.0, None),   # T0
    (1.02, 0.0003, -0.0001, 0.72),
])
def test_feq_reproduces_maxwellian_moments_to_order_4(rho, ux, uy, T):
    """G5: sum_l f_eq xi^p xi^q = rho E[(uh_x + sqrt(theta) Z)^p] E[(uh_y + sqrt(theta) Z)^q], p+q<=4."""
    a = oracle.scale_a()
    if T is None:
        T = oracle.t0()
    f = oracle.feq(rho, ux, uy, T)
    xi = a * oracle.velocities().astype(float)
    uhx, uhy, theta = a * ux, a * uy, a * a * T
    for p in range(5):
        for q in range(5 - p):
            terms = f * xi[:, 0] ** p * xi[:, 1] ** q
            m = float(np.sum(terms))
            exact = rho * shifted_gauss_moment(p, uhx, theta) * shifted_gauss_moment(q, uhy, theta)
            assert abs(m - exact) <= 1e-15 * float(np.abs(terms).sum()) * 16, (p, q, m, exact)


def test_feq_macro_roundtrip():
    """macroscopic(f_eq(rho,u,T)) = (rho,u,T)."""
    for rho, ux, uy, T in [(1.3, 0.05, -0.02, 1.1), (0.95, -0.01, 0.03, 0.69)]:
        m = oracle.macro(oracle.feq(rho, ux, uy, T))
        assert np.allclose(m, [rho, ux, uy, T], rtol=1e-14, atol=1e-15)


def test_feq_at_rest_reference_temperature_is_weights():
    """At u = 0, T = T0 (theta = 1) the equilibrium is rho * w_l."""
    f = oracle.feq(1.7, 0.0, 0.0, oracle.t0())
    assert np.allclose(f, 1.7 * oracle.weights(), rtol=1e-14, atol=0)


# ---------------------------------------------------------------- K_wall

@pytest.mark.parametrize("tw_rel", [1.05, 0.95, 1.0, 1.3])
def test_kwall_is_unit_density_rest_equilibrium(tw_rel):
    """App. B: sum K = 1, sum c K = 0, temperature of K = T_wall."""
    tw = tw_rel * oracle.t0()
    K = oracle.kwall(tw)
    m = oracle.macro(K)
    assert abs(m[0] - 1.0) < 1e-15
    assert abs(m[1]) < 1e-15 and abs(m[2]) < 1e-15
    assert abs(m[3] - tw) < 1e-14
    assert np.allclose(K, oracle.feq(1.0, 0.0, 0.0, tw), rtol=1e-13, atol=1e-17)


# ---------------------------------------------------------------- collide (Eq. 1)

def _near_eq_f(seed=1):
    rho, ux, uy, T = lbgen.perturbed_macro(1, 1, oracle.t0(), seed=seed)
    f = oracle.feq(rho[0, 0], ux[0, 0], uy[0, 0], T[0, 0])
    return f * (1.0 + 0.01 * lbgen.uniform_noise(Q, seed=seed + 100))


def test_collide_fixed_point_and_full_relaxation():
    """f = f_eq is a fixed point; dt = tau (omega = 1) gives f_eq."""
    feq = oracle.feq(1.1, 0.03, -0.04, 0.75)
    out = oracle.collide_site(feq, 1.25)
    assert np.allclose(out, feq, rtol=1e-14, atol=0)
    f = _near_eq_f()
    m = oracle.macro(f)
    assert np.allclose(oracle.collide_site(f, 1.0), oracle.feq(*m), rtol=1e-14, atol=0)


@pytest.mark.parametrize("omega", [1.0 / 0.8, 1.0, 0.5, 2.0])
def test_collide_conserves_mass_momentum_energy(omega):
    """Collide conserves rho, j and E = 1/2 sum |c|^2 f per site (moment matching)."""
    c = oracle.velocities().astype(float)
    c2 = (c ** 2).sum(axis=1)
    for seed in range(5):
        f = _near_eq_f(seed)
        g = oracle.collide_site(f, omega)
        assert abs(g.sum() - f.sum()) < 1e-14 * f.sum()
        assert np.allclose(c.T @ g, c.T @ f, rtol=0, atol=1e-15)
        assert abs(0.5 * c2 @ g - 0.5 * c2 @ f) < 1e-14 * (0.5 * c2 @ f)
        # it does change f (the non-conserved moments relax)
        assert np.abs(g - f).max() > 1e-6


def test_collide_linear_interpolation_in_omega():
    """Eq. 1 is affine in omega = dt/tau: f(omega) = f - omega (f - f_eq)."""
    f = _near_eq_f(9)
    g1 = oracle.collide_site(f, 1.0)   # = f_eq
    g = oracle.collide_site(f, 0.3)
    assert np.allclose(g, 0.7 * f + 0.3 * g1, rtol=1e-14, atol=1e-18)


def test_collide_commutes_with_x_mirror():
    c = oracle.velocities()
    mx = [next(k for k in range(Q) if c[k][0] == -c[l][0] and c[k][1] == c[l][1]) for l in range(Q)]
    f = _near_eq_f(4)
    g = oracle.collide_site(f, 1.25)
    gm = oracle.collide_site(f[mx], 1.25)
    assert np.allclose(gm, g[mx], rtol=1e-14, atol=0)


# ---------------------------------------------------------------- propagate / pbc

def test_propagate_delta_hops_by_c():
    """A single 1.0 at (l, x0, y0) appears only at (l, x0 + c_lx, y0 + c_ly) (Eq. 1 streaming)."""
    c = oracle.velocities()
    L = oracle.Lattice(12, 10, bc_y=oracle.PERIODIC)
    for l in (0, 1, 8, 18, 29, 36):
        st = np.zeros((Q, 12, 10))
        st[l, 5, 4] = 1.0
        L.set_state(st)
        L.pbc()
        L.propagate()
        out = L.get_state(1)
        nz = np.argwhere(out != 0)
        assert nz.tolist() == [[l, 5 + c[l][0], 4 + c[l][1]]]


def test_propagate_paper_offsets_on_buffers():
    """P:452-453 literally, on the full canonical buffers: nxt[s] = prv[s - 3NY + 1], nxt[NXNY + s] = prv[NXNY + s - 3NY]."""
    L = oracle.Lattice(8, 7, bc_y=oracle.WALL_ADIABATIC)
    L.set_state(lbgen.random_field(Q, 8, 7, seed=2))
    L.pbc()
    L.propagate()
    A = L.buffer(0).reshape(-1)
    B = L.buffer(1).reshape(-1)
    NX, NY = L.nx, L.ny
    for ix in range(3, 3 + 8):
        for iy in range(3, 3 + 7):
            s = ix * NY + iy
            assert B[s] == A[s - 3 * NY + 1]
            assert B[NX * NY + s] == A[NX * NY + s - 3 * NY]


def test_propagate_periodic_is_permutation_and_round_trips():
    """On a torus propagate is a permutation of each plane; propagate, swap l<->opp(l),
    propagate, swap back is the identity, bit-exactly."""
    lx, ly = 9, 7
    L = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC)
    st = lbgen.random_field(Q, lx, ly, seed=8)
    L.set_state(st)
    L.pbc()
    L.propagate()
    out = L.get_state(1)
    for l in range(Q):
        assert np.array_equal(np.sort(out[l].ravel()), np.sort(st[l].ravel()))
    opp = [oracle.opp(l) for l in range(Q)]
    L2 = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC)
    L2.set_state(out[opp])
    L2.pbc()
    L2.propagate()
    back = L2.get_state(1)[opp]
    assert np.array_equal(back, st)


def test_pbc_n1_is_wrap():
    lx, ly = 7, 6
    L = oracle.Lattice(lx, ly, bc_y=oracle.WALL_THERMAL)
    L.set_state(lbgen.random_field(Q, lx, ly, seed=4))
    A = L.buffer(0)
    A[:, :, :3] = 0.5   # y-halo garbage must be copied with the columns (G12)
    L.pbc()
    assert np.array_equal(A[:, 0:3, :], A[:, lx:lx + 3, :])
    assert np.array_equal(A[:, lx + 3:lx + 6, :], A[:, 3:6, :])


# ---------------------------------------------------------------- bc (G9)

def _label(cx, cy):
    c = oracle.velocities()
    return next(l for l in range(Q) if c[l][0] == cx and c[l][1] == cy)


def test_wall_hand_stepped_examples():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "wall_examples.txt")) if l.strip() and not l.strip().startswith("#")]
    assert len(rows) == 5
    for r in rows:
        cxs, cys, ixs, iys, cxe, cye, ixe, iye = map(int, r)
        L = oracle.Lattice(9, 6, bc_y=oracle.WALL_ADIABATIC)
        st = np.zeros((Q, 9, 6))
        st[_label(cxs, cys), ixs - 3, iys - 3] = 1.0
        L.set_state(st)
        L.pbc()
        L.propagate()
        L.bc()
        out = L.get_state(1)
        nz = np.argwhere(out != 0).tolist()
        assert nz == [[_label(cxe, cye), ixe - 3, iye - 3]], (r, nz)


def test_wall_crossing_pair_count():
    """26 (population, row) crossing pairs per wall: 15 + 8 + 3."""
    c = oracle.velocities()
    n = sum(1 for l in range(Q) for row in range(3) if row - c[l][1] < 0)
    assert n == 26
    assert sum(1 for l in range(Q) if c[l][1] > 0) == 15


def test_mirror_walls_are_a_permutation():
    """propagate + mirror (WALL_ADIABATIC) permutes the values of the whole lattice."""
    lx, ly = 8, 9
    L = oracle.Lattice(lx, ly, bc_y=oracle.WALL_ADIABATIC)
    st = lbgen.random_field(Q, lx, ly, seed=12)
    L.set_state(st)
    L.pbc()
    L.propagate()
    L.bc()
    out = L.get_state(1)
    assert np.array_equal(np.sort(out.ravel()), np.sort(st.ravel()))


def test_thermal_wall_sets_u0_and_twall():
    lx, ly = 6, 8
    T0 = oracle.t0()
    L = oracle.Lattice(lx, ly, bc_y=oracle.WALL_THERMAL, t_bottom=1.05 * T0, t_top=0.95 * T0)
    rho, ux, uy, T = lbgen.perturbed_macro(lx, ly, T0, seed=3)
    L.init_macro(rho, ux, uy, T)
    pre = L.get_state(0)
    L.pbc()
    L.propagate()
    L.bc()
    out = L.get_state(1)
    for x in range(lx):
        for y in list(range(3)) + list(range(ly - 3, ly)):
            m = oracle.macro(out[:, x, y])
            assert abs(m[1]) < 1e-15 and abs(m[2]) < 1e-15
            assert abs(m[3] - (1.05 if y < 3 else 0.95) * T0) < 1e-14
    assert pre.shape == out.shape


@pytest.mark.parametrize("bc", [oracle.WALL_THERMAL, oracle.WALL_ADIABATIC])
@pytest.mark.parametrize("ly", [6, 7, 11])
def test_bc_touches_only_the_three_rows_next_to_each_wall(bc, ly):
    """Reading G9 / SURVEY §8c O6: bc rewrites exactly the rows [0, 3) and
    [ly-3, ly) — the rows whose pull sources can lie beyond a wall (|c_y| <= 3).
    Every row in [3, ly-3) after propagate + bc equals, bit for bit, a
    brute-force periodic-x pull from the pre-step state written here with numpy
    indexing (independent of the oracle's propagate): a band that is too wide
    (or a bc writing interior rows) fails this; so does a band that is too
    narrow (the third row keeps raw y-halo zeros, caught below)."""
    lx = 9
    c = oracle.velocities()
    L = oracle.Lattice(lx, ly, bc_y=bc)
    st = lbgen.random_field(Q, lx, ly, seed=100 + ly)
    L.set_state(st)
    L.pbc()
    L.propagate()
    L.bc()
    out = L.get_state(1)
    for l in range(Q):
        cx, cy = int(c[l, 0]), int(c[l, 1])
        for y in range(3, ly - 3):
            assert 0 <= y - cy < ly
            want = st[l, (np.arange(lx) - cx) % lx, y - cy]
            assert np.array_equal(out[l, :, y], want), (l, y)
    # the band rows are all rewritten: no entry pulled from the zero y-halo survives
    for y in list(range(3)) + list(range(ly - 3, ly)):
        assert np.all(out[:, :, y] != 0.0), y
    if bc == oracle.WALL_THERMAL:
        # (ii) repopulates every band site (rho K_wall), so row 2 (the third
        # row) differs from its raw pull for at least one population
        for y in (2, ly - 3):
            raw = np.stack([st[l, (np.arange(lx) - c[l, 0]) % lx, min(max(y - c[l, 1], 0), ly - 1)]
                            for l in range(Q)])
            assert not np.array_equal(out[:, :, y], raw), y


def test_uniform_wall_equilibrium_is_fixed_point():
    """T_bottom = T_top = T', uniform (rho0, u=0, T') equilibrium is a fixed point of the walled step."""
    lx, ly = 8, 12
    Tw = 0.98 * oracle.t0()
    L = oracle.Lattice(lx, ly, bc_y=oracle.WALL_THERMAL, t_bottom=Tw, t_top=Tw)
    ones = np.ones((lx, ly))
    L.init_macro(1.02 * ones, 0 * ones, 0 * ones, Tw * ones)
    st0 = L.get_state(0)
    L.step(100)
    st = L.get_state(0)
    assert np.abs(st - st0).max() / st0.max() < 1e-12


# ---------------------------------------------------------------- full step

def test_periodic_step_conserves_invariants():
    """Fully periodic: global mass, momentum, energy conserved over 200 steps."""
    lx, ly = 32, 24
    L = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC)
    rho, ux, uy, T = lbgen.perturbed_macro(lx, ly, oracle.t0(), seed=21)
    L.init_macro(rho, ux, uy, T)
    inv0 = L.invariants(0)
    L.step(200)
    inv = L.invariants(0)
    assert np.all(np.isfinite(inv))
    assert np.abs(inv - inv0).max() / inv0[0] < 1e-13


@pytest.mark.parametrize("which", [0, 1])
def test_invariants_single_population_closed_form(which):
    """lbref_invariants (the checker behind every GPU monitor test), pinned to
    the definitions rho = sum f, j = sum c f, E = 1/2 sum |c|^2 f (Eq. 2,
    P:189-197; SURVEY §8b lb_invariants): a lattice holding one population of
    value v at label l (all else zero) must give exactly (v, v c_lx, v c_ly,
    v |c_l|^2 / 2) — a swapped j_x / j_y, a dropped 1/2 or a wrong |c|^2 fails.
    The labels' velocities are the paper-pinned table (P:452-453 and the
    shell-count test above); v and its products are exact in binary."""
    lx, ly = 5, 7
    c = oracle.velocities()
    for l in range(Q):
        L = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC)
        st = np.zeros((Q, lx, ly))
        v = 0.375 + l / 64.0
        st[l, l % lx, (3 * l) % ly] = v
        L.set_state(st)
        if which == 1:
            L.pbc()
            L.propagate()   # a permutation: the single value moves, the sums do not change
        inv = L.invariants(which)
        cx, cy = int(c[l, 0]), int(c[l, 1])
        assert inv[0] == v and inv[1] == v * cx and inv[2] == v * cy, l
        assert inv[3] == 0.5 * v * (cx * cx + cy * cy), l


def test_invariants_are_additive_over_sites():
    """Sum of the single-site closed forms over a whole random lattice: the
    invariants of the field equal, to rounding, the sum over sites of each
    site's (rho, j, E) computed here from the per-site moments of oracle.macro
    (pinned separately to Eq. 2) — rho u = j, and E = rho (|u|^2 + D T) / 2."""
    lx, ly = 6, 8
    st = lbgen.random_field(Q, lx, ly, seed=23)
    L = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC)
    L.set_state(st)
    inv = L.invariants(0)
    acc = np.zeros(4)
    for x in range(lx):
        for y in range(ly):
            rho, ux, uy, T = oracle.macro(st[:, x, y])
            acc += [rho, rho * ux, rho * uy, 0.5 * rho * (ux * ux + uy * uy + 2.0 * T)]
    assert np.allclose(inv, acc, rtol=1e-13, atol=1e-14 * acc[0])


def test_walled_rt_step_conserves_mass_and_stays_physical():
    lx, ly = 64, 32
    T0 = oracle.t0()
    L = oracle.Lattice(lx, ly)
    L.init_macro(*lbgen.rt_macro(lx, ly, T0))
    st = L.get_state(0)
    assert 1.9e-4 < st.min() and st.max() < 0.26
    m0 = L.invariants(0)[0]
    L.step(50)
    m = L.invariants(0)[0]
    assert abs(m - m0) / m0 < 1e-13
    assert L.get_state(0).min() > 0


# ---------------------------------------------------------------- Hermite projection (NEXT 1, G6)

def _monomials():
    """V[l, k] = cx^p cy^q for the 15 exponents p + q <= 4 (lattice units)."""
    c = oracle.velocities().astype(float)
    exps = [(p, q) for n in range(5) for p in range(n + 1) for q in [n - p]]
    return np.stack([c[:, 0] ** p * c[:, 1] ** q for p, q in exps], axis=1), exps


def test_projection_is_weighted_least_squares():
    """P f = W V (V^T W V)^-1 V^T f: the orthogonal projection onto {w_l p(c_l): deg p <= 4}
    under <g, h> = sum g h / w, computed in the monomial basis by linear algebra —
    independent of the oracle's Hermite-tensor contraction."""
    V, _ = _monomials()
    w = oracle.weights()
    for seed in range(4):
        f = lbgen.random_field(Q, 1, 1, seed=40 + seed).reshape(Q)
        beta = np.linalg.solve(V.T @ (w[:, None] * V), V.T @ f)
        ref = w * (V @ beta)
        # rounding: 37-term sums of Hermite values up to |xi|^4 ~ 170
        assert np.allclose(oracle.project(f), ref, rtol=0, atol=2e-13 * np.abs(ref).max())


def test_projection_properties():
    V, _ = _monomials()
    w = oracle.weights()
    f = _near_eq_f(5) * (1 + 0.2 * lbgen.uniform_noise(Q, seed=77))
    pf = oracle.project(f)
    assert np.allclose(oracle.project(pf), pf, rtol=0, atol=1e-15)          # idempotent
    assert np.allclose(V.T @ pf, V.T @ f, rtol=1e-13, atol=1e-15)           # moments p+q<=4 kept
    r = f - pf
    assert np.abs(V.T @ r).max() < 1e-14                                    # residual orthogonal
    assert np.abs(r).max() > 1e-5                                           # and nonzero
    feq = oracle.feq(1.1, 0.03, -0.02, 0.75)
    assert np.allclose(oracle.project(feq), feq, rtol=1e-13, atol=0)        # f_eq in the space
    assert np.allclose(oracle.project(w), w, rtol=1e-14, atol=0)


@pytest.mark.parametrize("omega", [1.25, 1.0, 0.6, 2.0])
def test_regularized_collide_conservation_and_limits(omega):
    c = oracle.velocities().astype(float)
    c2 = (c ** 2).sum(axis=1)
    f = _near_eq_f(11)
    g = oracle.collide_site_reg(f, omega)
    assert abs(g.sum() - f.sum()) < 1e-14 * f.sum()
    assert np.allclose(c.T @ g, c.T @ f, rtol=0, atol=1e-15)
    assert abs(c2 @ g - c2 @ f) < 1e-14 * (c2 @ f)
    m = oracle.macro(f)
    feq = oracle.feq(*m)
    if omega == 1.0:
        assert np.allclose(g, feq, rtol=1e-13, atol=0)
    assert np.allclose(oracle.collide_site_reg(feq, omega), feq, rtol=1e-13, atol=0)
    # linear in omega around f_eq: g = f_eq + (1 - omega)(P f - f_eq)
    pf = oracle.project(f)
    assert np.allclose(g, feq + (1 - omega) * (pf - feq), rtol=1e-13, atol=1e-18)


def test_regularized_equals_bgk_inside_hermite_space():
    """If f already lies in the order-<=4 Hermite space, regularised == BGK."""
    f = oracle.project(_near_eq_f(13))
    assert np.allclose(oracle.collide_site_reg(f, 1.25), oracle.collide_site(f, 1.25), rtol=1e-12, atol=0)


def test_regularized_periodic_step_conserves_invariants():
    lx, ly = 24, 20
    L = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC, collision=oracle.REGULARIZED)
    L.init_macro(*lbgen.perturbed_macro(lx, ly, oracle.t0(), seed=22))
    inv0 = L.invariants(0)
    L.step(50)
    inv = L.invariants(0)
    assert np.abs(inv - inv0).max() / inv0[0] < 1e-13


# ---------------------------------------------------------------- body force (NEXT 2, G7b)

@pytest.mark.parametrize("coll", [oracle.BGK, oracle.REGULARIZED])
@pytest.mark.parametrize("omega", [1.25, 1.0, 0.7])
def test_force_adds_exact_momentum_and_work(coll, omega):
    """One forced collision adds rho g to the momentum and rho (u.g + |g|^2/2) to
    E = 1/2 sum |c|^2 f, conserves mass — the balance laws of a body force."""
    c = oracle.velocities().astype(float)
    c2 = (c ** 2).sum(axis=1)
    gx, gy = 3e-5, -2e-4
    f = _near_eq_f(31)
    rho = f.sum()
    u = (c.T @ f) / rho
    g = oracle.collide_site_force(f, omega, gx, gy, coll)
    assert abs(g.sum() - rho) < 1e-14 * rho
    assert np.allclose(c.T @ g - c.T @ f, [rho * gx, rho * gy], rtol=1e-9, atol=1e-17)
    dE = 0.5 * c2 @ g - 0.5 * c2 @ f
    assert abs(dE - rho * (u @ [gx, gy] + 0.5 * (gx * gx + gy * gy))) < 1e-14 * (0.5 * c2 @ f)


def test_force_zero_reduces_to_unforced():
    f = _near_eq_f(32)
    assert np.array_equal(oracle.collide_site_force(f, 1.25, 0.0, 0.0, oracle.BGK), oracle.collide_site(f, 1.25))
    assert np.array_equal(oracle.collide_site_force(f, 1.25, 0.0, 0.0, oracle.REGULARIZED),
                          oracle.collide_site_reg(f, 1.25))


def test_uniform_fluid_free_fall_closed_form():
    """Periodic box, uniform fluid at rest, gravity g: every site stays identical
    and the momentum grows linearly, j(n) = n rho g (closed form)."""
    lx, ly, n = 6, 8, 40
    gy = -1e-4
    L = oracle.Lattice(lx, ly, bc_y=oracle.PERIODIC, gravity=(0.0, gy))
    ones = np.ones((lx, ly))
    L.init_macro(ones, 0 * ones, 0 * ones, oracle.t0() * ones)
    L.step(n)
    inv = L.invariants(0)
    sites = lx * ly
    assert abs(inv[0] - sites) < 1e-12 * sites
    assert abs(inv[2] - n * sites * gy) < 1e-10 * abs(n * sites * gy)
    st = L.get_state(0)
    assert np.abs(st - st[:, :1, :1]).max() < 1e-15
