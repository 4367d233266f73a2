"""Pins of the oracle's time stepping (§4.2; readings R1-R11 of
DESIGN.md): closed forms (Hertz contact duration, restitution from the
nondimensional ODE, static-stack overlaps, sliding-to-rolling), exact per-step
invariants, conservation laws, and brute force vs the CDG."""
import json
import math
import os

import numpy as np
import pytest
from scipy.integrate import solve_ivp
from scipy.special import beta

from paper_1301_1714_b200 import scenes as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_free_fall_worked_example(orc):
    """one semi-implicit Euler step from rest under g."""
    ex = GOLD["free_fall"][0]
    sp = S.SimParams(gravity=tuple(ex["g"]), dt=ex["dt"], box_hi=(100.0, 100.0, 100.0))
    sc = S.make_scene("ff", sp, [[50.0, 50.0, 50.0]], radius=[1.0], mass=[1.0])
    p = orc.make_params(sc.params, sc.radius)
    st = orc.State.from_scene(sc)
    r = orc.step(p, st, orc.History.empty(1, 4))
    assert r.rc == 0
    assert st.vel[0] == pytest.approx(ex["v"], abs=1e-6)
    assert 50.0 - st.pos[0, 2] == pytest.approx(ex["dx"], rel=1e-6)


# ------------------------------------------------ P7 head-on collision ----

def ode_restitution(alpha):
    """x'' + α x^{1/4} x' + x^{3/2} = 0, x(0)=0, x'(0)=1: the practical model's
    normal contact (Eqs. 4, 9, 10) nondimensionalised by δ_max-type scales
    (DESIGN.md §Pins). Returns (e, τ_c)."""
    def f(t, y):
        x = max(y[0], 0.0)
        return [y[1], -alpha * x**0.25 * y[1] - x**1.5]

    def hit(t, y):
        return y[0]
    hit.terminal, hit.direction = True, -1
    s = solve_ivp(f, [0, 50], [0.0, 1.0], events=hit, rtol=1e-12, atol=1e-14, method="DOP853",
                  first_step=1e-6)
    return -s.y_events[0][0][1], s.t_events[0][0]


def ode_restitution_clamped(alpha):
    """The same ODE with the contact unable to pull (reading R3 flag, SURVEY
    §8(c) A3): x'' = -max(0, x^{3/2} + α x^{1/4} x'). Returns (e, τ_c)."""
    def f(t, y):
        x = max(y[0], 0.0)
        return [y[1], -max(0.0, alpha * x**0.25 * y[1] + x**1.5)]

    def hit(t, y):
        return y[0]
    hit.terminal, hit.direction = True, -1
    s = solve_ivp(f, [0, 50], [0.0, 1.0], events=hit, rtol=1e-12, atol=1e-14, method="DOP853",
                  first_step=1e-6)
    return -s.y_events[0][0][1], s.t_events[0][0]


def run_head_on(orc, alpha, v0, steps_per_tc=1000, clamp_fn=False):
    m = float(S.sphere_mass([S.R])[0])
    mstar = m / 2
    K = float(np.float32(7.326e6)) * math.sqrt(float(np.float32(S.R)) / 2)
    tc_scale = (mstar / K) ** 0.4 * v0**-0.2
    dt = float(np.float32(3.218 * tc_scale / steps_per_tc))
    sc = S.two_body(v0, S.SimParams(damping=alpha, friction=0.5, dt=dt, clamp_fn=clamp_fn),
                    gap=0.0)
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(2, 8)
    steps, dmax = 0, 0.0
    for _ in range(4 * steps_per_tc):
        orc.step(p, st, h)
        d = 2 * st.radius[0] - np.linalg.norm(st.pos[1] - st.pos[0])
        if d > 0:
            steps += 1
            dmax = max(dmax, d)
        elif steps:
            break
    lo = int(np.argmin(st.pos[:, 0]))
    e = (st.vel[1 - lo, 0] - st.vel[lo, 0]) / v0
    return e, steps * p.dt, dmax, tc_scale, K, mstar, p.dt


def test_hertz_contact_duration_closed_form(orc):
    """α = 0: t_c = 2 (2/5) B(2/5,1/2) (5/4)^{2/5} (m*/K)^{2/5} v0^{-1/5},
    δ_max = (5 m* v0^2 / (4K))^{2/5}, e = 1 (energy conserved)."""
    const = 2 * 0.4 * beta(0.4, 0.5) * 1.25**0.4
    assert const == pytest.approx(3.218065, rel=1e-6)
    for v0 in (0.01, 0.1, 1.0):
        e, tc, dmax, scale, K, mstar, dt = run_head_on(orc, 0.0, v0)
        assert tc == pytest.approx(const * scale, abs=2 * dt)
        assert dmax == pytest.approx((5 * mstar * v0**2 / (4 * K)) ** 0.4, rel=2e-5)
        assert e == pytest.approx(1.0, abs=1e-6)


@pytest.mark.parametrize("alpha", [0.1, 0.2522, 0.5, 1.0])
def test_restitution_matches_ode(orc, alpha):
    """e(α) from the nondimensional ODE, independent of v0; first-order in dt
    (|Δe|/e <= 2e-3 at t_c/dt ~ 1000); duration τ_c (m*/K)^{2/5} v0^{-1/5}."""
    e_ode, tau = ode_restitution(alpha)
    for v0 in (0.01, 0.1, 1.0):
        e, tc, _, scale, _, _, dt = run_head_on(orc, alpha, v0)
        assert e == pytest.approx(e_ode, rel=2e-3)
        assert tc == pytest.approx(tau * scale, abs=2 * dt)


def test_restitution_anchor_values():
    """The ODE itself: α = 0 is the Hertz closed form; e(0.2522) ~ 0.70 is the
    reading-R19 default."""
    e0, tau0 = ode_restitution(0.0)
    assert e0 == pytest.approx(1.0, abs=1e-9)
    assert tau0 == pytest.approx(2 * 0.4 * beta(0.4, 0.5) * 1.25**0.4, rel=1e-9)
    assert ode_restitution(0.2522)[0] == pytest.approx(0.70, abs=1e-3)


# e(α) with F_n clamped >= 0, computed independently of this
# repository (DOP853 at rtol 1e-12)
E_CLAMPED = {0.1: 0.872291, 0.3: 0.677805, 0.5: 0.539421, 1.0: 0.330500}


@pytest.mark.parametrize("alpha", sorted(E_CLAMPED))
def test_clamped_restitution(orc, alpha):
    """Reading R3 flag (DEM_F_CLAMP_FN): no tensile normal force. The
    restitution is the clamped ODE's (SURVEY Appendix values), higher than
    the literal model's; the literal run at the same α keeps the ODE value
    without the clamp, so a dropped or inverted clamp fails one of the two."""
    e_ode, tau = ode_restitution_clamped(alpha)
    assert e_ode == pytest.approx(E_CLAMPED[alpha], abs=2e-6)
    assert e_ode > ode_restitution(alpha)[0] + 0.003
    for v0 in (0.01, 1.0):
        e, tc, _, scale, _, _, dt = run_head_on(orc, alpha, v0, clamp_fn=True)
        assert e == pytest.approx(e_ode, rel=2e-3)
        assert tc == pytest.approx(tau * scale, abs=2 * dt)
    e_lit = run_head_on(orc, alpha, 0.1, clamp_fn=False)[0]
    assert e_lit == pytest.approx(ode_restitution(alpha)[0], rel=2e-3)


# ------------------------------------------------------- P8 static stack --

def test_static_stack_overlaps(orc):
    """Settled column of n spheres: the contact with k spheres above it has
    δ_k = (k m g / (C_n sqrt(R*)))^{2/3}, R* = r/2 between spheres, r at the
    floor (Hertz: k_n δ = C_n sqrt(R* δ) δ = k m g)."""
    n = 10
    sc = S.stack(n, S.SimParams(damping=1.0))
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(n, 8)
    rc, err, F, T = orc.run(p, st, h, 150000)
    assert rc == 0
    y = np.sort(st.pos[:, 1])
    m, g, r = st.mass[0], -p.g[1], st.radius[0]
    d_pair = 2 * r - np.diff(y)
    k_above = np.arange(n - 1, 0, -1)
    want = (k_above * m * g / (p.Cn * np.sqrt(r / 2))) ** (2 / 3)
    assert d_pair == pytest.approx(want, rel=1e-7)
    assert r - y[0] == pytest.approx((n * m * g / (p.wCn * np.sqrt(r))) ** (2 / 3), rel=1e-7)


# ------------------------------------------------ P9 / P10 sliding sphere --

def slider(orc, truncate):
    sp = S.SimParams(truncate_dt=truncate)
    m = float(S.sphere_mass([S.R])[0])
    p0 = orc.make_params(sp, np.array([S.R], np.float32))
    d_eq = (m * (-p0.g[1]) / (p0.wCn * np.sqrt(np.float32(S.R)))) ** (2 / 3)
    L = 8 * S.D
    sc = S.make_scene("slide", sp.replace(box_hi=(L, L, L)),
                      [[0.5 * L, float(S.R) - d_eq, 0.5 * L]], vel=[[0.1, 0, 0]])
    p = orc.make_params(sc.params, sc.radius)
    return p, orc.State.from_scene(sc), orc.History.empty(1, 8)


def test_sliding_to_rolling(orc):
    """Angular momentum about the contact point is conserved, so the sphere
    ends rolling at (5/7) v0 after t = 2 v0/(7 μ g) (textbook; reading R4 flag)."""
    p, st, h = slider(orc, True)
    v0 = 0.1
    t_slip = 2 * v0 / (7 * p.mu * -p.g[1])
    orc.run(p, st, h, int(1.5 * t_slip / p.dt))
    assert st.vel[0, 0] == pytest.approx(5 / 7 * v0, rel=2e-5)
    assert -st.omega[0, 2] * st.radius[0] == pytest.approx(5 / 7 * v0, rel=2e-5)
    # during the slip phase the sphere is still sliding
    p, st, h = slider(orc, True)
    orc.run(p, st, h, int(0.7 * t_slip / p.dt))
    assert st.vel[0, 0] > -st.omega[0, 2] * st.radius[0] + 0.01 * v0


def test_wall_contact_impulse_invariant(orc):
    """P10: with g ∥ n, every sliding step has r|Δω| = (5/2)|Δv_t| (Eq. 3 with
    I = 0.4 m r^2), and the tangential impulse is μ times the normal one."""
    p, st, h = slider(orc, False)
    for k in range(1500):
        v, w = st.vel.copy(), st.omega.copy()
        r = orc.step(p, st, h)
        dv, dw = st.vel - v, st.omega - w
        dvt = math.hypot(dv[0, 0], dv[0, 2])
        assert st.radius[0] * np.linalg.norm(dw) == pytest.approx(2.5 * dvt, rel=1e-9)
        Fn = r.F[0, 1]
        Ft = math.hypot(r.F[0, 0], r.F[0, 2])
        assert Ft == pytest.approx(p.wmu * abs(Fn), rel=1e-9)


# --------------------------- tangential stiffness C_{k,t} (Eqs. 3, 6-9) ---

def hertz_rest(load, Cn, Rstar):
    """Static overlap of a Hertz contact carrying `load`: k_n δ = C_n sqrt(R* δ) δ
    = load (P8's closed form)."""
    return (load / (Cn * math.sqrt(Rstar))) ** (2 / 3)


def test_stuck_sphere_tangential_oscillation(orc):
    """A sphere resting on the floor (α = 0, static overlap of P8) is given a
    small horizontal velocity v0. Friction holds (|F_t| < μ|F_n|), so the
    contact point's slip s obeys m s'' = -(1 + m r^2/I) k_t s with I = 0.4 m r^2
    (Newton for v and ω, Eqs. 3, 6, 7), k_t = C_t sqrt(δ r) (Eq. 9, wall R* = r):
    v(t) = v0 (5/7 + (2/7) cos Ωt), Ω^2 = 3.5 k_t / m. With C_t = 3 C_n a swap of
    C_n and C_t changes Ω by 3^{2/3}."""
    m = float(S.sphere_mass([S.R])[0])
    sp = S.SimParams(damping=0.0, stiffness_t=3 * 7.326e6, dt=1e-7)
    p0 = orc.make_params(sp, np.array([S.R], np.float32))
    g, r = -p0.g[1], float(np.float32(S.R))
    d0 = hertz_rest(m * g, p0.wCn, r)
    L = 8 * S.D
    v0 = 1e-4
    sc = S.make_scene("stuck", sp.replace(box_hi=(L, L, L)),
                      [[0.5 * L, r - d0, 0.5 * L]], vel=[[v0, 0, 0]])
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(1, 8)
    assert p.wCt == pytest.approx(3 * p.wCn, rel=1e-7)
    kt = p.wCt * math.sqrt(d0 * r)
    Om = math.sqrt(3.5 * kt / st.mass[0])
    n = int(3 * 2 * math.pi / Om / p.dt)
    v = np.empty(n)
    for k in range(n):
        res = orc.step(p, st, h)
        assert math.hypot(res.F[0, 0], res.F[0, 2]) < p.wmu * abs(res.F[0, 1])  # stuck
        v[k] = st.vel[0, 0]
    t = p.dt * np.arange(1, n + 1)
    model = v0 * (5 / 7 + 2 / 7 * np.cos(Om * t))
    assert np.abs(v - model).max() <= 2e-3 * v0
    # spin: angular momentum about the contact point, I ω_z - m r v, is
    # conserved (every force passes through that point or the centre above
    # it), so ω_z = -(5/2)(v0 - v)/r
    v0f = float(sc.vel[0, 0])  # the fp32 input
    assert st.omega[0, 2] == pytest.approx(-2.5 * (v0f - st.vel[0, 0]) / r, rel=1e-6, abs=1e-12)
    # the same run with C_t = C_n is measurably different (the pin has teeth)
    sp2 = sp.replace(stiffness_t=7.326e6, box_hi=(L, L, L))
    sc2 = S.make_scene("stuck", sp2, [[0.5 * L, r - d0, 0.5 * L]], vel=[[v0, 0, 0]])
    p2 = orc.make_params(sc2.params, sc2.radius)
    st2, h2 = orc.State.from_scene(sc2), orc.History.empty(1, 8)
    for k in range(n // 6):
        orc.step(p2, st2, h2)
    assert abs(st2.vel[0, 0] - model[n // 6 - 1]) > 0.2 * v0


def test_stuck_stack_tangential_modes(orc):
    """Two spheres stacked on the floor (A below, B on top; α = 0, static
    overlaps of P8), B given a horizontal velocity v0. Both contacts stick, so
    the small-motion dynamics are linear: per sphere m v' = ΣF_x, I ω_z' = ΣT_z,
    and each contact's slip rate (Eq. 6, n vertical) and tangential spring
    (Eqs. 7, 9) give F = -k s. Particle pair: k_p = C_t sqrt(δ_p r/2) (Eq. 9,
    R* = r/2), wall: k_w = C_t,w sqrt(δ_w r). The oracle's trajectory must
    follow expm(A t) of that 6x6 linear system; C_t = 3 C_n for pairs and
    C_t,w = 2 C_n for the wall, so swapping C_n and C_t in either the pair or
    the wall composition moves a mode frequency by > 25%."""
    from scipy.linalg import expm
    m = float(S.sphere_mass([S.R])[0])
    Cn = 7.326e6
    sp = S.SimParams(damping=0.0, stiffness_t=3 * Cn, wall_stiffness_t=2 * Cn, dt=1e-7)
    p0 = orc.make_params(sp, np.array([S.R], np.float32))
    g, r = -p0.g[1], float(np.float32(S.R))
    dw = hertz_rest(2 * m * g, p0.wCn, r)
    dp = hertz_rest(m * g, p0.Cn, r / 2)
    L = 8 * S.D
    yA = r - dw
    yB = yA + 2 * r - dp
    v0 = 1e-4
    sc = S.make_scene("stack2", sp.replace(box_hi=(L, L, L)),
                      [[0.5 * L, yA, 0.5 * L], [0.5 * L, yB, 0.5 * L]], vel=[[0, 0, 0], [v0, 0, 0]])
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(2, 8)
    mA = st.mass[0]
    I = 0.4 * mA * r * r
    kw = p.wCt * math.sqrt(dw * r)
    kp = p.Ct * math.sqrt(dp * r / 2)
    # y = (vA, wA, vB, wB, s_w, s_p); contact normals vertical (n = -y from the
    # upper body), slip of the contact point: s_w' = vA + r wA,
    # s_p' = (vB - vA) + r (wB + wA). Tangential force on the upper body -k s
    # (and +k_p s_p on A); its torque about the upper centre r(n x F) = -r k s
    # along z, and on A from the pair r(n_A x F_A) = -r k_p s_p.
    A = np.zeros((6, 6))
    A[0, 4], A[0, 5] = -kw / mA, kp / mA
    A[1, 4], A[1, 5] = -r * kw / I, -r * kp / I
    A[2, 5] = -kp / mA
    A[3, 5] = -r * kp / I
    A[4, 0], A[4, 1] = 1.0, r
    A[5, 0], A[5, 1], A[5, 2], A[5, 3] = -1.0, r, 1.0, r
    y0 = np.array([0, 0, v0, 0, 0, 0], np.float64)
    wmax = np.abs(np.linalg.eigvals(A).imag).max()
    n = int(4 * 2 * math.pi / wmax / p.dt)
    every = max(1, n // 40)
    for k in range(1, n + 1):
        res = orc.step(p, st, h)
        assert res.rc == 0 and res.n_pair_contacts == 2 and res.n_wall_contacts == 1
        if k % every == 0:
            want = expm(A * (k * p.dt)) @ y0
            got = np.array([st.vel[0, 0], st.omega[0, 2], st.vel[1, 0], st.omega[1, 2]])
            scale = np.array([v0, v0 / r, v0, v0 / r])  # velocities, spins
            assert (np.abs(got - want[:4]) / scale).max() <= 2e-3, (k, got, want[:4])


# ------------------------------------------------------ P12/P13/P15 -------

def test_momentum_conservation(orc):
    """No walls touched, g = 0: Σ m v is constant (third law)."""
    c1 = S.C1()
    sp = S.SimParams(gravity=(0.0, 0.0, 0.0), box_hi=(0.016, 0.02, 0.016))
    sc = S.make_scene("free", sp, c1.pos + np.float32(2e-3), c1.vel, c1.omega)
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(sc.n, 16)
    P0 = (st.mass[:, None] * st.vel).sum(0)
    A = (st.mass[:, None] * np.abs(st.vel)).sum()
    contacts = 0
    for _ in range(300):
        r = orc.step(p, st, h)
        assert r.rc == 0 and r.n_wall_contacts == 0
        contacts += r.n_pair_contacts
    assert contacts > 300 * 1000 * 2  # a dense, colliding set
    assert np.abs((st.mass[:, None] * st.vel).sum(0) - P0).max() <= 1e-12 * A


def total_energy(orc, st, p):
    """KE + rotational KE + Hertz elastic energy (2/5) K δ^{5/2} of every
    contact (K = C_n sqrt(R*); walls R* = r)."""
    E = 0.5 * (st.mass * (st.vel**2).sum(1)).sum()
    E += 0.5 * (0.4 * st.mass * st.radius**2 * (st.omega**2).sum(1)).sum()
    x, r = st.pos, st.radius
    for i, j in orc.contacts_brute(x, r):
        d = r[i] + r[j] - np.linalg.norm(x[j] - x[i])
        E += 0.4 * p.Cn * math.sqrt(1 / (1 / r[i] + 1 / r[j])) * d**2.5
    for a in range(3):
        for dist in (x[:, a] - p.lo[a], p.hi[a] - x[:, a]):
            d = r - dist
            k = d > 0
            E += (0.4 * p.wCn * np.sqrt(r[k]) * d[k] ** 2.5).sum()
    return E


def test_energy_conservation_elastic_frictionless(orc):
    """α = 0, μ = 0 (so F_t = 0), elastic walls, g = 0: total energy shows no
    secular drift, and its oscillation shrinks with dt."""
    devs = []
    for dt in (2e-6, 1e-6):
        c1 = S.C1()
        sp = S.SimParams(gravity=(0.0, 0.0, 0.0), damping=0.0, friction=0.0, dt=dt)
        sc = S.make_scene("c1", sp.replace(box_hi=c1.params.box_hi), c1.pos,
                          c1.vel * np.float32(4), c1.omega)
        p = orc.make_params(sc.params, sc.radius)
        st, h = orc.State.from_scene(sc), orc.History.empty(sc.n, 16)
        E0 = total_energy(orc, st, p)
        every = int(round(100 * 2e-6 / dt))  # same physical sample times
        dev = []
        for k in range(20 * every):
            orc.step(p, st, h)
            if k % every == every - 1:
                dev.append(abs(total_energy(orc, st, p) / E0 - 1))
        devs.append(np.mean(dev))
    assert devs[0] < 3e-3 and devs[1] < 0.7 * devs[0]


def test_kissing_bound_and_history(orc):
    """P15: monodisperse contacts per particle <= 12 every step;
    history lists hold exactly the contacts of the step (reading R10)."""
    sc = S.C1()
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(sc.n, 16)
    for _ in range(30):
        r = orc.step(p, st, h)
        assert r.rc == 0
        pair = (h.pid < orc.WALL_PID0) & (np.arange(16)[None, :] < h.cnt[:, None])
        assert pair.sum(1).max() <= 12
        assert pair.sum() == r.n_pair_contacts
        assert h.cnt.sum() == r.n_pair_contacts + r.n_wall_contacts
        got = {(int(st.id[i]), int(st.id[j])) for i, j in orc.contacts_brute(st.pos, st.radius)}
    # after the last step the stored lists are those of the pre-integration
    # positions; the contact set was found by the CDG and is symmetric
    d = h.as_dict(st.id)
    pairs = {k for k in d if k[1] < orc.WALL_PID0}
    assert all((b, a) in pairs for a, b in pairs)
    assert len(got) > 0


def test_grid_step_equals_brute_force_step(orc):
    """a step through the CDG equals a step with all-pairs
    detection (same contacts; forces equal up to summation order)."""
    sc = S.random_gas(700, 9.0, 8, r_range=(0.3e-3, 0.5e-3), v_sigma=0.02)
    for brute in (False, True):
        p = orc.make_params(sc.params, sc.radius, brute=brute)
        st, h = orc.State.from_scene(sc), orc.History.empty(sc.n, 32)
        r = orc.step(p, st, h)
        if brute:
            rb, stb, hb = r, st, h
        else:
            rg, stg, hg = r, st, h
    assert rg.n_pair_contacts == rb.n_pair_contacts > 100
    assert np.array_equal(stg.id, stb.id)
    assert hg.as_dict(stg.id).keys() == hb.as_dict(stb.id).keys()
    scale = np.abs(rb.F).max()
    assert np.abs(rg.F - rb.F).max() <= 1e-12 * scale
    assert np.abs(stg.pos - stb.pos).max() <= 1e-15
    assert np.abs(stg.vel - stb.vel).max() <= 1e-12 * np.abs(stb.vel).max()


def test_sampled_step_equals_full_step(orc):
    """The one-by-one evaluation used for full-size parity reproduces the full
    step bitwise on the sampled slots."""
    sc = S.C1()
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(sc.n, 16)
    orc.step(p, st, h)  # some history
    st2, h2 = st.copy(), h.copy()
    full = orc.step(p, st, h)
    mask = np.random.default_rng(0).random(sc.n) < 0.1
    part = orc.step(p, st2, h2, only=mask)
    assert np.array_equal(full.SCCM, part.SCCM)
    for a, b in ((full.F, part.F), (full.T, part.T), (st.pos, st2.pos), (st.vel, st2.vel),
                 (st.omega, st2.omega), (h.cnt, h2.cnt), (h.dt, h2.dt)):
        assert np.array_equal(a[mask], b[mask])


# ------------------------------------ material pairs (Eqs. 5, 8-10 of (i, j)) --

def mat_table():
    """Three materials; every pair has its own C_n (and so its own contact
    duration) and its own α (and so its own restitution)."""
    Cn = {(0, 0): 4e6, (0, 1): 6e6, (0, 2): 8e6, (1, 1): 1.0e7, (1, 2): 1.2e7, (2, 2): 1.4e7}
    al = {(0, 0): 0.05, (0, 1): 0.1, (0, 2): 0.2, (1, 1): 0.3, (1, 2): 0.5, (2, 2): 0.75}
    t = [[None] * 3 for _ in range(3)]
    for (i, j), c in Cn.items():
        t[i][j] = t[j][i] = (c, c, al[(i, j)], 0.5)
    return tuple(tuple(r) for r in t), Cn, al


@pytest.mark.parametrize("a,b", [(0, 1), (1, 2), (2, 2), (2, 0)])
def test_material_pair_restitution_and_duration(orc, a, b):
    """A head-on pair of materials (a, b) rebounds with e(α(a, b)) of the ODE
    and stays in contact τ_c (m*/K)^{2/5} v0^{-1/5} with K = C_n(a, b) sqrt(R*):
    the pair's own table entry is used, whichever side is i."""
    table, Cn, al = mat_table()
    key = (min(a, b), max(a, b))
    v0 = 0.1
    m = float(S.sphere_mass([S.R])[0])
    mstar = m / 2
    K = float(np.float32(Cn[key])) * math.sqrt(float(np.float32(S.R)) / 2)
    tc_scale = (mstar / K) ** 0.4 * v0**-0.2
    dt = float(np.float32(3.218 * tc_scale / 1000))
    sc = S.two_body(v0, S.SimParams(dt=dt, materials=table), gap=0.0)
    sc.material = np.array([a, b], np.uint32)
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(2, 8)
    steps = 0
    for _ in range(4000):
        orc.step(p, st, h)
        if 2 * st.radius[0] - np.linalg.norm(st.pos[1] - st.pos[0]) > 0:
            steps += 1
        elif steps:
            break
    lo = int(np.argmin(st.pos[:, 0]))
    e = (st.vel[1 - lo, 0] - st.vel[lo, 0]) / v0
    e_ode, tau = ode_restitution(float(np.float32(al[key])))
    assert e == pytest.approx(e_ode, rel=2e-3)
    assert steps * p.dt == pytest.approx(tau * tc_scale, abs=2 * p.dt)
    assert sorted(st.mat.tolist()) == sorted([a, b])  # materials travel with the particles


def test_material_wall_restitution(orc):
    """A sphere of material b dropped on the floor rebounds with the wall
    table's α(b) (R* = r, m* = m: the wall limits of R11)."""
    table, _, _ = mat_table()
    walls = ((4e6, 4e6, 0.05, 0.5), (1e7, 1e7, 0.5, 0.5), (1.4e7, 1.4e7, 0.75, 0.5))
    for b in range(3):
        v0 = 0.1
        m = float(S.sphere_mass([S.R])[0])
        K = float(np.float32(walls[b][0])) * math.sqrt(float(np.float32(S.R)))
        tc_scale = (m / K) ** 0.4 * v0**-0.2
        dt = float(np.float32(3.218 * tc_scale / 1000))
        L = 8 * S.D
        sp = S.SimParams(dt=dt, gravity=(0.0, 0.0, 0.0), materials=table, wall_materials=walls,
                         box_hi=(L, L, L))
        sc = S.make_scene("drop", sp, [[0.5 * L, float(S.R), 0.5 * L]], vel=[[0.0, -v0, 0.0]])
        sc.material = np.array([b], np.uint32)
        p = orc.make_params(sc.params, sc.radius)
        st, h = orc.State.from_scene(sc), orc.History.empty(1, 8)
        for _ in range(4000):
            orc.step(p, st, h)
            if st.vel[0, 1] > 0 and st.pos[0, 1] > st.radius[0]:
                break
        e_ode, _ = ode_restitution(float(np.float32(walls[b][2])))
        assert st.vel[0, 1] / v0 == pytest.approx(e_ode, rel=2e-3)


def test_uniform_material_table_equals_scalars(orc):
    """A table whose every entry is the scalar parameters gives the scalar
    run bitwise (the table only selects coefficients)."""
    sc = S.random_gas(400, 8.0, 3, r_range=(0.3e-3, 0.5e-3), v_sigma=0.3)
    sp = sc.params
    c = (sp.stiffness_n, sp.stiffness_t, sp.damping, sp.friction)
    w = (sp.stiffness_n, sp.stiffness_t, sp.damping, sp.friction)
    spm = sp.replace(materials=tuple(tuple(c for _ in range(2)) for _ in range(2)),
                     wall_materials=(w, w))
    out = []
    for params, mat in ((sp, None), (spm, np.arange(sc.n, dtype=np.uint32) % 2)):
        p = orc.make_params(params, sc.radius)
        st = orc.State.from_arrays(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id, mat)
        h = orc.History.empty(sc.n, 16)
        for _ in range(5):
            assert orc.step(p, st, h).rc == 0
        out.append((st.pos.copy(), st.vel.copy(), st.omega.copy()))
    for a, b in zip(*out):
        assert np.array_equal(a, b)


# ------------------------------------------ plates (finite walls, R23) --

def plate_drop(orc, start, vel, plates, steps=4000, stop=None):
    """One sphere in a large gravity-free box with the given plates."""
    L = 40 * S.D
    sp = S.SimParams(gravity=(0.0, 0.0, 0.0), box_hi=(L, L, L), plates=plates)
    sc = S.make_scene("plate", sp, [start], vel=[vel])
    p = orc.make_params(sc.params, sc.radius)
    st, h = orc.State.from_scene(sc), orc.History.empty(1, 8)
    touched = 0
    for _ in range(steps):
        r = orc.step(p, st, h)
        assert r.rc == 0
        touched += r.n_wall_contacts
        if stop and stop(st):
            break
    return st, touched, p


def test_plate_face_restitution_both_sides(orc):
    """A sphere hitting a horizontal plate's face, from above or from below,
    rebounds with the wall e(α) of the ODE (R* = r, m* = m; two-sided)."""
    L = 40 * S.D
    c = (0.5 * L, 0.5 * L, 0.5 * L)
    pl = (S.plate(c, (0, 1, 0), (1, 0, 0), 5 * S.D, 5 * S.D),)
    e_ode, _ = ode_restitution(float(np.float32(0.2522)))
    for side in (+1, -1):
        y0 = c[1] + side * (float(S.R) + 1e-6)
        st, touched, _ = plate_drop(orc, (c[0] + 1.3 * S.D, y0, c[2] - 2.1 * S.D),
                                    (0.0, -side * 0.1, 0.0), pl,
                                    stop=lambda s: side * s.vel[0, 1] > 0
                                    and abs(s.pos[0, 1] - c[1]) > s.radius[0] + 1e-5)
        assert touched > 0
        assert side * st.vel[0, 1] / 0.1 == pytest.approx(e_ode, rel=3e-3)


def test_plate_edge_head_on(orc):
    """A sphere moving along -x at the plate's height onto its edge line
    (x = c_x + half_u) meets it head-on: horizontal normal, e(α) rebound, no
    vertical velocity picked up."""
    L = 40 * S.D
    c = (0.5 * L, 0.5 * L, 0.5 * L)
    a = 3 * S.D
    pl = (S.plate(c, (0, 1, 0), (1, 0, 0), a, 5 * S.D),)
    e_ode, _ = ode_restitution(float(np.float32(0.2522)))
    st, touched, _ = plate_drop(orc, (c[0] + a + float(S.R) + 1e-6, c[1], c[2]), (-0.1, 0.0, 0.0),
                                pl, stop=lambda s: s.vel[0, 0] > 0
                                and s.pos[0, 0] - c[0] - a > s.radius[0] + 1e-5)
    assert touched > 0
    assert st.vel[0, 0] / 0.1 == pytest.approx(e_ode, rel=3e-3)
    assert abs(st.vel[0, 1]) < 1e-12 and abs(st.vel[0, 2]) < 1e-12


def test_plate_corner_force_direction_and_miss(orc):
    """At rest overlapping a plate corner, the force points from the corner
    to the centre with the Hertz magnitude C_n sqrt(r δ) δ; a sphere passing
    beside the plate (beyond half_v + r) never touches it."""
    L = 40 * S.D
    c = np.array([0.5 * L] * 3)
    a, b = 3 * S.D, 2 * S.D
    pl = (S.plate(tuple(c), (0, 1, 0), (1, 0, 0), a, b),)
    corner = c + np.array([a, 0.0, b])
    dirn = np.array([1.0, 0.7, 0.4]) / np.linalg.norm([1.0, 0.7, 0.4])
    x0 = corner + dirn * (float(S.R) - 2e-6)
    sp = S.SimParams(gravity=(0.0, 0.0, 0.0), box_hi=(L, L, L), plates=pl)
    sc = S.make_scene("corner", sp, [tuple(x0)])
    p = orc.make_params(sc.params, sc.radius)
    st = orc.State.from_scene(sc)
    xs = st.pos[0].copy()
    res = orc.step(p, st, orc.History.empty(1, 8))
    corner32 = (c.astype(np.float32).astype(np.float64)
                + np.array([np.float32(a), 0.0, np.float32(b)], np.float64))
    d = xs - corner32
    dist = np.linalg.norm(d)
    delta = st.radius[0] - dist
    want = p.wCn * math.sqrt(st.radius[0] * delta) * delta * d / dist
    assert res.F[0] == pytest.approx(want, rel=1e-9)
    st, touched, _ = plate_drop(orc, (c[0], c[1] + 2 * S.D, c[2] + b + float(S.R) + 1e-5),
                                (0.0, -1.0, 0.0), pl, steps=1500)
    assert touched == 0 and st.pos[0, 1] < c[1] - 0.01 * S.D
