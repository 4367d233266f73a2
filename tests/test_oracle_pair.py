"""Pins of the oracle's contact model (§3, Eqs. 1-10): the printed
worked examples (A1-corrected where SPEC's own signs contradict it, see
golden/worked_examples.json), analytic limits, and exact invariants:
Newton's third law bitwise (P11), the friction law, tangentiality."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_stiffness_examples(orc):
    for ex in GOLD["stiffness"]:
        Rstar = 1.0 / (1.0 / ex["ri"] + 1.0 / ex["rj"])
        kn, kt = orc.stiffness(ex["C"], 3.0 * ex["C"], ex["delta"], Rstar)
        assert kn == ex["k"], ex["cite"]
        assert kt == 3.0 * ex["k"], ex["cite"]  # Eq. 8 differs from Eq. 9 only by C


def test_stiffness_wall_limit(orc):
    """r_j -> inf gives k_n = C sqrt(δ r_i); cross-check r_j = 1e12."""
    C, d, ri = 7.3e6, 2e-6, 5e-4
    kn_wall, _ = orc.stiffness(C, C, d, ri)
    kn_big, _ = orc.stiffness(C, C, d, 1.0 / (1.0 / ri + 1.0 / 1e12))
    assert kn_wall == pytest.approx(C * np.sqrt(d * ri), rel=1e-15)
    assert kn_big == pytest.approx(kn_wall, rel=1e-12)


def test_damping_examples(orc):
    for ex in GOLD["damping"]:
        mstar = 1.0 / (1.0 / ex["mi"] + 1.0 / ex["mj"])
        assert orc.damping(ex["alpha"], ex["kn"], mstar) == ex["eta"], ex["cite"]


def test_tangential_velocity_examples(orc):
    for ex in GOLD["tangential_velocity"]:
        assert orc.tangential_velocity(ex["v"], ex["rw"], ex["n"]).tolist() == ex["vt"], ex["cite"]


def test_tangential_displacement_examples(orc):
    for ex in GOLD["tangential_displacement"]:
        got = orc.tangential_displacement(ex["old"], ex["n"], ex["vt"], ex["dt"])
        assert got.tolist() == ex["new"], ex["cite"]


def test_friction_cap_examples(orc):
    for ex in GOLD["friction_cap"]:
        out, capped = orc.friction_cap(ex["Ft"], ex["limit"], 1.0)
        assert out == pytest.approx(ex["out"], abs=1e-15), ex["cite"]
        assert capped == ex["capped"], ex["cite"]


def test_simple_force_examples(orc):
    for ex in GOLD["simple_force"]:
        F = orc.pair_simple(ex["n"], ex["delta"], ex["u"], ex["ksp"], ex["kda"], ex["ksh"])
        assert F == pytest.approx(ex["F"], abs=1e-12), ex["cite"]


def test_simple_force_damps_approach(orc):
    """Reading R1: Eq. 1's damping and shear resist the relative motion."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = rng.normal(size=3)
        n /= np.linalg.norm(n)
        u = rng.normal(size=3)
        F = orc.pair_simple(n, 0.0, u, 0.0, 1.0, 1.0)
        assert np.dot(F, u) > 0  # F on i along u = v_j - v_i: it reduces |v_i - v_j|


def _random_contact(rng):
    n = rng.normal(size=3)
    n /= np.linalg.norm(n)
    ri, rj = rng.uniform(2e-4, 6e-4, 2)
    mi, mj = rng.uniform(1e-7, 2e-6, 2)
    delta = rng.uniform(1e-8, 3e-5)
    vi, vj = rng.normal(0, 0.1, (2, 3))
    wi, wj = rng.normal(0, 50, (2, 3))
    old = rng.normal(0, 1e-6, 3)
    old -= np.dot(old, n) * n
    return n, ri, rj, mi, mj, delta, vi, vj, wi, wj, old


def test_practical_stationary_pair_is_repulsive(orc):
    """SPEC.md:279 (A1-corrected orientation): at rest, α=0, no history, the
    force on i points from j to i and the torque vanishes."""
    n = np.array([1.0, 0.0, 0.0])
    F, Tc, d1 = orc.pair_practical(n, 1e-5, 2.5e-4, 6.5e-7, [0, 0, 0], [0, 0, 0], [0, 0, 0],
                                   7e6, 7e6, 0.0, 0.5, 2e-6)
    kn, _ = orc.stiffness(7e6, 7e6, 1e-5, 2.5e-4)
    assert F.tolist() == [-kn * 1e-5, 0.0, 0.0]
    assert Tc.tolist() == [0.0, 0.0, 0.0] and d1.tolist() == [0.0, 0.0, 0.0]


def test_practical_damping_adds_on_approach(orc):
    """approaching with α>0 pushes harder than α=0."""
    n = np.array([0.0, 0.0, 1.0])
    args = (n, 1e-5, 2.5e-4, 6.5e-7, [0, 0, 0.1], [0, 0, 0], [0, 0, 0], 7e6, 7e6)
    F0, _, _ = orc.pair_practical(*args, 0.0, 0.5, 2e-6)
    F1, _, _ = orc.pair_practical(*args, 0.5, 0.5, 2e-6)
    assert F1[2] < F0[2] < 0


def test_third_law_bitwise(orc):
    """P11: F_ij = -F_ji, δ_t,ij = -δ_t,ji bitwise, and the unscaled torque
    n x F_t is identical on both sides."""
    rng = np.random.default_rng(17)
    for _ in range(2000):
        n, ri, rj, mi, mj, delta, vi, vj, wi, wj, old = _random_contact(rng)
        Rs = 1.0 / (1.0 / ri + 1.0 / rj)
        Rs2 = 1.0 / (1.0 / rj + 1.0 / ri)
        ms = 1.0 / (1.0 / mi + 1.0 / mj)
        ms2 = 1.0 / (1.0 / mj + 1.0 / mi)
        assert Rs == Rs2 and ms == ms2
        for flags in (0, orc.F_TRUNCATE_DT, orc.F_CLAMP_FN):
            Fa, Ta, Da = orc.pair_practical(n, delta, Rs, ms, vi - vj, ri * wi + rj * wj, old,
                                            7e6, 5e6, 0.3, 0.5, 2e-6, flags)
            Fb, Tb, Db = orc.pair_practical(-n, delta, Rs, ms, vj - vi, rj * wj + ri * wi, -old,
                                            7e6, 5e6, 0.3, 0.5, 2e-6, flags)
            assert np.array_equal(Fa, -Fb)
            assert np.array_equal(Da, -Db)
            assert np.array_equal(Ta, Tb)


def test_friction_law_and_tangentiality(orc):
    """|F_t'| <= μ|F_n|; T·n = 0 and δ_t·n = 0."""
    rng = np.random.default_rng(23)
    mu = 0.4
    for _ in range(3000):
        n, ri, rj, mi, mj, delta, vi, vj, wi, wj, old = _random_contact(rng)
        Rs = 1.0 / (1.0 / ri + 1.0 / rj)
        ms = 1.0 / (1.0 / mi + 1.0 / mj)
        kn, kt = orc.stiffness(7e6, 7e6, delta, Rs)
        eta = orc.damping(0.3, kn, ms)
        v = vi - vj
        F, Tc, d1 = orc.pair_practical(n, delta, Rs, ms, v, ri * wi + rj * wj, old, 7e6, 7e6,
                                       0.3, mu, 2e-6)
        Fn = -kn * delta * n - eta * np.dot(v, n) * n
        Ft = F - Fn
        assert np.linalg.norm(Ft) <= mu * np.linalg.norm(Fn) * (1 + 1e-12)
        assert abs(np.dot(Tc, n)) <= 1e-12 * np.linalg.norm(Tc) + 1e-300
        assert abs(np.dot(d1, n)) <= 1e-12 * (np.linalg.norm(d1) + 1e-30)


def test_zero_overlap_continuity(orc):
    """k, η and hence F vanish as δ -> 0+."""
    n = np.array([0.0, 1.0, 0.0])
    F, Tc, _ = orc.pair_practical(n, 1e-15, 2.5e-4, 6.5e-7, [0, -0.1, 0.05], [0, 0, 0.01],
                                  [0, 0, 0], 7e6, 7e6, 0.3, 0.5, 2e-6)
    assert np.linalg.norm(F) < 1e-4 and np.linalg.norm(Tc) < 1e-4
    F2, _, _ = orc.pair_practical(n, 1e-5, 2.5e-4, 6.5e-7, [0, -0.1, 0.05], [0, 0, 0.01],
                                  [0, 0, 0], 7e6, 7e6, 0.3, 0.5, 2e-6)
    assert np.linalg.norm(F) < 0.1 * np.linalg.norm(F2)


def test_wall_is_infinite_particle(orc):
    """PAPER.md:129 / SPEC.md:290,306: a wall (R*=r_i, m*=m_i, v_j=ω_j=0) equals
    a static particle of radius R -> inf within O(1/R)."""
    rng = np.random.default_rng(29)
    for _ in range(200):
        n, ri, rj, mi, mj, delta, vi, vj, wi, wj, old = _random_contact(rng)
        Fw, Tw, Dw = orc.pair_practical(n, delta, ri, mi, vi, ri * wi, old, 7e6, 7e6, 0.3, 0.5, 2e-6)
        for big in (1e3, 1e6):
            Rb, Mb = big * ri, big**3 * mi
            Rs = 1.0 / (1.0 / ri + 1.0 / Rb)
            ms = 1.0 / (1.0 / mi + 1.0 / Mb)
            Fb, Tb, Db = orc.pair_practical(n, delta, Rs, ms, vi, ri * wi, old, 7e6, 7e6, 0.3,
                                            0.5, 2e-6)
            assert np.linalg.norm(Fb - Fw) <= 5.0 / big * np.linalg.norm(Fw)  # O(1/R)
