"""Pins of the oracle's exact-result part (§4.1-4.2 steps 2, 3, 6):
cell hash, stable sort (Eq. 11), per-cell offsets, the 27-cell set (Eq. 12),
and the contact set. Each pin is something other than the oracle itself:
printed worked examples (tests/golden), exact rational arithmetic, invariants
that characterise the result uniquely, and brute force."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_1301_1714_b200 import scenes

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def unit_params(orc, n=(5, 5, 5), h=1.0):
    """A grid of n cells of edge h starting at the origin."""
    sp = scenes.SimParams(box_lo=(0.0, 0.0, 0.0), box_hi=tuple(float(k * h) for k in n),
                          cell_edge=h)
    return orc.make_params(sp, np.array([0.25 * h], np.float32))


# ---------------------------------------------------------------- P1 hash --

def test_hash_worked_examples(orc):
    p = unit_params(orc, (5, 6, 7), 0.5)
    for ex in GOLD["hash"]:
        if ex.get("beyond_hi"):
            x = np.array([[10.0, 10.0, 10.0]])
            want = (4, 5, 6)
        else:
            x = np.array([ex["offset_h"]]) * 0.5
            want = tuple(ex["cell"])
        k = int(orc.hash_cells(p, x)[0])
        got = (k % 5, (k // 5) % 6, k // 30)
        assert got == want, ex["cite"]


def test_hash_matches_exact_floor(orc):
    """Away from cell faces (relative margin 1e-9), the fp64 expression of
    reading R15 equals floor((x - lo)/h) in exact rational arithmetic."""
    rng = np.random.default_rng(7)
    sc = scenes.C1()
    p = orc.make_params(sc.params, sc.radius)
    dims = orc.grid_dims(p)
    pts = rng.uniform(-0.001, 0.0125, (3000, 3)).astype(np.float32).astype(np.float64)
    CM = orc.hash_cells(p, pts)
    h = Fraction(p.h)
    checked = 0
    for x, k in zip(pts, CM):
        c = [int(k) % dims[0], (int(k) // dims[0]) % dims[1], int(k) // (dims[0] * dims[1])]
        for a in range(3):
            q = (Fraction(float(x[a])) - Fraction(p.lo[a])) / h
            frac = q - math.floor(q)
            if min(frac, 1 - frac) < Fraction(1, 10**9):
                continue
            want = min(max(math.floor(q), 0), dims[a] - 1)
            assert c[a] == want
            checked += 1
    assert checked > 8000


# ---------------------------------------------------------------- P2 sort --

def test_sort_worked_examples(orc):
    for ex in GOLD["sort"]:
        SCM, SCCM = orc.sort_map(np.array(ex["CM"], np.uint32))
        assert SCM.tolist() == ex["SCM"], ex["cite"]
        assert SCCM.tolist() == ex["SCCM"], ex["cite"]


@pytest.mark.parametrize("n,kmax,seed", [(1, 3, 0), (1000, 7, 1), (5000, 100000, 2), (4096, 1, 3)])
def test_sort_characterisation(orc, n, kmax, seed):
    """Eq. 11 + non-decreasing + permutation + ties in ascending index: these
    four properties determine the stable sort uniquely."""
    CM = np.random.default_rng(seed).integers(0, kmax, n).astype(np.uint32)
    SCM, SCCM = orc.sort_map(CM)
    assert np.array_equal(SCM, CM[SCCM])  # Eq. 11
    assert np.all(np.diff(SCM.astype(np.int64)) >= 0)
    assert np.array_equal(np.sort(SCCM), np.arange(n))
    ties = SCM[1:] == SCM[:-1]
    assert np.all(SCCM[1:][ties] > SCCM[:-1][ties])


# ------------------------------------------------------------- P3 offsets --

def test_offsets_worked_examples(orc):
    for ex in GOLD["offsets"]:
        off = orc.cell_offsets(np.array(ex["SCM"], np.uint32), ex["ncells"])
        assert off.tolist() == ex["off"], ex["cite"]


def test_offsets_range_invariant(orc):
    rng = np.random.default_rng(3)
    SCM = np.sort(rng.integers(0, 500, 3000)).astype(np.uint32)
    off = orc.cell_offsets(SCM, 600)
    assert off[0] == 0 and off[-1] == 3000
    sizes = np.diff(off.astype(np.int64))
    assert sizes.sum() == 3000 and np.all(sizes >= 0)
    for k in range(600):
        seg = SCM[off[k]:off[k + 1]]
        assert np.all(seg == k)
        assert np.count_nonzero(SCM == k) == seg.size


# ------------------------------------------------------ P4 neighbour set --

def test_neighbor_counts(orc):
    for ex in GOLD["neighbor_cells"]:
        p = unit_params(orc, tuple(ex["grid"]))
        g = ex["grid"]
        c = ex["cell"]
        k = c[0] + g[0] * (c[1] + g[1] * c[2])
        cells = orc.neighbor_cells(p, k)
        assert len(cells) == ex["count"], ex["cite"]
        assert cells == sorted(cells) and len(set(cells)) == len(cells)
        for q in cells:  # every member is within one cell in each axis (Eq. 12)
            qc = (q % g[0], (q // g[0]) % g[1], q // (g[0] * g[1]))
            assert all(abs(qc[a] - c[a]) <= 1 for a in range(3))


# ------------------------------------------------ P5 contact set -----------

def test_predicate_is_strict_and_exact(orc):
    """Touching exactly (d = r_i + r_j) is not a contact (SPEC.md:195 '>0');
    one ulp closer is."""
    r = np.array([0.5, 0.5])
    x = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    assert orc.contacts_brute(x, r).shape[0] == 0
    x[1, 0] = np.nextafter(1.0, 0.0)
    assert orc.contacts_brute(x, r).tolist() == [[0, 1]]


def test_predicate_matches_exact_rationals(orc):
    """Off the rounding band, the fp64 predicate of reading R14 agrees with
    d^2 < (r_i + r_j)^2 evaluated exactly."""
    rng = np.random.default_rng(11)
    n = 400
    x = rng.uniform(0.0, 0.004, (n, 3)).astype(np.float32).astype(np.float64)
    r = rng.uniform(4e-4, 6e-4, n).astype(np.float32).astype(np.float64)
    got = {tuple(p) for p in orc.contacts_brute(x, r).tolist()}
    checked = 0
    for i in range(0, n, 3):
        for j in range(i + 1, n):
            d2 = sum((Fraction(float(x[j, a])) - Fraction(float(x[i, a]))) ** 2 for a in range(3))
            S2 = (Fraction(float(r[i])) + Fraction(float(r[j]))) ** 2
            if abs(d2 - S2) <= S2 * Fraction(1, 10**12):
                continue
            assert ((i, j) in got) == (d2 < S2)
            checked += 1
    assert checked > 20000


@pytest.mark.parametrize("seed", range(6))
def test_grid_contacts_equal_brute_force(orc, seed):
    """Completeness of the CDG: pairs via steps 2-6 == all pairs."""
    sc = scenes.random_gas(1500, 10.0, seed, r_range=(0.25e-3, 0.5e-3))
    p = orc.make_params(sc.params, sc.radius)
    xb = sc.pos.astype(np.float64)
    rb = sc.radius.astype(np.float64)
    brute = orc.contacts_brute(xb, rb)
    grid = orc.contacts_grid(p, xb, rb)
    as_set = lambda a: {(min(i, j), max(i, j)) for i, j in a.tolist()}  # noqa: E731
    assert len(brute) > 100
    assert as_set(grid) == as_set(brute)


def test_grid_contacts_on_cell_faces(orc):
    """Pairs straddling cell faces at exactly touching-minus-epsilon distance."""
    h = 1.0e-3 * (1 + 2**-10)
    pts, rad = [], []
    for k in range(1, 8):
        for a in range(3):
            base = np.full(3, 2.5 * h)
            base[a] = k * h - 0.5e-3 + 1e-9
            other = base.copy()
            other[a] += 1.0e-3 - 2e-9
            pts += [base, other]
            rad += [0.5e-3, 0.5e-3]
    x = np.array(pts, np.float32).astype(np.float64)
    r = np.array(rad, np.float32).astype(np.float64)
    sp = scenes.SimParams(box_lo=(0, 0, 0), box_hi=(0.01, 0.01, 0.01))
    p = orc.make_params(sp, r.astype(np.float32))
    brute = {tuple(q) for q in orc.contacts_brute(x, r).tolist()}
    grid = {tuple(sorted(q)) for q in orc.contacts_grid(p, x, r).tolist()}
    assert len(brute) >= 21 and grid == brute


# ------------------------------------------------------------ P14 Eq. 13 --

def test_eq13_close_packing_formula():
    """Eq. 13: Lx/d * Ly/(sqrt(3)d/2) * Lz/(sqrt(2/3)d) = sqrt(2) LxLyLz/d^3."""
    gold = {e["name"]: e for e in GOLD["paper_constants"]}
    L = 1.0
    lhs = (L / 1.0) * (L / (math.sqrt(3) / 2)) * (L / math.sqrt(2.0 / 3.0))
    assert lhs == pytest.approx(gold["close_packed_per_cell"]["value"], rel=1e-15)


def test_fcc_generator_occupancy(orc):
    """The FCC workload's particles per interior cell match sqrt(2)(h/nn)^3,
    the number density behind Eq. 13."""
    sc = scenes.C2()
    p = orc.make_params(sc.params, sc.radius)
    dims = orc.grid_dims(p)
    CM = orc.hash_cells(p, sc.pos.astype(np.float64))
    cx = CM % dims[0]
    cy = (CM // dims[0]) % dims[1]
    cz = CM // (dims[0] * dims[1])
    # interior window of 14 cells per axis: 14 h = 19.9 lattice half-periods,
    # so plane aliasing of the window is < 0.5%
    lo, hi = 3, 17
    inner = (cx >= lo) & (cx < hi) & (cy >= lo) & (cy < hi) & (cz >= lo) & (cz < hi)
    per_cell = inner.sum() / (hi - lo) ** 3
    want = math.sqrt(2) * (p.h / sc.meta["nn"]) ** 3
    assert per_cell == pytest.approx(want, rel=0.02)
