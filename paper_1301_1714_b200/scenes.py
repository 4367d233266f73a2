"""Seeded synthetic inputs for the DEM timestep — shared by the product tests,
the bench and the oracle tests.

This module holds NO arithmetic of the method (no hashing, no forces, no
integration): only parameter sets and particle positions / velocities / radii /
masses drawn from seeded generators, returned as fp32 arrays exactly as the GPU
receives them. Both sides (CUDA path and oracle) consume the same arrays.

Workload recipe:
  * C1  jittered FCC 8x4x8 unit cells   =     1,024 spheres, box 12x16x12 d
  * C2  jittered FCC 16^3 unit cells    =    16,384 spheres, box 24x32x24 d
  * C3  jittered FCC 32x32x64           =   262,144 spheres, box 46x46x91 d
  * C4  pre-compressed SC settling bed  = 4,194,304 spheres (256x64x256), box 258x72x258 d
  * C5  polydisperse SC bed (per GPU)   = 2,097,152 spheres, r ~ U[0.25, 0.5] mm
FCC: nearest-neighbour spacing nn = 0.995 d, lattice constant a = sqrt(2) nn,
jitter U(+-0.01 d) per coordinate, lattice origin 0.6 d from the box corner,
v ~ N(0, 0.05 m/s)^3, omega ~ N(0, 50 rad/s)^3 — "particles are located so
densely that most particles are expected to have collisions with their closest
particles" (§6). Material defaults: DESIGN.md reading R19 (the
paper gives no constants).
"""
from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass, field

import numpy as np

D = 1.0e-3  # particle diameter [m] (reading R19)
R = 0.5 * D
RHO = 2500.0  # density [kg/m^3]


@dataclass
class SimParams:
    """The paper's problem statement: radius,
    spring parameters C_k, restitution parameter alpha, friction mu, gravity,
    time step, box walls; plus the simple model's constants (Eq. 1)."""

    model: str = "practical"  # "practical" (Eqs. 2-10) | "simple" (Eq. 1)
    dt: float = 2.0e-6
    gravity: tuple = (0.0, -9.81, 0.0)
    box_lo: tuple = (0.0, 0.0, 0.0)
    box_hi: tuple = (12 * D, 16 * D, 12 * D)
    stiffness_n: float = 7.326e6  # C_{k,n} [Pa]
    stiffness_t: float = 7.326e6  # C_{k,t} [Pa]
    damping: float = 0.2522  # alpha (e = 0.70)
    friction: float = 0.5  # mu
    wall_stiffness_n: float = -1.0  # < 0 -> particle value
    wall_stiffness_t: float = -1.0
    wall_damping: float = -1.0
    wall_friction: float = -1.0
    k_sp: float = 259.0  # simple model spring [N/m]
    k_da: float = 3.28e-3  # simple model damping [N s/m]
    k_sh: float = 3.28e-3  # simple model shear [N s/m]
    cell_edge: float = 0.0  # 0 -> 2 r_max (1 + 2^-10)
    max_contacts: int = 16  # K
    truncate_dt: bool = False  # reading R4 flag
    clamp_fn: bool = False  # reading R3 flag
    # Eqs. 5, 8-10 as functions of the pair: None, or an
    # (M, M, 4) symmetric table of (C_n, C_t, alpha, mu) per material pair and
    # optionally an (M, 4) table for particle-wall pairs (None: wall_* above)
    materials: tuple | None = None
    wall_materials: tuple | None = None
    # extra walls (reading R23): up to 10 finite two-sided rectangles, each
    # plate(centre, normal, u, half_u, half_v)
    plates: tuple | None = None

    def replace(self, **kw) -> "SimParams":
        return dataclasses.replace(self, **kw)


@dataclass
class Scene:
    name: str
    params: SimParams
    pos: np.ndarray  # (n,3) float32
    vel: np.ndarray  # (n,3) float32
    omega: np.ndarray  # (n,3) float32
    radius: np.ndarray  # (n,) float32
    mass: np.ndarray  # (n,) float32
    id: np.ndarray  # (n,) uint32
    meta: dict = field(default_factory=dict)
    material: np.ndarray | None = None  # (n,) uint32 material ids (params.materials)

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])


def sphere_mass(radius, density: float = RHO) -> np.ndarray:
    """m = rho (4/3) pi r^3, rounded to fp32 (an input, not method arithmetic)."""
    r = np.asarray(radius, dtype=np.float64)
    return (density * (4.0 / 3.0) * math.pi * r**3).astype(np.float32)


def make_scene(name, params, pos, vel=None, omega=None, radius=None, mass=None, ids=None,
               meta=None) -> Scene:
    pos = np.ascontiguousarray(np.asarray(pos, dtype=np.float32).reshape(-1, 3))
    n = pos.shape[0]
    z3 = np.zeros((n, 3), np.float32)
    vel = z3.copy() if vel is None else np.ascontiguousarray(np.asarray(vel, np.float32).reshape(n, 3))
    omega = z3.copy() if omega is None else np.ascontiguousarray(
        np.asarray(omega, np.float32).reshape(n, 3))
    if radius is None:
        radius = np.full(n, R, np.float32)
    radius = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float32), (n,)))
    mass = sphere_mass(radius) if mass is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(mass, np.float32), (n,)))
    ids = np.arange(n, dtype=np.uint32) if ids is None else np.asarray(ids, np.uint32)
    return Scene(name, params, pos, vel, omega, radius, mass, ids, dict(meta or {}))


# ----------------------------------------------------------------- lattices --

def fcc_lattice(ncx: int, ncy: int, ncz: int, nn: float, origin: float) -> np.ndarray:
    """FCC sites: basis {0, (0,1/2,1/2), (1/2,0,1/2), (1/2,1/2,0)} * a, a = sqrt(2) nn."""
    a = math.sqrt(2.0) * nn
    basis = np.array([[0, 0, 0], [0, 0.5, 0.5], [0.5, 0, 0.5], [0.5, 0.5, 0]], np.float64)
    i, j, k = np.meshgrid(np.arange(ncx), np.arange(ncy), np.arange(ncz), indexing="ij")
    cells = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.float64)
    pts = (cells[:, None, :] + basis[None, :, :]).reshape(-1, 3) * a + origin
    return pts


def sc_lattice(nx: int, ny: int, nz: int, spacing: float, origin: float) -> np.ndarray:
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    return np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.float64) * spacing + origin


def _shuffle(rng, *arrays):
    """Random initial memory order, so the first sort has real work to do."""
    p = rng.permutation(arrays[0].shape[0])
    return [a[p] for a in arrays]


def fcc_scene(name: str, ncells: tuple, box_d: tuple, seed: int, params: SimParams | None = None,
              nn: float = 0.995 * D, jitter: float = 0.01 * D, v_sigma: float = 0.05,
              w_sigma: float = 50.0, shuffle: bool = True) -> Scene:
    rng = np.random.default_rng(seed)
    pos = fcc_lattice(*ncells, nn=nn, origin=0.6 * D)
    pos = pos + rng.uniform(-jitter, jitter, pos.shape)
    n = pos.shape[0]
    vel = rng.normal(0.0, v_sigma, (n, 3))
    omg = rng.normal(0.0, w_sigma, (n, 3))
    if shuffle:
        pos, vel, omg = _shuffle(rng, pos, vel, omg)
    p = (params or SimParams()).replace(box_lo=(0.0, 0.0, 0.0),
                                        box_hi=tuple(float(b * D) for b in box_d))
    return make_scene(name, p, pos, vel, omg,
                      meta=dict(kind="fcc", nn=nn, jitter=jitter, ncells=ncells, seed=seed))


def C1(params: SimParams | None = None) -> Scene:
    """1,024 particles, practical model, settling in a small box under gravity."""
    return fcc_scene("C1", (8, 4, 8), (12, 16, 12), seed=1, params=params)


def C2(params: SimParams | None = None) -> Scene:
    """16,384 particles (the SDK sample's default size); simple vs practical."""
    return fcc_scene("C2", (16, 16, 16), (24, 32, 24), seed=2, params=params)


def C3(params: SimParams | None = None) -> Scene:
    """262,144 particles, dense random (jittered close) packing, friction + rotation."""
    return fcc_scene("C3", (32, 32, 64), (46, 46, 91), seed=3, params=params)


def settling_bed(name: str, nxyz: tuple, box_d: tuple, seed: int, spacing: float = 0.998 * D,
                 jitter: float = 0.005 * D, params: SimParams | None = None,
                 r_range: tuple | None = None, z0: float = 0.0) -> Scene:
    """Pre-compressed simple-cubic bed released from rest under gravity (-y).

    The bottom layer sits r - 0.001 d above the floor (in contact), neighbours
    are 0.998 d apart +- jitter, so the bed starts dense and settles.
    """
    rng = np.random.default_rng(seed)
    origin = 0.499 * spacing / 0.998
    pos = sc_lattice(*nxyz, spacing=spacing, origin=origin)
    pos = pos + rng.uniform(-jitter, jitter, pos.shape)
    pos[:, 2] += z0
    n = pos.shape[0]
    if r_range is None:
        radius = np.full(n, R)
    else:
        radius = rng.uniform(r_range[0], r_range[1], n)
    pos, radius = _shuffle(rng, pos, radius)
    p = (params or SimParams()).replace(box_lo=(0.0, 0.0, 0.0),
                                        box_hi=tuple(float(b * D) for b in box_d))
    return make_scene(name, p, pos, radius=radius,
                      meta=dict(kind="sc_bed", spacing=spacing, jitter=jitter, nxyz=nxyz, seed=seed))


def C4(params: SimParams | None = None, scale: int = 1) -> Scene:
    """4M-particle settling bed (256x64x256); `scale` shrinks x and z for tests."""
    nx, nz = 256 // scale, 256 // scale
    return settling_bed("C4" if scale == 1 else f"C4/{scale}", (nx, 64, nz),
                        (nx + 2, 72, nz + 2), seed=4, params=params)


def poly_bed(name: str, nxyz: tuple, box_d: tuple, seed: int, spacing: float = 0.75 * D,
             r_range: tuple = (0.25 * D, 0.5 * D), jitter: float = 0.005 * D, eps: float = 2e-3,
             params: SimParams | None = None, z0: float = 0.0) -> Scene:
    """Polydisperse bed on a jittered simple-cubic lattice (spacing ~ the mean
    diameter), released from rest under gravity. Radii are drawn from r_range
    and then capped so that no pair overlaps by more than eps of its gap:
    lattice sites are visited in 8 interleaved sub-lattices (sites of one are
    >= 2 spacings apart, so they never neighbour each other), and each drawn
    radius is limited to (d_ij - r_j)(1 + eps) over its 26 already-sized
    neighbours j (and the box faces) — a capped particle touches the
    neighbour that capped it.
    The bed starts loose (~1 contact per particle) and dense enough to
    compact within a few thousand steps."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = nxyz
    idx = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    pos = idx * spacing + 0.5 * D + rng.uniform(-jitter, jitter, idx.shape)
    pos[..., 2] += z0
    pos = pos.astype(np.float32).astype(np.float64)  # the fp32 centres the GPU will see
    draw = rng.uniform(r_range[0], r_range[1], (nx, ny, nz))
    box = np.array(box_d, np.float64) * D  # the walls cap radii the same way
    draw = np.minimum(draw, np.minimum(pos, box - pos).min(axis=-1) * (1.0 + eps))
    r = np.full((nx, ny, nz), np.nan)
    hi = np.array([nx - 1, ny - 1, nz - 1])
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)
            if (a, b, c) != (0, 0, 0)]
    for col in range(8):
        sl = (slice(col & 1, None, 2), slice((col >> 1) & 1, None, 2), slice((col >> 2) & 1, None, 2))
        ri, P, I = draw[sl].copy(), pos[sl], idx[sl]
        for o in offs:
            J = I + np.array(o)
            ok = np.all((J >= 0) & (J <= hi), axis=-1)
            Jc = np.clip(J, 0, hi)
            rj = r[Jc[..., 0], Jc[..., 1], Jc[..., 2]]
            dij = np.linalg.norm(pos[Jc[..., 0], Jc[..., 1], Jc[..., 2]] - P, axis=-1)
            use = ok & ~np.isnan(rj)
            ri = np.minimum(ri, np.where(use, (dij - np.where(use, rj, 0.0)) * (1.0 + eps), np.inf))
        r[sl] = ri
    pos, radius = _shuffle(rng, pos.reshape(-1, 3), r.ravel())
    p = (params or SimParams()).replace(box_lo=(0.0, 0.0, 0.0),
                                        box_hi=tuple(float(b * D) for b in box_d))
    return make_scene(name, p, pos, radius=radius,
                      meta=dict(kind="poly_bed", spacing=spacing, jitter=jitter, nxyz=nxyz,
                                seed=seed, r_range=r_range))


def C5(params: SimParams | None = None, rank: int = 0, scale: int = 1) -> Scene:
    """2M particles per GPU, polydisperse r ~ U[0.25, 0.5] mm (capped, see
    poly_bed), K = 32; bench.py compacts it before timing."""
    nx = 512 // scale
    p = (params or SimParams()).replace(max_contacts=32)
    box = (int(math.ceil(nx * 0.75)) + 2, 50, 50)
    return poly_bed("C5" if scale == 1 else f"C5/{scale}", (nx, 64, 64), box,
                    seed=5 + rank, params=p)


CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5}


# ------------------------------------------------- small scenes for pins ----

def random_gas(n: int, box_d: float, seed: int, r_range=(0.4 * D, 0.6 * D), v_sigma=0.1,
               w_sigma=20.0, params: SimParams | None = None, margin: float = 0.0) -> Scene:
    """Uniform random centres (overlaps allowed) with polydisperse radii."""
    rng = np.random.default_rng(seed)
    L = box_d * D
    pos = rng.uniform(margin * D, L - margin * D, (n, 3))
    radius = rng.uniform(r_range[0], r_range[1], n)
    vel = rng.normal(0.0, v_sigma, (n, 3))
    omg = rng.normal(0.0, w_sigma, (n, 3))
    p = (params or SimParams()).replace(box_lo=(0.0, 0.0, 0.0), box_hi=(L, L, L))
    return make_scene(f"gas{n}", p, pos, vel, omg, radius=radius, meta=dict(seed=seed))


def flag_gas(clamp_fn: bool = False, truncate_dt: bool = False, seed: int = 21) -> Scene:
    """A fast, spinning, overlapping gas with strong damping, low friction and
    C_t = 2.5 C_n: many contacts hit the Eq. 5 cap (so DEM_F_TRUNCATE_DT
    rewrites δ_t) and many separate with a tensile F_n (so DEM_F_CLAMP_FN
    zeroes it). For the flag parity tests."""
    sp = SimParams(max_contacts=32, stiffness_t=2.5 * 7.326e6, damping=0.8, friction=0.2,
                   clamp_fn=clamp_fn, truncate_dt=truncate_dt)
    return random_gas(3000, 14.0, seed, r_range=(0.3 * D, 0.5 * D), v_sigma=0.4, w_sigma=200.0,
                      params=sp)


def two_body(v0: float, params: SimParams, gap: float = 1e-6, box_d: float = 8.0) -> Scene:
    """Head-on pair along x approaching at relative speed v0 (no gravity)."""
    L = box_d * D
    c = 0.5 * L
    x0 = c - R - 0.5 * gap
    x1 = c + R + 0.5 * gap
    pos = [[x0, c, c], [x1, c, c]]
    vel = [[0.5 * v0, 0, 0], [-0.5 * v0, 0, 0]]
    p = params.replace(gravity=(0.0, 0.0, 0.0), box_lo=(0.0, 0.0, 0.0), box_hi=(L, L, L))
    return make_scene("two_body", p, pos, vel)


def stack(n: int, params: SimParams, gap: float = 0.0) -> Scene:
    """n equal spheres in a vertical column on the floor (y up)."""
    L = 6 * D
    H = (n + 3) * D
    ys = R + np.arange(n) * (D + gap)
    pos = np.stack([np.full(n, 0.5 * L), ys, np.full(n, 0.5 * L)], axis=1)
    p = params.replace(box_lo=(0.0, 0.0, 0.0), box_hi=(L, H, L))
    return make_scene(f"stack{n}", p, pos)


# ---------------------------------------------------------------- materials --

def material_table(M: int, seed: int = 0, walls: bool = True):
    """A symmetric (M, M, 4) table of (C_n, C_t, alpha, mu) around the R19
    defaults (C x [0.5, 2], alpha in [0.1, 0.5], mu in [0.2, 0.8]) and an
    (M, 4) particle-wall table, as nested tuples (SimParams fields)."""
    rng = np.random.default_rng(seed)
    t = np.empty((M, M, 4))
    for i in range(M):
        for j in range(i, M):
            c = (7.326e6 * rng.uniform(0.5, 2.0), 7.326e6 * rng.uniform(0.5, 2.0),
                 rng.uniform(0.1, 0.5), rng.uniform(0.2, 0.8))
            t[i, j] = t[j, i] = c
    w = np.stack([(7.326e6 * rng.uniform(0.5, 2.0), 7.326e6 * rng.uniform(0.5, 2.0),
                   rng.uniform(0.1, 0.5), rng.uniform(0.2, 0.8)) for _ in range(M)])
    def tup(a):
        return tuple(tup(b) for b in a) if a.ndim > 1 else tuple(float(x) for x in a)

    return tup(t), (tup(w) if walls else None)


def mixed_gas(n: int, box_d: float, seed: int, M: int = 3, **kw) -> Scene:
    """random_gas with M materials: random per-particle material ids and a
    random symmetric pair table (material_table)."""
    mats, walls = material_table(M, seed)
    params = kw.pop("params", None) or SimParams()
    sc = random_gas(n, box_d, seed, params=params.replace(materials=mats, wall_materials=walls),
                    **kw)
    sc.material = np.random.default_rng(seed + 1000).integers(0, M, n).astype(np.uint32)
    sc.name = f"mixed{n}x{M}"
    return sc


# ------------------------------------------------------------------ plates --

def plate(centre, normal, u, half_u: float, half_v: float) -> tuple:
    """A finite two-sided rectangular wall (reading R23): centre, unit normal,
    unit in-plane axis u, half-lengths along u and v = normal x u."""
    n = np.asarray(normal, np.float64)
    uu = np.asarray(u, np.float64)
    assert abs(np.linalg.norm(n) - 1) < 1e-6 and abs(np.linalg.norm(uu) - 1) < 1e-6
    assert abs(n @ uu) < 1e-6 and half_u > 0 and half_v > 0
    return tuple(float(x) for x in (*centre, *normal, *u, half_u, half_v, 0.0))


def slit_box(nxyz: tuple = (64, 32, 64), seed: int = 6, slit_d: float = 6.0,
             params: SimParams | None = None) -> Scene:
    """The paper's §5 experiment: equal spheres falling from a
    box through a slit at its bottom onto the floor. The paper gives no
    dimensions; this geometry is a stated choice: a simple-cubic
    block of nx*ny*nz spheres (spacing 1.02 d, jitter ±0.01 d horizontally, the bottom
    layer resting on the box bottom) in an
    open-topped box whose bottom, 40 d above the floor, has a slit of slit_d
    diameters along x through its middle; box and bottom are plates (R23), the
    floor and the outer walls are the domain faces. nxyz = (64, 32, 64) gives
    the paper's 2^17 = 131,072 particles."""
    nx, ny, nz = nxyz
    sp_ = 1.02 * D
    rng = np.random.default_rng(seed)
    W_x, W_z = nx * sp_ + 2 * D, nz * sp_ + 2 * D  # inner box widths
    H_box = ny * sp_ + 8 * D                        # box wall height
    y_b = 40 * D                                    # box bottom
    Lx, Lz = W_x + 40 * D, W_z + 40 * D
    Ly = y_b + H_box + 10 * D
    x0, z0 = 0.5 * (Lx - W_x), 0.5 * (Lz - W_z)
    zc = z0 + 0.5 * W_z
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    pos = np.stack([x0 + D + (i.ravel() + 0.5) * sp_,
                    y_b + R - 0.002 * D + j.ravel() * sp_,
                    z0 + D + (k.ravel() + 0.5) * sp_], axis=1)
    pos = pos + rng.uniform(-0.01 * D, 0.01 * D, pos.shape) * np.array([1.0, 0.1, 1.0])
    half_slit = 0.5 * slit_d * D
    hb = 0.5 * (0.5 * W_z - half_slit)  # half-width of each bottom plate along z
    plates = (
        # bottom, either side of the slit (normal +y, u = x)
        plate((x0 + 0.5 * W_x, y_b, z0 + hb), (0, 1, 0), (1, 0, 0), 0.5 * W_x, hb),
        plate((x0 + 0.5 * W_x, y_b, zc + half_slit + hb), (0, 1, 0), (1, 0, 0), 0.5 * W_x, hb),
        # sides (normal +-x and +-z), from the bottom up
        plate((x0, y_b + 0.5 * H_box, zc), (1, 0, 0), (0, 1, 0), 0.5 * H_box, 0.5 * W_z),
        plate((x0 + W_x, y_b + 0.5 * H_box, zc), (1, 0, 0), (0, 1, 0), 0.5 * H_box, 0.5 * W_z),
        plate((x0 + 0.5 * W_x, y_b + 0.5 * H_box, z0), (0, 0, 1), (1, 0, 0), 0.5 * W_x, 0.5 * H_box),
        plate((x0 + 0.5 * W_x, y_b + 0.5 * H_box, z0 + W_z), (0, 0, 1), (1, 0, 0), 0.5 * W_x,
              0.5 * H_box),
    )
    p = (params or SimParams()).replace(box_lo=(0.0, 0.0, 0.0), box_hi=(Lx, Ly, Lz),
                                        plates=plates)
    n = pos.shape[0]
    return make_scene(f"slit{n}", p, pos, meta=dict(kind="slit", nxyz=nxyz, slit_d=slit_d,
                                                   y_bottom=y_b, seed=seed))
