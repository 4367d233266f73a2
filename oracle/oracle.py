"""ctypes wrapper of the fp64 CPU oracle (TEST INFRASTRUCTURE, not product code).

Every entry point forwards to oracle/dem_oracle.cpp, whose functions cite the
paper passage they follow. Inputs are the fp32 values the GPU sees, upcast
exactly to fp64 (SURVEY §8(c) "Inputs"); parameters are rounded to fp32 first
for the same reason.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

MODEL_PRACTICAL, MODEL_SIMPLE = 0, 1
F_TRUNCATE_DT, F_CLAMP_FN, F_BRUTE = 1, 2, 1 << 16
WALL_PID0 = 0xFFFFFFF0
OK, EINVAL, EOVERFLOW, ENONFINITE, EESCAPED, ECOINCIDENT = 0, -1, -6, -7, -8, -9

_D = C.c_double
_P = C.c_void_p


class OrcParams(C.Structure):
    _fields_ = [("model", C.c_int32), ("flags", C.c_uint32), ("dt", _D), ("g", _D * 3),
                ("lo", _D * 3), ("hi", _D * 3), ("h", _D), ("Cn", _D), ("Ct", _D),
                ("alpha", _D), ("mu", _D), ("wCn", _D), ("wCt", _D), ("walpha", _D),
                ("wmu", _D), ("ksp", _D), ("kda", _D), ("ksh", _D), ("nmat", C.c_int32),
                ("mat", _P), ("wmat", _P), ("nplates", C.c_int32), ("plates", _P)]


class OrcState(C.Structure):
    _fields_ = [("x", _P), ("v", _P), ("w", _P), ("r", _P), ("m", _P), ("id", _P), ("mat", _P)]


class OrcHist(C.Structure):
    _fields_ = [("K", C.c_int32), ("cnt", _P), ("pid", _P), ("dt", _P)]


class OrcOut(C.Structure):
    _fields_ = [("CM", _P), ("SCCM", _P), ("off", _P), ("F", _P), ("T", _P), ("Fabs", _P),
                ("Tabs", _P), ("err", C.c_int64 * 3), ("n_pair_contacts", C.c_int64),
                ("n_wall_contacts", C.c_int64), ("n_candidates", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.build()
        L = C.CDLL(path)
        L.orc_grid_dims.argtypes = [C.POINTER(OrcParams), C.POINTER(C.c_int64)]
        L.orc_hash.argtypes = [C.POINTER(OrcParams), C.c_int64, _P, _P]
        L.orc_sort.argtypes = [C.c_int64, _P, _P, _P]
        L.orc_offsets.argtypes = [C.c_int64, _P, C.c_int64, _P]
        L.orc_neighbor_cells.argtypes = [C.POINTER(OrcParams), C.c_int64, _P]
        L.orc_contacts_brute.argtypes = [C.c_int64, _P, _P, C.c_int64, _P, _P]
        L.orc_contacts_brute.restype = C.c_int64
        L.orc_contacts_grid.argtypes = [C.POINTER(OrcParams), C.c_int64, _P, _P, C.c_int64, _P, _P]
        L.orc_contacts_grid.restype = C.c_int64
        L.orc_stiffness.argtypes = [_D, _D, _D, _D, C.POINTER(_D), C.POINTER(_D)]
        L.orc_damping.argtypes = [_D, _D, _D]
        L.orc_damping.restype = _D
        L.orc_tangential_velocity.argtypes = [_P, _P, _P, _P]
        L.orc_tangential_displacement.argtypes = [_P, _P, _P, _D, _P]
        L.orc_friction_cap.argtypes = [_P, _D, _D]
        L.orc_pair_practical.argtypes = [_P, _D, _D, _D, _P, _P, _P, _D, _D, _D, _D, _D,
                                         C.c_uint32, _P, _P, _P, _P]
        L.orc_pair_simple.argtypes = [_P, _D, _P, _D, _D, _D, _P, _P]
        L.orc_step.argtypes = [C.POINTER(OrcParams), C.c_int64, C.POINTER(OrcState),
                               C.POINTER(OrcHist), C.POINTER(OrcOut)]
        L.orc_step_sampled.argtypes = [C.POINTER(OrcParams), C.c_int64, C.POINTER(OrcState),
                                       C.POINTER(OrcHist), C.POINTER(OrcOut), _P]
        L.orc_run.argtypes = [C.POINTER(OrcParams), C.c_int64, C.POINTER(OrcState),
                              C.POINTER(OrcHist), C.c_int64, C.POINTER(OrcOut)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_P)


def _f32(x) -> float:
    """Parameters are fp32 on the GPU; the oracle uses the same fp32 values."""
    return float(np.float32(x))


def default_cell_edge(radius: np.ndarray) -> float:
    """h = 2 r_max (1 + 2^-10) in fp64 (reading R15); exact for fp32 r_max."""
    rmax = float(np.max(np.asarray(radius, np.float32))) if len(radius) else 0.0
    return 2.0 * rmax * (1.0 + 2.0**-10)


def make_params(sp, radius: np.ndarray | None = None, brute: bool = False) -> OrcParams:
    """Build the oracle's parameter struct from a scenes.SimParams."""
    p = OrcParams()
    p.model = MODEL_PRACTICAL if sp.model == "practical" else MODEL_SIMPLE
    p.flags = ((F_TRUNCATE_DT if sp.truncate_dt else 0) | (F_CLAMP_FN if sp.clamp_fn else 0)
               | (F_BRUTE if brute else 0))
    p.dt = _f32(sp.dt)
    for a in range(3):
        p.g[a] = _f32(sp.gravity[a])
        p.lo[a] = _f32(sp.box_lo[a])
        p.hi[a] = _f32(sp.box_hi[a])
    if sp.cell_edge > 0:
        p.h = _f32(sp.cell_edge)
    else:
        p.h = default_cell_edge(radius)
    p.Cn, p.Ct, p.alpha, p.mu = (_f32(sp.stiffness_n), _f32(sp.stiffness_t), _f32(sp.damping),
                                 _f32(sp.friction))

    def wall(v, dflt):
        return _f32(v) if v >= 0 else dflt

    p.wCn = wall(sp.wall_stiffness_n, p.Cn)
    p.wCt = wall(sp.wall_stiffness_t, p.Ct)
    p.walpha = wall(sp.wall_damping, p.alpha)
    p.wmu = wall(sp.wall_friction, p.mu)
    p.ksp, p.kda, p.ksh = _f32(sp.k_sp), _f32(sp.k_da), _f32(sp.k_sh)
    # material pairs (Eqs. 5, 8-10 as functions of (i, j)): fp32-rounded like
    # every parameter; the arrays are kept alive on the struct
    mats = getattr(sp, "materials", None)
    p.nmat = 1
    if mats is not None and len(mats) > 1:
        t = np.ascontiguousarray(np.asarray(mats, np.float32).astype(np.float64))
        M = t.shape[0]
        assert t.shape == (M, M, 4), "materials: (M, M, 4) of (C_n, C_t, alpha, mu)"
        p.nmat = M
        p._mat = t
        p.mat = _ptr(t)
        wm = getattr(sp, "wall_materials", None)
        if wm is not None:
            w = np.ascontiguousarray(np.asarray(wm, np.float32).astype(np.float64))
            assert w.shape == (M, 4)
            p._wmat = w
            p.wmat = _ptr(w)
    # plates (reading R23): 12 fp32-rounded numbers each
    plates = getattr(sp, "plates", None)
    p.nplates = 0
    if plates:
        a = np.ascontiguousarray(np.asarray(plates, np.float32).astype(np.float64))
        assert a.ndim == 2 and a.shape[1] == 12 and a.shape[0] <= 10
        p.nplates = a.shape[0]
        p._plates = a
        p.plates = _ptr(a)
    return p


def grid_dims(p: OrcParams):
    d = (C.c_int64 * 3)()
    rc = lib().orc_grid_dims(C.byref(p), d)
    if rc != 0:
        raise ValueError("invalid grid (each dimension must be >= 3 cells)")
    return int(d[0]), int(d[1]), int(d[2])


def hash_cells(p: OrcParams, pos) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(pos, np.float64).reshape(-1, 3))
    CM = np.empty(x.shape[0], np.uint32)
    rc = lib().orc_hash(C.byref(p), x.shape[0], _ptr(x), _ptr(CM))
    if rc != 0:
        raise ValueError("invalid grid")
    return CM


def sort_map(CM) -> tuple[np.ndarray, np.ndarray]:
    CM = np.ascontiguousarray(np.asarray(CM, np.uint32))
    SCM = np.empty_like(CM)
    SCCM = np.empty_like(CM)
    lib().orc_sort(CM.shape[0], _ptr(CM), _ptr(SCM), _ptr(SCCM))
    return SCM, SCCM


def cell_offsets(SCM, ncells: int) -> np.ndarray:
    SCM = np.ascontiguousarray(np.asarray(SCM, np.uint32))
    off = np.empty(ncells + 1, np.uint32)
    lib().orc_offsets(SCM.shape[0], _ptr(SCM), ncells, _ptr(off))
    return off


def neighbor_cells(p: OrcParams, cell: int) -> list[int]:
    out = np.empty(27, np.int64)
    k = lib().orc_neighbor_cells(C.byref(p), int(cell), _ptr(out))
    return [int(c) for c in out[:k]]


def _pairs(fn, n, *args):
    cap = max(1024, 16 * n)
    while True:
        pi = np.empty(cap, np.uint32)
        pj = np.empty(cap, np.uint32)
        m = fn(*args, cap, _ptr(pi), _ptr(pj))
        if m >= 0:
            return np.stack([pi[:m], pj[:m]], axis=1)
        if m == -2:
            raise ValueError("invalid grid")
        cap *= 4


def contacts_brute(pos, radius) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(pos, np.float64).reshape(-1, 3))
    r = np.ascontiguousarray(np.asarray(radius, np.float64))
    return _pairs(lib().orc_contacts_brute, x.shape[0], x.shape[0], _ptr(x), _ptr(r))


def contacts_grid(p: OrcParams, pos, radius) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(pos, np.float64).reshape(-1, 3))
    r = np.ascontiguousarray(np.asarray(radius, np.float64))
    return _pairs(lib().orc_contacts_grid, x.shape[0], C.byref(p), x.shape[0], _ptr(x), _ptr(r))


# -------------------------------------------------------- pair pieces ------

def _v(a):
    return np.ascontiguousarray(np.asarray(a, np.float64).reshape(3))


def stiffness(Cn, Ct, delta, Rstar):
    kn, kt = _D(), _D()
    lib().orc_stiffness(Cn, Ct, delta, Rstar, C.byref(kn), C.byref(kt))
    return kn.value, kt.value


def damping(alpha, kn, mstar):
    return lib().orc_damping(alpha, kn, mstar)


def tangential_velocity(v, rw, n):
    v, rw, n = _v(v), _v(rw), _v(n)
    out = np.empty(3)
    lib().orc_tangential_velocity(_ptr(v), _ptr(rw), _ptr(n), _ptr(out))
    return out


def tangential_displacement(dt_old, n, vt, dt):
    a, n, vt = _v(dt_old), _v(n), _v(vt)
    out = np.empty(3)
    lib().orc_tangential_displacement(_ptr(a), _ptr(n), _ptr(vt), dt, _ptr(out))
    return out


def friction_cap(Ft, fn_mag, mu):
    Ft = _v(Ft).copy()
    capped = lib().orc_friction_cap(_ptr(Ft), fn_mag, mu)
    return Ft, bool(capped)


def pair_practical(n, delta, Rstar, mstar, v, rw, dt_old, Cn, Ct, alpha, mu, dt, flags=0):
    n, v, rw, d0 = _v(n), _v(v), _v(rw), _v(dt_old)
    F, Tc, d1 = np.empty(3), np.empty(3), np.empty(3)
    lib().orc_pair_practical(_ptr(n), delta, Rstar, mstar, _ptr(v), _ptr(rw), _ptr(d0), Cn, Ct,
                             alpha, mu, dt, flags, _ptr(F), _ptr(Tc), _ptr(d1), None)
    return F, Tc, d1


def pair_simple(n, delta, u, ksp, kda, ksh):
    n, u = _v(n), _v(u)
    F = np.empty(3)
    lib().orc_pair_simple(_ptr(n), delta, _ptr(u), ksp, kda, ksh, _ptr(F), None)
    return F


# ---------------------------------------------------------------- state ----

@dataclass
class State:
    """Particle properties in fp64, in the current memory order."""
    pos: np.ndarray
    vel: np.ndarray
    omega: np.ndarray
    radius: np.ndarray
    mass: np.ndarray
    id: np.ndarray
    mat: np.ndarray | None = None  # material ids (materials tables), None -> 0

    @property
    def n(self):
        return int(self.pos.shape[0])

    @staticmethod
    def from_arrays(pos, vel, omega, radius, mass, ids, mat=None) -> "State":
        f = lambda a, s: np.array(a, dtype=np.float64, copy=True).reshape(s)  # noqa: E731
        n = np.asarray(pos).reshape(-1, 3).shape[0]
        return State(f(pos, (n, 3)), f(vel, (n, 3)), f(omega, (n, 3)), f(radius, (n,)),
                     f(mass, (n,)), np.array(ids, dtype=np.uint32, copy=True),
                     None if mat is None else np.array(mat, dtype=np.uint32, copy=True))

    @staticmethod
    def from_scene(sc) -> "State":
        return State.from_arrays(sc.pos, sc.vel, sc.omega, sc.radius, sc.mass, sc.id,
                                 getattr(sc, "material", None))

    def copy(self) -> "State":
        return State(*(a.copy() for a in (self.pos, self.vel, self.omega, self.radius, self.mass,
                                          self.id)), None if self.mat is None else self.mat.copy())

    def rounded_fp32(self) -> "State":
        """The state rounded to fp32 and back (the 'x~' shadow of SURVEY T3)."""
        r = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731
        return State(r(self.pos), r(self.vel), r(self.omega), r(self.radius), r(self.mass),
                     self.id.copy(), None if self.mat is None else self.mat.copy())


@dataclass
class History:
    """Per-slot tangential-displacement lists (Eq. 7's δ_t,old), slot-major."""
    cnt: np.ndarray  # (n,) uint32
    pid: np.ndarray  # (n,K) uint32
    dt: np.ndarray  # (n,K,3) float64

    @property
    def K(self):
        return int(self.pid.shape[1])

    @staticmethod
    def empty(n: int, K: int) -> "History":
        return History(np.zeros(n, np.uint32), np.zeros((n, K), np.uint32),
                       np.zeros((n, K, 3), np.float64))

    def copy(self) -> "History":
        return History(self.cnt.copy(), self.pid.copy(), self.dt.copy())

    def as_dict(self, ids: np.ndarray) -> dict:
        """{(id_i, pid_j): δ_t} for comparison with other representations."""
        out = {}
        for s in range(self.cnt.shape[0]):
            for k in range(int(self.cnt[s])):
                out[(int(ids[s]), int(self.pid[s, k]))] = self.dt[s, k].copy()
        return out

    @staticmethod
    def from_pairs(ids: np.ndarray, K: int, id_i, id_j, dt3) -> "History":
        """Build slot lists from (id_i, id_j, δ_t) triples; order within a slot
        follows the triples' order."""
        n = ids.shape[0]
        h = History.empty(n, K)
        id_i = np.asarray(id_i, np.int64)
        if id_i.size == 0:
            return h
        ids64 = ids.astype(np.int64)
        if ids64.max(initial=-1) < n and np.unique(ids64).size == n:
            slot_of = np.empty(n, np.int64)
            slot_of[ids64] = np.arange(n)
            slot = slot_of[id_i]
        else:
            lut = {int(v): s for s, v in enumerate(ids)}
            slot = np.array([lut[int(a)] for a in id_i], np.int64)
        order = np.argsort(slot, kind="stable")
        ss = slot[order]
        k = np.arange(ss.size) - np.searchsorted(ss, ss, side="left")
        if k.max() >= K:
            raise ValueError("more than K history entries for a particle")
        h.pid[ss, k] = np.asarray(id_j, np.uint32)[order]
        h.dt[ss, k] = np.asarray(dt3, np.float64).reshape(-1, 3)[order]
        h.cnt[:] = np.bincount(ss, minlength=n).astype(np.uint32)
        return h


@dataclass
class StepResult:
    rc: int
    CM: np.ndarray
    SCCM: np.ndarray
    off: np.ndarray
    F: np.ndarray
    T: np.ndarray
    Fabs: np.ndarray
    Tabs: np.ndarray
    err: tuple
    n_pair_contacts: int
    n_wall_contacts: int
    n_candidates: int


def _structs(st: State, h: History):
    s = OrcState(_ptr(st.pos), _ptr(st.vel), _ptr(st.omega), _ptr(st.radius), _ptr(st.mass),
                 _ptr(st.id), None if st.mat is None else _ptr(st.mat))
    hh = OrcHist(h.K, _ptr(h.cnt), _ptr(h.pid), _ptr(h.dt))
    return s, hh


def step(p: OrcParams, st: State, h: History, only=None) -> StepResult:
    """One timestep in place: on return st/h hold the new state in sorted order.
    `only`: boolean mask over the NEW sorted slots; when given, only those
    slots are evaluated and advanced (the rest are reordered, not advanced)."""
    n = st.n
    ncells = math.prod(grid_dims(p))
    CM = np.empty(n, np.uint32)
    SCCM = np.empty(n, np.uint32)
    off = np.empty(ncells + 1, np.uint32)
    F = np.empty((n, 3))
    T = np.empty((n, 3))
    Fabs = np.empty(n)
    Tabs = np.empty(n)
    s, hh = _structs(st, h)
    o = OrcOut(_ptr(CM), _ptr(SCCM), _ptr(off), _ptr(F), _ptr(T), _ptr(Fabs), _ptr(Tabs))
    if only is None:
        rc = lib().orc_step(C.byref(p), n, C.byref(s), C.byref(hh), C.byref(o))
    else:
        mask = np.ascontiguousarray(np.asarray(only, dtype=np.uint8))
        assert mask.shape == (n,)
        rc = lib().orc_step_sampled(C.byref(p), n, C.byref(s), C.byref(hh), C.byref(o),
                                    _ptr(mask))
    return StepResult(rc, CM, SCCM, off, F, T, Fabs, Tabs, tuple(o.err), o.n_pair_contacts,
                      o.n_wall_contacts, o.n_candidates)


def run(p: OrcParams, st: State, h: History, nsteps: int):
    """nsteps in place; returns (rc, err, F, T of the last step)."""
    n = st.n
    F = np.empty((n, 3))
    T = np.empty((n, 3))
    s, hh = _structs(st, h)
    o = OrcOut(None, None, None, _ptr(F), _ptr(T), None, None)
    rc = lib().orc_run(C.byref(p), n, C.byref(s), C.byref(hh), nsteps, C.byref(o))
    return rc, tuple(o.err), F, T
