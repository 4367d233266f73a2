"""ctypes binding of libdem.so (include/dem.h) — argument marshalling only.

Every step of the DEM timestep runs in the CUDA kernels of libdem.so; this
module converts Python/NumPy/torch arguments into the C ABI's plain pointers
and sizes and turns error codes into exceptions. There is no CPU fallback: if
libdem.so is missing or no CUDA device is present, creating a ``Dem`` raises.

Names mirror the C ABI: ``dem_create`` -> ``Dem(...)`` (also ``dem_create``),
``dem_set_particles`` -> ``Dem.set_particles`` (also ``dem_set_particles(h,..)``),
and so on.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DEM_LIB") or os.path.join(HERE, "libdem.so")
# the ablation kernels (the paper's fused thread-per-particle mapping, half
# lists, one lane per particle) live in a second build of the same sources
ABLATIONS_PATH = os.environ.get("DEM_LIB_ABLATIONS") or os.path.join(HERE, "libdem_ablations.so")

DEM_ABI_VERSION = 4
DEM_OK, DEM_EINVAL, DEM_EABI, DEM_ENOMEM, DEM_ECUDA, DEM_ENCCL = 0, -1, -2, -3, -4, -5
DEM_EOVERFLOW, DEM_ENONFINITE, DEM_EESCAPED, DEM_ECOINCIDENT, DEM_ESTATE = -6, -7, -8, -9, -10
DEM_EPEER = -11
DEM_MODEL_PRACTICAL, DEM_MODEL_SIMPLE = 0, 1
DEM_F_TRUNCATE_DT, DEM_F_CLAMP_FN, DEM_F_DIAG, DEM_F_ASYNC, DEM_F_NO_GRAPH = 1, 2, 4, 8, 16
DEM_F_THREAD_PER_PARTICLE = 32
DEM_F_HALF_LISTS = 64
DEM_F_FORCE_DENSE = 128
DEM_F_FORCE_LIGHT = 256
DEM_F_GENERAL_DETECT = 512
DEM_F_FULL_SORT = 1024
DEM_F_FORCE_LANES = 2048
DEM_F_FORCE_WS = 4096
DEM_F_SPLIT_SWEEP = 8192
DEM_MEM_HOST, DEM_MEM_DEVICE = 0, 1
DEM_ORDER_INTERNAL, DEM_ORDER_ID = 0, 1
KERNELS = ("hash", "scan", "scatter", "rank", "sweep", "other", "detect", "finish")
WALL_PID0 = 0xFFFFFFF0

_f = C.c_float
_F3 = _f * 3


class DemAllocator(C.Structure):
    _fields_ = [("ctx", C.c_void_p),
                ("alloc", C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)),
                ("free", C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p))]


class DemParams(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("model", C.c_int32), ("dt", _f), ("gravity", _F3),
                ("box_lo", _F3), ("box_hi", _F3), ("radius", _f), ("density", _f),
                ("stiffness_n", _f), ("stiffness_t", _f), ("damping", _f), ("friction", _f),
                ("wall_stiffness_n", _f), ("wall_stiffness_t", _f), ("wall_damping", _f),
                ("wall_friction", _f), ("k_sp", _f), ("k_da", _f), ("k_sh", _f),
                ("cell_edge", _f), ("max_contacts", C.c_uint32), ("flags", C.c_uint32),
                ("device", C.c_int32), ("stream", C.c_void_p),
                ("allocator", C.POINTER(DemAllocator)), ("rank", C.c_int32),
                ("world_size", C.c_int32),
                ("n_materials", C.c_uint32), ("material_pairs", C.c_void_p),
                ("material_walls", C.c_void_p), ("n_plates", C.c_uint32),
                ("plates", C.c_void_p)]


class DemParticles(C.Structure):
    _fields_ = [("mem_kind", C.c_int32), ("pos", C.c_void_p), ("vel", C.c_void_p),
                ("omega", C.c_void_p), ("radius", C.c_void_p), ("mass", C.c_void_p),
                ("id", C.c_void_p), ("force", C.c_void_p), ("torque", C.c_void_p),
                ("material", C.c_void_p)]


class DemStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("ncells", C.c_int64), ("dims", C.c_int32 * 3),
                ("cell_edge", C.c_double), ("steps", C.c_int64), ("contacts", C.c_int64),
                ("max_contacts_seen", C.c_int64), ("launches", C.c_int64),
                ("graph_launches", C.c_int64), ("kernel_ms", C.c_double * 8),
                ("kernel_count", C.c_int64 * 8), ("force_cfg", C.c_int32),
                ("full_sorts", C.c_int32), ("max_speed", C.c_double),
                ("fused_sweep", C.c_int32), ("reserved", C.c_int32)]


class DemAnalysis(C.Structure):
    _fields_ = [("n", C.c_int64), ("candidates", C.c_int64), ("max_candidates", C.c_int64),
                ("contacts", C.c_int64), ("max_contacts", C.c_int64),
                ("warp_candidate_slots", C.c_int64), ("warp_contact_slots", C.c_int64),
                ("max_per_cell", C.c_int64), ("occupied_cells", C.c_int64),
                ("contact_hist", C.c_int64 * 33), ("movers", C.c_int64)]


class DemError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str):
        super().__init__(f"{where}: {detail} (code {code})")
        self.code = code


_libs = {}


def lib(path: str = LIB_PATH) -> C.CDLL:
    """Load libdem.so (or the ablation build); raise loudly if it has not been built."""
    if path not in _libs:
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with "
                              "`python -m paper_1301_1714_b200.build` (nvcc, sm_100a)")
        L = C.CDLL(path)
        P, I64, I32, VP = C.c_void_p, C.c_int64, C.c_int32, C.c_void_p
        L.dem_create.argtypes = [C.POINTER(DemParams), C.POINTER(VP)]
        L.dem_destroy.argtypes = [VP]
        L.dem_set_particles.argtypes = [VP, I64, C.POINTER(DemParticles)]
        L.dem_set_contacts.argtypes = [VP, I32, I64, P, P, P]
        L.dem_step.argtypes = [VP, I64]
        L.dem_sync.argtypes = [VP]
        L.dem_get_state.argtypes = [VP, I32, I64, C.POINTER(DemParticles), C.POINTER(I64)]
        L.dem_get_contacts.argtypes = [VP, I32, I64, P, P, P, C.POINTER(I64)]
        L.dem_get_grid.argtypes = [VP, I64, P, P, P, C.POINTER(I64)]
        L.dem_get_stats.argtypes = [VP, C.POINTER(DemStats)]
        L.dem_profile.argtypes = [VP, I32]
        L.dem_analyze.argtypes = [VP, C.POINTER(DemAnalysis)]
        L.dem_exchange_handle.argtypes = [VP, P]
        L.dem_exchange_ptr.argtypes = [VP, C.POINTER(VP)]
        L.dem_connect.argtypes = [VP, P, P]
        L.dem_connect_ptrs.argtypes = [VP, VP, VP]
        L.dem_strerror.argtypes = [C.c_int]
        L.dem_strerror.restype = C.c_char_p
        L.dem_last_error.argtypes = [VP]
        L.dem_last_error.restype = C.c_char_p
        _libs[path] = L
    return _libs[path]


def _f32(x) -> float:
    return float(np.float32(x))


def params_from(sp, *, flags: int = 0, device: int = -1, stream=None, allocator=None,
                radius: Optional[float] = None, density: float = 2500.0, rank: int = 0,
                world: int = 1) -> DemParams:
    """dem_params from a scenes.SimParams-like object."""
    p = DemParams()
    p.abi_version = DEM_ABI_VERSION
    p.model = DEM_MODEL_PRACTICAL if sp.model == "practical" else DEM_MODEL_SIMPLE
    p.dt = sp.dt
    for a in range(3):
        p.gravity[a] = sp.gravity[a]
        p.box_lo[a] = sp.box_lo[a]
        p.box_hi[a] = sp.box_hi[a]
    p.radius = 0.5e-3 if radius is None else radius
    p.density = density
    p.stiffness_n, p.stiffness_t = sp.stiffness_n, sp.stiffness_t
    p.damping, p.friction = sp.damping, sp.friction
    p.wall_stiffness_n, p.wall_stiffness_t = sp.wall_stiffness_n, sp.wall_stiffness_t
    p.wall_damping, p.wall_friction = sp.wall_damping, sp.wall_friction
    p.k_sp, p.k_da, p.k_sh = sp.k_sp, sp.k_da, sp.k_sh
    p.cell_edge = sp.cell_edge
    p.max_contacts = sp.max_contacts
    p.flags = (flags | (DEM_F_TRUNCATE_DT if sp.truncate_dt else 0)
               | (DEM_F_CLAMP_FN if sp.clamp_fn else 0))
    p.device = device
    p.stream = stream
    p.allocator = allocator
    p.rank, p.world_size = rank, world
    mats = getattr(sp, "materials", None)
    if mats is not None and len(mats) > 1:  # (M, M, 4) C_n, C_t, alpha, mu per pair
        t = np.ascontiguousarray(np.asarray(mats, np.float32))
        p.n_materials = t.shape[0]
        p._mat = t  # kept alive with the struct
        p.material_pairs = t.ctypes.data
        wm = getattr(sp, "wall_materials", None)
        if wm is not None:
            w = np.ascontiguousarray(np.asarray(wm, np.float32))
            p._wmat = w
            p.material_walls = w.ctypes.data
    plates = getattr(sp, "plates", None)
    if plates:  # (n, 12) finite two-sided rectangles (R23)
        a = np.ascontiguousarray(np.asarray(plates, np.float32))
        p.n_plates = a.shape[0]
        p._plates = a
        p.plates = a.ctypes.data
    return p


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Arg:
    """Holds an array alive and exposes its pointer for the ABI."""

    def __init__(self, x, dtype, shape_last=None, device=False):
        self.obj = None
        self.ptr = None
        if x is None:
            return
        if device:
            import torch
            t = x if _is_torch(x) else torch.as_tensor(x)
            want = {np.float32: torch.float32, np.uint32: torch.int32}[dtype]
            if dtype == np.uint32 and t.dtype in (torch.int32, torch.uint32):
                t = t.view(torch.int32) if t.dtype == torch.uint32 else t
            elif t.dtype != want:
                t = t.to(want)
            t = t.contiguous()
            assert t.is_cuda, "device arrays must be CUDA tensors"
            self.obj = t
            self.ptr = t.data_ptr()
        else:
            a = np.ascontiguousarray(np.asarray(x, dtype=dtype))
            self.obj = a
            self.ptr = a.ctypes.data


class Dem:
    """One DEM particle set on one GPU: dem_create / dem_destroy.

    ``torch_allocator=True`` routes device allocations through torch's
    caching allocator and ``stream`` (a torch.cuda.Stream) orders the work on
    it; both are optional plumbing — the kernels are the library's.
    """

    def __init__(self, sp, *, flags: int = 0, device: int = 0, stream=None,
                 torch_allocator: bool = True, radius: Optional[float] = None,
                 density: float = 2500.0, rank: int = 0, world: int = 1):
        ablation = flags & (DEM_F_THREAD_PER_PARTICLE | DEM_F_HALF_LISTS | DEM_F_FORCE_LANES |
                            DEM_F_FORCE_WS)
        L = self.L = lib(ABLATIONS_PATH if ablation else LIB_PATH)
        self._keep = []
        alloc_p = None
        stream_ptr = None
        if stream is not None:
            stream_ptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
            stream_ptr = stream_ptr or None
        if torch_allocator:
            import torch

            dev = device

            def _alloc(ctx, nbytes, st):
                return torch.cuda.caching_allocator_alloc(int(nbytes), dev, st or 0)

            def _free(ctx, ptr, nbytes, st):
                try:
                    torch.cuda.caching_allocator_delete(ptr)
                except Exception:  # interpreter teardown: torch is already gone
                    pass

            A = DemAllocator()
            A.ctx = None
            A.alloc = DemAllocator._fields_[1][1](_alloc)
            A.free = DemAllocator._fields_[2][1](_free)
            self._keep += [A, _alloc, _free]
            alloc_p = C.pointer(A)
        self.params = params_from(sp, flags=flags, device=device, stream=stream_ptr,
                                  allocator=alloc_p, radius=radius, density=density, rank=rank,
                                  world=world)
        self.rank, self.world = rank, world
        self.flags = self.params.flags
        self.nmat = max(1, int(self.params.n_materials))
        h = C.c_void_p()
        rc = L.dem_create(C.byref(self.params), C.byref(h))
        if rc != DEM_OK:
            raise DemError(rc, "dem_create", L.dem_last_error(None).decode())
        self.h = h
        self.n = 0

    # ------------------------------------------------------------------
    def _check(self, rc: int, where: str):
        if rc != DEM_OK:
            raise DemError(rc, where, self.L.dem_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.dem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---------------------------------------------------------- set ----
    def set_particles(self, pos, vel=None, omega=None, radius=None, mass=None, id=None,
                      material=None):
        """dem_set_particles: numpy arrays (host) or CUDA tensors (device). A slab
        rank keeps its own particles of the given set. `material`: per-particle
        material ids (with SimParams.materials)."""
        device = _is_torch(pos) and pos.is_cuda
        n = int(pos.shape[0]) if pos is not None else 0
        args = [_Arg(pos, np.float32, device=device), _Arg(vel, np.float32, device=device),
                _Arg(omega, np.float32, device=device), _Arg(radius, np.float32, device=device),
                _Arg(mass, np.float32, device=device), _Arg(id, np.uint32, device=device)]
        mat = _Arg(material, np.uint32, device=device)
        P = DemParticles(DEM_MEM_DEVICE if device else DEM_MEM_HOST, *(a.ptr for a in args),
                         None, None, mat.ptr)
        self._check(self.L.dem_set_particles(self.h, n, C.byref(P)), "dem_set_particles")
        self.n = n if self.world == 1 else int(self.stats()["n"])

    def set_contacts(self, id_i, id_j, dt3):
        """dem_set_contacts: (id_i, id_j, δ_t) triples (Eq. 7's δ_t,old)."""
        device = _is_torch(id_i) and id_i.is_cuda
        m = int(len(id_i))
        a = _Arg(id_i, np.uint32, device=device)
        b = _Arg(id_j, np.uint32, device=device)
        d = _Arg(dt3, np.float32, device=device)
        self._check(self.L.dem_set_contacts(self.h, DEM_MEM_DEVICE if device else DEM_MEM_HOST,
                                           m, a.ptr, b.ptr, d.ptr), "dem_set_contacts")

    # --------------------------------------------------------- step ----
    def step(self, nsteps: int = 1):
        """dem_step: advance nsteps timesteps."""
        self._check(self.L.dem_step(self.h, int(nsteps)), "dem_step")
        if self.world > 1:
            self.n = int(self.stats()["n"])

    def sync(self):
        self._check(self.L.dem_sync(self.h), "dem_sync")

    def profile(self, enable: bool = True):
        self._check(self.L.dem_profile(self.h, 1 if enable else 0), "dem_profile")

    # -------------------------------------------------------- slabs ----
    def exchange_handle(self) -> bytes:
        """dem_exchange_handle: 64-byte CUDA IPC handle of this rank's exchange region."""
        buf = C.create_string_buffer(64)
        self._check(self.L.dem_exchange_handle(self.h, buf), "dem_exchange_handle")
        return buf.raw

    def exchange_ptr(self) -> int:
        p = C.c_void_p()
        self._check(self.L.dem_exchange_ptr(self.h, C.byref(p)), "dem_exchange_ptr")
        return p.value

    def connect(self, left: Optional[bytes], right: Optional[bytes]):
        """dem_connect: the neighbours' IPC handles (None at the domain ends)."""
        lb = C.create_string_buffer(left, 64) if left else None
        rb = C.create_string_buffer(right, 64) if right else None
        self._check(self.L.dem_connect(self.h, lb, rb), "dem_connect")

    def connect_local(self, left: Optional["Dem"], right: Optional["Dem"]):
        """dem_connect_ptrs: same-process neighbours."""
        self._check(self.L.dem_connect_ptrs(self.h, left.exchange_ptr() if left else None,
                                           right.exchange_ptr() if right else None),
                    "dem_connect_ptrs")

    def connect_group(self, group=None):
        """Exchange IPC handles over torch.distributed (any backend) and connect."""
        from .slabs import neighbour_handles
        self.connect(*neighbour_handles(self.rank, self.world, self.exchange_handle(), group))

    # ---------------------------------------------------------- get ----
    def get_state(self, order: int = DEM_ORDER_INTERNAL, forces: bool = False,
                  out: Optional[dict] = None) -> dict:
        """dem_get_state into host numpy arrays (or the CUDA tensors in `out`)."""
        n = self.n
        if out is None:
            out = dict(pos=np.empty((n, 3), np.float32), vel=np.empty((n, 3), np.float32),
                       omega=np.empty((n, 3), np.float32), radius=np.empty(n, np.float32),
                       mass=np.empty(n, np.float32), id=np.empty(n, np.uint32))
            if forces:
                out["force"] = np.empty((n, 3), np.float32)
                out["torque"] = np.empty((n, 3), np.float32)
            if self.nmat > 1:
                out["material"] = np.empty(n, np.uint32)
            device = False
        else:
            device = any(_is_torch(v) for v in out.values() if v is not None)

        def ptr(k):
            v = out.get(k)
            if v is None:
                return None
            return v.data_ptr() if device else v.ctypes.data

        P = DemParticles(DEM_MEM_DEVICE if device else DEM_MEM_HOST, ptr("pos"), ptr("vel"),
                         ptr("omega"), ptr("radius"), ptr("mass"), ptr("id"), ptr("force"),
                         ptr("torque"), ptr("material"))
        nout = C.c_int64()
        self._check(self.L.dem_get_state(self.h, order, n, C.byref(P), C.byref(nout)),
                    "dem_get_state")
        return out

    def get_contacts(self, out=None):
        """dem_get_contacts -> (id_i, id_j, dt3) host arrays. With `out` =
        (id_i, id_j, dt3) caller buffers (e.g. pinned) of enough capacity, one
        call fills them and views of the first m entries are returned."""
        m = C.c_int64()
        if out is not None:
            oi, oj, od = out
            cap = min(len(oi), len(oj), len(od))
            rc = self.L.dem_get_contacts(self.h, DEM_MEM_HOST, cap, oi.ctypes.data, oj.ctypes.data,
                                        od.ctypes.data, C.byref(m))
            if rc == DEM_OK:
                k = int(m.value)
                return oi[:k], oj[:k], od[:k]
            if rc != DEM_EINVAL:
                self._check(rc, "dem_get_contacts")
        rc = self.L.dem_get_contacts(self.h, DEM_MEM_HOST, 0, None, None, None, C.byref(m))
        if rc not in (DEM_OK, DEM_EINVAL):
            self._check(rc, "dem_get_contacts")
        cap = int(m.value)
        id_i = np.empty(cap, np.uint32)
        id_j = np.empty(cap, np.uint32)
        dt3 = np.empty((cap, 3), np.float32)
        self._check(self.L.dem_get_contacts(self.h, DEM_MEM_HOST, cap, id_i.ctypes.data,
                                           id_j.ctypes.data, dt3.ctypes.data, C.byref(m)),
                    "dem_get_contacts")
        k = int(m.value)
        return id_i[:k], id_j[:k], dt3[:k]

    def get_grid(self):
        """dem_get_grid -> (key = CM of the current state, perm = SCCM of the
        last sort, off = cell offsets of the last sort)."""
        nc = C.c_int64()
        self._check(self.L.dem_get_grid(self.h, 0, None, None, None, C.byref(nc)), "dem_get_grid")
        ncells = int(nc.value)
        key = np.empty(self.n, np.uint32)
        perm = np.empty(self.n, np.uint32)
        off = np.empty(ncells + 1, np.uint32)
        self._check(self.L.dem_get_grid(self.h, max(self.n, ncells + 1), key.ctypes.data,
                                       perm.ctypes.data, off.ctypes.data, C.byref(nc)),
                    "dem_get_grid")
        return key, perm, off

    def stats(self) -> dict:
        s = DemStats()
        self._check(self.L.dem_get_stats(self.h, C.byref(s)), "dem_get_stats")
        return dict(n=s.n, ncells=s.ncells, dims=tuple(s.dims), cell_edge=s.cell_edge,
                    steps=s.steps, contacts=s.contacts, max_contacts_seen=s.max_contacts_seen,
                    launches=s.launches, graph_launches=s.graph_launches,
                    kernel_ms={k: s.kernel_ms[i] for i, k in enumerate(KERNELS)},
                    kernel_count={k: s.kernel_count[i] for i, k in enumerate(KERNELS)},
                    force_cfg={-1: None, 0: "dense", 1: "light", 2: "lanes", 3: "ws"}[s.force_cfg],
                    full_sorts=s.full_sorts, max_speed=s.max_speed,
                    fused_sweep=bool(s.fused_sweep))


    def analyze(self) -> dict:
        """The paper's §6 quantities for the last step (dem_analyze), raw
        counts plus the ratios the paper argues with."""
        a = DemAnalysis()
        self._check(self.L.dem_analyze(self.h, C.byref(a)), "dem_analyze")
        n = max(a.n, 1)
        return dict(
            n=a.n, candidates=a.candidates, max_candidates=a.max_candidates,
            contacts=a.contacts, max_contacts=a.max_contacts,
            warp_candidate_slots=a.warp_candidate_slots,
            warp_contact_slots=a.warp_contact_slots, max_per_cell=a.max_per_cell,
            occupied_cells=a.occupied_cells, contact_hist=list(a.contact_hist),
            movers=a.movers,
            candidates_mean=a.candidates / n, contacts_mean=a.contacts / n,
            # contacts among candidates: the paper's "about a quarter"
            contact_fraction=a.contacts / max(a.candidates, 1),
            # lane efficiency of the thread-per-particle mapping (SIMT divergence)
            tpp_candidate_lane_efficiency=a.candidates / max(a.warp_candidate_slots, 1),
            tpp_contact_lane_efficiency=a.contacts / max(a.warp_contact_slots, 1))


# C-ABI-named aliases ----------------------------------------------------------
def dem_create(sp, **kw) -> Dem:
    return Dem(sp, **kw)


def dem_destroy(h: Dem):
    h.close()


def dem_set_particles(h: Dem, *a, **kw):
    return h.set_particles(*a, **kw)


def dem_set_contacts(h: Dem, *a, **kw):
    return h.set_contacts(*a, **kw)


def dem_step(h: Dem, nsteps: int = 1):
    return h.step(nsteps)


def dem_get_state(h: Dem, *a, **kw):
    return h.get_state(*a, **kw)


def dem_get_contacts(h: Dem):
    return h.get_contacts()


def dem_get_grid(h: Dem):
    return h.get_grid()


def dem_analyze(h: Dem):
    return h.analyze()


def dem_get_stats(h: Dem):
    return h.stats()


def exported_symbols() -> list[str]:
    """Every function include/dem.h declares (parsed from the header)."""
    import re
    hdr = open(os.path.join(os.path.dirname(HERE), "include", "dem.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(dem_\w+)\(", hdr, re.M)))
