"""Thin ctypes binding of ``include/lbm.h`` (argument marshalling only; every step of the LB
path runs in the CUDA kernels of ``liblbm_b200.so``).

Function names mirror the C ABI (``lbm_create``, ``lbm_init_equilibrium``, ``lbm_step``,
``lbm_get_macroscopic`` ...). :class:`Simulation` is a small convenience wrapper that owns a
handle and accepts numpy arrays (host) or torch CUDA tensors (device).

There is no fallback: if the shared library is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LBM_B200_LIB selects an experiment build variant (same ABI); default: the in-tree library
LIBPATH = os.environ.get("LBM_B200_LIB") or os.path.join(HERE, "liblbm_b200.so")

LBM_OK, LBM_EINVAL, LBM_EUNSUPPORTED, LBM_ECUDA, LBM_ENCCL, LBM_ENAN, LBM_EOOM = 0, -1, -2, -3, -4, -5, -6
D3Q19, D3Q27 = 19, 27
SRT, TRT, MRT, CUMULANT, IDENTITY, SMAGORINSKY, KBC, KBC_EXACT, GEN_SRT, GEN_TRT, GEN_MRT, GEN_SMAGORINSKY = range(12)
F64, F32 = 0, 1
PULL, AA, ESOTWIST, PUSH = 0, 1, 2, 3
FLUID, NOSLIP, UBB = 0, 1, 2
HOST, DEVICE, HOST_ASYNC = 0, 1, 2
HALO_ZEROCOPY, HALO_PACKED, HALO_FUSED = 0, 1, 2
PATH_AUTO, PATH_PLAIN, PATH_STAGED = 0, 1, 2
EQ_COMPRESSIBLE, EQ_INCOMPRESSIBLE, EQ_MOMENT_MATCHED = 0, 1, 2
BOUNDARY_FLAGS, BOUNDARY_LINKS, BOUNDARY_INLINE = 0, 1, 2
BOUNDARY_MODES = {"flags": BOUNDARY_FLAGS, "links": BOUNDARY_LINKS, "inline": BOUNDARY_INLINE}
EQUILIBRIA = {"compressible": EQ_COMPRESSIBLE, "incompressible": EQ_INCOMPRESSIBLE, "moment_matched": EQ_MOMENT_MATCHED}
KERNEL_PATHS = {"auto": PATH_AUTO, "plain": PATH_PLAIN, "staged": PATH_STAGED}

COLLISIONS = {"srt": SRT, "trt": TRT, "mrt": MRT, "cumulant": CUMULANT, "identity": IDENTITY,
              "smagorinsky": SMAGORINSKY, "kbc": KBC, "kbc_exact": KBC_EXACT,
              "gen_srt": GEN_SRT, "gen_trt": GEN_TRT, "gen_mrt": GEN_MRT, "gen_smagorinsky": GEN_SMAGORINSKY}
DTYPES = {"f64": F64, "float64": F64, "fp64": F64, "f32": F32, "float32": F32, "fp32": F32}
PATTERNS = {"pull": PULL, "aa": AA, "esotwist": ESOTWIST, "push": PUSH}


class lbm_config(C.Structure):
    _fields_ = [
        ("stencil", C.c_int32), ("collision", C.c_int32), ("dtype", C.c_int32), ("pattern", C.c_int32),
        ("n_rates", C.c_int32), ("rates", C.c_double * 8), ("force", C.c_double * 3),
        ("global_", C.c_int64 * 3), ("periodic", C.c_int32 * 3), ("flags", C.c_void_p),
        ("ubb_velocity", C.c_double * 3), ("rank", C.c_int32), ("nranks", C.c_int32),
        ("nccl_id", C.c_void_p), ("n_local_slabs", C.c_int32), ("device", C.c_int32),
        ("stream", C.c_void_p), ("halo_mode", C.c_int32), ("use_graph", C.c_int32),
        ("block_x", C.c_int32), ("check_nan_every", C.c_int32), ("nccl_self", C.c_int32),
        ("equilibrium", C.c_int32), ("boundary_mode", C.c_int32),
        ("n_row_rates", C.c_int32), ("row_rates", C.c_double * 15),
        ("pdf_dev", C.c_void_p * 2), ("flags_dev", C.c_void_p), ("halo_dev", C.c_void_p),
    ]


class lbm_kernel_args(C.Structure):
    _fields_ = [
        ("stencil", C.c_int32), ("collision", C.c_int32), ("dtype", C.c_int32),
        ("src", C.c_void_p), ("dst", C.c_void_p), ("flags", C.c_void_p),
        ("shape", C.c_int64 * 3), ("ghost", C.c_int32), ("z_begin", C.c_int64), ("z_end", C.c_int64),
        ("rates", C.c_double * 8), ("force", C.c_double * 3), ("ubb_velocity", C.c_double * 3),
        ("stream", C.c_void_p), ("equilibrium", C.c_int32),
    ]


class LBMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


if not os.path.exists(LIBPATH):
    raise ImportError(f"{LIBPATH} is missing: build it with `python -m paper_2001_11806_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIBPATH)

_P, _I32, _I64, _D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_SIGS = {
    "lbm_config_default": ([C.POINTER(lbm_config)], None),
    "lbm_create": ([C.POINTER(lbm_config), C.POINTER(C.c_void_p)], C.c_int),
    "lbm_destroy": ([_P], C.c_int),
    "lbm_local_extent": ([_P, _P], C.c_int),
    "lbm_init_equilibrium": ([_P, _P, _P, _I32], C.c_int),
    "lbm_init_random": ([_P, C.c_uint64, _D, _D, _I32, _D], C.c_int),
    "lbm_step": ([_P, _I64], C.c_int),
    "lbm_sync": ([_P], C.c_int),
    "lbm_steps_done": ([_P], _I64),
    "lbm_get_macroscopic": ([_P, _P, _P, _I32], C.c_int),
    "lbm_get_populations": ([_P, _P, _I32, _I32], C.c_int),
    "lbm_set_populations": ([_P, _P, _I32, _I32], C.c_int),
    "lbm_pack_face": ([_P, _I64, _I32, _P, _I32], C.c_int),
    "lbm_get_populations_at": ([_P, _P, _I64, _P], C.c_int),
    "lbm_kernel_time_ms": ([_P, _P, _P], C.c_int),
    "lbm_launch_count": ([_P], _I64),
    "lbm_nccl_unique_id": ([_P], C.c_int),
    "lbm_slab_plan": ([_I64, _I32, _I32, _P], C.c_int),
    "lbm_crossing_directions": ([_I32, _I32, _P], C.c_int),
    "lbm_stencil_table": ([_I32, _P, _P], C.c_int),
    "lbm_halo_schedule": ([_I32, _I64, _I32, _I32, _P, _I32], C.c_int),
    "lbm_halo_schedule_phase": ([_I32, _I32, _I64, _I32, _I32, _P, _I32], C.c_int),
    "lbm_kernel_pull": ([C.POINTER(lbm_kernel_args)], C.c_int),
    "lbm_kernel_aa": ([C.POINTER(lbm_kernel_args), _I32], C.c_int),
    "lbm_kernel_push": ([C.POINTER(lbm_kernel_args)], C.c_int),
    "lbm_kernel_collide": ([C.POINTER(lbm_kernel_args)], C.c_int),
    "lbm_prepare_flags": ([_P, _I64, _I64, _I64, _I32, _P, _P], C.c_int),
    "lbm_strerror": ([C.c_int], C.c_char_p),
    "lbm_last_error": ([_P], C.c_char_p),
    "lbm_version": ([], C.c_char_p),
    "lbm_set_kernel_path": ([_I32], C.c_int),
    "lbm_probe_copy": ([_I32, _I32, _I32, _I64, _I64, _I64, _I32, _I32, _P], C.c_int),
    "lbm_boundary_links": ([_P, _P, _P, _P, _I64], _I64),
    "lbm_set_link_velocities": ([_P, _P, _I64], C.c_int),
    "lbm_get_kernel_path": ([], _I32),
    "lbm_buffer_sizes": ([C.POINTER(lbm_config), _P], C.c_int),
    "lbm_step_phases_ms": ([_P, _P], C.c_int),
    "lbm_boundary_impl": ([_P], C.c_int),
    "lbm_detect_faces": ([C.POINTER(lbm_config), _P], C.c_int),
    "lbm_probe_update": ([_I32, _I32, _I32, _I64, _I64, _I64, _I32, _I32, _P], C.c_int),
    "lbm_probe_fma": ([_I32, _I32, _P], C.c_int),
    "lbm_state_bytes": ([_P], _I64),
    "lbm_save_state": ([_P, _P, _I32, _P], C.c_int),
    "lbm_load_state": ([_P, _P, _I32, _I64], C.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res
    globals()[_name] = _fn

EXPORTED = tuple(_SIGS)


def _check(status: int, h=None, what: str = "") -> None:
    if status < 0:
        msg = (lbm_last_error(h) or b"").decode() or lbm_strerror(status).decode()
        raise LBMError(status, f"{what}: {msg}")


def _ptr(a) -> int:
    """Address of a numpy array (host) or a torch tensor (device or host)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    assert a.is_contiguous()
    return a.data_ptr()


def probe_copy(stencil: int, dtype: str, shifted: bool, shape, reps: int = 10, device: int = 0) -> float:
    """Copy-q roofline probe (include/lbm.h lbm_probe_copy): GB/s of the LB memory streams without collision."""
    out = C.c_double()
    nx, ny, nz = shape
    _check(lbm_probe_copy(stencil, DTYPES[dtype], int(shifted), nx, ny, nz, reps, device, C.byref(out)),
           what="lbm_probe_copy")
    return out.value


def probe_update(stencil: int, dtype: str, mode: int, shape, reps: int = 10, device: int = 0) -> float:
    """Update-q (in-place AA streams) roofline probe (include/lbm.h lbm_probe_update): GB/s."""
    out = C.c_double()
    nx, ny, nz = shape
    _check(lbm_probe_update(stencil, DTYPES[dtype], int(mode), nx, ny, nz, reps, device, C.byref(out)),
           what="lbm_probe_update")
    return out.value


def probe_fma(dtype: str, device: int = 0) -> float:
    """FMA-chain ALU ceiling (include/lbm.h lbm_probe_fma): TFLOP/s of DFMA (f64) or FFMA (f32)."""
    out = C.c_double()
    _check(lbm_probe_fma(DTYPES[dtype], device, C.byref(out)), what="lbm_probe_fma")
    return out.value


def set_kernel_path(path) -> None:
    """Bulk kernel path, process-wide: "auto" | "plain" | "staged" (include/lbm.h)."""
    _check(lbm_set_kernel_path(KERNEL_PATHS[path] if isinstance(path, str) else int(path)), what="lbm_set_kernel_path")


def kernel_path() -> str:
    v = int(lbm_get_kernel_path())
    return {b: a for a, b in KERNEL_PATHS.items()}[v]


def slab_plan(nz: int, nranks: int, rank: int):
    out = np.zeros(4, np.int64)
    _check(lbm_slab_plan(nz, nranks, rank, out.ctypes.data), what="lbm_slab_plan")
    return tuple(int(v) for v in out)


def crossing_directions(stencil: int, direction: int):
    out = np.zeros(9, np.int32)
    n = lbm_crossing_directions(stencil, direction, out.ctypes.data)
    _check(n, what="lbm_crossing_directions")
    return out[:n].tolist()


def stencil_table(stencil: int):
    c = np.zeros(3 * stencil, np.int32)
    w = np.zeros(stencil, np.float64)
    _check(lbm_stencil_table(stencil, c.ctypes.data, w.ctypes.data), what="lbm_stencil_table")
    return c.reshape(stencil, 3), w


PHASE_PULL, PHASE_AA_FILL, PHASE_AA_RETURN, PHASE_ESO_AFTER_EVEN, PHASE_ESO_AFTER_ODD = 0, 1, 2, 3, 4


def halo_schedule(stencil: int, nz_local: int, rank: int, nranks: int, phase: int = PHASE_PULL):
    """Zero-copy halo operations of one exchange phase in NCCL posting order: (kind, peer, q, plane)
    with kind 0 = send, 1 = recv, q the slot (plane of the q-th population array); plane 0 /
    nz_local+1 are the ghost planes."""
    out = np.zeros((64, 4), np.int32)
    n = lbm_halo_schedule_phase(stencil, phase, nz_local, rank, nranks, out.ctypes.data, 64)
    _check(n, what="lbm_halo_schedule_phase")
    return [tuple(int(v) for v in r) for r in out[:n]]


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lbm_nccl_unique_id(C.addressof(buf)), what="lbm_nccl_unique_id")
    return bytes(buf)


class Simulation:
    """Owns one lbm handle. ``rates`` follow include/lbm.h; ``flags`` is a host uint8 array of
    shape (nz, ny, nx) for the GLOBAL lattice; ``stream`` is a cudaStream_t (int) or None."""

    def __init__(self, shape: Sequence[int], stencil: int = 19, collision: str = "srt",
                 rates: Sequence[float] = (1.8,), dtype: str = "f64", pattern: str = "pull",
                 force: Sequence[float] = (0.0, 0.0, 0.0), flags: Optional[np.ndarray] = None,
                 ubb_velocity: Sequence[float] = (0.0, 0.0, 0.0), periodic=(1, 1, 1),
                 rank: int = 0, nranks: int = 1, nccl_id: Optional[bytes] = None,
                 n_local_slabs: int = 1, device: int = 0, stream: Optional[int] = None,
                 halo_mode: int = HALO_ZEROCOPY, use_graph: bool = False, block_x: int = 0,
                 check_nan_every: int = 0, nccl_self: bool = False, equilibrium: str = "compressible",
                 boundary_mode: str = "flags", borrow: bool = False):
        """borrow=True: the population arrays, device flag bytes and halo buffer are torch tensors owned by
        this object and lent to the library (lbm_config.pdf_dev / flags_dev / halo_dev, include/lbm.h
        "Ownership"); ``self.buffers`` holds them."""
        cfg = lbm_config()
        lbm_config_default(C.byref(cfg))
        nx, ny, nz = shape
        cfg.stencil = stencil
        cfg.collision = COLLISIONS[collision] if isinstance(collision, str) else collision
        cfg.dtype = DTYPES[dtype] if isinstance(dtype, str) else dtype
        cfg.pattern = PATTERNS[pattern] if isinstance(pattern, str) else pattern
        if len(rates) == 15:  # MRT with one rate per moment
            cfg.n_rates = 0
            cfg.n_row_rates = 15
            for i, r in enumerate(rates):
                cfg.row_rates[i] = r
        else:
            cfg.n_rates = len(rates)
            for i, r in enumerate(rates):
                cfg.rates[i] = r
        for d in range(3):
            cfg.force[d] = force[d]
            cfg.ubb_velocity[d] = ubb_velocity[d]
            cfg.periodic[d] = int(periodic[d])
        cfg.global_[0], cfg.global_[1], cfg.global_[2] = nx, ny, nz
        self._flags = None
        if flags is not None:
            self._flags = np.ascontiguousarray(flags, dtype=np.uint8)
            assert self._flags.shape == (nz, ny, nx)
            cfg.flags = self._flags.ctypes.data
        cfg.rank, cfg.nranks = rank, nranks
        self._id = None
        if nccl_id is not None:
            self._id = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            cfg.nccl_id = C.addressof(self._id)
        cfg.n_local_slabs = n_local_slabs
        cfg.device = device
        cfg.stream = stream
        cfg.halo_mode = halo_mode
        cfg.use_graph = int(use_graph)
        cfg.block_x = block_x
        cfg.check_nan_every = check_nan_every
        cfg.nccl_self = int(nccl_self)
        cfg.equilibrium = EQUILIBRIA[equilibrium] if isinstance(equilibrium, str) else int(equilibrium)
        cfg.boundary_mode = BOUNDARY_MODES[boundary_mode] if isinstance(boundary_mode, str) else int(boundary_mode)
        self.buffers = {}
        if borrow:
            import torch
            sizes = np.zeros(3, np.int64)
            _check(lbm_buffer_sizes(C.byref(cfg), sizes.ctypes.data), None, "lbm_buffer_sizes")
            dev = torch.device("cuda", device)
            narr = 2 if cfg.pattern in (PULL, PUSH) else 1
            for a in range(narr):
                t = torch.empty(int(sizes[0]), dtype=torch.uint8, device=dev)
                self.buffers[f"pdf{a}"] = t
                cfg.pdf_dev[a] = t.data_ptr()
            if sizes[1]:
                self.buffers["flags"] = torch.empty(int(sizes[1]), dtype=torch.uint8, device=dev)
                cfg.flags_dev = self.buffers["flags"].data_ptr()
            if sizes[2]:
                self.buffers["halo"] = torch.empty(int(sizes[2]), dtype=torch.uint8, device=dev)
                cfg.halo_dev = self.buffers["halo"].data_ptr()
        self.cfg = cfg
        self.Q = stencil
        self.device = device
        h = C.c_void_p()
        st = lbm_create(C.byref(cfg), C.byref(h))
        _check(st, None, "lbm_create")
        self.h = h
        ext = np.zeros(4, np.int64)
        _check(lbm_local_extent(self.h, ext.ctypes.data), self.h, "lbm_local_extent")
        self.z0, self.nz_local, self.nx, self.ny = (int(v) for v in ext)
        self.cells = self.nx * self.ny * self.nz_local

    # -- index-list boundaries -------------------------------------------------------
    def boundary_links(self):
        """(cells, dirs, types) of the boundary links (empty in flag mode)."""
        n = int(lbm_boundary_links(self.h, None, None, None, 0))
        _check(n, self.h, "lbm_boundary_links")
        cells, dirs, types = np.zeros(n, np.int64), np.zeros(n, np.int32), np.zeros(n, np.int32)
        if n:
            _check(int(lbm_boundary_links(self.h, cells.ctypes.data, dirs.ctypes.data, types.ctypes.data, n)), self.h,
                   "lbm_boundary_links")
        return cells, dirs, types

    def set_link_velocities(self, uw: np.ndarray) -> None:
        uw = np.ascontiguousarray(uw, np.float64)
        assert uw.ndim == 2 and uw.shape[1] == 3
        _check(lbm_set_link_velocities(self.h, uw.ctypes.data, uw.shape[0]), self.h, "lbm_set_link_velocities")

    # -- lifecycle ------------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            lbm_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- calls ------------------------------------------------------------------------
    def _device_arg(self, t, numel: int, what: str):
        """Validate a torch tensor passed as device memory: CUDA, float64, contiguous, on the handle's
        device, exactly `numel` elements (the C library reads / writes that many doubles)."""
        if not (hasattr(t, "is_cuda") and t.is_cuda):
            raise TypeError(f"{what}: expected a numpy array (host) or a CUDA tensor (device)")
        import torch
        if t.dtype != torch.float64:
            raise TypeError(f"{what}: device tensor must be float64, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{what}: device tensor must be contiguous")
        if t.numel() != numel:
            raise ValueError(f"{what}: device tensor has {t.numel()} elements, expected {numel}")
        if t.device.index != self.device:
            raise ValueError(f"{what}: tensor on cuda:{t.device.index}, handle on cuda:{self.device}")

    def init_equilibrium(self, rho, u):
        where = HOST if isinstance(rho, np.ndarray) else DEVICE
        if where == HOST:
            rho = np.ascontiguousarray(rho, np.float64)
            u = np.ascontiguousarray(u, np.float64)
            assert rho.size == self.cells and u.size == 3 * self.cells
        else:
            self._device_arg(rho, self.cells, "rho")
            self._device_arg(u, 3 * self.cells, "u")
        _check(lbm_init_equilibrium(self.h, _ptr(rho), _ptr(u), where), self.h, "lbm_init_equilibrium")

    def init_random(self, seed: int, rho_amp: float, u_amp: float, profile: int = 0, profile_amp: float = 0.0):
        _check(lbm_init_random(self.h, seed, rho_amp, u_amp, profile, profile_amp), self.h, "lbm_init_random")

    def step(self, n: int = 1):
        _check(lbm_step(self.h, n), self.h, "lbm_step")

    def sync(self):
        _check(lbm_sync(self.h), self.h, "lbm_sync")

    @property
    def steps_done(self) -> int:
        return int(lbm_steps_done(self.h))

    @property
    def launches(self) -> int:
        return int(lbm_launch_count(self.h))

    def macroscopic(self, rho=None, u=None):
        """Returns (rho, u) as numpy (nz, ny, nx) / (3, nz, ny, nx) unless device outputs are given."""
        if rho is None:
            rho = np.empty((self.nz_local, self.ny, self.nx))
            u = np.empty((3, self.nz_local, self.ny, self.nx))
        where = HOST if isinstance(rho, np.ndarray) else DEVICE
        if where == HOST:
            assert rho.dtype == np.float64 and u.dtype == np.float64 and rho.flags["C_CONTIGUOUS"] and u.flags["C_CONTIGUOUS"]
            assert rho.size == self.cells and u.size == 3 * self.cells
        else:
            self._device_arg(rho, self.cells, "rho")
            self._device_arg(u, 3 * self.cells, "u")
        _check(lbm_get_macroscopic(self.h, _ptr(rho), _ptr(u), where), self.h, "lbm_get_macroscopic")
        return rho, u

    def populations(self, raw: bool = False, out=None):
        if out is None:
            out = np.empty((self.Q, self.nz_local, self.ny, self.nx))
        where = HOST if isinstance(out, np.ndarray) else DEVICE
        if where == HOST:
            assert out.dtype == np.float64 and out.flags["C_CONTIGUOUS"] and out.size == self.Q * self.cells
        else:
            self._device_arg(out, self.Q * self.cells, "out")
        _check(lbm_get_populations(self.h, _ptr(out), where, int(raw)), self.h, "lbm_get_populations")
        return out

    def set_populations(self, f, raw: bool = False):
        where = HOST if isinstance(f, np.ndarray) else DEVICE
        if where == HOST:
            f = np.ascontiguousarray(f, np.float64)
            assert f.size == self.Q * self.cells
        else:
            self._device_arg(f, self.Q * self.cells, "f")
        _check(lbm_set_populations(self.h, _ptr(f), where, int(raw)), self.h, "lbm_set_populations")

    def populations_at(self, cells) -> np.ndarray:
        """Canonical populations (Q, n) at local linear cell indices."""
        idx = np.ascontiguousarray(cells, np.int64)
        out = np.empty((self.Q, idx.size))
        _check(lbm_get_populations_at(self.h, idx.ctypes.data, idx.size, out.ctypes.data), self.h,
               "lbm_get_populations_at")
        return out

    def pack_face(self, z: int, direction: int):
        nq = 5 if self.Q == 19 else 9
        out = np.empty(nq * self.nx * self.ny)
        _check(lbm_pack_face(self.h, z, direction, out.ctypes.data, HOST), self.h, "lbm_pack_face")
        return out

    def enable_kernel_timing(self):
        _check(lbm_kernel_time_ms(self.h, None, None), self.h, "lbm_kernel_time_ms")

    @property
    def boundary_impl(self) -> str:
        """What the handle's boundary handling runs: none | split | inline | links | faces | links_fused."""
        v = int(lbm_boundary_impl(self.h))
        _check(v, self.h, "lbm_boundary_impl")
        return ["none", "split", "inline", "links", "faces", "links_fused"][v]

    def step_phases_ms(self):
        """{boundary, exchange, interior}: (begin, end) in ms of the last timed decomposed step."""
        out = np.zeros(6)
        _check(lbm_step_phases_ms(self.h, out.ctypes.data), self.h, "lbm_step_phases_ms")
        return {"boundary": (out[0], out[1]), "exchange": (out[2], out[3]), "interior": (out[4], out[5])}

    def save_state(self):
        """Checkpoint: (host bytes of the stored state incl. ghost planes, step count); bit-exact resume."""
        n = int(lbm_state_bytes(self.h))
        _check(n, self.h, "lbm_state_bytes")
        buf = np.empty(n, np.uint8)
        steps = C.c_int64()
        _check(lbm_save_state(self.h, buf.ctypes.data, HOST, C.byref(steps)), self.h, "lbm_save_state")
        return buf, steps.value

    def load_state(self, buf: np.ndarray, steps: int):
        n = int(lbm_state_bytes(self.h))
        buf = np.ascontiguousarray(buf, np.uint8)
        if buf.size != n:
            raise ValueError(f"state has {buf.size} bytes, this handle needs {n}")
        _check(lbm_load_state(self.h, buf.ctypes.data, HOST, int(steps)), self.h, "lbm_load_state")

    def kernel_time_ms(self):
        ms = C.c_double()
        n = C.c_int64()
        _check(lbm_kernel_time_ms(self.h, C.byref(ms), C.byref(n)), self.h, "lbm_kernel_time_ms")
        return ms.value, n.value
