"""ctypes binding of ``libtsmpc.so`` (C ABI declared in ``include/tsmpc.h``).

The shared library is built in-tree by :func:`build_library` (nvcc, sm_100a)
and loaded from this package directory.  There is deliberately no fallback: if
the library or a CUDA device is missing, every solver entry point raises
:class:`~.errors.DeviceError`.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess
import threading
import weakref

import numpy as np

from .errors import DeviceError, DimensionError, TreeSmpcError, ValidationError

PKG_DIR = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libtsmpc.so"
CSRC = PKG_DIR / "csrc"
SOURCES = ["tsmpc_apg.cu", "tsmpc_sparse.cu", "tsmpc_sparse_host.cu", "tsmpc_nccl.cu", "tsmpc_cache.cu",
           "tsmpc_aux.cu", "tsmpc_capi.cu"]

OK, ERR_DIMENSION, ERR_VALIDATION, ERR_CUDA, ERR_NCCL, ERR_ARGUMENT = 0, -1, -2, -3, -4, -5
RECORD_RESIDUALS, SKIP_GAP, KEEP_DEVICE, WARM_DEVICE, GAP_TRACE = 1, 2, 4, 8, 16

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


class Problem(ctypes.Structure):
    _fields_ = [
        ("n_x", ctypes.c_int32), ("n_u", ctypes.c_int32), ("n_v", ctypes.c_int32),
        ("n_d", ctypes.c_int32), ("n_e", ctypes.c_int32), ("N", ctypes.c_int32),
        ("n_nodes", ctypes.c_int32),
        ("A", _dp), ("B", _dp), ("L", _dp), ("Bbar", _dp), ("Phi", _dp), ("Psi", _dp),
        ("Wu", _dp), ("E", _dp), ("E_pinvT", _dp),
        ("u_min", _dp), ("u_max", _dp), ("x_min", _dp), ("x_max", _dp), ("x_s", _dp),
        ("W_alpha", ctypes.c_double), ("Wx", ctypes.c_double), ("gamma_d", ctypes.c_double),
        ("sig_stage", _dp), ("zeta_stage", _dp), ("psi_stage", _dp),
        ("stage_starts", _ip), ("anc", _ip), ("child_start", _ip), ("child_stop", _ip),
        ("prob", _dp),
        ("Ls", _dp), ("lam_s", _dp), ("Ms", _dp),
    ]


class Result(ctypes.Structure):
    _fields_ = [
        ("u0", _dp), ("x", _dp), ("u", _dp), ("x_avg", _dp), ("u_avg", _dp),
        ("dual_sig", _dp), ("dual_zeta", _dp), ("dual_psi", _dp), ("resid_trace", _dp),
        ("residual_inf", ctypes.c_double), ("gap", ctypes.c_double),
        ("device_ms", ctypes.c_double), ("iterations", ctypes.c_int32),
        ("device_total_ms", ctypes.c_double), ("kernel_launches", ctypes.c_int64),
        ("gap_trace", _dp),
    ]


# name -> (restype, argtypes); the exported symbol set of include/tsmpc.h
SIGNATURES = {
    "tsmpc_plan_create": (ctypes.c_void_p, [ctypes.POINTER(Problem), ctypes.c_int]),
    "tsmpc_plan_destroy": (None, [ctypes.c_void_p]),
    "tsmpc_set_cache": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
    "tsmpc_solve": (ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.c_int32, ctypes.c_double,
                                   _dp, _dp, _dp, _dp, _dp, ctypes.c_int32,
                                   ctypes.POINTER(Result)]),
    "tsmpc_solve_step": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp]),
    "tsmpc_prox": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, _dp, _dp, _dp,
                                  ctypes.c_double, ctypes.c_int32, _dp, _dp, _dp]),
    "tsmpc_dual_operator_begin": (ctypes.c_int, [ctypes.c_void_p, _dp]),
    "tsmpc_dual_operator_set_ones": (ctypes.c_int, [ctypes.c_void_p]),
    "tsmpc_dual_operator_step": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp]),
    "tsmpc_plan_info": (ctypes.c_int, [ctypes.c_void_p, _ip, ctypes.c_int32]),
    "tsmpc_last_error": (ctypes.c_char_p, []),
    "tsmpc_plan_path": (ctypes.c_char_p, [ctypes.c_void_p]),
    "tsmpc_set_stopping": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int32]),
    "tsmpc_plan_trial": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]),
    "tsmpc_plans_create_multi": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.POINTER(ctypes.c_int32),
                                                ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "tsmpc_solve_multi": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, _dp, ctypes.c_int32,
                                         ctypes.c_double, _dp, _dp, ctypes.c_int32, ctypes.POINTER(Result)]),
    "tsmpc_set_cache_operators": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, _dp, _dp, _dp, _dp, _dp,
                                                 _dp]),
    "tsmpc_set_forecast": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, _dp]),
    "tsmpc_get_cache": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp]),
    "tsmpc_nccl_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8)]),
    "tsmpc_plan_peer_handles": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint8)]),
    "tsmpc_plan_peer_open": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint8), ctypes.c_int32]),
    "tsmpc_plan_peer_close": (ctypes.c_int, [ctypes.c_void_p]),
    "tsmpc_plan_create_shard": (ctypes.c_void_p, [ctypes.POINTER(Problem), ctypes.c_int, ctypes.c_int32,
                                                  ctypes.c_int32, ctypes.POINTER(ctypes.c_uint8)]),
    "tsmpc_solve_group": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, _dp, ctypes.c_int32,
                                         ctypes.c_double, _dp, _dp, ctypes.c_int32, ctypes.POINTER(Result)]),
    "tsmpc_plan_edges": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, _ip, ctypes.c_int64]),
    "tsmpc_describe_shard": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.c_int32, ctypes.c_int64,
                                            ctypes.c_int32, ctypes.c_int32, _ip, ctypes.c_int32, _ip,
                                            ctypes.c_int64]),
    "tsmpc_describe_sparse": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.c_int32, ctypes.c_int64,
                                             _ip, ctypes.c_int32]),
    "tsmpc_device_count": (ctypes.c_int, []),
    "tsmpc_host_alloc": (ctypes.c_void_p, [ctypes.c_int64]),
    "tsmpc_host_free": (None, [ctypes.c_void_p]),
    "tsmpc_debug_timers": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                                          ctypes.c_int32]),
    "tsmpc_describe_tree": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.c_int32, ctypes.c_int32,
                                           _ip, ctypes.c_int32]),
}

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-ldl"]


def _compile(srcs, out: pathlib.Path, extra=()) -> None:
    """nvcc each translation unit to an object in parallel (build/ next to csrc),
    then link the shared library."""
    import concurrent.futures as cf
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = CSRC.parent / "build" / out.stem
    objdir.mkdir(parents=True, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f not in ("-shared", "-ldl")]

    def one(src):
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc, *cflags, *extra, "-c", "-o", str(obj), str(src)]
        res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if res.returncode != 0:
            raise DeviceError(f"nvcc failed ({' '.join(cmd)}):\n{res.stderr[-4000:]}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(one, srcs))
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(out),
           *map(str, objs), "-ldl"]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        raise DeviceError(f"nvcc link failed ({' '.join(cmd)}):\n{res.stderr[-4000:]}")


def build_variant(name: str, defines: list[str]) -> pathlib.Path:
    """A-B experiment build: libtsmpc_<name>.so with extra -D defines (tools/ab_variants.sh)."""
    out = PKG_DIR / f"libtsmpc_{name}.so"
    _compile([CSRC / s for s in SOURCES], out, tuple(f"-D{d}" for d in defines))
    return out


def build_library(force: bool = False, verbose: bool = False, timers: bool = False) -> pathlib.Path:
    """Compile ``libtsmpc.so`` in-tree for sm_100a (cross-compiles without a GPU).

    ``timers=True`` builds the phase-timer profiling variant ``libtsmpc_timers.so``
    (load it with ``TSMPC_LIB=.../libtsmpc_timers.so``).
    """
    srcs = [CSRC / s for s in SOURCES]
    if timers:
        out = PKG_DIR / "libtsmpc_timers.so"
        _compile(srcs, out, ("-DTSMPC_TIMERS",))
        return out
    deps = srcs + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [PKG_DIR.parent / "include" / "tsmpc.h"]
    if not force and LIB_PATH.exists():
        newest = max(p.stat().st_mtime for p in deps)
        if LIB_PATH.stat().st_mtime >= newest:
            return LIB_PATH
    _compile(srcs, LIB_PATH)
    return LIB_PATH


_LIB = None


def load_library() -> ctypes.CDLL:
    """Load (never silently skip) the native library and bind its signatures."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = pathlib.Path(os.environ.get("TSMPC_LIB", str(LIB_PATH)))
    if not path.exists():
        raise DeviceError(f"{path} is missing: run __graft_entry__.build() "
                          "(or paper_1604_01074_b200._native.build_library())")
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def last_error() -> str:
    msg = load_library().tsmpc_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == ERR_VALIDATION:
        raise ValidationError(msg)
    if rc in (ERR_CUDA, ERR_NCCL):
        raise DeviceError(msg)
    raise TreeSmpcError(msg)


def device_count() -> int:
    return int(load_library().tsmpc_device_count())


class _PinnedPool:
    """Reusable page-locked blocks (``tsmpc_host_alloc``) backing result arrays.

    A block returns to the pool when the last array viewing it is collected, so
    steady-state solves reuse the same few blocks and their device->host copies
    run at DMA speed (pageable destinations go through the driver's bounce
    buffer at a fraction of that).  At most ``keep`` bytes are kept idle.
    """

    def __init__(self, keep: int = 1 << 30):
        self.keep = keep
        self._free: dict[int, list[int]] = {}
        self._idle = 0
        self._lock = threading.Lock()
        self.disabled = bool(os.environ.get("TSMPC_PAGEABLE"))

    def arrays(self, shapes) -> list[np.ndarray] | None:
        """float64 arrays of the given shapes in one pinned block (None if
        page-locked memory is unavailable)."""
        if self.disabled:
            return None
        sizes = [int(np.prod(sh)) * 8 for sh in shapes]
        offs, total = [], 0
        for n in sizes:
            offs.append(total)
            total += (n + 127) // 128 * 128
        total = max(total, 128)
        with self._lock:
            lst = self._free.get(total)
            ptr = lst.pop() if lst else None
            if ptr is not None:
                self._idle -= total
        if ptr is None:
            ptr = load_library().tsmpc_host_alloc(total)
            if not ptr:
                self.disabled = True  # no device / no page-locked memory: pageable arrays
                return None
        buf = (ctypes.c_char * total).from_address(ptr)
        weakref.finalize(buf, self._release, ptr, total).atexit = False
        return [np.frombuffer(buf, dtype=np.float64, count=n // 8, offset=o).reshape(sh)
                if n else np.empty(sh) for sh, n, o in zip(shapes, sizes, offs)]

    def _release(self, ptr: int, nbytes: int) -> None:
        with self._lock:
            if self._idle + nbytes <= self.keep:
                self._free.setdefault(nbytes, []).append(ptr)
                self._idle += nbytes
                return
        load_library().tsmpc_host_free(ptr)


PINNED = _PinnedPool()


def dptr(a) -> "ctypes._Pointer | None":
    """float64 C-contiguous pointer (None passes NULL)."""
    if a is None:
        return None
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise TypeError("expected a C-contiguous float64 array")
    return a.ctypes.data_as(_dp)


def iptr(a):
    if not (isinstance(a, np.ndarray) and a.dtype == np.int64 and a.flags.c_contiguous):
        raise TypeError("expected a C-contiguous int64 array")
    return a.ctypes.data_as(_ip)
