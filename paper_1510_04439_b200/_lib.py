"""ctypes binding of libdfpca_cuda.so (include/dfpca_cuda.h).

The library is built in-tree (paper_1510_04439_b200/build.py).  Loading fails
loudly if it is missing; a context is created lazily on first use and fails
loudly if there is no CUDA device -- the product path has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent


def _point_at_wheel_libs():
    """The library dlopens libnccl / libcusolver by soname (or from
    DFPCA_NCCL_LIB / DFPCA_CUSOLVER_LIB).  In a Python environment they
    usually ship inside the nvidia-* wheels, off the loader path: resolve them
    from the installed packages at run time (a caller's setting wins)."""
    import importlib.util
    for env, pkg, so in (("DFPCA_NCCL_LIB", "nvidia.nccl", "libnccl.so.2"),
                         ("DFPCA_CUSOLVER_LIB", "nvidia.cusolver", "libcusolver.so.11")):
        if os.environ.get(env):
            continue
        try:
            spec = importlib.util.find_spec(pkg)
        except (ImportError, ValueError):
            spec = None
        for d in (spec.submodule_search_locations or []) if spec else []:
            cand = Path(d) / "lib" / so
            if cand.exists():
                os.environ[env] = str(cand)
                break


_point_at_wheel_libs()
LIB_PATH = Path(os.environ.get("DFPCA_CUDA_LIB", _HERE / "libdfpca_cuda.so"))

MAX_DIM = 3


class DfpcaGrid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("shape", C.c_int64 * MAX_DIM),
                ("axes", C.POINTER(C.c_double) * MAX_DIM), ("mask", C.POINTER(C.c_uint8))]


class DfpcaPlan(C.Structure):
    _fields_ = [("n_blocks", C.c_int64), ("blocks_lo", C.POINTER(C.c_int64)),
                ("blocks_hi", C.POINTER(C.c_int64)), ("halo", C.POINTER(C.c_int64))]


# (name, restype, argtypes) -- every symbol declared in include/dfpca_cuda.h
P = C.c_void_p
PD = C.POINTER(C.c_double)
PI64 = C.POINTER(C.c_int64)
SIGNATURES = [
    ("dfpca_context_create", C.c_int, [C.c_int, C.POINTER(P)]),
    ("dfpca_context_destroy", C.c_int, [P]),
    ("dfpca_context_reserve", C.c_int, [P, C.c_uint64]),
    ("dfpca_last_error", C.c_int, [P, C.POINTER(C.c_int), C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]),
    ("dfpca_last_error_location", C.c_int, [P, PI64, PI64]),
    ("dfpca_stage_time", C.c_int, [P, C.c_char_p, PD]),
    ("dfpca_kernel_launches", C.c_int64, [P]),
    ("dfpca_profile_enable", C.c_int, [P, C.c_int]),
    ("dfpca_kernel_stat", C.c_int, [P, C.c_int64, C.POINTER(C.c_char_p), PD, PI64]),
    ("dfpca_host_register", C.c_int, [P, C.c_int64]),
    ("dfpca_host_unregister", C.c_int, [P]),
    ("dfpca_linear_bin", C.c_int, [P, C.POINTER(DfpcaGrid), C.c_int64, PI64, PD, PD, C.c_int, C.c_int,
                                   C.POINTER(P)]),
    ("dfpca_binned_info", C.c_int, [P, PI64, PI64, PI64, PI64, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("dfpca_binned_download", C.c_int, [P, P, PD, PD, PD, PI64, PD, PD, PD, PD, PD, PI64]),
    ("dfpca_binned_upload", C.c_int, [P, C.POINTER(DfpcaGrid), C.c_int64, PI64, C.c_int, PD, PD, PD, C.c_int,
                                      C.c_int64, PI64, PD, PD, PD, PD, PD, C.POINTER(P)]),
    ("dfpca_binned_free", C.c_int, [P]),
    ("dfpca_local_linear", C.c_int, [P, P, C.POINTER(DfpcaGrid), PD, C.c_int, C.POINTER(DfpcaPlan), PD,
                                     C.POINTER(P)]),
    ("dfpca_covariance", C.c_int, [P, P, C.POINTER(DfpcaGrid), PD, PD, C.POINTER(DfpcaPlan), C.POINTER(P)]),
    ("dfpca_pair_grids", C.c_int, [P, P, PD, PD]),
    ("dfpca_surface_info", C.c_int, [P, C.POINTER(C.c_int), PI64]),
    ("dfpca_surface_download", C.c_int, [P, P, PD]),
    ("dfpca_surface_gather", C.c_int, [P, P, C.c_int64, PI64, PD]),
    ("dfpca_surface_upload", C.c_int, [P, C.POINTER(DfpcaGrid), C.c_int, PD, C.c_int64, C.POINTER(P)]),
    ("dfpca_surface_free", C.c_int, [P]),
    ("dfpca_randomized_eig", C.c_int, [P, P, C.POINTER(DfpcaGrid), C.c_int64, C.c_int64, C.c_uint64, PD, PD,
                                       PD, PD, PI64]),
    ("dfpca_eig_residuals", C.c_int, [P, P, C.POINTER(DfpcaGrid), C.c_int64, PD, PD, PD]),
    ("dfpca_dense_eig", C.c_int, [P, P, C.POINTER(DfpcaGrid), C.c_int64, PD, PD, PD, PD, PI64]),
    ("dfpca_nccl_unique_id", C.c_int, [P]),
    ("dfpca_nccl_init", C.c_int, [P, C.c_int, C.c_int, P]),
    ("dfpca_nccl_selftest", C.c_int, [P, PI64]),
    ("dfpca_covariance_sharded", C.c_int, [P, P, C.POINTER(DfpcaGrid), PD, PD, C.POINTER(DfpcaPlan),
                                           C.POINTER(P)]),
    ("dfpca_covariance_emulated", C.c_int, [P, P, C.POINTER(DfpcaGrid), PD, PD, C.POINTER(DfpcaPlan), C.c_int,
                                            C.POINTER(P)]),
    ("dfpca_covariance_slab_dryrun", C.c_int, [P, P, C.POINTER(DfpcaGrid), PD, PD, C.POINTER(DfpcaPlan), C.c_int,
                                               C.c_int, C.POINTER(P)]),
    ("dfpca_fpca_emulated", C.c_int, [P, P, C.POINTER(DfpcaGrid), PD, PD, C.c_int, C.c_int64, C.c_int64, C.c_uint64,
                                      PD, PD, PD, PD, PI64, C.POINTER(C.c_int)]),
    ("dfpca_surface_rows", C.c_int, [P, PI64, PI64]),
    ("dfpca_dataset_upload", C.c_int, [P, C.c_int, C.c_int64, PI64, PD, PD, C.POINTER(P)]),
    ("dfpca_dataset_free", C.c_int, [P]),
    ("dfpca_cv_units", C.c_int, [C.c_int64, PI64, C.c_int, C.c_int64, C.c_uint64, PI64, C.c_int64, PI64]),
    ("dfpca_cv_objective", C.c_int, [P, P, C.POINTER(DfpcaGrid), C.c_int, C.c_int64, PI64, PD, PD, PI64]),
    ("dfpca_estimate_sigma2", C.c_int, [P, C.POINTER(DfpcaGrid), PD, P, PD, PD]),
    ("dfpca_scores", C.c_int, [P, C.POINTER(DfpcaGrid), C.c_int64, PI64, PD, PD, PD, C.c_int64, PD, PD, C.c_double,
                               C.c_int, PD, C.POINTER(C.c_int32)]),
    ("dfpca_reconstruct", C.c_int, [P, C.POINTER(DfpcaGrid), PD, C.c_int64, PD, C.c_int64, PD, PD]),
    ("dfpca_read_long_format", C.c_int, [P, C.c_char_p, C.POINTER(P)]),
    ("dfpca_parse_long_format", C.c_int, [P, C.c_char_p, C.c_char_p, C.c_int64, C.POINTER(P)]),
    ("dfpca_table_info", C.c_int, [P, C.POINTER(C.c_int), PI64, PI64, PI64]),
    ("dfpca_table_copy", C.c_int, [P, P, PI64, PD, PD, PI64, C.c_char_p]),
    ("dfpca_linear_bin_table", C.c_int, [P, P, C.POINTER(DfpcaGrid), C.c_int, C.c_int, C.POINTER(P)]),
    ("dfpca_table_free", C.c_int, [P]),
    ("dfpca_shard_bounds", C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int, PI64]),
    ("dfpca_shard_blocks", C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, PI64, C.c_int64, PI64]),
    ("dfpca_simulate", C.c_int, [C.c_int, C.POINTER(DfpcaGrid), C.c_int64, C.c_int64, C.c_uint64, PI64, PD, PD]),
]

_lib = None
_ctx = None
_lock = threading.Lock()
_error_factory = None


def set_error_factory(f):
    global _error_factory
    _error_factory = f


def load(path: Path | str | None = None):
    """Loads the shared library (no device needed) and declares prototypes."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"libdfpca_cuda.so not built ({p}); run python -m paper_1510_04439_b200.build")
    lib = C.CDLL(str(p))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def lib():
    return load()


def ctx(device: int | None = None):
    """Process-wide context on `device` (default: LOCAL_RANK or 0)."""
    global _ctx
    with _lock:
        if _ctx is None:
            dev = device if device is not None else int(os.environ.get("DFPCA_DEVICE",
                                                                       os.environ.get("LOCAL_RANK", 0)))
            h = P()
            st = lib().dfpca_context_create(dev, C.byref(h))
            if st != 0 or not h:
                raise RuntimeError(f"dfpca: cannot create a CUDA context on device {dev} (status {st}); "
                                   "the GPU path has no CPU fallback")
            _ctx = h
        return _ctx


def last_error():
    cls, name, msg = C.c_int(), C.c_char_p(), C.c_char_p()
    lib().dfpca_last_error(ctx(), C.byref(cls), C.byref(name), C.byref(msg))
    n = name.value.decode() if name.value else "Unknown"
    m = msg.value.decode() if msg.value else ""
    if _error_factory is None:
        return RuntimeError(f"{n}: {m}")
    return _error_factory(cls.value, n, m)


def last_error_location():
    s, o = C.c_int64(), C.c_int64()
    lib().dfpca_last_error_location(ctx(), C.byref(s), C.byref(o))
    return s.value, o.value


def check(status: int):
    if status != 0:
        raise last_error()


def stage_ms(stage: str) -> float:
    v = C.c_double()
    lib().dfpca_stage_time(ctx(), stage.encode(), C.byref(v))
    return v.value


def kernel_launches() -> int:
    return int(lib().dfpca_kernel_launches(ctx()))


def profile(on: bool):
    lib().dfpca_profile_enable(ctx(), int(on))


def kernel_stats() -> dict:
    out = {}
    i = 0
    while True:
        name, ms, cnt = C.c_char_p(), C.c_double(), C.c_int64()
        if lib().dfpca_kernel_stat(ctx(), i, C.byref(name), C.byref(ms), C.byref(cnt)) != 0:
            break
        out[name.value.decode()] = (ms.value, cnt.value)
        i += 1
    return out


def pin(arr) -> bool:
    """Page-lock a numpy array's buffer (for pinned H2D/D2H copies)."""
    return lib().dfpca_host_register(arr.ctypes.data, arr.nbytes) == 0


def unpin(arr):
    lib().dfpca_host_unregister(arr.ctypes.data)
