"""ctypes binding of the C-ABI in include/feti_b200.h (libfeti_b200.so).

This is the only way the Python host side reaches the device: there is no
CPU fallback.  Loading fails loudly when the in-tree library is missing.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfeti_b200.so")

FETI_OK = 0
FETI_ERR_ARG = 1
FETI_ERR_LIFECYCLE = 2
FETI_ERR_CUDA = 3
FETI_ERR_CAPACITY = 4
FETI_ERR_SINGULAR = 5
FETI_ERR_INTERNAL = 6
FETI_ERR_NOT_SPD = 7
FETI_ERR_BREAKDOWN = 8
FETI_ERR_NOT_CONVERGED = 9
FETI_FACTOR_HOST = 0
FETI_FACTOR_DEVICE = 1
FETI_STRATEGY_EXPLICIT = 0
FETI_STRATEGY_IMPLICIT = 1
FETI_PATH_SYRK = 0
FETI_PATH_TRSM = 1

EXPORTED = (
    "feti_abi_version", "feti_last_error", "feti_create", "feti_destroy", "feti_add_subdomain",
    "feti_finalize", "feti_set_factor", "feti_assemble", "feti_local_operator", "feti_apply",
    "feti_apply_device", "feti_get_stats", "feti_host_alloc", "feti_host_free",
    "feti_debug_kernel_attributes", "feti_coarse_setup", "feti_project_device", "feti_coarse_apply_device",
    "feti_apply_implicit", "feti_apply_implicit_device", "feti_enable_device_factorization", "feti_set_stiffness",
    "feti_factorize", "feti_solve_many", "feti_enable_sparse_factorization", "feti_set_sparse_pattern",
    "feti_set_preconditioner", "feti_precond_apply", "feti_precond_apply_device",
    "feti_exchange_setup", "feti_exchange_connect", "feti_apply_exchange_device", "feti_exchange_status",
    "feti_set_strategy", "feti_set_stiffness_values", "feti_pcpg_solve", "feti_enable_dual_rhs",
    "feti_set_forces", "feti_dual_rhs", "feti_set_path",
)
FETI_IPC_HANDLE_BYTES = 64


class FetiStats(C.Structure):
    _fields_ = [
        ("ms_wait_upload", C.c_double), ("ms_unpack", C.c_double), ("ms_diag_inverse", C.c_double),
        ("ms_block_scale", C.c_double), ("ms_trsm", C.c_double), ("ms_syrk", C.c_double),
        ("ms_assemble", C.c_double), ("ms_apply", C.c_double),
        ("flops_trsm_alg", C.c_double), ("flops_syrk_alg", C.c_double),
        ("flops_trsm_exec", C.c_double), ("flops_syrk_exec", C.c_double),
        ("flops_scale_exec", C.c_double), ("apply_bytes_alg", C.c_double),
        ("apply_bytes_exec", C.c_double), ("factor_bytes", C.c_double),
        ("bytes_persistent", C.c_int64), ("bytes_temporary", C.c_int64),
        ("n_subdomains", C.c_int64), ("n_multipliers", C.c_int64),
        ("launches_assemble", C.c_int32), ("launches_apply", C.c_int32),
        ("ms_factorize", C.c_double), ("ms_correct", C.c_double), ("flops_factor_exec", C.c_double),
        ("launches_factorize", C.c_int32), ("pad_", C.c_int32), ("ms_preprocess", C.c_double),
        ("flops_factor_alg", C.c_double), ("ms_pcpg", C.c_double), ("pcpg_iterations", C.c_int64),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load() -> C.CDLL:
    """Load (once) the in-tree CUDA library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2502_08382_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i64p = C.POINTER(C.c_int64)
    f64p = C.POINTER(C.c_double)
    sig = {
        "feti_abi_version": ([], C.c_int),
        "feti_last_error": ([], C.c_char_p),
        "feti_create": ([C.c_int, C.POINTER(P)], C.c_int),
        "feti_destroy": ([P], C.c_int),
        "feti_add_subdomain": ([P, C.c_int64, C.c_int64, i64p, f64p, i64p, i64p, i64p, C.c_int64, i64p],
                               C.c_int),
        "feti_finalize": ([P, C.c_int64], C.c_int),
        "feti_set_factor": ([P, C.c_int64, P, C.c_int64, C.c_int], C.c_int),
        "feti_assemble": ([P], C.c_int),
        "feti_local_operator": ([P, C.c_int64, f64p], C.c_int),
        "feti_apply": ([P, f64p, f64p], C.c_int),
        "feti_apply_device": ([P, P, P, P], C.c_int),
        "feti_get_stats": ([P, C.POINTER(FetiStats)], C.c_int),
        "feti_host_alloc": ([C.c_size_t, C.POINTER(P)], C.c_int),
        "feti_debug_kernel_attributes": ([C.c_char_p, C.c_int], C.c_int),
        "feti_coarse_setup": ([P, i64p, f64p, f64p, C.c_int64], C.c_int),
        "feti_project_device": ([P, P, P, P], C.c_int),
        "feti_coarse_apply_device": ([P, P, P, P], C.c_int),
        "feti_apply_implicit": ([P, f64p, f64p], C.c_int),
        "feti_set_strategy": ([P, C.c_int], C.c_int),
        "feti_set_path": ([P, C.c_int], C.c_int),
        "feti_set_stiffness_values": ([P, C.c_int64, P, P, P, P], C.c_int),
        "feti_pcpg_solve": ([P, f64p, f64p, C.c_double, C.c_int64, C.c_int, f64p, P, P], C.c_int),
        "feti_enable_dual_rhs": ([P], C.c_int),
        "feti_set_forces": ([P, C.c_int64, P, P, P], C.c_int),
        "feti_dual_rhs": ([P, P, f64p], C.c_int),
        "feti_apply_implicit_device": ([P, P, P, P], C.c_int),
        "feti_enable_device_factorization": ([P], C.c_int),
        "feti_set_stiffness": ([P, C.c_int64, C.c_int64, i64p, i64p, f64p, C.c_int64, f64p, C.c_int64, C.c_double,
                                i64p], C.c_int),
        "feti_factorize": ([P], C.c_int),
        "feti_solve_many": ([P, C.c_int64, i64p, f64p, f64p], C.c_int),
        "feti_host_free": ([P], C.c_int),
        "feti_enable_sparse_factorization": ([P], C.c_int),
        "feti_set_preconditioner": ([P, C.c_int64, f64p], C.c_int),
        "feti_exchange_setup": ([P, C.c_int, C.c_int, C.c_char_p], C.c_int),
        "feti_exchange_connect": ([P, C.c_char_p], C.c_int),
        "feti_apply_exchange_device": ([P, P, P, P], C.c_int),
        "feti_exchange_status": ([P], C.c_int),
        "feti_precond_apply": ([P, f64p, f64p], C.c_int),
        "feti_precond_apply_device": ([P, P, P, P], C.c_int),
        "feti_set_sparse_pattern": ([P, C.c_int64, C.c_int64, i64p, i64p, i64p, C.c_int64, i64p], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


class FetiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(rc: int) -> None:
    if rc != FETI_OK:
        msg = load().feti_last_error().decode(errors="replace")
        raise FetiError(rc, msg)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def f64ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class PinnedArray:
    """float64 numpy view over cudaHostAlloc'ed (page-locked) memory."""

    def __init__(self, n: int):
        lib = load()
        ptr = C.c_void_p()
        check(lib.feti_host_alloc(max(int(n), 1) * 8, C.byref(ptr)))
        self._ptr = ptr
        buf = (C.c_double * max(int(n), 1)).from_address(ptr.value)
        self.array = np.frombuffer(buf, dtype=np.float64, count=int(n))

    def free(self):
        if self._ptr is not None and self._ptr.value:
            load().feti_host_free(self._ptr)
        self._ptr = None
        self.array = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def kernel_attributes() -> str:
    buf = C.create_string_buffer(4096)
    check(load().feti_debug_kernel_attributes(buf, 4096))
    return buf.value.decode()
