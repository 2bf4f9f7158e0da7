"""ctypes loader for libliecl_b200.so (the C-ABI in include/liecl_b200.h).

The product path has no CPU fallback: if the CUDA library is missing or no
B200 is visible, every entry point raises `NativeUnavailable` -- loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LIECL_B200_LIB") or os.path.join(HERE, "lib", "libliecl_b200.so")  # env: A/B builds

# status codes (include/liecl_b200.h)
OK, INVALID_INPUT, CAPACITY, DEGENERACY, TIMEOUT, PARSE, CUDA, NOMEM, INTERNAL = 0, 1, 2, 3, 4, 5, 6, 7, 9
METHOD_STANDARD_RANK, METHOD_MATRIX_INVERSION, METHOD_ORTHONORM, METHOD_ORTHONORM_DIMONLY = 0, 1, 2, 3

# every symbol include/liecl_b200.h declares (tests check the .so exports them all)
EXPORTED = [
    "liecl_b200_abi_version", "liecl_b200_last_error", "liecl_b200_ctx_create", "liecl_b200_ctx_destroy",
    "liecl_b200_ctx_kernel_count", "liecl_b200_ctx_set_stream", "liecl_b200_ctx_set_timing",
    "liecl_b200_ctx_kernel_times", "liecl_b200_closure_dense", "liecl_b200_closure_dense_gram",
    "liecl_b200_closure_pauli", "liecl_b200_closure_pauli_sums", "liecl_b200_pauli_sums_fetch",
    "liecl_b200_project_residual_dense", "liecl_b200_commutator_dense", "liecl_b200_inner_product_dense",
    "liecl_b200_norm_dense", "liecl_b200_linear_combination_dense", "liecl_b200_from_pauli", "liecl_b200_session_create_dense", "liecl_b200_session_destroy",
    "liecl_b200_session_set_basis", "liecl_b200_session_prefetch_basis", "liecl_b200_session_prefetch_candidates", "liecl_b200_session_run_pairs", "liecl_b200_session_run_rows",
    "liecl_b200_session_size", "liecl_b200_session_field", "liecl_b200_session_get_basis",
    "liecl_b200_session_get_vectors", "liecl_b200_session_screen_pairs",
    "liecl_b200_session_get_log",
    "liecl_b200_session_check_candidates",
    "liecl_b200_nccl_unique_id", "liecl_b200_shard_range", "liecl_b200_session_set_shards",
    # round 2: device-resident results, GramState / check_matrix_inversion, Pauli-sum single queries
    "liecl_b200_dense_fetch", "liecl_b200_pauli_sums_fetch_gram",
    "liecl_b200_gram_schur_complement", "liecl_b200_gram_expand", "liecl_b200_gram_refresh",
    "liecl_b200_gram_inverse_error", "liecl_b200_check_matrix_inversion_dense",
    "liecl_b200_project_residual_pauli", "liecl_b200_linear_combination_pauli", "liecl_b200_overlaps_pauli",
    "liecl_b200_pauli_from_terms", "liecl_b200_scale_terms", "liecl_b200_norm_pauli",
    "liecl_b200_check_matrix_inversion_pauli",
    "liecl_b200_session_set_loop_shards", "liecl_b200_loop_shard_range", "liecl_b200_session_run_closure",
    "liecl_b200_session_warnings", "liecl_b200_session_comm_bytes", "liecl_b200_parse_pauli_sum",
    "liecl_b200_realize_generators",
]

# int (*liecl_b200_reduce_fn)(double* values, int64_t count, void* user)
ReduceFn = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_void_p)


class NativeUnavailable(RuntimeError):
    pass


class Config(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_dim", C.c_uint64), ("threads", C.c_uint32),
                ("record_log", C.c_uint32), ("deadline_seconds", C.c_double), ("batch_max", C.c_int64),
                ("field", C.c_uint32), ("stop_when_complete", C.c_uint32), ("conditioning_floor", C.c_double),
                ("gram_refresh_interval", C.c_uint64), ("rank_tolerance", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("commutators_evaluated", C.c_uint64), ("independence_checks", C.c_uint64),
                ("accepted", C.c_uint64), ("dimension", C.c_uint64), ("warnings", C.c_uint64),
                ("wall_seconds", C.c_double), ("batches", C.c_uint64), ("survivors", C.c_uint64),
                ("rechecks", C.c_uint64), ("kernels", C.c_uint64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class Decision(C.Structure):
    _fields_ = [("l", C.c_int64), ("m", C.c_int64), ("null_cand", C.c_int32), ("independent", C.c_int32),
                ("rechecked", C.c_int32), ("pad", C.c_int32), ("residual_norm", C.c_double)]


_lib = None
_lock = threading.RLock()  # context() reports errors through load()


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the shared library (no CUDA call is made by loading)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise NativeUnavailable(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(no CPU fallback exists for the B200 path)")
            lib = C.CDLL(path)
            lib.liecl_b200_last_error.restype = C.c_char_p
            lib.liecl_b200_ctx_kernel_count.restype = C.c_uint64
            lib.liecl_b200_ctx_destroy.restype = None
            lib.liecl_b200_session_destroy.restype = None
            _lib = lib
    return _lib


def last_error() -> str:
    return load().liecl_b200_last_error().decode(errors="replace")


class _Context:
    """Owns one liecl_b200_ctx; destroyed when the last reference goes."""

    def __init__(self, device: int):
        lib = load()
        self.ptr = C.c_void_p()
        if lib.liecl_b200_ctx_create(C.c_int(device), C.byref(self.ptr)) != OK:
            raise NativeUnavailable(f"liecl_b200_ctx_create(device={device}) failed: {last_error()}")
        self._lib = lib

    def __del__(self):
        try:
            if self.ptr:
                self._lib.liecl_b200_ctx_destroy(self.ptr)
                self.ptr = C.c_void_p()
        except Exception:  # interpreter shutdown
            pass


_tls = threading.local()


def context_ref(device: int = 0) -> _Context:
    """This thread's context for `device` (include/liecl_b200.h: one context
    per device and caller thread -- a context's stream, workspaces and cached
    engines are not shared between concurrent callers). Holders that outlive
    the call (sessions) keep the returned object."""
    ctxs = getattr(_tls, "contexts", None)
    if ctxs is None:
        ctxs = _tls.contexts = {}
    if device not in ctxs:
        ctxs[device] = _Context(device)
    return ctxs[device]


def context(device: int = 0) -> C.c_void_p:
    """This thread's context pointer for `device` (see context_ref)."""
    return context_ref(device).ptr


def new_context(device: int = 0) -> C.c_void_p:
    """A private context (own stream and workspaces), e.g. one per thread driving
    its own session; release with destroy_context."""
    lib = load()
    ctx = C.c_void_p()
    if lib.liecl_b200_ctx_create(C.c_int(device), C.byref(ctx)) != OK:
        raise NativeUnavailable(f"liecl_b200_ctx_create(device={device}) failed: {last_error()}")
    return ctx


def destroy_context(ctx) -> None:
    load().liecl_b200_ctx_destroy(ctx)


def kernel_count(device: int = 0) -> int:
    return int(load().liecl_b200_ctx_kernel_count(context(device)))


class KernelTime(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("milliseconds", C.c_double), ("flops", C.c_double)]


KERNEL_CLASSES = ("zgemm_project", "zgemm_subtract", "commutator", "other")


def set_stream(stream_ptr: int | None, device: int = 0) -> None:
    """Launch on a caller-owned cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)."""
    st = load().liecl_b200_ctx_set_stream(context(device), C.c_void_p(stream_ptr) if stream_ptr else None)
    if st != OK:
        raise NativeUnavailable(last_error())


def set_timing(enable: bool, device: int = 0) -> None:
    load().liecl_b200_ctx_set_timing(context(device), C.c_int32(int(enable)))


def kernel_times(device: int = 0) -> dict:
    """Per-class CUDA-event totals since the last call (then reset)."""
    out = (KernelTime * 4)()
    st = load().liecl_b200_ctx_kernel_times(context(device), out)
    if st != OK:
        raise NativeUnavailable(last_error())
    return {name: {"launches": out[k].launches, "ms": out[k].milliseconds, "flops": out[k].flops}
            for k, name in enumerate(KERNEL_CLASSES)}
