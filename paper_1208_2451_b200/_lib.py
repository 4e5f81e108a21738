"""ctypes binding of libprrp_b200.so (C ABI declared in include/prrp_b200.h).

Loading fails loudly: without the in-tree library or a CUDA device every
compute entry point raises DeviceUnavailable (no CPU fallback)."""
import ctypes
import os

from .errors import (DeviceUnavailable, DimensionMismatch, NonConvergence,
                     RankDeficient, SingularFactor, SingularMatrix)

# PRRP_B200_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("PRRP_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libprrp_b200.so")

PRRP_OK = 0
PRRP_ERR_DIM = 1
PRRP_ERR_ARG = 2
PRRP_ERR_RANK_DEFICIENT = 3
PRRP_ERR_NONCONVERGENCE = 4
PRRP_ERR_SINGULAR_MATRIX = 5
PRRP_ERR_SINGULAR_FACTOR = 6
PRRP_ERR_CUDA = 7
PRRP_ERR_UNSUPPORTED = 8
PRRP_ERR_NCCL = 9


class PrrpErr(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("panel", ctypes.c_int32), ("index", ctypes.c_int32),
                ("column", ctypes.c_int32), ("tree_level", ctypes.c_int32), ("tree_index", ctypes.c_int32),
                ("worst", ctypes.c_double), ("msg", ctypes.c_char * 160)]


class PrrpStats(ctypes.Structure):
    _fields_ = [("original_max", ctypes.c_double), ("intermediate_max", ctypes.c_double),
                ("finish_max", ctypes.c_double), ("panel_multiplier_max", ctypes.c_double),
                ("total_swaps", ctypes.c_int64)]


KCLASSES = ("panel", "trsm", "finalize", "permute", "schur", "compose", "blockrow", "gepp", "other")


class PrrpTiming(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 9), ("launches", ctypes.c_int32 * 9),
                ("schur_flops", ctypes.c_double), ("total_ms", ctypes.c_double)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

SIGNATURES = {
    "prrp_b200_abi_version": ([], ctypes.c_int),
    "prrp_b200_device_probe": ([_P, _P, _P], ctypes.c_int),
    "prrp_luprrp": ([_P, _I64, _I64, _I64, _I32, _D, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_luprrp_timed": ([_P, _I64, _I64, _I64, _I32, _D, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_b200_dmma_peak": ([_D, _P, _P], ctypes.c_int),
    "prrp_caluprrp": ([_P, _I64, _I64, _I64, _I32, _D, _I32, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_b200_graph_kernels": ([], ctypes.c_int64),
    "prrp_b200_qrcp_time": ([_P, _I64, _I32, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_caluprrp_timed": ([_P, _I64, _I64, _I64, _I32, _D, _I32, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_strong_rrqr": ([_P, _I64, _I32, _I64, _I32, _D, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_householder_qr": ([_P, _I64, _I32, _I64, _P, _P, _P, _P], ctypes.c_int),
    "prrp_qrcp": ([_P, _I64, _I32, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_lu_residual": ([_P, _I64, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P], ctypes.c_int),
    "prrp_lu_solve": ([_P, _I64, _I64, _P, _P, _I64, _P, _I64, _I32, _P, _P], ctypes.c_int),
    "prrp_multiplier_block": ([_P, _I64, _I32, _I64, _P, _I64, _P, _P, _P], ctypes.c_int),
    "prrp_schur_update": ([_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I32, _P, _P, _P], ctypes.c_int),
    "prrp_gepp_blockrow": ([_P, _I64, _I32, _I64, _P, _P, _P, _P], ctypes.c_int),
    "prrp_calu": ([_P, _I64, _I64, _I64, _I32, _I32, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_gepp_select": ([_P, _I64, _I64, _I32, _P, _P, _P, _P], ctypes.c_int),
    "prrp_gepp": ([_P, _I64, _I64, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_gepp_steps": ([_P, _I64, _I64, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_calu_dist_create": ([_P, _P, _I64, _I64, _I64, _I64, _I32, _D, _I32, _I32, _I32, _P, _P, _P],
                              ctypes.c_int),
    "prrp_calu_dist_buffers": ([_P, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_calu_dist_msg_bytes": ([_P, _I32], ctypes.c_int64),
    "prrp_calu_dist_select": ([_P, _I32, _P, _P], ctypes.c_int),
    "prrp_calu_dist_apply": ([_P, _I32, _I32, _P, _P], ctypes.c_int),
    "prrp_calu_dist_stats": ([_P, _P, _P], ctypes.c_int),
    "prrp_calu_dist_finish": ([_P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_calu_dist_destroy": ([_P], None),
    "prrp_residual_extended": ([_P, _I64, _I64, _I64, _P, _P, _P, _P, _P], ctypes.c_int),
    "prrp_abs_sums": ([_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P], ctypes.c_int),
}

_lib = None


def load_library(path=LIB_PATH):
    """Load the shared library and bind every exported symbol (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceUnavailable(f"{path} is missing: run paper_1208_2451_b200/build.py (nvcc, sm_100a)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def device_lib():
    """The library, after checking a CUDA device is present."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device: the LU_PRRP path runs only on the GPU (no CPU fallback)")
    return load_library()


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def raise_for(rc, err, what):
    """Map a status code + error record onto the reference's exceptions."""
    if rc == PRRP_OK:
        return
    msg = err.msg.decode(errors="replace")
    exc = None
    if rc == PRRP_ERR_DIM:
        exc = DimensionMismatch(msg or f"{what}: dimension mismatch")
    elif rc == PRRP_ERR_ARG:
        exc = ValueError(msg or f"{what}: invalid argument")
    elif rc == PRRP_ERR_RANK_DEFICIENT:
        exc = RankDeficient(f"leading R block numerically singular at diagonal {err.index}", index=err.index)
    elif rc == PRRP_ERR_NONCONVERGENCE:
        exc = NonConvergence(f"swap cap exceeded, worst multiplier {err.worst}", worst=err.worst)
    elif rc == PRRP_ERR_SINGULAR_MATRIX:
        exc = SingularMatrix(f"zero pivot column {err.column}", column=err.column)
    elif rc == PRRP_ERR_SINGULAR_FACTOR:
        exc = SingularFactor(f"zero diagonal at index {err.index}", index=err.index)
    elif rc == PRRP_ERR_UNSUPPORTED:
        exc = NotImplementedError(f"{what}: {msg}")
    else:
        exc = RuntimeError(f"{what}: status {rc}: {msg}")
    if err.panel >= 0 and isinstance(exc, ArithmeticError):
        exc.panel = int(err.panel)
    if err.tree_level >= 0 and isinstance(exc, ArithmeticError):
        exc.tree_node = (int(err.tree_level), int(err.tree_index))
    raise exc
