"""ctypes binding of libttiga_b200.so (the C ABI declared in include/ttiga_b200.h).

There is deliberately no fallback: if the library is missing or no CUDA
device is present, every entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTB_LIB") or os.path.join(HERE, "libttiga_b200.so")  # TTB_LIB: A/B builds


class NativeUnavailable(RuntimeError):
    """The sm_100a library or the CUDA device is missing (no CPU fallback exists)."""


class NativeError(RuntimeError):
    """A native entry point returned a non-zero status."""


vp, i32, i64, f64 = C.c_void_p, C.c_int, C.c_longlong, C.c_double

SIGNATURES = {
    "ttb_launch_count": (i64, [i32]),
    "ttb_dgemm": (i32, [vp, i32, i32, i32, i32, i32, f64, vp, i64, i64, vp, i64, i64, f64, vp, i64, i64, i32]),
    "ttb_permute": (i32, [vp, i32, vp, vp, vp, vp]),
    "ttb_dot": (i32, [vp, i64, vp, vp, vp, vp, i32]),
    "ttb_qr_workspace": (i64, [i32, i32]),
    "ttb_geqrf": (i32, [vp, i32, i32, vp, i64, vp, vp]),
    "ttb_orgqr": (i32, [vp, i32, i32, i32, vp, i64, vp, i64, vp, i32]),
    "ttb_extract_r": (i32, [vp, i32, i32, vp, i64, vp]),
    "ttb_qr_small_fits": (i32, [i32, i32]),
    "ttb_qr_small": (i32, [vp, i32, i32, vp, i64, vp, i64, vp]),
    "ttb_svd_jacobi": (i32, [vp, i32, vp, i64, vp, i64, vp, vp, i64, i32, vp, vp]),
    "ttb_lu_solve": (i32, [vp, i32, vp, i64, vp, i32, vp, i64, i32, vp]),
    "ttb_potrf": (i32, [vp, i32, vp, i64, vp]),
    "ttb_band_lu_solve": (i32, [vp, i32, i32, i32, vp, i64, i32, vp, i64]),
    "ttb_potrs": (i32, [vp, i32, vp, i64, vp]),
    "ttb_maxvol_workspace": (i64, [i32, i32]),
    "ttb_maxvol": (i32, [vp, i32, i32, vp, f64, i32, vp, vp, vp]),
    "ttb_basis_eval": (i32, [vp, i32, vp, vp, i32, i32, vp, vp, vp, vp, vp]),
    "ttb_geo_eval": (i32, [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, f64,
                           i32, i32, i32, i32, vp, vp]),
    "ttb_geo_min_det": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp,
                              vp]),
    "ttb_fullgrid_assemble": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "ttb_stencil_spmv": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp]),
    "ttb_op_core": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, i32, i32, i32, vp]),
    "ttb_vec_core": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, i32, i32, vp]),
    "ttb_op_core_flat": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp, i32, i32, i32, vp]),
    "ttb_vec_core_flat": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, i32, i32, vp]),
    "ttb_field_table": (i32, [vp, i32, i32, i32, vp, i32, vp, vp, i32, vp]),
    "ttb_l1_error": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, vp, i32, i32, i32,
                           vp, i32, vp, i32, vp, vp, vp, vp, i32, vp, vp, vp]),
    "ttb_band_matvec": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp]),
    "ttb_band_apply": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, i32]),
    "ttb_local_dense": (i32, [vp, i32, i32, i32, i32, i32, vp, vp, vp]),
    "ttb_local_band_build": (i32, [vp, i32, i32, i32, i32, i32, vp, vp, vp]),
    "ttb_band_chol_solve": (i32, [vp, i64, i32, vp, vp, vp]),
    "ttb_jacobi_diag": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp]),
    "ttb_tt_gather3": (i32, [vp, i32, vp, vp, i32, i32, vp, i32, i32, vp, i32, vp]),
    "ttb_fiber_index": (i32, [vp, i32, i32, i32, i32, i32, vp, vp, vp]),
    "ttb_nested_index": (i32, [vp, i32, i32, i32, i32, vp, vp, vp]),
    "ttb_local_matvec": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "ttb_pcg_workspace": (i64, [i32, i32, i32, i32, i32]),
    "ttb_local_pcg": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, f64, i32, i32, vp, vp, vp]),
    "ttb_abs_floor": (i32, [vp, i64, vp, vp]),
    "ttb_i8gemm": (i32, [vp, i32, i32, i32, vp, vp, vp]),
    "ttb_ozaki_workspace": (i64, [i32, i32, i32]),
    "ttb_ozaki_kernel_events": (i32, [i32]),
    "ttb_ozaki_kernel_events_read": (i32, [i32, vp, vp]),
    "ttb_ozaki_applies": (i32, [i32, i32, i32]),
    "ttb_dgemm_ozaki": (i32, [vp, i32, i32, i32, i32, vp, i64, vp, i64, vp, i64, vp]),
    "ttb_dgemm_ozaki_ex": (i32, [vp, i32, i32, i32, i32, f64, vp, i64, vp, i64, f64, vp, i64, vp]),
    "ttb_dgemm_ozaki_trilA": (i32, [vp, i32, i32, vp, i64, vp, i64, vp, i64, vp]),
    "ttb_dgemm_ozaki_triuB": (i32, [vp, i32, i32, vp, i64, vp, i64, vp, i64, vp]),
    "ttb_ozaki_gram_workspace": (i64, [i32, i32]),
    "ttb_ozaki_gram": (i32, [vp, i32, i32, vp, i64, vp, i64, vp]),
    "ttb_ozaki_gram_rows_workspace": (i64, [i32, i32]),
    "ttb_ozaki_gram_rows": (i32, [vp, i32, i32, vp, i64, vp, i64, vp]),
    "ttb_trtri_lower": (i32, [vp, i32, vp, i64, vp, i64, vp]),
    "ttb_tri_from_potrf": (i32, [vp, i32, vp, i64, vp, i64, vp]),
    "ttb_norm2_est": (i32, [vp, i32, vp, i64, i32, vp, vp]),
    "ttb_band_gemm": (i32, [vp, i32, i32, i32, i32, i32, vp, vp, vp]),
    "ttb_band_gemm_ozaki_workspace": (i64, [i32, i32, i32, i32, i32, i32]),
    "ttb_matvec_core_ozaki_workspace": (i64, [i32, i32, i32, i32, i32, i32]),
    "ttb_matvec_core_ozaki": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp]),
    "ttb_band_gemm_ozaki": (i32, [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, i32]),
    "ttb_local_gemm_workspace": (i64, [i32, i32, i32, i32, i32, i32]),
    "ttb_local_gemm_ws_init": (i32, [vp, i32, i32, i32, i32, i32, vp]),
    "ttb_local_matvec_gemm": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "ttb_pcg_gemm_workspace": (i64, [i32, i32, i32, i32, i32, i32]),
    "ttb_local_pcg_gemm": (i32, [vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, f64, i32, i32, vp, vp,
                                 vp]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load the shared library without touching the GPU (usable on CPU-only hosts)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(f"{path} not built; run `python -m paper_2509_13224_b200.build_native`")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_LIB = None
_DEV_INDEX = None
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def lib():
    global _LIB
    if _LIB is None:
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the TT-IGA hot path runs only on the GPU (no CPU fallback)")
        _LIB = load_library()
    return _LIB


_current_device = torch._C._cuda_getDevice if hasattr(torch._C, "_cuda_getDevice") else torch.cuda.current_device


def stream():
    """Current torch stream of the device the library runs on, as the raw handle (an int: ctypes passes it
    as void* through the argtypes; no per-call object construction)."""
    global _DEV_INDEX
    if _DEV_INDEX is None:
        _DEV_INDEX = torch.cuda.current_device()
    if _raw_stream is not None and _current_device() == _DEV_INDEX:
        return _raw_stream(_DEV_INDEX)
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    """Device address of a tensor as an int (None for a null pointer)."""
    if t is None:
        return None
    return t.data_ptr()


_FNS = {}


def call(name, *args):
    """Invoke an entry point with the current torch stream prepended; raise on non-zero status."""
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(lib(), name)
    rc = fn(stream(), *args)
    if rc != 0:
        raise NativeError(f"{name} returned {rc}")
    return rc


def call_raw(name, *args):
    """Invoke an entry point that takes no stream (workspace queries)."""
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(lib(), name)
    return fn(*args)


DEV = None


def device():
    global DEV
    if DEV is None:
        lib()
        DEV = torch.device("cuda", torch.cuda.current_device())
    return DEV
