"""ctypes binding of the C-ABI library ``libhelmsolve_b200.so`` (include/helmsolve_b200.h).

The library is built in-tree for sm_100a (``make -C paper_2306_17486_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the library or a GPU is
missing, every compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhelmsolve_b200.so")

HS_OK, HS_EDIMENSION, HS_ESINGULAR, HS_EBREAKDOWN, HS_ENONFINITE, HS_ECONFIG, HS_ECUDA = range(7)
HS_APPLY_C64_F32, HS_APPLY_C64_F64, HS_APPLY_C128 = 0, 1, 2

c_int_p = ctypes.POINTER(ctypes.c_int)
c_double_p = ctypes.POINTER(ctypes.c_double)


class HsLevel(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int),
        ("ny", ctypes.c_int),
        ("h", ctypes.c_double),
        ("wall_x", ctypes.c_double),
        ("wall_y", ctypes.c_double),
        ("mass", ctypes.c_void_p),
    ]


class HsHierarchy(ctypes.Structure):
    _fields_ = [
        ("num_levels", ctypes.c_int),
        ("n_models", ctypes.c_int),
        ("levels", HsLevel * 8),
        ("relax_pre", ctypes.c_int),
        ("relax_post", ctypes.c_int),
        ("damping_pre", ctypes.c_double),
        ("damping_post", ctypes.c_double),
        ("coarse_iters", ctypes.c_int),
        ("coarse_damping", ctypes.c_double),
    ]


class HsSolveArgs(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int),
        ("max_iter", ctypes.c_int),
        ("restart", ctypes.c_int),
        ("b", ctypes.c_void_p),
        ("x0", ctypes.c_void_p),
        ("x", ctypes.c_void_p),
        ("tol", ctypes.c_void_p),
        ("c_true", ctypes.c_void_p),
        ("model_of", ctypes.c_void_p),
        ("hist", ctypes.c_void_p),
        ("hist_len", ctypes.c_void_p),
        ("iterations", ctypes.c_void_p),
        ("converged", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("iter_cap", ctypes.c_void_p),
    ]


class HsConv(ctypes.Structure):
    _fields_ = [
        ("cin", ctypes.c_int),
        ("cout", ctypes.c_int),
        ("stride", ctypes.c_int),
        ("transposed", ctypes.c_int),
        ("softplus", ctypes.c_int),
        ("w", ctypes.c_void_p),
        ("b", ctypes.c_void_p),
    ]


class HsNetDesc(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_int),
        ("channels", ctypes.c_int * 8),
        ("ix", ctypes.c_int),
        ("iy", ctypes.c_int),
        ("nx", ctypes.c_int),
        ("ny", ctypes.c_int),
        ("out_scale", ctypes.c_float),
        ("enc_stem", HsConv),
        ("enc_res_a", HsConv * 8),
        ("enc_res_b", HsConv * 8),
        ("enc_down", HsConv * 8),
        ("sol_stem", HsConv),
        ("sol_res_a", HsConv * 8),
        ("sol_res_b", HsConv * 8),
        ("sol_down", HsConv * 8),
        ("sol_up", HsConv * 8),
        ("sol_ures_a", HsConv * 8),
        ("sol_ures_b", HsConv * 8),
        ("sol_head", HsConv),
        ("implicit_w", ctypes.c_void_p),
    ]


class HsTrainDesc(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_int),
        ("channels", ctypes.c_int * 8),
        ("nx", ctypes.c_int),
        ("ny", ctypes.c_int),
        ("batch", ctypes.c_int),
        ("h", ctypes.c_double),
    ]


class HsAdam(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float), ("eps", ctypes.c_float)]


# (name, restype, argtypes) for every symbol include/helmsolve_b200.h declares
_VP, _I, _D, _SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
SIGNATURES = {
    "hs_abi_version": (_I, []),
    "hs_last_error": (ctypes.c_char_p, []),
    "hs_helm_apply": (_I, [_VP, _VP, _VP, _VP, _I, _I, _I, _D, _D, _D, _I, _VP]),
    "hs_restrict": (_I, [_VP, _VP, _I, _I, _I, _I, _VP]),
    "hs_prolong": (_I, [_VP, _VP, _I, _I, _I, _I, _I, _I, _VP]),
    "hs_jacobi": (_I, [_VP, _VP, _VP, ctypes.POINTER(HsLevel), _VP, _I, _D, _VP]),
    "hs_vcycle_workspace_bytes": (_SZ, [ctypes.POINTER(HsHierarchy), _I]),
    "hs_vcycle": (_I, [ctypes.POINTER(HsHierarchy), _VP, _VP, _VP, _VP, _I, _VP, _SZ, _VP, _VP]),
    "hs_fgmres_workspace_bytes": (_SZ, [ctypes.POINTER(HsHierarchy), _VP, _I, _I, _I, _I, _I]),
    "hs_fgmres_solve": (_I, [ctypes.POINTER(HsHierarchy), _VP, ctypes.POINTER(HsSolveArgs), _VP, _SZ, _VP]),
    "hs_net_create": (_I, [ctypes.POINTER(_VP), ctypes.POINTER(HsNetDesc), _VP]),
    "hs_net_destroy": (None, [_VP]),
    "hs_net_encode_workspace_bytes": (_SZ, [_VP, _I]),
    "hs_net_encode": (_I, [_VP, _VP, _I, _VP, _VP, _SZ, _VP]),
    "hs_net_set_encodings": (_I, [_VP, _I, _VP]),
    "hs_net_workspace_bytes": (_SZ, [_VP, _I]),
    "hs_net_forward": (_I, [_VP, _VP, _VP, _VP, _I, _VP, _SZ, _VP]),
    "hs_green_spectrum": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "hs_green_spectrum_eps": (_I, [_VP, _I, _I, _I, ctypes.c_double, _VP, _VP]),
    "hs_implicit_apply": (_I, [_VP, _VP, _VP, _I, _I, _I, _I, _VP]),
    "hs_conv2d": (_I, [_VP, ctypes.POINTER(HsConv), _VP, _VP, _VP, _I, _I, _I, _VP]),
    "hs_profile_enable": (None, [ctypes.c_uint]),
    "hs_profile_reset": (None, []),
    "hs_profile_query": (_I, [_I, c_double_p, c_double_p, ctypes.POINTER(ctypes.c_longlong)]),
    "hs_launch_count": (ctypes.c_longlong, []),
    "hs_profile_records": (_I, [c_int_p, c_int_p, c_double_p, _I]),
    "hs_set_conv_path": (None, [_I]),
    "hs_resize_bilinear": (_I, [_VP, _VP, _I, _I, _I, _I, _I, _VP]),
    "hs_gaussian_smooth": (_I, [_VP, _VP, _VP, _I, _I, _I, _D, _VP]),
    "hs_normalise_range": (_I, [_VP, _VP, _VP, _I, ctypes.c_longlong, _D, _D, _VP]),
    "hs_train_param_count": (_SZ, [ctypes.POINTER(HsTrainDesc)]),
    "hs_trainer_create": (_I, [ctypes.POINTER(_VP), ctypes.POINTER(HsTrainDesc), _VP, _VP]),
    "hs_trainer_destroy": (None, [_VP]),
    "hs_trainer_step": (_I, [_VP, _VP, _I, _VP, _VP, _VP, ctypes.POINTER(HsAdam), c_double_p, _VP]),
    "hs_trainer_read": (_I, [_VP, _I, _VP, _VP]),
    "hs_trainer_grads": (_I, [_VP, _VP, _I, _VP]),
    "hs_trainer_apply": (_I, [_VP, ctypes.POINTER(HsAdam), _VP]),
    "hs_trainer_write": (_I, [_VP, _I, _VP, _I, _VP]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the ctypes library; raises if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is not built; run `make -C {HERE}` (needs nvcc, sm_100a)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name, None)
                if fn is None:
                    continue  # checked by tests/test_abi.py against the header
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


(PROF_CONV, PROF_CONV_L0, PROF_VCYCLE, PROF_ARNOLDI, PROF_CNN, PROF_IMPLICIT, PROF_VC_UP0, PROF_TRAIN_WGRAD,
 PROF_CONV_WIDE, PROF_KRYLOV) = range(10)


def profile_query(tag: int):
    """(total_ms, total_work, launches) of a tag since the last reset."""
    ms, work, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
    check(load().hs_profile_query(tag, ctypes.byref(ms), ctypes.byref(work), ctypes.byref(n)), "profile")
    return ms.value, work.value, n.value


def profile_records(max_records: int = 100000):
    """[(tag, label, ms)] of every timed launch since the last reset, in launch order."""
    tags = (ctypes.c_int * max_records)()
    labels = (ctypes.c_int * max_records)()
    ms = (ctypes.c_double * max_records)()
    n = load().hs_profile_records(tags, labels, ms, max_records)
    if n < 0:
        check(-n, "profile records")
    return [(tags[i], labels[i], ms[i]) for i in range(n)]


def last_error() -> str:
    msg = load().hs_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str):
    """Map an HS_* return code onto the reference's exception classes."""
    if rc == HS_OK:
        return
    from . import errors

    msg = f"{what}: {last_error()}"
    if rc == HS_EDIMENSION:
        raise errors.DimensionError(msg)
    if rc == HS_ESINGULAR:
        raise errors.SingularityError(msg)
    if rc == HS_EBREAKDOWN:
        raise errors.SolverError(msg)
    if rc == HS_ENONFINITE:
        raise errors.NumericalError(msg)
    if rc == HS_ECONFIG:
        raise errors.ConfigurationError(msg)
    raise RuntimeError(msg)
