"""ctypes loader for libssi.so (include/ssi.h). Argument marshalling only.

The product path has no CPU fallback: if the shared library is missing or was built for
another target, every entry point raises.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libssi.so")

SSI_OK = 0
SSI_F32, SSI_F64 = 0, 1
SSI_COV_FP64, SSI_COV_INT8X3, SSI_COV_SPECTRAL = 0, 1, 2


class PoleTableC(C.Structure):
    _fields_ = [("n_orders", C.c_int32), ("cap", C.c_int32), ("l", C.c_int32),
                ("n_min", C.c_int32), ("n_step", C.c_int32),
                ("count", C.c_void_p), ("f", C.c_void_p), ("xi", C.c_void_p),
                ("mu_re", C.c_void_p), ("mu_im", C.c_void_p), ("mpc", C.c_void_p),
                ("mpd", C.c_void_p), ("shape", C.c_void_p)]


class CriteriaC(C.Structure):
    _fields_ = [("xi_max", C.c_double), ("mpc_min", C.c_double), ("mpd_max", C.c_double),
                ("alpha_f", C.c_double), ("alpha_xi", C.c_double), ("alpha_mac", C.c_double)]


class ClusterInfoC(C.Structure):
    _fields_ = [("n_stable", C.c_int32), ("n_retained", C.c_int32), ("fcm_iters", C.c_int32),
                ("phys", C.c_int32), ("n_components", C.c_int32), ("n_clusters", C.c_int32),
                ("n_merges", C.c_int32), ("overflow", C.c_int32), ("V", C.c_double * 10)]


SSI_MAX_LAGS = 64

# name -> (restype, argtypes)
P, I32, I64, U64, SZ, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t, C.c_double
SIGNATURES = {
    "ssi_covariances": (I32, [P, I32, I64, I32, I64, I32, I32, I32, I64, I64, I32, P, P, SZ, P]),
    "ssi_covariances_ws": (I32, [I64, I32, I32, I32, I32, C.POINTER(SZ)]),
    "ssi_cov_spectral_plan": (I32, [I64, I32, I32, I32, C.POINTER(I32), C.POINTER(I64)]),
    "ssi_cov_normalize": (I32, [P, I32, I32, I32, I64, P]),
    "ssi_cov_spectral_phases": (I32, [P, I32, I64, I32, I64, I32, I32, I64, I64, I32, P, P, SZ, I32, P]),
    "ssi_toeplitz": (I32, [P, I32, I32, P, I64, P]),
    "ssi_rsvd": (I32, [P, I64, I32, I32, I32, U64, U64, I32, P, I64, P, P, SZ, P]),
    "ssi_rsvd_ws": (I32, [I32, I32, I32, C.POINTER(SZ)]),
    "ssi_rsvd_toeplitz": (I32, [P, I32, I32, I32, I32, U64, U64, I32, P, I64, P, P, SZ, P]),
    "ssi_rsvd_toeplitz_ws": (I32, [I32, I32, I32, I32, C.POINTER(SZ)]),
    "ssi_philox_words": (I32, [U64, U64, I64, P, P]),
    "ssi_gaussian_sketch": (I32, [I32, I32, U64, U64, P, I64, P]),
    "ssi_modal_sweep": (I32, [P, I64, P, I32, I32, I32, I32, I32, D, C.POINTER(PoleTableC), P, SZ, P]),
    "ssi_modal_sweep_ws": (I32, [I32, I32, I32, I32, I32, C.POINTER(SZ)]),
    "ssi_stab3d": (I32, [C.POINTER(PoleTableC), I32, C.POINTER(CriteriaC), P, P, P]),
    "ssi_cluster_stage1": (I32, [C.POINTER(PoleTableC), I32, C.POINTER(CriteriaC), P, I32, D, I32, P, P, P, P, P,
                                 P, SZ, P]),
    "ssi_cluster_stage1_ws": (I32, [I32, I32, C.POINTER(SZ)]),
    "ssi_cluster_stage2": (I32, [C.POINTER(PoleTableC), I32, P, P, I32, D, I32, I32, P, P, P, P, P, P, P, P, P, P,
                                 SZ, P]),
    "ssi_cluster_stage2_ws": (I32, [I32, I32, C.POINTER(SZ)]),
    "ssi_track": (I32, [P, P, I32, P, P, P, I32, I32, I32, D, D, P, P, P]),
    "ssi_preprocess": (I32, [P, I32, I64, I32, I64, D, I32, I32, I32, D, D, P, I32, I64, P, SZ, P]),
    "ssi_preprocess_ws": (I32, [I64, I32, I32, I32, C.POINTER(SZ)]),
    "ssi_lowpass_design": (I32, [I32, D, D, D, P, P]),
    "ssi_frame_simulate": (I32, [I32, D, D, D, I32, I32, D, I64, I64, D, U64, U64, P, I32, I64, P, P, SZ, P]),
    "ssi_frame_simulate_ws": (I32, [I32, I64, I64, C.POINTER(SZ)]),
    "ssi_frame_model": (I32, [I32, D, D, D, I32, I32, D, P, P, P, P, P]),
    "ssi_fetch_device_status": (I32, [P, C.POINTER(I32)]),
    "ssi_clear_status": (I32, [P, P]),
    "ssi_status_string": (C.c_char_p, [I32]),
    "ssi_last_error": (C.c_char_p, []),
    "ssi_version": (C.c_char_p, []),
}

_lib = None


class SSIError(RuntimeError):
    def __init__(self, fn, code):
        lib = get()
        msg = lib.ssi_status_string(code).decode()
        detail = lib.ssi_last_error().decode()
        super().__init__(f"{fn}: status {code} ({msg}) {detail}")
        self.code = code


def get():
    """Load libssi.so once; raise if it is absent (no fallback by design)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: run `python -m paper_2411_05510_b200.build` "
                              "(nvcc, sm_100a). There is no CPU fallback.")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def call(name, *args):
    code = getattr(get(), name)(*args)
    if code != SSI_OK:
        raise SSIError(name, code)
    return code
