"""ctypes binding of libbsq.so (include/bsq.h).

There is no fallback: importing the step without the built library, or
creating a context without a CUDA device, raises.  Build with
``python -m paper_1909_04153_b200.build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# BSQ_LIB: load another build of the library (A/B timing of variants only)
LIB_PATH = os.environ.get("BSQ_LIB") or os.path.join(PKG, "lib", "libbsq.so")

BSQ_OK, BSQ_ERR_BAD_ARG, BSQ_ERR_CUDA, BSQ_ERR_SINGULAR, BSQ_ERR_NO_DEVICE, BSQ_ERR_NCCL = range(6)
WALL, MAKER, SPONGE = 0, 1, 2
FP64, FP32 = 0, 1
THOMAS, CR = 0, 1
Y_PIPELINE, Y_SPIKE = 0, 1

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
MAX_OFF, MAX_RESET, MAX_FOLD, MAX_FLUSH = range(4)


class Desc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("solver", ctypes.c_int32),
                ("side_kind", ctypes.c_int32 * 4), ("cross_correction", ctypes.c_int32),
                ("sponge_lo", ctypes.c_int32 * 4), ("sponge_len", ctypes.c_int32 * 4),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double),
                ("dx2", ctypes.c_double), ("dy2", ctypes.c_double),
                ("g", ctypes.c_double), ("b_disp", ctypes.c_double), ("bp13", ctypes.c_double),
                ("c_f", ctypes.c_double), ("theta", ctypes.c_double), ("h_eps", ctypes.c_double),
                ("h_dry", ctypes.c_double), ("ws", ctypes.c_double),
                ("south_internal", ctypes.c_int32), ("north_internal", ctypes.c_int32),
                ("row0", ctypes.c_int32), ("ny_global", ctypes.c_int32),
                ("y_coupling", ctypes.c_int32), ("exact_tiny", ctypes.c_int32)]


class Static(ctypes.Structure):
    _fields_ = [("bed_eff", _dp), ("depth", _dp), ("depth_dx", _dp), ("depth_dy", _dp),
                ("bed_face_x", _dp), ("bed_face_y", _dp), ("cw_south", _dp)]


# phased step (y-strip sharding) and device array ids -- include/bsq.h
PH_GHOST, PH_STAGE, PH_SOLVE1F, PH_SOLVE1B, PH_CORRECT, PH_SOLVE2F, PH_SOLVE2B, PH_FINAL = range(8)
PH_STAGE_INNER, PH_STAGE_EDGE, PH_CORRECT_INNER, PH_CORRECT_EDGE, PH_FINAL_LAUNCH = range(8, 13)
ARR_Q2 = 10
ARR_RESULT = 11
ARR_W, ARR_P, ARR_Q, ARR_W_NEW, ARR_P_NEW, ARR_Q_NEW, ARR_DW_IN, ARR_DW_OUT, ARR_X_IN, ARR_X_OUT = \
    range(10)


class StepParams(ctypes.Structure):
    _fields_ = [("t", ctypes.c_double), ("dt", ctypes.c_double),
                ("euler", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("wc", ctypes.c_double), ("wp", ctypes.c_double), ("wp2", ctypes.c_double),
                ("sc", ctypes.c_double), ("sp", ctypes.c_double), ("sp2", ctypes.c_double),
                ("maker_eta_t", ctypes.c_double * 4), ("maker_flux_t", ctypes.c_double * 4),
                ("maker_eta_n", ctypes.c_double * 4), ("maker_flux_n", ctypes.c_double * 4),
                ("sponge_fac", _dp * 4),
                ("spec", ctypes.c_int32), ("adaptive", ctypes.c_int32),
                ("step_index", ctypes.c_int64),
                ("cfl_target", ctypes.c_double), ("alpha", ctypes.c_double),
                ("dt_min", ctypes.c_double), ("dt_max", ctypes.c_double),
                ("dt_init", ctypes.c_double), ("chain", ctypes.c_double),
                ("dt_fixed", ctypes.c_double), ("dt_prev", ctypes.c_double)]


class StepResult(ctypes.Structure):
    _fields_ = [("max_rate", ctypes.c_double), ("max_speed", ctypes.c_double),
                ("max_depth", ctypes.c_double), ("max_dev", ctypes.c_double),
                ("clamped", ctypes.c_double),
                ("stage_bad", ctypes.c_int64 * 5), ("state_bad", ctypes.c_int64 * 3)]


# every symbol include/bsq.h declares: (name, restype, argtypes)
SIGNATURES = [
    ("bsq_workspace_bytes", ctypes.c_size_t, [ctypes.POINTER(Desc)]),
    ("bsq_create", ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(Static), ctypes.c_void_p,
                                  ctypes.c_size_t, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    ("bsq_destroy", ctypes.c_int, [ctypes.c_void_p]),
    ("bsq_last_error", ctypes.c_char_p, []),
    ("bsq_device_count", ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    ("bsq_upload_state", ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp]),
    ("bsq_download_state", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _dp, _dp, _dp]),
    ("bsq_download_history", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _dp]),
    ("bsq_step", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(StepParams),
                                ctypes.POINTER(StepResult)]),
    ("bsq_commit", ctypes.c_int, [ctypes.c_void_p]),
    ("bsq_stage_rates", ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, _dp, _dp]),
    ("bsq_solve_momentum", ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
    ("bsq_speed_extrema", ctypes.c_int, [ctypes.c_void_p, _dp]),
    ("bsq_fill_ghosts", ctypes.c_int, [ctypes.c_void_p, _dp, _dp]),
    ("bsq_set_timing", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("bsq_kernel_times", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_float),
                                        ctypes.POINTER(ctypes.c_char_p),
                                        ctypes.POINTER(ctypes.c_int)]),
    ("bsq_kernels_per_step", ctypes.c_int, [ctypes.c_void_p]),
    ("bsq_phase", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(StepParams),
                                 ctypes.POINTER(StepResult)]),
    ("bsq_factor_tail", ctypes.c_int, [ctypes.c_void_p, _dp]),
    ("bsq_array_layout", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_size_t),
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int)]),
    ("bsq_pivot_flags", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_int)]),
    ("bsq_spike_coeffs", ctypes.c_int, [ctypes.c_void_p, _dp]),
    ("bsq_set_spike_table", ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.c_int, ctypes.c_int]),
    ("bsq_spike_fix", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    ("bsq_set_gauges", ctypes.c_int, [ctypes.c_void_p, _ip, _ip, ctypes.c_int]),
    ("bsq_gauge_values", ctypes.c_int, [ctypes.c_void_p, _dp]),
    ("bsq_max_tracker", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    ("bsq_download_max", ctypes.c_int, [ctypes.c_void_p, _dp]),
    ("bsq_maker_sums", ctypes.c_int, [_dp, ctypes.c_int, ctypes.c_double, _dp]),
    ("bsq_check_quotients", ctypes.c_int, [ctypes.c_int, _dp, _dp, ctypes.c_long, _dp]),
    ("bsq_append_rows", ctypes.c_longlong, [ctypes.c_char_p, _dp, ctypes.c_long, ctypes.c_long,
                                            ctypes.c_long, ctypes.c_int]),
]

_lib = None


def lib():
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1909_04153_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def iptr(a):
    return a.ctypes.data_as(_ip)


def ptr(a):
    return a.ctypes.data_as(_dp)


def check(rc: int, what: str = "") -> None:
    if rc == BSQ_OK:
        return
    msg = lib().bsq_last_error().decode(errors="replace")
    if rc == BSQ_ERR_SINGULAR:
        raise ZeroDivisionError(msg)
    if rc == BSQ_ERR_BAD_ARG:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise RuntimeError(f"libbsq error {rc} in {what}: {msg}")
