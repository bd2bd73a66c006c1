"""ctypes binding of libduodec_b200.so (the C ABI in include/duodec_b200.h).

The shared library is built in-tree by paper_2503_00784_b200/build.py.  There
is no fallback: if the library is missing, importing the native path raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libduodec_b200.so"
if os.environ.get("DD_LIB_AB"):  # A/B timing scripts only: an alternative build of the same ABI
    LIB_PATH = Path(os.environ["DD_LIB_AB"]).resolve()

DD_OK, DD_E_ARG, DD_E_CUDA, DD_E_STATE, DD_E_CAPACITY = 0, -1, -2, -3, -4
DD_MODE_DUO, DD_MODE_SPS, DD_MODE_VANILLA = 0, 1, 2
DD_BUDGET_FIXED, DD_BUDGET_CALIBRATED = 0, 1
DD_TP_HANDLE_BYTES = 64
DD_PREC_BF16, DD_PREC_FP32ACC = 0, 1


class ModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int),
                ("n_kv_heads", C.c_int), ("head_dim", C.c_int), ("ffn_dim", C.c_int),
                ("vocab", C.c_int), ("rms_eps", C.c_float), ("rope_theta", C.c_float),
                ("max_seq", C.c_int), ("page_size", C.c_int), ("precision", C.c_int)]


class PlantDesc(C.Structure):
    _fields_ = [("plant_seed", C.c_uint64), ("alpha", C.c_double), ("gain", C.c_float),
                ("emb_std", C.c_float)]


class VerifyArgs(C.Structure):
    _fields_ = [("mode", C.c_int), ("tail_len", C.c_int), ("n_firsts", C.c_int),
                ("firsts", C.c_int32 * 16), ("seed", C.c_uint64), ("counter", C.c_uint64),
                ("temperature", C.c_double), ("greedy", C.c_int), ("q_onehot", C.c_int)]


class VerifyOut(C.Structure):
    _fields_ = [("prefix_all_accepted", C.c_int), ("reject_index", C.c_int),
                ("resample", C.c_int), ("bundle_accepted", C.c_int), ("seq_index", C.c_int),
                ("fallback", C.c_int), ("sps_accepted", C.c_int), ("next_token", C.c_int),
                ("n_draws", C.c_int), ("pad", C.c_int), ("counter_out", C.c_uint64)]


class EngineConfigC(C.Structure):
    _fields_ = [("mode", C.c_int), ("budget", C.c_int), ("max_sequences", C.c_int),
                ("max_new_tokens", C.c_int), ("temperature", C.c_double), ("greedy", C.c_int),
                ("draft_seed", C.c_uint64), ("verify_seed", C.c_uint64),
                ("budget_policy", C.c_int), ("budget_hard_cap", C.c_int),
                ("calib_probe_len", C.c_int), ("calib_trials", C.c_int), ("threaded", C.c_int),
                ("jitter_seed", C.c_uint64), ("jitter_max_us", C.c_int)]


class IterationRecordC(C.Structure):
    _fields_ = [("draft_ms", C.c_double), ("target_ms", C.c_double), ("verify_ms", C.c_double),
                ("comm_ms", C.c_double), ("tokens_processed", C.c_int),
                ("sequence_count", C.c_int), ("accepted", C.c_int), ("width", C.c_int)]


class GenerationResultC(C.Structure):
    _fields_ = [("tokens", C.POINTER(C.c_int32)), ("max_tokens", C.c_int),
                ("n_tokens", C.c_int), ("iterations", C.POINTER(IterationRecordC)),
                ("max_iterations", C.c_int), ("n_iterations", C.c_int), ("ttft_ms", C.c_double),
                ("total_ms", C.c_double), ("tps", C.c_double), ("prefill_ms", C.c_double),
                ("budget_used", C.c_int), ("device_ms", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("gpu_launches", C.c_uint64),
                ("device_ttft_ms", C.c_double)]


# every entry point of include/duodec_b200.h: name -> (restype, argtypes)
_vp = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_u16p = C.POINTER(C.c_uint16)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
SIGNATURES = {
    "dd_ctx_create": (C.c_int, [C.POINTER(ModelDesc), C.c_int, C.POINTER(_vp)]),
    "dd_ctx_destroy": (None, [_vp]),
    "dd_ctx_create_tp": (C.c_int, [C.POINTER(ModelDesc), C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "dd_tp_export": (C.c_int, [_vp, C.c_char_p]),
    "dd_tp_connect": (C.c_int, [_vp, C.c_char_p]),
    "dd_tp_connect_local": (C.c_int, [C.POINTER(_vp), C.c_int]),
    "dd_last_error": (C.c_char_p, [_vp]),
    "dd_weights_init": (C.c_int, [_vp, C.c_uint64, C.POINTER(PlantDesc)]),
    "dd_prefill": (C.c_int, [_vp, _i32p, C.c_int]),
    "dd_score": (C.c_int, [_vp, _i32p, C.c_int]),
    "dd_kv_len": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "dd_kv_truncate": (C.c_int, [_vp, C.c_int]),
    "dd_kv_compact": (C.c_int, [_vp, _i32p, _i32p, C.c_int]),
    "dd_read_logits": (C.c_int, [_vp, _f32p, C.c_int, C.c_int]),
    "dd_upload_q": (C.c_int, [_vp, _f32p, C.c_int, C.c_int]),
    "dd_verify": (C.c_int, [_vp, C.POINTER(VerifyArgs), C.POINTER(VerifyOut)]),
    "dd_verify_probs": (C.c_int, [_vp, _f64p, _i32p, C.c_int, C.POINTER(VerifyArgs),
                                  C.POINTER(VerifyOut)]),
    "dd_time_pass": (C.c_int, [_vp, C.c_int, C.c_int, _f32p]),
    "dd_profile_pass": (C.c_int, [_vp, C.c_int, _f32p]),
    "dd_pass_weight_bytes": (C.c_uint64, [_vp]),
    "dd_time_gemms": (C.c_int, [_vp, C.c_int, C.c_int, _f32p, C.POINTER(C.c_int)]),
    "dd_read_weights": (C.c_int, [_vp, C.c_int, C.c_int, _u16p, C.c_size_t]),
    "dd_test_gemm": (C.c_int, [_u16p, _u16p, C.c_int, C.c_int, C.c_int, _f32p]),
    "dd_debug_pass_trace": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_uint64), C.c_size_t,
                                      C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "dd_pass_balance": (C.c_int, [_vp]),
    "dd_debug_pass_timeline": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_uint64), C.c_size_t,
                                         C.POINTER(C.c_int)]),
    "dd_debug_prefill_trace": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_uint64), C.c_size_t,
                                         C.POINTER(C.c_int)]),
    "dd_debug_pass_progress": (C.c_void_p, []),
    "dd_debug_gemm_trace": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_uint64), C.c_int,
                                      C.POINTER(C.c_int)]),
    "dd_draft_create": (C.c_int, [C.POINTER(ModelDesc), C.c_uint64, C.POINTER(PlantDesc), C.c_int,
                                  C.POINTER(C.c_int), C.c_int, C.POINTER(_vp)]),
    "dd_draft_destroy": (None, [_vp]),
    "dd_draft_logits": (C.c_int, [_vp, _i32p, C.c_int, _f32p]),
    "dd_draft_time_token": (C.c_int, [_vp, C.c_int, _f32p]),
    "dd_draft_dist": (C.c_int, [_vp, _i32p, C.c_int, C.c_double, C.c_int, _f32p,
                                C.POINTER(C.c_int)]),
    "dd_draft_dynamic": (C.c_int, [_vp, _i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                   C.c_uint64, C.POINTER(C.c_uint64), _i32p, _i32p,
                                   C.POINTER(C.c_int), _f64p, C.POINTER(C.c_int)]),
    "dd_engine_run": (C.c_int, [_vp, _vp, C.POINTER(EngineConfigC), _i32p, C.c_int,
                                C.POINTER(GenerationResultC)]),
    "dd_engine_run_tp": (C.c_int, [C.POINTER(_vp), C.c_int, _vp, C.POINTER(EngineConfigC), _i32p,
                                   C.c_int, C.POINTER(GenerationResultC)]),
    "dd_calibrate": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, _f64p,
                               C.POINTER(C.c_int)]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the native library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing; run paper_2503_00784_b200/build.py")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("DD_LIB_AB") and not hasattr(L, name):
                continue  # an older build in an A/B timing run
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
