"""ctypes binding of the C ABI in include/saber_cuda.h (libsaber_b200.so).

The shared library is built in-tree by ``make -C paper_2506_19677_b200`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing, importing this module raises, and with no sm_100 device every compute
call returns SABER_ECUDA.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SABER_LIB", os.path.join(HERE, "libsaber_b200.so"))

(SABER_OK, SABER_EINVAL, SABER_EDOMAIN, SABER_EFIT, SABER_ECUDA, SABER_ECAPACITY, SABER_EINTERNAL,
 SABER_ERETRY) = range(8)
STATUS_NAMES = ["SABER_OK", "SABER_EINVAL", "SABER_EDOMAIN", "SABER_EFIT", "SABER_ECUDA",
                "SABER_ECAPACITY", "SABER_EINTERNAL", "SABER_ERETRY"]
ABI_VERSION = 2


class saber_model(C.Structure):
    _fields_ = [("family", C.c_int32), ("params", C.c_double * 3)]


class saber_mix(C.Structure):
    _fields_ = [("frac", C.c_double * 4), ("present", C.c_int32 * 4)]


class saber_traj_row(C.Structure):
    _fields_ = [
        ("goodput", C.c_double), ("ratio_mean", C.c_double), ("ratio_std", C.c_double),
        ("cv", C.c_double), ("n", C.c_int64), ("completed", C.c_int64), ("met", C.c_int64),
        ("decisions", C.c_int64), ("n_kind", C.c_int64 * 5), ("decision_hash", C.c_uint64),
        ("issued_by_task", C.c_int64 * 4), ("met_by_task", C.c_int64 * 4),
        ("ticks", C.c_int64), ("passes", C.c_int64), ("decode_updates", C.c_int64),
        ("prefill_updates", C.c_int64), ("refresh_entries", C.c_int64),
        ("gate_candidates", C.c_int64), ("ledger_scanned", C.c_int64), ("rng_draws", C.c_int64),
        ("last_arrival", C.c_double), ("horizon", C.c_double),
        ("latency_q", C.c_double * 3),
    ]


class saber_decision(C.Structure):
    _fields_ = [("time", C.c_double), ("request_id", C.c_uint64), ("kind", C.c_int32),
                ("load_before", C.c_int32), ("has_pred", C.c_int32), ("has_req", C.c_int32),
                ("pred_speed", C.c_double), ("req_speed", C.c_double)]


class saber_sweep_desc(C.Structure):
    _fields_ = [
        ("mixes", C.POINTER(C.c_int32)), ("n_mixes", C.c_int32),
        ("rps", C.POINTER(C.c_double)), ("n_rps", C.c_int32),
        ("caps", C.POINTER(C.c_int32)), ("n_caps", C.c_int32),
        ("with_saber", C.c_int32),
        ("num_requests", C.c_int32), ("length_jitter", C.c_double),
        ("window_size", C.c_int32), ("tick", C.c_double),
        ("has_model", C.c_int32), ("model", saber_model), ("ground_truth", saber_model),
        ("prefill_rate", C.c_double), ("has_horizon", C.c_int32), ("horizon", C.c_double),
        ("repeats", C.c_int32), ("seed", C.c_uint64),
        ("device", C.c_int32), ("shard_index", C.c_int32), ("shard_count", C.c_int32),
    ]


class saber_mix_summary(C.Structure):
    _fields_ = [("saber_mean_goodput", C.c_double), ("best_static_mean_goodput", C.c_double),
                ("delta", C.c_double), ("saber_pooled_cv", C.c_double),
                ("best_static_pooled_cv", C.c_double), ("saber_rps_mean_cv", C.c_double),
                ("best_static_rps_mean_cv", C.c_double)]


class saber_row_stats(C.Structure):
    _fields_ = [("goodput", C.c_double), ("ratio_mean", C.c_double), ("ratio_std", C.c_double),
                ("cv", C.c_double)]


class saber_sweep_out(C.Structure):
    _fields_ = [
        ("rows", C.POINTER(saber_traj_row)), ("completion_times", C.POINTER(C.c_double)),
        ("summary", C.POINTER(saber_mix_summary)), ("best_cap_by_rps", C.POINTER(C.c_int32)),
        ("n_rows", C.c_int64), ("device_ms", C.c_double), ("kernel_launches", C.c_int32),
        ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
        ("row_stats", C.POINTER(saber_row_stats)),
    ]


class saber_sweep_buffers(C.Structure):
    _fields_ = [("rows", C.c_void_p), ("rows_bytes", C.c_size_t),
                ("completion_times", C.c_void_p), ("completion_bytes", C.c_size_t),
                ("n_rows", C.c_int64), ("rows_this_shard", C.c_int64)]


class saber_request(C.Structure):
    _fields_ = [("arrival_time", C.c_double), ("sla_seconds", C.c_double), ("deadline", C.c_double),
                ("input_tokens", C.c_int32), ("max_output_tokens", C.c_int32), ("task", C.c_int32),
                ("group", C.c_int32)]


class saber_request_state(C.Structure):
    _fields_ = [("admit_time", C.c_double), ("completion_time", C.c_double),
                ("generated_tokens", C.c_double), ("recorded_required_speed", C.c_double),
                ("state", C.c_int32), ("met_sla", C.c_int32), ("demoted", C.c_int32),
                ("pad_", C.c_int32)]


class saber_workload_spec(C.Structure):
    _fields_ = [("mix", saber_mix), ("rps", C.c_double), ("num_requests", C.c_int32),
                ("seed", C.c_uint64), ("length_jitter", C.c_double)]


class saber_traj_spec(C.Structure):
    _fields_ = [
        ("mix", saber_mix), ("rps", C.c_double), ("num_requests", C.c_int32),
        ("workload_seed", C.c_uint64), ("length_jitter", C.c_double),
        ("requests", C.POINTER(saber_request)),
        ("mode", C.c_int32), ("window_size", C.c_int32), ("tick", C.c_double),
        ("static_batch_size", C.c_int32),
        ("has_model", C.c_int32), ("model", saber_model), ("ground_truth", saber_model),
        ("prefill_rate", C.c_double), ("has_horizon", C.c_int32), ("horizon", C.c_double),
        ("seed", C.c_uint64),
    ]


class saber_run_batch_desc(C.Structure):
    _fields_ = [("specs", C.POINTER(saber_traj_spec)), ("n_traj", C.c_int32), ("device", C.c_int32)]


class saber_run_batch_out(C.Structure):
    _fields_ = [
        ("rows", C.POINTER(saber_traj_row)),
        ("arrival_times", C.POINTER(C.c_double)), ("admit_times", C.POINTER(C.c_double)),
        ("completion_times", C.POINTER(C.c_double)), ("demoted", C.POINTER(C.c_uint8)),
        ("max_n", C.c_int32),
        ("decisions", C.POINTER(saber_decision)), ("decision_cap", C.c_int64),
        ("n_decisions", C.POINTER(C.c_int64)),
        ("device_ms", C.c_double), ("kernel_launches", C.c_int32),
        ("requests", C.POINTER(saber_request)), ("states", C.POINTER(saber_request_state)),
        ("cdf_latency", C.POINTER(C.c_double)), ("cdf_fraction", C.POINTER(C.c_double)),
        ("group_issued", C.POINTER(C.c_int32)), ("group_met", C.POINTER(C.c_int32)),
        ("max_groups", C.c_int32),
    ]


class saber_fit_desc(C.Structure):
    _fields_ = [("loads", C.POINTER(C.c_int32)), ("speeds", C.POINTER(C.c_double)),
                ("offsets", C.POINTER(C.c_int64)), ("n_curves", C.c_int32),
                ("family_mask", C.c_int32), ("calibrate", C.c_int32), ("device", C.c_int32)]


class saber_fit_out(C.Structure):
    _fields_ = [("params", C.POINTER(C.c_double)), ("r2", C.POINTER(C.c_double)),
                ("status", C.POINTER(C.c_int32)), ("best_family", C.POINTER(C.c_int32)),
                ("iterations", C.POINTER(C.c_int32)), ("device_ms", C.c_double),
                ("kernel_launches", C.c_int32), ("trials", C.POINTER(C.c_int32))]


SABER_MC_STATS = 8
SABER_MC_BINS = 64


class saber_mc_desc(C.Structure):
    _fields_ = [
        ("n_traj", C.c_int64),
        ("mixes", C.POINTER(C.c_int32)), ("n_mixes", C.c_int32),
        ("rps", C.POINTER(C.c_double)), ("n_rps", C.c_int32),
        ("caps", C.POINTER(C.c_int32)), ("n_caps", C.c_int32),
        ("with_saber", C.c_int32),
        ("num_requests", C.c_int32), ("length_jitter", C.c_double),
        ("window_size", C.c_int32), ("tick", C.c_double),
        ("has_model", C.c_int32), ("model", saber_model), ("ground_truth", saber_model),
        ("prefill_rate", C.c_double),
        ("seed", C.c_uint64), ("burst_factor", C.c_double), ("mean_calm", C.c_double),
        ("mean_burst", C.c_double), ("scheduler_seed", C.c_uint64), ("scheduler_seeds", C.c_int32),
        ("device", C.c_int32), ("shard_index", C.c_int32), ("shard_count", C.c_int32),
        ("chunk", C.c_int64),
    ]


class saber_mc_out(C.Structure):
    _fields_ = [("cell_stats", C.POINTER(C.c_int64)), ("cell_hist", C.POINTER(C.c_int64)),
                ("rows", C.POINTER(saber_traj_row)), ("device_ms", C.c_double),
                ("sim_kernel_ms", C.c_double), ("kernel_launches", C.c_int32)]


class saber_profile_spec(C.Structure):
    _fields_ = [("ground_truth", saber_model), ("prefill_rate", C.c_double), ("mix", saber_mix),
                ("num_requests", C.c_int32), ("seed", C.c_uint64), ("length_jitter", C.c_double),
                ("l_max", C.c_int32)]


class saber_profile_desc(C.Structure):
    _fields_ = [("specs", C.POINTER(saber_profile_spec)), ("n_profiles", C.c_int32),
                ("device", C.c_int32)]


class saber_profile_out(C.Structure):
    _fields_ = [("sample_offsets", C.POINTER(C.c_int64)), ("loads", C.POINTER(C.c_int32)),
                ("speeds", C.POINTER(C.c_double)), ("capacity", C.c_int64),
                ("status", C.POINTER(C.c_int32)), ("device_ms", C.c_double)]


# (name, restype, argtypes) for every symbol include/saber_cuda.h declares.
_P = C.POINTER
SYMBOLS = [
    ("saber_cuda_sweep_rows", C.c_int64, [_P(saber_sweep_desc)]),
    ("saber_cuda_sweep", C.c_int, [_P(saber_sweep_desc), _P(saber_sweep_out)]),
    ("saber_cuda_sweep_plan_create", C.c_int, [_P(saber_sweep_desc), _P(C.c_void_p)]),
    ("saber_cuda_sweep_plan_run", C.c_int, [C.c_void_p, C.c_void_p]),
    ("saber_cuda_sweep_plan_summarize", C.c_int, [C.c_void_p, C.c_void_p]),
    ("saber_cuda_sweep_plan_launch", C.c_int, [C.c_void_p, C.c_void_p]),
    ("saber_cuda_sweep_plan_summarize_launch", C.c_int, [C.c_void_p, C.c_void_p]),
    ("saber_cuda_sweep_plan_wait", C.c_int, [C.c_void_p]),
    ("saber_cuda_sweep_plan_launch_sim", C.c_int, [C.c_void_p, C.c_void_p]),
    ("saber_cuda_sweep_plan_metrics_launch", C.c_int, [C.c_void_p, C.c_void_p]),
    ("saber_cuda_sweep_plan_buffers", C.c_int, [C.c_void_p, _P(saber_sweep_buffers)]),
    ("saber_cuda_sweep_plan_fetch", C.c_int, [C.c_void_p, _P(saber_sweep_out)]),
    ("saber_cuda_sweep_plan_stats", C.c_int, [C.c_void_p, _P(C.c_double), _P(C.c_double),
                                              _P(C.c_int32)]),
    ("saber_cuda_sweep_plan_destroy", None, [C.c_void_p]),
    ("saber_cuda_sweep_plan_reseed", C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p]),
    ("saber_cuda_sweep_plan_fetch_async", C.c_int, [C.c_void_p, _P(saber_sweep_out), C.c_void_p]),
    ("saber_cuda_run_batch", C.c_int, [_P(saber_run_batch_desc), _P(saber_run_batch_out)]),
    ("saber_cuda_fit_batch", C.c_int, [_P(saber_fit_desc), _P(saber_fit_out)]),
    ("saber_cuda_profile_samples", C.c_int64, [_P(saber_profile_spec)]),
    ("saber_cuda_profile_batch", C.c_int, [_P(saber_profile_desc), _P(saber_profile_out)]),
    ("saber_cuda_mc_cells", C.c_int64, [_P(saber_mc_desc)]),
    ("saber_cuda_mc_sweep", C.c_int, [_P(saber_mc_desc), _P(saber_mc_out)]),
    ("saber_cuda_mc_trace", C.c_int, [_P(saber_mc_desc), C.c_int64, _P(saber_request),
                                      _P(saber_traj_spec)]),
    ("saber_cuda_predict_table", C.c_int, [_P(saber_model), C.c_int32, _P(C.c_double)]),
    ("saber_cuda_generate", C.c_int, [_P(saber_workload_spec), C.c_int32, C.c_int32,
                                      _P(saber_request), C.c_int32]),
    ("saber_cuda_release_cache", C.c_int, [C.c_int32]),
    ("saber_cuda_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("saber_cuda_nccl_init", C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, _P(C.c_void_p)]),
    ("saber_cuda_nccl_destroy", None, [C.c_void_p]),
    ("saber_cuda_sweep_plan_gather", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    ("saber_cuda_sweep_multi", C.c_int, [_P(saber_sweep_desc), _P(C.c_int32), C.c_int32,
                                         _P(saber_sweep_out)]),
    ("saber_cuda_profile_planned_loads", C.c_int32, [C.c_int32, C.c_int32]),
    ("saber_cuda_trace_from_csv", C.c_int, [C.c_char_p, C.c_size_t, _P(saber_request), C.c_int32,
                                            _P(C.c_int32)]),
    ("saber_cuda_trace_to_csv", C.c_int, [_P(saber_request), C.c_int32, C.c_char_p, C.c_size_t,
                                          _P(C.c_size_t)]),
    ("saber_cuda_last_error", C.c_char_p, []),
    ("saber_cuda_abi_version", C.c_int32, []),
    ("saber_cuda_device_count", C.c_int32, []),
    ("saber_cuda_fp64_peak", C.c_int, [C.c_int32, _P(C.c_double)]),
]

_lib = None


def lib():
    """The loaded libsaber_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                              "(the engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SYMBOLS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SaberError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


def check(status: int):
    if status != SABER_OK:
        raise SaberError(status, lib().saber_cuda_last_error().decode())
