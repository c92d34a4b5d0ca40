"""Python mirror of the reference's public API for the hot path.

Names, argument meaning and error behaviour follow proj/core/include/saber/
(simloop.hpp, estimator.hpp, calibration.hpp, workload.hpp, types.hpp), so a
caller of the reference finds the same surface:

    sweep(grid, base, jobs=0)       -> SweepResult      simloop.hpp:96-99
    run(config)                     -> RunOutput        simloop.hpp:49
    run_with_requests(config, reqs) -> RunOutput        simloop.hpp:53-54
    generate(spec)                  -> List[Request]    workload.hpp:31
    trace_from_csv / trace_to_csv                       workload.hpp:38-39
    fit(samples, family)            -> SpeedModel       estimator.hpp:61
    calibrate(samples)              -> CalibrationReport calibration.hpp:54
    predict(model, load), max_speed(model)              estimator.hpp:39-42

Every call goes through the C ABI (include/saber_cuda.h) into the sm_100a
kernels; nothing here computes a simulation or a fit on the CPU.
Exceptions: InvalidArgument (std::invalid_argument), DomainError
(std::domain_error), FitError, CalibrationError, and SaberError for device
failures.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N

# ----------------------------------------------------------------- constants
TASK_NAMES = ["code_qna", "code_generation", "code_summary", "code_translation"]
TASK_INDEX = {n: i for i, n in enumerate(TASK_NAMES)}
FAMILIES = ["usl", "logistic", "linear"]
DECISION_KINDS = ["admit_high", "admit_low", "reject_own", "reject_active", "demote"]


class ModelFamily:
    Usl, Logistic, Linear = 0, 1, 2


class SchedulerMode:
    Saber, Static = 0, 1


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ValueError):
    """std::domain_error"""


class FitError(RuntimeError):
    """saber::FitError (estimator.hpp:46-58)."""

    def __init__(self, what, family, best_params, best_sse):
        super().__init__(what)
        self.family = family
        self.best_params = list(best_params)
        self.best_sse = best_sse


class CalibrationError(RuntimeError):
    """saber::CalibrationError (calibration.hpp:15-18)."""


def _check(status: int):
    if status == N.SABER_OK:
        return
    msg = N.lib().saber_cuda_last_error().decode()
    if status == N.SABER_EINVAL:
        raise InvalidArgument(msg)
    if status == N.SABER_EDOMAIN:
        raise DomainError(msg)
    raise N.SaberError(status, msg)


# --------------------------------------------------------------------- types
@dataclass
class TaskProfile:
    name: str
    avg_input_tokens: int
    avg_output_tokens: int
    sla_seconds: float


def task_catalog() -> List[TaskProfile]:
    """types.cpp:10-18"""
    return [TaskProfile("code_qna", 186, 43, 1.0), TaskProfile("code_generation", 463, 387, 8.0),
            TaskProfile("code_summary", 31, 30, 1.0), TaskProfile("code_translation", 670, 617, 12.0)]


@dataclass
class WorkloadMix:
    proportions: Dict[str, float] = field(default_factory=dict)


def preset_mix(mix_id: str) -> WorkloadMix:
    """types.cpp:27-47"""
    if mix_id == "w1":
        return WorkloadMix({"code_translation": 0.4, "code_generation": 0.4, "code_qna": 0.1,
                            "code_summary": 0.1})
    if mix_id == "w2":
        return WorkloadMix({"code_qna": 0.4, "code_summary": 0.4, "code_generation": 0.1,
                            "code_translation": 0.1})
    if mix_id == "w3":
        return WorkloadMix({"code_qna": 0.25, "code_generation": 0.25, "code_summary": 0.25,
                            "code_translation": 0.25})
    raise InvalidArgument(f"unknown mix preset: {mix_id}")


@dataclass
class SpeedModel:
    family: int = ModelFamily.Usl
    params: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    fit_r2: Optional[float] = None


@dataclass
class WorkloadSpec:
    mix: WorkloadMix = field(default_factory=lambda: preset_mix("w3"))
    rps: float = 1.0
    num_requests: int = 100
    seed: int = 0
    length_jitter: float = 0.2


@dataclass
class SchedulerConfig:
    mode: int = SchedulerMode.Saber
    window_size: int = 8
    tick: float = 0.01
    static_batch_size: int = 0


@dataclass
class EngineConfig:
    ground_truth: SpeedModel = field(
        default_factory=lambda: SpeedModel(ModelFamily.Usl, (100.0, 0.05, 0.001)))
    prefill_rate: float = 2000.0


@dataclass
class SimConfig:
    workload: WorkloadSpec = field(default_factory=WorkloadSpec)
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    model: Optional[SpeedModel] = None
    engine: EngineConfig = field(default_factory=EngineConfig)
    horizon: Optional[float] = None
    repeats: int = 3
    seed: int = 0


class RequestState:
    """types.hpp:43"""
    QueuedHigh, QueuedLow, Executing, Completed = 0, 1, 2, 3


@dataclass
class Request:
    """types.hpp:45-59 (id == index)."""
    id: int
    task: str
    arrival_time: float
    input_tokens: int
    max_output_tokens: int
    sla_seconds: float
    deadline: float
    generated_tokens: float = 0.0
    state: int = RequestState.QueuedHigh
    admit_time: Optional[float] = None
    completion_time: Optional[float] = None
    recorded_required_speed: Optional[float] = None
    demoted: bool = False


@dataclass
class RunRecord:
    request_id: int
    task: str
    arrival_time: float
    admit_time: Optional[float]
    completion_time: Optional[float]
    sla: float
    met_sla: bool
    final_tier: str


@dataclass
class Decision:
    time: float
    request_id: int
    kind: int
    load_before: int
    pred_speed: Optional[float]
    req_speed: Optional[float]


@dataclass
class TaskMetrics:
    """metrics.hpp:55-59"""
    issued: int
    goodput: float
    cdf_points: List[Tuple[float, float]]


@dataclass
class MetricsReport:
    """metrics.hpp:63-69 (goodput, ratio stats, per_task) plus the engine's
    decision statistics and event counters."""
    goodput: float
    ratio_mean: float
    ratio_std: float
    cv: float
    completed: int
    decision_count: int
    decision_kinds: List[int]
    decision_hash: int
    counters: Dict[str, int]
    per_task: Dict[str, TaskMetrics] = field(default_factory=dict)


@dataclass
class RunOutput:
    """simloop.hpp:37-43 (the engine event trace is not produced)."""
    records: List[RunRecord]
    decisions: Optional[List[Decision]]
    metrics: MetricsReport
    requests: List[Request] = field(default_factory=list)


@dataclass
class SweepGrid:
    mixes: List[str] = field(default_factory=list)
    rps_list: List[float] = field(default_factory=list)
    caps: List[int] = field(default_factory=list)
    with_saber: bool = False


@dataclass
class SweepRow:
    mix: str
    rps: float
    scheduler: int
    static_cap: int
    repeat_seed: int
    goodput: float
    ratio_mean: float
    ratio_std: float
    cv: float


@dataclass
class MixSummary:
    saber_mean_goodput: float
    best_static_mean_goodput: float
    delta: float
    saber_pooled_cv: float
    best_static_pooled_cv: float
    saber_rps_mean_cv: float
    best_static_rps_mean_cv: float
    best_cap_by_rps: Dict[float, int]


@dataclass
class SweepResult:
    rows: List[SweepRow]
    summary: Dict[str, MixSummary]
    # engine extras: the raw per-trajectory rows (decision hashes, counters)
    traj_rows: Optional[np.ndarray] = None
    device_ms: float = 0.0


def default_rps_sweep() -> List[float]:
    """workload.cpp:81-85"""
    return [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 15, 20]


# ----------------------------------------------------------------- helpers
def _model(m: SpeedModel) -> N.saber_model:
    x = N.saber_model()
    x.family = int(m.family)
    p = list(m.params) + [0.0] * (3 - len(m.params))
    for i in range(3):
        x.params[i] = float(p[i])
    return x


def _mix(m: WorkloadMix) -> N.saber_mix:
    x = N.saber_mix()
    for name, frac in m.proportions.items():
        if name not in TASK_INDEX:
            raise InvalidArgument(f"mix references unknown task: {name}")
        x.frac[TASK_INDEX[name]] = float(frac)
        x.present[TASK_INDEX[name]] = 1
    return x


def _row_dtype():
    fields = []
    for name, ct in N.saber_traj_row._fields_:
        length = getattr(ct, "_length_", None)
        base = ct._type_ if length else ct
        np_t = np.uint64 if name == "decision_hash" else (np.int64 if base is C.c_int64 else np.float64)
        fields.append((name, np_t, (length,)) if length else (name, np_t))
    return np.dtype(fields)


ROW_DTYPE = _row_dtype()
ROW_STATS_DTYPE = np.dtype([("goodput", np.float64), ("ratio_mean", np.float64),
                            ("ratio_std", np.float64), ("cv", np.float64)])
assert ROW_DTYPE.itemsize == C.sizeof(N.saber_traj_row)

COUNTER_NAMES = ["ticks", "passes", "decode_updates", "prefill_updates", "refresh_entries",
                 "gate_candidates", "ledger_scanned", "rng_draws"]


def _spec_from_config(cfg: SimConfig, requests: Optional[Sequence[Request]] = None,
                      keepalive=None) -> N.saber_traj_spec:
    s = N.saber_traj_spec()
    w = cfg.workload
    s.mix = _mix(w.mix)
    s.rps = float(w.rps)
    s.num_requests = int(w.num_requests if requests is None else len(requests))
    s.workload_seed = int(w.seed) & 0xFFFFFFFFFFFFFFFF
    s.length_jitter = float(w.length_jitter)
    if requests is not None:
        arr = (N.saber_request * max(1, len(requests)))()
        rank = {name: g for g, name in enumerate(sorted({r.task for r in requests}))}
        for i, r in enumerate(requests):
            if r.id != i:
                raise InvalidArgument("run: request ids must be 0..n-1")
            q = arr[i]
            q.arrival_time = r.arrival_time
            q.sla_seconds = r.sla_seconds
            q.deadline = r.deadline
            q.input_tokens = r.input_tokens
            q.max_output_tokens = r.max_output_tokens
            q.task = TASK_INDEX.get(r.task, -1)
            q.group = rank[r.task]
        s.requests = arr
        if keepalive is not None:
            keepalive.append(arr)
    sc = cfg.scheduler
    s.mode = int(sc.mode)
    s.window_size = int(sc.window_size)
    s.tick = float(sc.tick)
    s.static_batch_size = int(sc.static_batch_size)
    s.has_model = 1 if cfg.model is not None else 0
    if cfg.model is not None:
        s.model = _model(cfg.model)
    s.ground_truth = _model(cfg.engine.ground_truth)
    s.prefill_rate = float(cfg.engine.prefill_rate)
    s.has_horizon = 1 if cfg.horizon is not None else 0
    s.horizon = float(cfg.horizon) if cfg.horizon is not None else 0.0
    s.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    return s


# ----------------------------------------------------------------- run path
@dataclass
class BatchResult:
    rows: np.ndarray                     # ROW_DTYPE [n_traj]
    completion_times: np.ndarray         # [n_traj][max_n] NaN = never
    arrival_times: Optional[np.ndarray] = None
    admit_times: Optional[np.ndarray] = None
    demoted: Optional[np.ndarray] = None
    decisions: Optional[List[np.ndarray]] = None
    device_ms: float = 0.0
    kernel_launches: int = 0
    # full RunOutput from the engine (records=True)
    requests: Optional[np.ndarray] = None      # REQUEST_DTYPE [n_traj][max_n]
    states: Optional[np.ndarray] = None        # STATE_DTYPE [n_traj][max_n]
    cdf_latency: Optional[np.ndarray] = None   # [n_traj][max_n]
    cdf_fraction: Optional[np.ndarray] = None
    group_issued: Optional[np.ndarray] = None  # [n_traj][max_groups]
    group_met: Optional[np.ndarray] = None


DECISION_DTYPE = np.dtype([("time", np.float64), ("request_id", np.uint64), ("kind", np.int32),
                           ("load_before", np.int32), ("has_pred", np.int32), ("has_req", np.int32),
                           ("pred_speed", np.float64), ("req_speed", np.float64)])
assert DECISION_DTYPE.itemsize == C.sizeof(N.saber_decision)
REQUEST_DTYPE = np.dtype([("arrival_time", np.float64), ("sla_seconds", np.float64),
                          ("deadline", np.float64), ("input_tokens", np.int32),
                          ("max_output_tokens", np.int32), ("task", np.int32), ("group", np.int32)])
assert REQUEST_DTYPE.itemsize == C.sizeof(N.saber_request)
STATE_DTYPE = np.dtype([("admit_time", np.float64), ("completion_time", np.float64),
                        ("generated_tokens", np.float64), ("recorded_required_speed", np.float64),
                        ("state", np.int32), ("met_sla", np.int32), ("demoted", np.int32),
                        ("pad_", np.int32)])
assert STATE_DTYPE.itemsize == C.sizeof(N.saber_request_state)


def run_batch(configs: Sequence[SimConfig], requests: Optional[Sequence[Optional[Sequence[Request]]]] = None,
              records: bool = False, decisions: bool = False, decision_cap: int = 1 << 16,
              device: int = 0) -> BatchResult:
    """Many independent run()/run_with_requests() trajectories in one launch.
    records=True also returns every request's final state, its record and the
    per-task-group CDFs, all computed on the device."""
    T = len(configs)
    if T == 0:
        raise InvalidArgument("run_batch: no trajectories")
    keep: list = []
    specs = (N.saber_traj_spec * T)()
    max_group = 3
    for k, cfg in enumerate(configs):
        reqs = requests[k] if requests is not None else None
        specs[k] = _spec_from_config(cfg, reqs, keep)
        if reqs is not None:
            max_group = max(max_group, len({r.task for r in reqs}) - 1)
    max_n = max(int(s.num_requests) for s in specs)
    max_groups = max_group + 1
    while True:
        rows = np.zeros(T, dtype=ROW_DTYPE)
        comp = np.full((T, max_n), np.nan)
        arr = np.full((T, max_n), np.nan) if records else None
        adm = np.full((T, max_n), np.nan) if records else None
        dem = np.zeros((T, max_n), dtype=np.uint8) if records else None
        dec = np.zeros((T, decision_cap), dtype=DECISION_DTYPE) if decisions else None
        ndec = np.zeros(T, dtype=np.int64) if decisions else None
        d = N.saber_run_batch_desc()
        d.specs = specs
        d.n_traj = T
        d.device = device
        o = N.saber_run_batch_out()
        P = C.POINTER
        o.rows = rows.ctypes.data_as(P(N.saber_traj_row))
        o.completion_times = comp.ctypes.data_as(P(C.c_double))
        o.max_n = max_n
        ext = {}
        if records:
            o.arrival_times = arr.ctypes.data_as(P(C.c_double))
            o.admit_times = adm.ctypes.data_as(P(C.c_double))
            o.demoted = dem.ctypes.data_as(P(C.c_uint8))
            ext = dict(requests=np.zeros((T, max_n), dtype=REQUEST_DTYPE),
                       states=np.zeros((T, max_n), dtype=STATE_DTYPE),
                       cdf_latency=np.full((T, max_n), np.nan),
                       cdf_fraction=np.full((T, max_n), np.nan),
                       group_issued=np.zeros((T, max_groups), dtype=np.int32),
                       group_met=np.zeros((T, max_groups), dtype=np.int32))
            o.requests = ext["requests"].ctypes.data_as(P(N.saber_request))
            o.states = ext["states"].ctypes.data_as(P(N.saber_request_state))
            o.cdf_latency = ext["cdf_latency"].ctypes.data_as(P(C.c_double))
            o.cdf_fraction = ext["cdf_fraction"].ctypes.data_as(P(C.c_double))
            o.group_issued = ext["group_issued"].ctypes.data_as(P(C.c_int32))
            o.group_met = ext["group_met"].ctypes.data_as(P(C.c_int32))
            o.max_groups = max_groups
        if decisions:
            o.decisions = dec.ctypes.data_as(P(N.saber_decision))
            o.decision_cap = decision_cap
            o.n_decisions = ndec.ctypes.data_as(P(C.c_int64))
        st = N.lib().saber_cuda_run_batch(C.byref(d), C.byref(o))
        if st == N.SABER_ECAPACITY and decisions and int(rows["decisions"].max()) > decision_cap:
            decision_cap = int(rows["decisions"].max())  # exactly the longest log
            continue
        _check(st)
        break
    decs = [dec[k, : ndec[k]].copy() for k in range(T)] if decisions else None
    return BatchResult(rows, comp, arr, adm, dem, decs, o.device_ms, o.kernel_launches, **ext)


def _opt(v) -> Optional[float]:
    return None if math.isnan(v) else float(v)


def _run_output(cfg: SimConfig, res: BatchResult, k: int, requests=None) -> RunOutput:
    """RunOutput of trajectory k, every value read off the engine's outputs."""
    row = res.rows[k]
    n = int(row["n"])
    recs, reqs = [], []
    per_task: Dict[str, TaskMetrics] = {}
    if res.states is not None:
        if requests is not None:
            group_name = sorted({r.task for r in requests})
        else:
            group_name = sorted(TASK_NAMES)
        for i in range(n):
            q = res.requests[k, i]
            x = res.states[k, i]
            task = requests[i].task if requests is not None else TASK_NAMES[int(q["task"])]
            r = Request(i, task, float(q["arrival_time"]), int(q["input_tokens"]),
                        int(q["max_output_tokens"]), float(q["sla_seconds"]), float(q["deadline"]),
                        float(x["generated_tokens"]), int(x["state"]), _opt(x["admit_time"]),
                        _opt(x["completion_time"]), _opt(x["recorded_required_speed"]),
                        bool(x["demoted"]))
            reqs.append(r)
            recs.append(RunRecord(i, task, r.arrival_time, r.admit_time, r.completion_time,
                                  r.sla_seconds, bool(x["met_sla"]), "low" if r.demoted else "high"))
        start = 0
        for g, name in enumerate(group_name):
            issued = int(res.group_issued[k, g])
            if issued == 0:
                continue
            seg = slice(start, start + issued)
            lat, frac = res.cdf_latency[k, seg], res.cdf_fraction[k, seg]
            pts = [(float(a), float(b)) for a, b in zip(lat, frac) if not math.isnan(b)]
            per_task[name] = TaskMetrics(issued, float(res.group_met[k, g]) / float(issued), pts)
            start += issued
    decs = None
    if res.decisions is not None:
        decs = [Decision(float(x["time"]), int(x["request_id"]), int(x["kind"]), int(x["load_before"]),
                         float(x["pred_speed"]) if x["has_pred"] else None,
                         float(x["req_speed"]) if x["has_req"] else None) for x in res.decisions[k]]
    m = MetricsReport(float(row["goodput"]), float(row["ratio_mean"]), float(row["ratio_std"]),
                      float(row["cv"]), int(row["completed"]), int(row["decisions"]),
                      [int(v) for v in row["n_kind"]], int(row["decision_hash"]),
                      {c: int(row[c]) for c in COUNTER_NAMES}, per_task)
    return RunOutput(recs, decs, m, reqs)


def run(config: SimConfig, decisions: bool = True, device: int = 0) -> RunOutput:
    """simloop.cpp:113-116: generate() then the tick loop, on the GPU."""
    res = run_batch([config], records=True, decisions=decisions, device=device)
    return _run_output(config, res, 0)


def run_with_requests(config: SimConfig, requests: Sequence[Request], decisions: bool = True,
                      device: int = 0) -> RunOutput:
    """simloop.cpp:50-111 over a caller-supplied workload (replay)."""
    if len(requests) == 0:
        raise InvalidArgument("run: no requests")
    res = run_batch([config], [requests], records=True, decisions=decisions, device=device)
    return _run_output(config, res, 0, requests)


def generate(spec: WorkloadSpec, device: int = 0) -> List[Request]:
    """workload.cpp:52-79 on the device (bit-identical arrivals and lengths)."""
    w = N.saber_workload_spec()
    w.mix = _mix(spec.mix)
    w.rps = float(spec.rps)
    w.num_requests = int(spec.num_requests)
    w.seed = int(spec.seed) & 0xFFFFFFFFFFFFFFFF
    w.length_jitter = float(spec.length_jitter)
    n = max(1, int(spec.num_requests))
    out = np.zeros(n, dtype=REQUEST_DTYPE)
    _check(N.lib().saber_cuda_generate(C.byref(w), 1, device,
                                       out.ctypes.data_as(C.POINTER(N.saber_request)), n))
    return [Request(i, TASK_NAMES[int(q["task"])], float(q["arrival_time"]), int(q["input_tokens"]),
                    int(q["max_output_tokens"]), float(q["sla_seconds"]), float(q["deadline"]))
            for i, q in enumerate(out)]


def trace_from_csv(text: str) -> List[Request]:
    """workload.cpp:97-138 (saber_cuda_trace_from_csv): the replay workload of a
    trace CSV; raises InvalidArgument with the reference's messages."""
    raw = text.encode()
    n = C.c_int32(0)
    st = N.lib().saber_cuda_trace_from_csv(raw, len(raw), None, 0, C.byref(n))
    if st != N.SABER_ECAPACITY:
        _check(st)
    buf = (N.saber_request * max(1, n.value))()
    _check(N.lib().saber_cuda_trace_from_csv(raw, len(raw), buf, n.value, C.byref(n)))
    return [Request(i, TASK_NAMES[q.task], q.arrival_time, q.input_tokens, q.max_output_tokens,
                    q.sla_seconds, q.deadline) for i, q in enumerate(buf[: n.value])]


def trace_to_csv(requests: Sequence[Request]) -> str:
    """workload.cpp:87-95 (saber_cuda_trace_to_csv)."""
    arr = (N.saber_request * max(1, len(requests)))()
    for i, r in enumerate(requests):
        if r.task not in TASK_INDEX:
            raise InvalidArgument(f"trace csv: unknown task {r.task}")
        arr[i].arrival_time = r.arrival_time
        arr[i].input_tokens = r.input_tokens
        arr[i].max_output_tokens = r.max_output_tokens
        arr[i].task = TASK_INDEX[r.task]
    need = C.c_size_t(0)
    st = N.lib().saber_cuda_trace_to_csv(arr, len(requests), None, 0, C.byref(need))
    if st != N.SABER_ECAPACITY:
        _check(st)
    buf = C.create_string_buffer(need.value + 1)
    _check(N.lib().saber_cuda_trace_to_csv(arr, len(requests), buf, need.value + 1, C.byref(need)))
    return buf.value.decode()


# ---------------------------------------------------------------- sweep path
def _sweep_desc(grid: SweepGrid, base: SimConfig, device: int, shard_index: int, shard_count: int,
                keep: list) -> N.saber_sweep_desc:
    d = N.saber_sweep_desc()
    mix_ids = []
    for m in grid.mixes:
        if m not in ("w1", "w2", "w3"):
            raise InvalidArgument(f"unknown mix preset: {m}")
        mix_ids.append(int(m[1:]))
    mixes = (C.c_int32 * max(1, len(mix_ids)))(*mix_ids)
    rps = (C.c_double * max(1, len(grid.rps_list)))(*[float(r) for r in grid.rps_list])
    caps = (C.c_int32 * max(1, len(grid.caps)))(*[int(c) for c in grid.caps])
    keep += [mixes, rps, caps]
    d.mixes, d.n_mixes = mixes, len(mix_ids)
    d.rps, d.n_rps = rps, len(grid.rps_list)
    d.caps, d.n_caps = caps, len(grid.caps)
    d.with_saber = 1 if grid.with_saber else 0
    d.num_requests = base.workload.num_requests
    d.length_jitter = base.workload.length_jitter
    d.window_size = base.scheduler.window_size
    d.tick = base.scheduler.tick
    d.has_model = 1 if base.model is not None else 0
    if base.model is not None:
        d.model = _model(base.model)
    d.ground_truth = _model(base.engine.ground_truth)
    d.prefill_rate = base.engine.prefill_rate
    d.has_horizon = 1 if base.horizon is not None else 0
    d.horizon = float(base.horizon) if base.horizon is not None else 0.0
    d.repeats = base.repeats
    d.seed = int(base.seed) & 0xFFFFFFFFFFFFFFFF
    d.device = device
    d.shard_index = shard_index
    d.shard_count = shard_count
    return d


class NcclComm:
    """One rank of the engine's NCCL communicator (saber_cuda_nccl_*): the
    final statistics reduce of a sharded sweep (SweepPlan.gather)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(N.lib().saber_cuda_nccl_unique_id(buf))
        return buf.raw

    def __init__(self, uid: bytes, n_ranks: int, rank: int, device: int):
        h = C.c_void_p()
        _check(N.lib().saber_cuda_nccl_init(uid, n_ranks, rank, device, C.byref(h)))
        self.handle, self.n_ranks, self.rank = h, n_ranks, rank

    def close(self):
        if self.handle:
            N.lib().saber_cuda_nccl_destroy(self.handle)
            self.handle = None


class SweepPlan:
    """Staged sweep (saber_cuda_sweep_plan_*): create once, run many times."""

    def __init__(self, grid: SweepGrid, base: SimConfig, device: int = 0, shard_index: int = 0,
                 shard_count: int = 1):
        self.grid = grid
        self.base = base
        self._keep = []
        self.last_h2d_bytes = self.last_d2h_bytes = 0
        d = _sweep_desc(grid, base, device, shard_index, shard_count, self._keep)
        self.desc = d
        self.n_rows = int(N.lib().saber_cuda_sweep_rows(C.byref(d)))
        h = C.c_void_p()
        _check(N.lib().saber_cuda_sweep_plan_create(C.byref(d), C.byref(h)))
        self.handle = h

    def run(self, stream: int = 0):
        _check(N.lib().saber_cuda_sweep_plan_run(self.handle, C.c_void_p(stream)))

    def summarize(self, stream: int = 0):
        _check(N.lib().saber_cuda_sweep_plan_summarize(self.handle, C.c_void_p(stream)))

    def launch(self, stream: int = 0):
        """Enqueue run() without waiting (pair with wait())."""
        _check(N.lib().saber_cuda_sweep_plan_launch(self.handle, C.c_void_p(stream)))

    def launch_sim(self, stream: int = 0):
        """launch() without the per-row metrics (pair with metrics_launch())."""
        _check(N.lib().saber_cuda_sweep_plan_launch_sim(self.handle, C.c_void_p(stream)))

    def metrics_launch(self, stream: int = 0):
        """Enqueue the per-row metrics of the last launch_sim()."""
        _check(N.lib().saber_cuda_sweep_plan_metrics_launch(self.handle, C.c_void_p(stream)))

    def summarize_launch(self, stream: int = 0):
        """Enqueue summarize() without waiting (pair with wait())."""
        _check(N.lib().saber_cuda_sweep_plan_summarize_launch(self.handle, C.c_void_p(stream)))

    def gather(self, comm: "NcclComm", root: int = 0, stream: int = 0):
        """Enqueue the NCCL reduce of this shard's rows onto `root` (every rank)."""
        _check(N.lib().saber_cuda_sweep_plan_gather(self.handle, comm.handle, root, C.c_void_p(stream)))

    def wait(self):
        """Synchronise the enqueued work, check the kernels' error flag."""
        _check(N.lib().saber_cuda_sweep_plan_wait(self.handle))

    def buffers(self) -> N.saber_sweep_buffers:
        b = N.saber_sweep_buffers()
        _check(N.lib().saber_cuda_sweep_plan_buffers(self.handle, C.byref(b)))
        return b

    def stats(self):
        a, b, c = C.c_double(), C.c_double(), C.c_int32()
        _check(N.lib().saber_cuda_sweep_plan_stats(self.handle, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def fetch(self, completion=False, summary=True):
        rows = np.zeros(self.n_rows, dtype=ROW_DTYPE)
        o = N.saber_sweep_out()
        o.rows = rows.ctypes.data_as(C.POINTER(N.saber_traj_row))
        comp = None
        if completion:
            comp = np.empty((self.n_rows, self.desc.num_requests))
            o.completion_times = comp.ctypes.data_as(C.POINTER(C.c_double))
        summ = best = None
        if summary:
            summ = (N.saber_mix_summary * self.desc.n_mixes)()
            best = np.zeros((self.desc.n_mixes, self.desc.n_rps), dtype=np.int32)
            o.summary = summ
            o.best_cap_by_rps = best.ctypes.data_as(C.POINTER(C.c_int32))
        _check(N.lib().saber_cuda_sweep_plan_fetch(self.handle, C.byref(o)))
        self.last_h2d_bytes, self.last_d2h_bytes = int(o.h2d_bytes), int(o.d2h_bytes)
        return rows, comp, summ, best

    def reseed(self, seed: int, stream: int = 0):
        """Host prologue for base seed `seed` + async upload on `stream`."""
        _check(N.lib().saber_cuda_sweep_plan_reseed(self.handle, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                                    C.c_void_p(stream)))

    def fetch_stats_async(self, stats: np.ndarray, summ, best: np.ndarray, stream: int = 0):
        """Enqueue the SweepResult payload's copies into caller buffers (pinned
        for a truly asynchronous copy); read them after `stream` synchronises."""
        o = N.saber_sweep_out()
        o.row_stats = stats.ctypes.data_as(C.POINTER(N.saber_row_stats))
        o.summary = summ
        o.best_cap_by_rps = best.ctypes.data_as(C.POINTER(C.c_int32))
        _check(N.lib().saber_cuda_sweep_plan_fetch_async(self.handle, C.byref(o), C.c_void_p(stream)))
        self.last_h2d_bytes, self.last_d2h_bytes = int(o.h2d_bytes), int(o.d2h_bytes)

    def fetch_stats(self):
        """The SweepResult payload: per-row statistics (saber_row_stats) plus
        the summary and best caps (what the drop-in sweep() returns)."""
        stats = np.zeros(self.n_rows, dtype=ROW_STATS_DTYPE)
        summ = (N.saber_mix_summary * self.desc.n_mixes)()
        best = np.zeros((self.desc.n_mixes, self.desc.n_rps), dtype=np.int32)
        o = N.saber_sweep_out()
        o.row_stats = stats.ctypes.data_as(C.POINTER(N.saber_row_stats))
        o.summary = summ
        o.best_cap_by_rps = best.ctypes.data_as(C.POINTER(C.c_int32))
        _check(N.lib().saber_cuda_sweep_plan_fetch(self.handle, C.byref(o)))
        self.last_h2d_bytes, self.last_d2h_bytes = int(o.h2d_bytes), int(o.d2h_bytes)
        return stats, summ, best

    def close(self):
        if self.handle:
            N.lib().saber_cuda_sweep_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sweep_row_keys(grid: SweepGrid, base: SimConfig):
    """(mix, rps, mode, cap, seed) per row in the reference's grid order (simloop.cpp:137-152)."""
    keys = []
    for m in grid.mixes:
        for r in grid.rps_list:
            for c in grid.caps:
                for i in range(base.repeats):
                    keys.append((m, float(r), SchedulerMode.Static, int(c), base.seed + i))
            if grid.with_saber:
                for i in range(base.repeats):
                    keys.append((m, float(r), SchedulerMode.Saber, 0, base.seed + i))
    return keys


def sweep(grid: SweepGrid, base: SimConfig, jobs: int = 0, device: int = 0,
          completion: bool = False) -> SweepResult:
    """simloop.cpp:130-277 on the GPU.  `jobs` is accepted for API parity; the
    device decides its own parallelism and the output never depends on it."""
    del jobs
    if not grid.mixes or not grid.rps_list or (not grid.caps and not grid.with_saber):
        raise InvalidArgument("sweep: empty grid")
    if grid.with_saber and base.model is None:
        raise InvalidArgument("sweep: saber variant requires a model")
    plan = SweepPlan(grid, base, device=device)
    try:
        plan.run()
        plan.summarize()
        rows, comp, summ, best = plan.fetch(completion=completion)
        dev_ms = plan.stats()[0]
    finally:
        plan.close()
    res = _sweep_result(grid, base, rows, summ, best, dev_ms)
    if completion:
        res.completion_times = comp
    return res


def sweep_multi(grid: SweepGrid, base: SimConfig, devices: Sequence[int]) -> SweepResult:
    """sweep() over several GPUs of this process (saber_cuda_sweep_multi): one
    shard per device, NCCL reduce onto the first, summary there."""
    keep: list = []
    d = _sweep_desc(grid, base, int(devices[0]), 0, 1, keep)
    n_rows = int(N.lib().saber_cuda_sweep_rows(C.byref(d)))
    rows = np.zeros(n_rows, dtype=ROW_DTYPE)
    summ = (N.saber_mix_summary * max(1, len(grid.mixes)))()
    best = np.zeros((len(grid.mixes), len(grid.rps_list)), dtype=np.int32)
    o = N.saber_sweep_out()
    o.rows = rows.ctypes.data_as(C.POINTER(N.saber_traj_row))
    o.summary = summ
    o.best_cap_by_rps = best.ctypes.data_as(C.POINTER(C.c_int32))
    devs = (C.c_int32 * len(devices))(*[int(x) for x in devices])
    _check(N.lib().saber_cuda_sweep_multi(C.byref(d), devs, len(devices), C.byref(o)))
    return _sweep_result(grid, base, rows, summ, best, o.device_ms)


def _sweep_result(grid, base, rows, summ, best, dev_ms):
    cols = [rows[f].tolist() for f in ("goodput", "ratio_mean", "ratio_std", "cv")]
    out_rows = [SweepRow(m, r, mode, cap, seed, g, rm, rs, cv)
                for (m, r, mode, cap, seed), g, rm, rs, cv in zip(sweep_row_keys(grid, base), *cols)]
    summary = {}
    for k, m in enumerate(grid.mixes):
        s = summ[k]
        caps = {float(r): int(best[k, j]) for j, r in enumerate(grid.rps_list)} if grid.caps else {}
        summary[m] = MixSummary(s.saber_mean_goodput, s.best_static_mean_goodput, s.delta,
                                s.saber_pooled_cv, s.best_static_pooled_cv, s.saber_rps_mean_cv,
                                s.best_static_rps_mean_cv, caps)
    return SweepResult(out_rows, summary, rows, dev_ms)


# ---------------------------------------------------------------- estimator
def predict(model: SpeedModel, load: int) -> float:
    """estimator.cpp:234-237 (host table builder shared with the engine)."""
    if load < 1:
        raise DomainError("predict: load must be >= 1")
    tab = (C.c_double * load)()
    _check(N.lib().saber_cuda_predict_table(C.byref(_model(model)), load, tab))
    return tab[load - 1]


def max_speed(model: SpeedModel) -> float:
    return predict(model, 1)


def device_count() -> int:
    return int(N.lib().saber_cuda_device_count())


def fp64_peak_tflops(device: int = 0) -> float:
    v = C.c_double()
    _check(N.lib().saber_cuda_fp64_peak(device, C.byref(v)))
    return v.value


# ------------------------------------------------------------------ fitting
@dataclass
class LoadSpeedSample:
    load: int
    speed: float


@dataclass
class FamilyFit:
    family: int
    ok: bool
    model: Optional[SpeedModel]
    error: str = ""


@dataclass
class CalibrationReport:
    best: SpeedModel
    fits: List[FamilyFit]


@dataclass
class FitBatchResult:
    params: np.ndarray       # [3 families][n_curves][3]
    r2: np.ndarray           # [3][n_curves] fit_r2, or FitError best_sse
    status: np.ndarray       # [3][n_curves] 0 ok, -1 not fitted, > 0 FitError reason (1..4)
    best_family: Optional[np.ndarray]  # [n_curves] (calibrate): -(2+d) only d < 3 loads, -1 none
    iterations: np.ndarray   # [3][n_curves] LM iterations over the 5 starts
    device_ms: float
    kernel_launches: int
    trials: Optional[np.ndarray] = None  # [3][n_curves] LM damping trials over the 5 starts


def fit_batch(loads, speeds, offsets, family_mask: int = 0x7, calibrate: bool = False,
              device: int = 0) -> FitBatchResult:
    """Many independent fit()/calibrate() calls in one launch (SoA curves:
    curve c owns samples [offsets[c], offsets[c+1]))."""
    loads = np.ascontiguousarray(loads, dtype=np.int32)
    speeds = np.ascontiguousarray(speeds, dtype=np.float64)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    n = len(offsets) - 1
    params = np.zeros((3, n, 3))
    r2 = np.zeros((3, n))
    status = np.zeros((3, n), dtype=np.int32)
    best = np.zeros(n, dtype=np.int32) if calibrate else None
    iters = np.zeros((3, n), dtype=np.int32)
    trials = np.zeros((3, n), dtype=np.int32)
    d = N.saber_fit_desc()
    P = C.POINTER
    d.loads = loads.ctypes.data_as(P(C.c_int32))
    d.speeds = speeds.ctypes.data_as(P(C.c_double))
    d.offsets = offsets.ctypes.data_as(P(C.c_int64))
    d.n_curves = n
    d.family_mask = family_mask
    d.calibrate = 1 if calibrate else 0
    d.device = device
    o = N.saber_fit_out()
    o.params = params.ctypes.data_as(P(C.c_double))
    o.r2 = r2.ctypes.data_as(P(C.c_double))
    o.status = status.ctypes.data_as(P(C.c_int32))
    if calibrate:
        o.best_family = best.ctypes.data_as(P(C.c_int32))
    o.iterations = iters.ctypes.data_as(P(C.c_int32))
    o.trials = trials.ctypes.data_as(P(C.c_int32))
    _check(N.lib().saber_cuda_fit_batch(C.byref(d), C.byref(o)))
    return FitBatchResult(params, r2, status, best, iters, o.device_ms, o.kernel_launches, trials)


def _samples_arrays(samples):
    loads = np.array([s.load if isinstance(s, LoadSpeedSample) else s[0] for s in samples], np.int32)
    speeds = np.array([s.speed if isinstance(s, LoadSpeedSample) else s[1] for s in samples], np.float64)
    return loads, speeds


def fit_error_message(kind: int, family: int) -> str:
    """FitError::what() for the engine's reason code (saber_cuda.h SABER_FITERR_*)."""
    if kind == 1:
        return f"too few samples or distinct loads to fit {FAMILIES[family]}"
    if kind == 2:
        return f"optimizer did not converge for {FAMILIES[family]}"
    if kind == 3:
        return "fitted linear model is increasing in load"
    return "fitted model is not non-increasing in load"


def fit(samples, family: int, device: int = 0) -> SpeedModel:
    """estimator.cpp:241-346 on the GPU; raises FitError like the reference."""
    loads, speeds = _samples_arrays(samples)
    res = fit_batch(loads, speeds, [0, len(loads)], family_mask=1 << family, device=device)
    p = res.params[family, 0]
    if res.status[family, 0] != 0:
        raise FitError(fit_error_message(int(res.status[family, 0]), family), family, p,
                       res.r2[family, 0])
    return SpeedModel(family, tuple(float(x) for x in p), float(res.r2[family, 0]))


def calibrate(samples, device: int = 0) -> CalibrationReport:
    """calibration.cpp:137-168 on the GPU."""
    loads, speeds = _samples_arrays(samples)
    res = fit_batch(loads, speeds, [0, len(loads)], calibrate=True, device=device)
    b = int(res.best_family[0])
    if b <= -2:
        raise CalibrationError(f"calibrate: insufficient distinct loads ({-2 - b} < 3)")
    if b == -1:
        raise CalibrationError("calibrate: no model family produced a fit")
    fits = []
    for f in range(3):
        ok = res.status[f, 0] == 0
        fits.append(FamilyFit(f, bool(ok), SpeedModel(f, tuple(float(x) for x in res.params[f, 0]),
                                                      float(res.r2[f, 0])) if ok else None,
                              "" if ok else fit_error_message(int(res.status[f, 0]), f)))
    return CalibrationReport(fits[b].model, fits)


# ------------------------------------------------- bursty Monte-Carlo (config 5)
@dataclass
class BurstyArrivals:
    """2-state MMPP of BASELINE config 5; see csrc/bursty.h."""
    seed: int = 2026
    burst_factor: float = 5.0
    mean_calm: float = 8.0
    mean_burst: float = 2.0


@dataclass
class McResult:
    cell_stats: np.ndarray      # [n_cells][8]: trajectories, requests, met, completed,
    #                             decisions, admitted, hash-low-bit sum, ticks
    cell_hist: np.ndarray       # [n_cells][65]: latency/SLA bins (4/octave from 2^-6) + never
    rows: Optional[np.ndarray]  # [n_traj] ROW_DTYPE (this shard's rows filled)
    device_ms: float
    sim_kernel_ms: float
    kernel_launches: int


def _mc_desc(n_traj, grid: SweepGrid, base: SimConfig, arrivals: BurstyArrivals, scheduler_seeds,
             device, shard_index, shard_count, chunk, keep):
    d = N.saber_mc_desc()
    mix_ids = (C.c_int32 * len(grid.mixes))(*[int(m[1:]) for m in grid.mixes])
    rps = (C.c_double * len(grid.rps_list))(*[float(r) for r in grid.rps_list])
    caps = (C.c_int32 * max(1, len(grid.caps)))(*[int(c) for c in grid.caps])
    keep += [mix_ids, rps, caps]
    d.n_traj = n_traj
    d.mixes, d.n_mixes = mix_ids, len(grid.mixes)
    d.rps, d.n_rps = rps, len(grid.rps_list)
    d.caps, d.n_caps = caps, len(grid.caps)
    d.with_saber = 1 if grid.with_saber else 0
    d.num_requests = base.workload.num_requests
    d.length_jitter = base.workload.length_jitter
    d.window_size = base.scheduler.window_size
    d.tick = base.scheduler.tick
    d.has_model = 1 if base.model is not None else 0
    if base.model is not None:
        d.model = _model(base.model)
    d.ground_truth = _model(base.engine.ground_truth)
    d.prefill_rate = base.engine.prefill_rate
    d.seed = arrivals.seed
    d.burst_factor = arrivals.burst_factor
    d.mean_calm = arrivals.mean_calm
    d.mean_burst = arrivals.mean_burst
    d.scheduler_seed = int(base.seed) & 0xFFFFFFFFFFFFFFFF
    d.scheduler_seeds = scheduler_seeds
    d.device, d.shard_index, d.shard_count, d.chunk = device, shard_index, shard_count, chunk
    return d


def mc_sweep(n_traj: int, grid: SweepGrid, base: SimConfig, arrivals: BurstyArrivals = None,
             scheduler_seeds: int = 1024, rows: bool = False, device: int = 0, shard_index: int = 0,
             shard_count: int = 1, chunk: int = 0) -> McResult:
    """Bursty Monte-Carlo sweep (saber_cuda_mc_sweep): trajectory k simulates
    cell k % n_cells on its own Philox MMPP trace."""
    keep = []
    d = _mc_desc(n_traj, grid, base, arrivals or BurstyArrivals(), scheduler_seeds, device,
                 shard_index, shard_count, chunk, keep)
    cells = int(N.lib().saber_cuda_mc_cells(C.byref(d)))
    stats = np.zeros((cells, N.SABER_MC_STATS), dtype=np.int64)
    hist = np.zeros((cells, N.SABER_MC_BINS + 1), dtype=np.int64)
    rws = np.zeros(n_traj, dtype=ROW_DTYPE) if rows else None
    o = N.saber_mc_out()
    o.cell_stats = stats.ctypes.data_as(C.POINTER(C.c_int64))
    o.cell_hist = hist.ctypes.data_as(C.POINTER(C.c_int64))
    if rows:
        o.rows = rws.ctypes.data_as(C.POINTER(N.saber_traj_row))
    _check(N.lib().saber_cuda_mc_sweep(C.byref(d), C.byref(o)))
    return McResult(stats, hist, rws, o.device_ms, o.sim_kernel_ms, o.kernel_launches)


def mc_trace(k: int, n_traj: int, grid: SweepGrid, base: SimConfig, arrivals: BurstyArrivals = None,
             scheduler_seeds: int = 1024):
    """Host twin: trajectory k's requests and SimConfig, bit-identical to what
    the device simulates (for replay through run_with_requests)."""
    keep = []
    d = _mc_desc(n_traj, grid, base, arrivals or BurstyArrivals(), scheduler_seeds, 0, 0, 1, 0, keep)
    n = base.workload.num_requests
    reqs = (N.saber_request * n)()
    spec = N.saber_traj_spec()
    _check(N.lib().saber_cuda_mc_trace(C.byref(d), k, reqs, C.byref(spec)))
    out = [Request(i, TASK_NAMES[r.task], r.arrival_time, r.input_tokens, r.max_output_tokens,
                   r.sla_seconds, r.deadline) for i, r in enumerate(reqs)]
    cfg = SimConfig()
    cfg.workload = WorkloadSpec(WorkloadMix({TASK_NAMES[t]: spec.mix.frac[t] for t in range(4)
                                             if spec.mix.present[t]}), spec.rps, n, 0,
                                spec.length_jitter)
    cfg.scheduler = SchedulerConfig(spec.mode, spec.window_size, spec.tick, spec.static_batch_size)
    cfg.model = SpeedModel(spec.model.family, tuple(spec.model.params)) if spec.has_model else None
    cfg.engine = EngineConfig(SpeedModel(spec.ground_truth.family, tuple(spec.ground_truth.params)),
                              spec.prefill_rate)
    cfg.seed = spec.seed
    return out, cfg


# ---------------------------------------------------------------- profiling
def _profile_spec(engine: EngineConfig, spec: WorkloadSpec, l_max: int) -> N.saber_profile_spec:
    s = N.saber_profile_spec()
    s.ground_truth = _model(engine.ground_truth)
    s.prefill_rate = engine.prefill_rate
    s.mix = _mix(spec.mix)
    s.num_requests = spec.num_requests
    s.seed = int(spec.seed) & 0xFFFFFFFFFFFFFFFF
    s.length_jitter = spec.length_jitter
    s.l_max = l_max
    return s


def profile_batch(items, device: int = 0):
    """Many profile() calls in one launch: items = [(EngineConfig, WorkloadSpec, l_max)].
    Returns a list of (loads, speeds) arrays; raises CalibrationError like the
    reference when a profile yields fewer than 3 distinct loads."""
    P = len(items)
    specs = (N.saber_profile_spec * P)(*[_profile_spec(e, w, l) for e, w, l in items])
    total = 0
    for k in range(P):
        c = int(N.lib().saber_cuda_profile_samples(C.byref(specs[k])))
        if c < 0:
            raise CalibrationError("profile: " + N.lib().saber_cuda_last_error().decode())
        total += c
    offs = np.zeros(P + 1, dtype=np.int64)
    loads = np.zeros(max(1, total), dtype=np.int32)
    speeds = np.zeros(max(1, total))
    status = np.zeros(P, dtype=np.int32)
    d = N.saber_profile_desc(specs, P, device)
    o = N.saber_profile_out()
    o.sample_offsets = offs.ctypes.data_as(C.POINTER(C.c_int64))
    o.loads = loads.ctypes.data_as(C.POINTER(C.c_int32))
    o.speeds = speeds.ctypes.data_as(C.POINTER(C.c_double))
    o.capacity = total
    o.status = status.ctypes.data_as(C.POINTER(C.c_int32))
    _check(N.lib().saber_cuda_profile_batch(C.byref(d), C.byref(o)))
    out = []
    for k in range(P):
        if status[k] != 0:
            raise CalibrationError("profile: insufficient distinct loads (< 3)")
        out.append((loads[offs[k]:offs[k + 1]].copy(), speeds[offs[k]:offs[k + 1]].copy()))
    return out


def profile(engine_config: EngineConfig, profiling_spec: WorkloadSpec, l_max: int = 50,
            device: int = 0) -> List[LoadSpeedSample]:
    """calibration.cpp:58-135 on the GPU."""
    loads, speeds = profile_batch([(engine_config, profiling_spec, l_max)], device)[0]
    return [LoadSpeedSample(int(l), float(s)) for l, s in zip(loads, speeds)]
