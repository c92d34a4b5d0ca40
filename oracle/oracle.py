"""ctypes view of the CPU checkers — TEST INFRASTRUCTURE ONLY.

Loads oracle/liboracle.so (the C restatement, prefix ``orc_``) or
oracle/_ref/libsaber_ref.so (the compiled reference, prefix ``ref_``) and
exposes both behind one Python class so a test can run a case through either.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libsaber_ref.so")

QNA, GENERATION, SUMMARY, TRANSLATION = 0, 1, 2, 3
TASK_NAMES = ["code_qna", "code_generation", "code_summary", "code_translation"]
USL, LOGISTIC, LINEAR = 0, 1, 2
SABER, STATIC = 0, 1
KIND_NAMES = ["admit_high", "admit_low", "reject_own", "reject_active", "demote"]


class OrcModel(C.Structure):
    _fields_ = [("family", C.c_int32), ("p", C.c_double * 3)]


class OrcMix(C.Structure):
    _fields_ = [("frac", C.c_double * 4), ("present", C.c_int32 * 4)]


class OrcSimConfig(C.Structure):
    _fields_ = [
        ("mix", OrcMix),
        ("rps", C.c_double),
        ("num_requests", C.c_int32),
        ("workload_seed", C.c_uint64),
        ("jitter", C.c_double),
        ("mode", C.c_int32),
        ("window", C.c_int32),
        ("tick", C.c_double),
        ("cap", C.c_int32),
        ("has_model", C.c_int32),
        ("model", OrcModel),
        ("ground_truth", OrcModel),
        ("prefill_rate", C.c_double),
        ("has_horizon", C.c_int32),
        ("horizon", C.c_double),
        ("seed", C.c_uint64),
    ]


class OrcRequest(C.Structure):
    _fields_ = [
        ("arrival_time", C.c_double),
        ("sla_seconds", C.c_double),
        ("deadline", C.c_double),
        ("input_tokens", C.c_int32),
        ("max_output_tokens", C.c_int32),
        ("task", C.c_int32),
    ]


class OrcDecision(C.Structure):
    _fields_ = [
        ("time", C.c_double),
        ("request_id", C.c_uint64),
        ("kind", C.c_int32),
        ("load_before", C.c_int32),
        ("has_pred", C.c_int32),
        ("has_req", C.c_int32),
        ("pred_speed", C.c_double),
        ("req_speed", C.c_double),
    ]


class OrcTrajOut(C.Structure):
    _fields_ = [
        ("goodput", C.c_double),
        ("ratio_mean", C.c_double),
        ("ratio_std", C.c_double),
        ("cv", C.c_double),
        ("completed", C.c_int64),
        ("met", C.c_int64),
        ("decisions", C.c_int64),
        ("n_kind", C.c_int64 * 5),
        ("decision_hash", C.c_uint64),
        ("issued_by_task", C.c_int64 * 4),
        ("met_by_task", C.c_int64 * 4),
        ("ticks", C.c_int64),
        ("passes", C.c_int64),
        ("decode_updates", C.c_int64),
        ("prefill_updates", C.c_int64),
        ("refresh_entries", C.c_int64),
        ("gate_candidates", C.c_int64),
        ("ledger_scanned", C.c_int64),
        ("rng_draws", C.c_int64),
        ("last_arrival", C.c_double),
        ("horizon", C.c_double),
    ]


class OrcRecord(C.Structure):
    _fields_ = [
        ("arrival_time", C.c_double),
        ("admit_time", C.c_double),
        ("completion_time", C.c_double),
        ("sla", C.c_double),
        ("task", C.c_int32),
        ("input_tokens", C.c_int32),
        ("max_output_tokens", C.c_int32),
        ("demoted", C.c_int32),
    ]


PRESETS = {
    "w1": {TRANSLATION: 0.4, GENERATION: 0.4, QNA: 0.1, SUMMARY: 0.1},
    "w2": {QNA: 0.4, SUMMARY: 0.4, GENERATION: 0.1, TRANSLATION: 0.1},
    "w3": {QNA: 0.25, GENERATION: 0.25, SUMMARY: 0.25, TRANSLATION: 0.25},
}


def make_mix(mix) -> OrcMix:
    m = OrcMix()
    d = PRESETS[mix] if isinstance(mix, str) else mix
    for t, f in d.items():
        m.frac[t] = f
        m.present[t] = 1
    return m


def make_model(family: int, p: Sequence[float]) -> OrcModel:
    m = OrcModel()
    m.family = family
    for i, v in enumerate(list(p) + [0.0] * (3 - len(p))):
        m.p[i] = v
    return m


DEFAULT_GT = (USL, (100.0, 0.05, 0.001))
# calibrate(profile(EngineConfig{}, {w3, n=1000, seed 42}, 50)).best
CALIBRATED_USL = (USL, (99.999999999997357, 0.049999999999992085, 0.0010000000000001078))


def make_config(mix="w1", rps=4.0, n=100, seed=42, workload_seed=None, mode=SABER,
                cap=0, window=8, tick=0.01, model=CALIBRATED_USL, gt=DEFAULT_GT,
                prefill_rate=2000.0, jitter=0.2, horizon=None) -> OrcSimConfig:
    c = OrcSimConfig()
    c.mix = make_mix(mix)
    c.rps = rps
    c.num_requests = n
    c.workload_seed = seed if workload_seed is None else workload_seed
    c.jitter = jitter
    c.mode = mode
    c.window = window
    c.tick = tick
    c.cap = cap
    c.has_model = 1 if (model is not None and mode == SABER) else 0
    if model is not None:
        c.model = make_model(*model)
    c.ground_truth = make_model(*gt)
    c.prefill_rate = prefill_rate
    c.has_horizon = 0 if horizon is None else 1
    c.horizon = 0.0 if horizon is None else horizon
    c.seed = seed
    return c


class OracleError(RuntimeError):
    pass


@dataclass
class RunResult:
    out: OrcTrajOut
    records: Optional[list] = None
    decisions: Optional[list] = None


class Oracle:
    """One of the two CPU checkers ('restatement' or 'reference')."""

    def __init__(self, which: str = "restatement"):
        path, prefix = (RESTATEMENT_SO, "orc_") if which == "restatement" else (REFERENCE_SO, "ref_")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.which = which
        self.lib = C.CDLL(path)
        self.p = prefix
        f = self._f
        f("last_error").restype = C.c_char_p
        P = C.POINTER
        f("generate").argtypes = [P(OrcSimConfig), P(OrcRequest)]
        f("run").argtypes = [P(OrcSimConfig), P(OrcTrajOut), P(OrcRecord), P(OrcDecision),
                             C.c_int64, P(C.c_int64)]
        f("run_with_requests").argtypes = [P(OrcSimConfig), P(OrcRequest), C.c_int32, P(OrcTrajOut),
                                           P(OrcRecord), P(OrcDecision), C.c_int64, P(C.c_int64)]
        f("predict").argtypes = [P(OrcModel), C.c_int32, P(C.c_double)]
        f("fit").argtypes = [P(C.c_int32), P(C.c_double), C.c_int32, C.c_int32, P(C.c_double),
                             P(C.c_double), P(C.c_int32)]
        f("calibrate").argtypes = [P(C.c_int32), P(C.c_double), C.c_int32, P(C.c_int32),
                                   P(C.c_double), P(C.c_double), P(C.c_int32), P(C.c_double),
                                   P(C.c_double)]
        f("profile").argtypes = [P(OrcModel), C.c_double, P(OrcMix), C.c_int32, C.c_uint64,
                                 C.c_double, C.c_int32, P(C.c_int32), P(C.c_double), C.c_int64,
                                 P(C.c_int64)]
        f("sweep").argtypes = [P(OrcSimConfig), P(C.c_int32), C.c_int32, P(C.c_double), C.c_int32,
                               P(C.c_int32), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                               P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double),
                               P(C.c_double), P(C.c_int32)]
        for name in ("generate", "run", "run_with_requests", "predict", "fit", "calibrate",
                     "profile", "sweep"):
            f(name).restype = C.c_int

    def latency_quantiles(self, cfg: OrcSimConfig, ps=(0.5, 0.9, 0.99)) -> list:
        """Reference only: p-quantiles of latency over every issued request,
        read off saber::cdf (metrics.cpp:61-85) of saber::run(cfg)'s records."""
        if self.which != "reference":
            raise OracleError("latency_quantiles: reference harness only")
        f = self._f("latency_quantiles")
        f.argtypes = [C.POINTER(OrcSimConfig), C.POINTER(C.c_double), C.c_int32,
                      C.POINTER(C.c_double)]
        f.restype = C.c_int
        pa = (C.c_double * len(ps))(*ps)
        q = (C.c_double * len(ps))()
        self._check(f(C.byref(cfg), pa, len(ps), q))
        return list(q)

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self._f("last_error")().decode())

    # ---- API -------------------------------------------------------------
    def generate(self, cfg: OrcSimConfig) -> list:
        buf = (OrcRequest * cfg.num_requests)()
        self._check(self._f("generate")(C.byref(cfg), buf))
        return list(buf)

    def run(self, cfg: OrcSimConfig, records=False, decisions=False, dec_cap=1 << 20) -> RunResult:
        out = OrcTrajOut()
        recs = (OrcRecord * cfg.num_requests)() if records else None
        decs = (OrcDecision * dec_cap)() if decisions else None
        nd = C.c_int64(0)
        self._check(self._f("run")(C.byref(cfg), C.byref(out), recs, decs, dec_cap if decisions else 0,
                                   C.byref(nd)))
        return RunResult(out, list(recs) if records else None,
                         list(decs)[: nd.value] if decisions else None)

    def run_with_requests(self, cfg: OrcSimConfig, reqs: Sequence[OrcRequest], records=False,
                          decisions=False, dec_cap=1 << 20) -> RunResult:
        n = len(reqs)
        arr = (OrcRequest * n)(*reqs)
        out = OrcTrajOut()
        recs = (OrcRecord * n)() if records else None
        decs = (OrcDecision * dec_cap)() if decisions else None
        nd = C.c_int64(0)
        self._check(self._f("run_with_requests")(C.byref(cfg), arr, n, C.byref(out), recs, decs,
                                                 dec_cap if decisions else 0, C.byref(nd)))
        return RunResult(out, list(recs) if records else None,
                         list(decs)[: nd.value] if decisions else None)

    def predict(self, family, params, load) -> float:
        m = make_model(family, params)
        v = C.c_double()
        self._check(self._f("predict")(C.byref(m), load, C.byref(v)))
        return v.value

    def fit(self, loads, speeds, family):
        loads = np.ascontiguousarray(loads, dtype=np.int32)
        speeds = np.ascontiguousarray(speeds, dtype=np.float64)
        params = (C.c_double * 3)()
        v = C.c_double()
        err = C.c_int32()
        self._check(self._f("fit")(loads.ctypes.data_as(C.POINTER(C.c_int32)),
                                   speeds.ctypes.data_as(C.POINTER(C.c_double)), len(loads), family,
                                   params, C.byref(v), C.byref(err)))
        return list(params), v.value, bool(err.value)

    def calibrate(self, loads, speeds):
        loads = np.ascontiguousarray(loads, dtype=np.int32)
        speeds = np.ascontiguousarray(speeds, dtype=np.float64)
        bf = C.c_int32()
        bp = (C.c_double * 3)()
        br2 = C.c_double()
        ok = (C.c_int32 * 3)()
        fp = (C.c_double * 9)()
        fr2 = (C.c_double * 3)()
        self._check(self._f("calibrate")(loads.ctypes.data_as(C.POINTER(C.c_int32)),
                                         speeds.ctypes.data_as(C.POINTER(C.c_double)), len(loads),
                                         C.byref(bf), bp, C.byref(br2), ok, fp, fr2))
        return {"best_family": bf.value, "best_params": list(bp), "best_r2": br2.value,
                "ok": list(ok), "params": [list(fp[3 * i:3 * i + 3]) for i in range(3)],
                "r2": list(fr2)}

    def profile(self, gt=DEFAULT_GT, prefill_rate=2000.0, mix="w3", num_requests=1000, seed=42,
                jitter=0.2, l_max=50):
        cap = num_requests + l_max + 8
        loads = (C.c_int32 * cap)()
        speeds = (C.c_double * cap)()
        n = C.c_int64()
        m = make_model(*gt)
        mx = make_mix(mix)
        self._check(self._f("profile")(C.byref(m), prefill_rate, C.byref(mx), num_requests, seed,
                                       jitter, l_max, loads, speeds, cap, C.byref(n)))
        return np.array(loads[: n.value], dtype=np.int32), np.array(speeds[: n.value])

    def sweep(self, base: OrcSimConfig, mixes, rps, caps, with_saber, repeats, jobs=0):
        mix_ids = (C.c_int32 * len(mixes))(*[int(m[1:]) for m in mixes])
        rps_a = (C.c_double * len(rps))(*rps)
        caps_a = (C.c_int32 * max(1, len(caps)))(*caps)
        per_rps = len(caps) * repeats + (repeats if with_saber else 0)
        n_rows = len(mixes) * len(rps) * per_rps
        g = (C.c_double * n_rows)()
        rm = (C.c_double * n_rows)()
        rs = (C.c_double * n_rows)()
        cv = (C.c_double * n_rows)()
        summ = (C.c_double * (7 * len(mixes)))()
        best = (C.c_int32 * (len(mixes) * len(rps)))()
        self._check(self._f("sweep")(C.byref(base), mix_ids, len(mixes), rps_a, len(rps), caps_a,
                                     len(caps), 1 if with_saber else 0, repeats, jobs, g, rm, rs, cv,
                                     summ, best))
        return {"goodput": np.array(g[:]), "ratio_mean": np.array(rm[:]),
                "ratio_std": np.array(rs[:]), "cv": np.array(cv[:]),
                "summary": np.array(summ[:]).reshape(len(mixes), 7),
                "best_cap": np.array(best[:]).reshape(len(mixes), len(rps))}


def sweep_decisions(base: OrcSimConfig, mixes, rps, caps, with_saber, repeats, jobs=0):
    """Per-row decision counts and digests of a sweep, from the compiled
    reference's run() over the sweep's cells (ref_sweep_decisions)."""
    lib = C.CDLL(REFERENCE_SO)
    f = lib.ref_sweep_decisions
    mix_ids = (C.c_int32 * len(mixes))(*[int(m[1:]) for m in mixes])
    rps_a = (C.c_double * len(rps))(*rps)
    caps_a = (C.c_int32 * max(1, len(caps)))(*caps)
    n_rows = len(mixes) * len(rps) * (len(caps) * repeats + (repeats if with_saber else 0))
    dec = np.zeros(n_rows, dtype=np.int64)
    hs = np.zeros(n_rows, dtype=np.uint64)
    rc = f(C.byref(base), mix_ids, len(mixes), rps_a, len(rps), caps_a, len(caps),
           1 if with_saber else 0, repeats, jobs, dec.ctypes.data_as(C.c_void_p),
           hs.ctypes.data_as(C.c_void_p))
    if rc != 0:
        lib.ref_last_error.restype = C.c_char_p
        raise OracleError(lib.ref_last_error().decode())
    return dec, hs


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)


def restatement_available() -> bool:
    return os.path.exists(RESTATEMENT_SO)


def fmt17(v: float) -> str:
    """%.17g, the reference's format_double (text_io.cpp:9-13)."""
    return "%.17g" % v


def decisions_to_csv(decs) -> str:
    """Byte-for-byte restatement of decisions_to_csv (scheduler.cpp:148-157)."""
    out = ["time,request_id,decision,load_before,pred_speed,req_speed\n"]
    for d in decs:
        out.append(",".join([fmt17(d.time), str(d.request_id), KIND_NAMES[d.kind],
                             str(d.load_before), fmt17(d.pred_speed) if d.has_pred else "",
                             fmt17(d.req_speed) if d.has_req else ""]) + "\n")
    return "".join(out)
