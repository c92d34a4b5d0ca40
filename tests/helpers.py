"""Shared test helpers: build the same case for the engine (api types) and the
CPU checkers (oracle structs)."""
import math
import random

import numpy as np

import oracle as O
import paper_2506_19677_b200 as S

CAL_USL = (0, (99.999999999997357, 0.049999999999992085, 0.0010000000000001078))
CAL_LOG = (1, (200.0, 0.046625169303483933, -6.3061840170033063))
CAL_LIN = (2, (-1.292318089365694, 72.295958816519274, 0.0))
GT = (0, (100.0, 0.05, 0.001))


def sim_config(mix="w1", rps=4.0, n=100, seed=42, mode=0, cap=0, window=8, tick=0.01,
               model=CAL_USL, gt=GT, prefill_rate=2000.0, jitter=0.2, horizon=None,
               workload_seed=None):
    cfg = S.SimConfig()
    cfg.workload = S.WorkloadSpec(S.preset_mix(mix) if isinstance(mix, str) else mix, rps, n,
                                  seed if workload_seed is None else workload_seed, jitter)
    cfg.scheduler = S.SchedulerConfig(mode, window, tick, cap)
    cfg.model = S.SpeedModel(model[0], tuple(model[1])) if (model is not None and mode == 0) else None
    cfg.engine = S.EngineConfig(S.SpeedModel(gt[0], tuple(gt[1])), prefill_rate)
    cfg.horizon = horizon
    cfg.seed = seed
    return cfg


def orc_config(cfg: "S.SimConfig"):
    mix = {S.TASK_INDEX[k]: v for k, v in cfg.workload.mix.proportions.items()}
    m = cfg.model
    c = O.make_config(mix=mix, rps=cfg.workload.rps, n=cfg.workload.num_requests, seed=cfg.seed,
                      workload_seed=cfg.workload.seed, mode=cfg.scheduler.mode,
                      cap=cfg.scheduler.static_batch_size, window=cfg.scheduler.window_size,
                      tick=cfg.scheduler.tick,
                      model=(m.family, m.params) if m is not None else None,
                      gt=(cfg.engine.ground_truth.family, cfg.engine.ground_truth.params),
                      prefill_rate=cfg.engine.prefill_rate, jitter=cfg.workload.length_jitter,
                      horizon=cfg.horizon)
    return c


def orc_requests(reqs):
    out = []
    for r in reqs:
        q = O.OrcRequest()
        q.arrival_time = r.arrival_time
        q.sla_seconds = r.sla_seconds
        q.deadline = r.deadline
        q.input_tokens = r.input_tokens
        q.max_output_tokens = r.max_output_tokens
        q.task = S.TASK_INDEX.get(r.task, -1)
        out.append(q)
    return out


ROW_FIELDS_EXACT = ["completed", "met", "decisions", "decision_hash"]
COUNTERS = ["ticks", "passes", "decode_updates", "prefill_updates", "refresh_entries",
            "gate_candidates", "ledger_scanned", "rng_draws"]


def same_float(a, b):
    return (math.isnan(a) and math.isnan(b)) or a == b


def compare_row(row, o, counters=True):
    """Engine row vs oracle orc_traj_out: bit-exact on every field."""
    errs = []
    for f in ROW_FIELDS_EXACT:
        if int(row[f]) != int(getattr(o, f)):
            errs.append(f"{f}: {int(row[f])} != {int(getattr(o, f))}")
    for f in ("goodput", "ratio_mean", "ratio_std", "cv"):
        if not same_float(float(row[f]), float(getattr(o, f))):
            errs.append(f"{f}: {float(row[f])!r} != {float(getattr(o, f))!r}")
    if list(row["n_kind"]) != list(o.n_kind):
        errs.append(f"n_kind {list(row['n_kind'])} != {list(o.n_kind)}")
    if list(row["issued_by_task"]) != list(o.issued_by_task):
        errs.append("issued_by_task")
    if list(row["met_by_task"]) != list(o.met_by_task):
        errs.append("met_by_task")
    if counters and o.ticks >= 0:
        for f in COUNTERS:
            if int(row[f]) != int(getattr(o, f)):
                errs.append(f"{f}: {int(row[f])} != {int(getattr(o, f))}")
    return errs


def random_configs(count, seed=1234, n_choices=(1, 7, 50, 100, 130), allow_logistic=True,
                   windows=(1, 2, 3, 8, 8, 16)):
    rng = random.Random(seed)
    out = []
    models = [CAL_USL, CAL_LIN] + ([CAL_LOG, (1, (90.0, 0.06, 35.0))] if allow_logistic else []) + \
             [(0, (100.0, 0.05, 0.001)), (0, (80.0, 0.12, 0.002))]
    for _ in range(count):
        mode = rng.choice([0, 0, 1])
        out.append(sim_config(
            mix=rng.choice(["w1", "w2", "w3"]), rps=rng.choice([0.5, 1, 2, 4, 8, 15, 20, 35]),
            n=rng.choice(n_choices), seed=rng.randrange(1 << 40), mode=mode,
            cap=rng.choice([1, 3, 10, 40, 100]), window=rng.choice(windows),
            tick=rng.choice([0.01, 0.01, 0.05, 0.003]), model=rng.choice(models),
            gt=rng.choice([GT, (0, (80.0, 0.12, 0.002)), (1, (120.0, 0.1, 30.0))]),
            prefill_rate=rng.choice([2000.0, 2000.0, 0.0, 500.0]), jitter=rng.choice([0.2, 0.0, 0.5])))
    return out


def quantiles_from_records(records):
    """The reference's cdf (metrics.cpp:61-85) over all issued requests:
    smallest latency x with (#latencies <= x) / issued >= p."""
    issued = len(records)
    lat = sorted(r.completion_time - r.arrival_time for r in records if not math.isnan(r.completion_time))
    out = []
    for p in (0.5, 0.9, 0.99):
        got = float("nan")
        for i, x in enumerate(lat):
            if (i + 1) / issued >= p:
                got = x
                break
        out.append(got)
    return out
