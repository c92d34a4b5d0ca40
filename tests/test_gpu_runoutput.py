"""The full RunOutput of run() / run_with_requests() and generate() from the
engine (ABI 2), against the compiled reference (oracle/_ref): every generated
Request field bit-exact, the final request states (admit / completion times,
tiers, fluid progress at a horizon cut, recorded required speed) and the
per-task MetricsReport (issued, goodput, cdf() points, metrics.cpp:61-140)
restated here from the reference's own records."""
import math

import numpy as np
import pytest

import oracle as O
import paper_2506_19677_b200 as S
from helpers import orc_config, orc_requests, sim_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not O.reference_available():
        pytest.skip("oracle/_ref not built")
    return O.Oracle("reference")


def _cdf(lat_sorted, issued):
    """metrics.cpp:61-85 restated: one point per distinct latency."""
    pts = []
    for i, x in enumerate(lat_sorted):
        if i + 1 == len(lat_sorted) or lat_sorted[i + 1] != x:
            pts.append((x, (i + 1) / issued))
    return pts


def _expected_per_task(records, names):
    out = {}
    for name in sorted(set(names)):
        idx = [i for i, nm in enumerate(names) if nm == name]
        lat = sorted(records[i].completion_time - records[i].arrival_time for i in idx
                     if not math.isnan(records[i].completion_time))
        met = sum(1 for i in idx if not math.isnan(records[i].completion_time)
                  and records[i].completion_time - records[i].arrival_time <= records[i].sla)
        out[name] = (len(idx), met / len(idx), _cdf(lat, len(idx)))
    return out


def _same(a, b):
    return (a is None and (b is None or math.isnan(b))) or a == b


@pytest.mark.parametrize("mix,rps,n,seed,jit", [("w1", 4.0, 100, 42, 0.2), ("w2", 17.0, 333, 7, 0.0),
                                                ("w3", 0.3, 57, 2**63 + 5, 0.9)])
def test_generate_matches_reference(ref, mix, rps, n, seed, jit):
    cfg = sim_config(mix, rps, n, seed, jitter=jit)
    got = S.generate(cfg.workload)
    want = ref.generate(orc_config(cfg))
    assert len(got) == len(want) == n
    for i, (g, w) in enumerate(zip(got, want)):
        assert g.id == i
        assert (g.arrival_time, g.sla_seconds, g.deadline, g.input_tokens, g.max_output_tokens) == \
            (w.arrival_time, w.sla_seconds, w.deadline, w.input_tokens, w.max_output_tokens), i
        assert S.TASK_INDEX[g.task] == w.task


CASES = [
    dict(mix="w1", rps=4.0, n=100, seed=42),                                   # config 1
    dict(mix="w1", rps=30.0, n=200, seed=3, horizon=4.0),                      # SABER cut mid-run
    dict(mix="w3", rps=8.0, n=150, seed=11, mode=1, cap=30, horizon=3.3,
         prefill_rate=400.0),                                                  # static, slots in prefill
    dict(mix="w2", rps=12.0, n=64, seed=5, mode=1, cap=10),                    # static to completion
]


@pytest.mark.parametrize("case", CASES)
def test_run_output_matches_reference(ref, case):
    cfg = sim_config(**case)
    out = S.run(cfg)
    r = ref.run(orc_config(cfg), records=True, decisions=True)
    n = cfg.workload.num_requests
    assert len(out.records) == len(out.requests) == n
    names = [O.TASK_NAMES[x.task] for x in r.records]
    for i, (q, rec, w) in enumerate(zip(out.requests, out.records, r.records)):
        assert q.task == rec.task == names[i]
        assert q.arrival_time == w.arrival_time and q.max_output_tokens == w.max_output_tokens
        assert _same(q.admit_time, w.admit_time) and _same(q.completion_time, w.completion_time), i
        assert q.demoted == bool(w.demoted) and rec.final_tier == ("low" if w.demoted else "high")
        done = not math.isnan(w.completion_time)
        assert rec.met_sla == (done and w.completion_time - w.arrival_time <= w.sla)
        if done:
            assert q.state == S.RequestState.Completed and q.generated_tokens == q.max_output_tokens
        elif q.admit_time is not None:
            assert q.state == S.RequestState.Executing
            assert 0.0 <= q.generated_tokens < q.max_output_tokens
        else:
            assert q.state in (S.RequestState.QueuedHigh, S.RequestState.QueuedLow)
            assert q.generated_tokens == 0.0 and q.recorded_required_speed is None
        if q.admit_time is not None:  # Engine::admit: required_speed(r, now), generated == 0
            want = math.inf if q.admit_time >= q.deadline else \
                (q.max_output_tokens - 0.0) / (q.deadline - q.admit_time)
            assert q.recorded_required_speed == want
    assert out.metrics.goodput == r.out.goodput
    exp = _expected_per_task(r.records, names)
    assert set(out.metrics.per_task) == set(exp)
    for name, (issued, gp, pts) in exp.items():
        tm = out.metrics.per_task[name]
        assert (tm.issued, tm.goodput) == (issued, gp), name
        assert tm.cdf_points == pts, name
    assert [(d.time, d.request_id, d.kind) for d in out.decisions] == \
        [(d.time, d.request_id, d.kind) for d in r.decisions]


def test_replay_custom_task_names(ref):
    """Per-task metrics keyed by names outside the catalog (run_with_requests)."""
    cfg = sim_config("w1", 25.0, 120, 9)
    reqs = S.generate(cfg.workload)
    for i in range(0, len(reqs), 3):
        reqs[i].task = "alpha" if i % 2 else "zeta"
    out = S.run_with_requests(cfg, reqs)
    r = ref.run_with_requests(orc_config(cfg), orc_requests(reqs), records=True)
    names = [q.task for q in reqs]
    exp = _expected_per_task(r.records, names)
    assert list(out.metrics.per_task) == sorted(exp)
    for name, (issued, gp, pts) in exp.items():
        tm = out.metrics.per_task[name]
        assert (tm.issued, tm.goodput, tm.cdf_points) == (issued, gp, pts), name


def test_decision_buffer_grows_to_the_log():
    """A trajectory with more decisions than the initial buffer reruns with a
    buffer of exactly its log length instead of failing."""
    cfg = sim_config("w1", 40.0, 300, 1)
    res = S.run_batch([cfg], records=True, decisions=True, decision_cap=64)
    assert len(res.decisions[0]) == int(res.rows[0]["decisions"]) > 64
