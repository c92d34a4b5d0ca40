"""The reference CLI surface on the engine:
paper_2506_19677_b200/bin/saber_sim_b200 — the engine's own command-line tool,
linked only against libsaber_b200.so, writing every file with its own writers.

CPU: the argument grammar and exit codes of proj/tools/saber_sim.cpp (usage =
2, runtime = 3), SABER_SIM_SEED, and a loud failure without a device.  GPU:
every output file of `run`, `sweep` and `calibrate` byte-identical to the
reference's own tool (oracle/_ref/saber_sim_ref: the reference library's
calibrate / run / sweep and writers behind the same flags), and `run --trace`
(trace CSV replay) identical to the generated run it was written from.
"""
import hashlib
import json
import os
import subprocess

import pytest

import paper_2506_19677_b200 as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2506_19677_b200", "bin", "saber_sim_b200")
REF = os.path.join(ROOT, "oracle", "_ref", "saber_sim_ref")
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")
USL = {"family": "usl", "fit_r2": 1.0,
       "params": [99.999999999997357, 0.049999999999992085, 0.0010000000000001078]}


def _run(binary, *args, env=None):
    e = dict(os.environ)
    e.pop("SABER_SIM_SEED", None)
    if env:
        e.update(env)
    return subprocess.run([binary, *args], capture_output=True, text=True, env=e, timeout=900)


def cli(*args, env=None):
    return _run(CLI, *args, env=env)


def ref(*args, env=None):
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/saber_sim_ref not built")
    return _run(REF, *args, env=env)


@pytest.fixture()
def model(tmp_path):
    p = tmp_path / "usl.json"
    p.write_text(json.dumps(USL))
    return str(p)


def test_cli_links_only_the_engine():
    out = subprocess.run(["ldd", CLI], capture_output=True, text=True).stdout
    assert "libsaber_b200.so" in out and "saber_ref" not in out


@pytest.mark.parametrize("args,needle", [
    ([], "usage"),
    (["bogus", "--out", "x"], "unknown subcommand"),
    (["run"], "--out is required"),
    (["run", "--out", "o", "--scheduler", "fifo"], "expected saber or static"),
    (["run", "--out", "o", "--rps", "4"], "saber scheduler requires --model"),
    (["run", "--out", "o", "--scheduler", "static"], "static scheduler requires --cap"),
    (["run", "--out", "o", "--rps", "-1"], "must be positive"),
    (["run", "--out", "o", "--rps", "4x"], "malformed number"),
    (["run", "--out", "o", "--frobnicate", "1"], "unknown option"),
    (["run", "--out", "o", "--model", "/nonexistent.json"], "--model"),
    (["run", "--out", "o", "--mix", "/nonexistent.json"], "--mix"),
    (["run", "--out", "o", "--config", "/nonexistent.json"], "--config"),
    (["sweep", "--out", "o", "--mixes", "w1,w4"], "unknown preset"),
    (["sweep", "--out", "o", "--rps", "5-1"], "empty or backward range"),
    (["sweep", "--out", "o", "--rps", "1,,2"], "malformed number"),
    (["sweep", "--out", "o", "--caps", "1.5"], "positive integers"),
    (["sweep", "--out", "o", "--with-saber"], "--with-saber requires --model"),
    (["calibrate", "--out", "o", "--samples", "2", "--lmax", "50"], "insufficient distinct loads"),
    (["calibrate", "--out", "o", "--jitter", "1.5"], "[0, 1]"),
])
def test_usage_errors_exit_2(tmp_path, args, needle):
    r = cli(*[a if a != "o" else str(tmp_path / "o") for a in args])
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert needle in (r.stderr + r.stdout)


def test_reference_tool_agrees_on_usage_errors(tmp_path, model):
    """Same exit code from the reference's own tool for a sample of the cases."""
    for args in (["run", "--out", str(tmp_path / "o"), "--scheduler", "fifo"],
                 ["sweep", "--out", str(tmp_path / "o"), "--rps", "5-1"],
                 ["calibrate", "--out", str(tmp_path / "o"), "--samples", "2"]):
        assert ref(*args).returncode == cli(*args).returncode == 2


def test_bad_seed_environment_is_a_usage_error(tmp_path, model):
    r = cli("run", "--out", str(tmp_path / "o"), "--model", model, env={"SABER_SIM_SEED": "abc"})
    assert r.returncode == 2 and "SABER_SIM_SEED" in r.stderr


def test_bad_model_json_is_a_usage_error(tmp_path):
    p = tmp_path / "m.json"
    p.write_text('{"family": "cubic", "params": [1, 2, 3]}')
    r = cli("run", "--out", str(tmp_path / "o"), "--model", str(p))
    assert r.returncode == 2 and "unknown model family: cubic" in r.stderr


@pytest.mark.skipif(S.device_count() > 0, reason="no-GPU behaviour")
def test_runtime_failure_without_a_device_exits_3(tmp_path, model):
    r = cli("run", "--out", str(tmp_path / "o"), "--model", model, "--mix", "w1")
    assert r.returncode == 3 and "no CUDA device" in r.stderr
    assert not (tmp_path / "o" / "records.csv").exists()


def test_reference_tool_matches_config1_golden(tmp_path, model):
    """The baseline tool itself: BASELINE config 1 equals the golden fixture."""
    out = tmp_path / "r"
    r = ref("run", "--out", str(out), "--mix", "w1", "--rps", "4", "--requests", "100",
            "--scheduler", "saber", "--model", model, "--seed", "42")
    assert r.returncode == 0, r.stderr
    g = json.load(open(GOLDEN))["config1"]
    assert hashlib.sha256((out / "decisions.csv").read_bytes()).hexdigest() == g["decisions_csv_sha256"]


def _same_files(a, b, names):
    for n in names:
        assert (a / n).read_bytes() == (b / n).read_bytes(), n


RUN_CASES = [
    ["--mix", "w1", "--rps", "4", "--requests", "100", "--scheduler", "saber", "--seed", "42"],
    ["--mix", "w2", "--rps", "12", "--requests", "200", "--scheduler", "static", "--cap", "30",
     "--seed", "7"],
    ["--mix", "w3", "--rps", "3.5", "--requests", "60", "--scheduler", "saber", "--window", "3",
     "--tick", "0.05", "--prefill-rate", "0", "--horizon", "40", "--seed", "1234567"],
    ["--mix", "w1", "--rps", "30", "--requests", "250", "--scheduler", "saber", "--horizon", "5",
     "--seed", "3"],
    # the wide kernel: more requests than the register masks, a 24-wide window
    ["--mix", "w2", "--rps", "15", "--requests", "700", "--scheduler", "saber", "--window", "24",
     "--seed", "5"],
]


@pytest.mark.gpu
@pytest.mark.parametrize("extra", RUN_CASES)
def test_run_outputs_byte_identical(tmp_path, model, extra):
    a, b = tmp_path / "b200", tmp_path / "ref"
    ra = cli("run", "--out", str(a), "--model", model, *extra)
    rb = ref("run", "--out", str(b), "--model", model, *extra)
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    assert ra.stdout == rb.stdout
    _same_files(a, b, ["records.csv", "decisions.csv", "metrics.json"])


@pytest.mark.gpu
def test_run_with_config_file_and_env_seed(tmp_path, model):
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"workload": {"mix": {"code_qna": 0.5, "code_translation": 0.5},
                                            "rps": 6.0, "num_requests": 90, "seed": 11},
                               "scheduler": {"mode": "saber", "window_size": 5},
                               "model": USL, "seed": 11}))
    for env in (None, {"SABER_SIM_SEED": "99"}):
        a, b = tmp_path / f"b200{env is None}", tmp_path / f"ref{env is None}"
        ra = cli("run", "--out", str(a), "--config", str(cfg), env=env)
        rb = ref("run", "--out", str(b), "--config", str(cfg), env=env)
        assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
        _same_files(a, b, ["records.csv", "decisions.csv", "metrics.json"])


@pytest.mark.gpu
def test_sweep_outputs_byte_identical(tmp_path, model):
    args = ["--mixes", "w3,w1", "--rps", "1-3,8", "--caps", "10-30:10", "--with-saber",
            "--model", model, "--repeats", "3", "--requests", "80", "--seed", "42"]
    a, b = tmp_path / "b200", tmp_path / "ref"
    ra = cli("sweep", "--out", str(a), *args)
    rb = ref("sweep", "--out", str(b), *args)
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    assert ra.stdout == rb.stdout
    _same_files(a, b, ["results.csv", "summary.json"])


@pytest.mark.gpu
def test_calibrate_outputs(tmp_path):
    """Profile samples and the selected (USL) model are byte-identical; the
    logistic entry of models.json uses the device exp."""
    a, b = tmp_path / "b200", tmp_path / "ref"
    ra = cli("calibrate", "--out", str(a), "--samples", "1000", "--seed", "42")
    rb = ref("calibrate", "--out", str(b), "--samples", "1000", "--seed", "42")
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    assert ra.stdout == rb.stdout
    _same_files(a, b, ["samples.csv", "best_model.json"])
    ma, mb = json.load(open(a / "models.json")), json.load(open(b / "models.json"))
    assert [f["family"] for f in ma["fits"]] == [f["family"] for f in mb["fits"]]
    assert [f["ok"] for f in ma["fits"]] == [f["ok"] for f in mb["fits"]]
    for fa, fb in zip(ma["fits"], mb["fits"]):
        if fa["family"] != "logistic":
            assert fa == fb


@pytest.mark.gpu
def test_trace_replay_equals_generated_run(tmp_path, model):
    """run --trace (workload.cpp:97-138 ingestion): the trace written from a
    generated workload replays to the same records, decisions and metrics."""
    spec = S.WorkloadSpec(S.preset_mix("w2"), 9.0, 150, 5, 0.2)
    trace = tmp_path / "t.csv"
    trace.write_text(S.trace_to_csv(S.generate(spec)))
    a, b = tmp_path / "trace", tmp_path / "gen"
    common = ["--scheduler", "saber", "--model", model, "--seed", "5"]
    ra = cli("run", "--out", str(a), "--trace", str(trace), *common)
    rb = ref("run", "--out", str(b), "--mix", "w2", "--rps", "9", "--requests", "150", *common)
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    _same_files(a, b, ["records.csv", "decisions.csv", "metrics.json"])
