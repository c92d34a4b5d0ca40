"""The reference CLI surface on the engine (tools/saber_sim_cuda.cpp, built by
oracle/Makefile into oracle/_ref/saber_sim_cuda).

CPU: argument grammar and exit codes of proj/tools/saber_sim.cpp (usage = 2,
runtime = 3), SABER_SIM_SEED, and the `--backend ref` path pinned to the
config-1 golden decisions.csv.  GPU: every output file of `run`, `sweep` and
`calibrate` byte-identical between the CUDA backend and the reference's own
CPU functions (same binary, same writers).
"""
import hashlib
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "oracle", "_ref", "saber_sim_cuda")
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")
USL = {"family": "usl", "fit_r2": 1.0,
       "params": [99.999999999997357, 0.049999999999992085, 0.0010000000000001078]}

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="oracle/_ref/saber_sim_cuda not built")


def cli(*args, env=None):
    e = dict(os.environ)
    e.pop("SABER_SIM_SEED", None)
    if env:
        e.update(env)
    return subprocess.run([CLI, *args], capture_output=True, text=True, env=e, timeout=600)


@pytest.fixture()
def model(tmp_path):
    p = tmp_path / "usl.json"
    p.write_text(json.dumps(USL))
    return str(p)


@pytest.mark.parametrize("args,needle", [
    ([], "usage"),
    (["bogus", "--out", "x"], "unknown subcommand"),
    (["run"], "--out is required"),
    (["run", "--out", "o", "--scheduler", "fifo"], "expected saber or static"),
    (["run", "--out", "o", "--rps", "4"], "saber scheduler requires --model"),
    (["run", "--out", "o", "--rps", "-1"], "must be positive"),
    (["run", "--out", "o", "--rps", "4x"], "malformed number"),
    (["run", "--out", "o", "--frobnicate", "1"], "unknown option"),
    (["sweep", "--out", "o", "--mixes", "w1,w4"], "unknown preset"),
    (["sweep", "--out", "o", "--rps", "5-1"], "empty or backward range"),
    (["sweep", "--out", "o", "--caps", "1.5"], "positive integers"),
    (["sweep", "--out", "o", "--with-saber"], "--with-saber requires --model"),
    (["calibrate", "--out", "o", "--samples", "2", "--lmax", "50"], "insufficient distinct loads"),
])
def test_usage_errors_exit_2(tmp_path, args, needle):
    r = cli(*[a if a != "o" else str(tmp_path / "o") for a in args])
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert needle in (r.stderr + r.stdout)


def test_bad_seed_environment_is_a_usage_error(tmp_path, model):
    r = cli("run", "--out", str(tmp_path / "o"), "--model", model, "--backend", "ref",
            env={"SABER_SIM_SEED": "abc"})
    assert r.returncode == 2 and "SABER_SIM_SEED" in r.stderr


def test_ref_backend_matches_config1_golden(tmp_path, model):
    """BASELINE config 1 through the CLI (reference functions): the golden
    decisions.csv of the compiled reference (tests/golden)."""
    out = tmp_path / "r"
    r = cli("run", "--out", str(out), "--mix", "w1", "--rps", "4", "--requests", "100",
            "--scheduler", "saber", "--model", model, "--seed", "42", "--backend", "ref")
    assert r.returncode == 0, r.stderr
    g = json.load(open(GOLDEN))["config1"]
    assert hashlib.sha256((out / "decisions.csv").read_bytes()).hexdigest() == g["decisions_csv_sha256"]
    assert "goodput 0.35999999999999999" in r.stdout


def _same_files(a, b, names):
    for n in names:
        assert (a / n).read_bytes() == (b / n).read_bytes(), n


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [
    ["--mix", "w1", "--rps", "4", "--requests", "100", "--scheduler", "saber", "--seed", "42"],
    ["--mix", "w2", "--rps", "12", "--requests", "200", "--scheduler", "static", "--cap", "30",
     "--seed", "7"],
    ["--mix", "w3", "--rps", "3.5", "--requests", "60", "--scheduler", "saber", "--window", "3",
     "--tick", "0.05", "--prefill-rate", "0", "--horizon", "40", "--seed", "1234567"],
])
def test_run_outputs_byte_identical(tmp_path, model, extra):
    a, b = tmp_path / "cuda", tmp_path / "ref"
    ra = cli("run", "--out", str(a), "--model", model, *extra)
    rb = cli("run", "--out", str(b), "--model", model, "--backend", "ref", *extra)
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    assert ra.stdout == rb.stdout
    _same_files(a, b, ["records.csv", "decisions.csv", "metrics.json"])


@pytest.mark.gpu
def test_sweep_outputs_byte_identical(tmp_path, model):
    args = ["--mixes", "w1,w3", "--rps", "1-3,8", "--caps", "10-30:10", "--with-saber",
            "--model", model, "--repeats", "3", "--requests", "80", "--seed", "42"]
    a, b = tmp_path / "cuda", tmp_path / "ref"
    ra = cli("sweep", "--out", str(a), *args)
    rb = cli("sweep", "--out", str(b), "--backend", "ref", *args)
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    _same_files(a, b, ["results.csv", "summary.json"])


@pytest.mark.gpu
def test_calibrate_outputs(tmp_path):
    """Profile samples and the selected (USL) model are byte-identical; the
    logistic entry of models.json uses the device exp."""
    a, b = tmp_path / "cuda", tmp_path / "ref"
    ra = cli("calibrate", "--out", str(a), "--samples", "1000", "--seed", "42")
    rb = cli("calibrate", "--out", str(b), "--samples", "1000", "--seed", "42", "--backend", "ref")
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    assert ra.stdout == rb.stdout
    _same_files(a, b, ["samples.csv", "best_model.json"])
