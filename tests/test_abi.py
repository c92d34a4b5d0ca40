"""CPU: the C-ABI library builds, loads, exports exactly what include/saber_cuda.h
declares, its structs match the ctypes mirror, and it validates inputs with
the reference's error semantics — and never falls back to the CPU."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

import paper_2506_19677_b200 as S
from paper_2506_19677_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "saber_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(saber_cuda_\w+)\s*\(", src)))


def test_header_declares_the_python_symbol_table():
    assert declared_functions() == sorted(name for name, _, _ in N.SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(N.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (saber_cuda_\w+)", out))
    assert exported == set(declared_functions())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


STRUCTS = ["saber_model", "saber_mix", "saber_traj_row", "saber_decision", "saber_sweep_desc",
           "saber_mix_summary", "saber_sweep_out", "saber_sweep_buffers", "saber_request",
           "saber_traj_spec", "saber_run_batch_desc", "saber_run_batch_out", "saber_fit_desc",
           "saber_fit_out", "saber_request_state", "saber_workload_spec", "saber_mc_desc",
           "saber_mc_out", "saber_profile_spec", "saber_profile_desc", "saber_profile_out"]


def test_struct_layouts_match_header():
    prog = "#include <stdio.h>\n#include <stddef.h>\n#include \"saber_cuda.h\"\nint main(){\n"
    for s in STRUCTS:
        prog += f'printf("{s} %zu\\n", sizeof({s}));\n'
    for name, _ in N.saber_traj_row._fields_:
        prog += f'printf("row.{name} %zu\\n", offsetof(saber_traj_row, {name}));\n'
    for name, _ in N.saber_sweep_desc._fields_:
        prog += f'printf("desc.{name} %zu\\n", offsetof(saber_sweep_desc, {name}));\n'
    for name, _ in N.saber_traj_spec._fields_:
        prog += f'printf("spec.{name} %zu\\n", offsetof(saber_traj_spec, {name}));\n'
    for name, _ in N.saber_run_batch_out._fields_:
        prog += f'printf("rbo.{name} %zu\\n", offsetof(saber_run_batch_out, {name}));\n'
    for name, _ in N.saber_request_state._fields_:
        prog += f'printf("rst.{name} %zu\\n", offsetof(saber_request_state, {name}));\n'
    prog += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(l.split() for l in lines if l)
    for s in STRUCTS:
        assert int(got[s]) == C.sizeof(getattr(N, s)), s
    for prefix, cls in (("row", N.saber_traj_row), ("desc", N.saber_sweep_desc),
                        ("spec", N.saber_traj_spec), ("rbo", N.saber_run_batch_out),
                        ("rst", N.saber_request_state)):
        for name, _ in cls._fields_:
            assert int(got[f"{prefix}.{name}"]) == getattr(cls, name).offset, (prefix, name)


def test_abi_version():
    assert N.lib().saber_cuda_abi_version() == N.ABI_VERSION == 2


def test_validation_mirrors_reference_errors():
    """simloop.cpp:130-136 / types.cpp:94-100: invalid_argument before any work."""
    base = S.SimConfig()
    with pytest.raises(S.InvalidArgument, match="empty grid"):
        S.sweep(S.SweepGrid(["w1"], [1.0], [], False), base)
    with pytest.raises(S.InvalidArgument, match="requires a model"):
        S.sweep(S.SweepGrid(["w1"], [1.0], [], True), base)
    with pytest.raises(S.InvalidArgument, match="unknown mix preset"):
        S.sweep(S.SweepGrid(["w9"], [1.0], [10], False), base)
    for grid in (S.SweepGrid(["w1", "w1"], [1.0], [10], False),
                 S.SweepGrid(["w1"], [2.0, 2.0], [10], False),
                 S.SweepGrid(["w1"], [1.0], [10, 20, 10], False)):
        with pytest.raises(S.InvalidArgument, match="duplicate"):
            S.sweep(grid, base)
    bad = S.SimConfig()
    bad.scheduler.tick = 0.0
    bad.model = S.SpeedModel(0, (100, 0.05, 0.001))
    with pytest.raises(S.InvalidArgument, match="tick"):
        S.run_batch([bad])
    bad = S.SimConfig()
    bad.scheduler.mode = S.SchedulerMode.Static
    with pytest.raises(S.InvalidArgument, match="positive batch size"):
        S.run_batch([bad])
    bad = S.SimConfig()  # saber mode without a model
    with pytest.raises(S.InvalidArgument, match="requires a speed model"):
        S.run_batch([bad])
    bad = S.SimConfig(model=S.SpeedModel(0, (100, 0.05, 0.001)))
    bad.workload.length_jitter = 1.0
    with pytest.raises(S.InvalidArgument, match="length_jitter"):
        S.run_batch([bad])
    with pytest.raises(S.DomainError):
        S.predict(S.SpeedModel(0, (100, 0, 0)), 0)


def test_predict_table_known_answers():
    """estimator.cpp:16-31 via the host table builder the engine uses."""
    assert S.predict(S.SpeedModel(0, (100, 0, 0)), 17) == 100
    assert S.predict(S.SpeedModel(0, (100, 0.1, 0)), 2) == 100 / 1.1
    assert S.predict(S.SpeedModel(0, (100, 0.05, 0.001)), 50) == 100 / 5.9
    assert S.predict(S.SpeedModel(1, (120, 0.1, 30)), 30) == 60
    assert S.predict(S.SpeedModel(2, (-2, 10)), 2) == 6
    assert S.predict(S.SpeedModel(2, (-2, 10)), 100) == 1e-6
    assert S.max_speed(S.SpeedModel(1, (120, 0.1, 30))) == pytest.approx(113.74157243058988, abs=1e-12)


@pytest.mark.skipif(S.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_a_device():
    cfg = S.SimConfig(model=S.SpeedModel(0, (100, 0.05, 0.001)))
    with pytest.raises(S.SaberError, match="SABER_ECUDA"):
        S.run_batch([cfg])
    with pytest.raises(S.SaberError, match="SABER_ECUDA"):
        S.sweep(S.SweepGrid(["w1"], [1.0], [10], False), S.SimConfig())


def test_sweep_row_count_and_keys():
    grid = S.SweepGrid(["w1", "w3"], [2.0, 15.0], [10, 30], True)
    base = S.SimConfig(repeats=3, seed=42)
    d = N.saber_sweep_desc()
    d.n_mixes, d.n_rps, d.n_caps, d.with_saber, d.repeats = 2, 2, 2, 1, 3
    assert N.lib().saber_cuda_sweep_rows(C.byref(d)) == 2 * 2 * (2 * 3 + 3)
    keys = S.sweep_row_keys(grid, base)
    assert len(keys) == 36
    assert keys[0] == ("w1", 2.0, S.SchedulerMode.Static, 10, 42)
    assert keys[6] == ("w1", 2.0, S.SchedulerMode.Saber, 0, 42)
    assert keys[9] == ("w1", 15.0, S.SchedulerMode.Static, 10, 42)
