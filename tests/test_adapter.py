"""The reference-side drop-in (include/saber_cuda_adapter.hpp): the reference's
own API and saber::cuda::* on the same inputs, compared field by field and
byte by byte (decisions.csv, records.csv, metrics.json, results.csv,
summary.json) by oracle/_ref/adapter_check."""
import os
import subprocess

import pytest

import paper_2506_19677_b200 as S

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "adapter_check")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/adapter_check not built")


@pytest.mark.skipif(S.device_count() > 0, reason="no-GPU behaviour")
def test_adapter_fails_loudly_without_a_device():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_adapter_matches_reference_byte_for_byte():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER OK" in r.stdout
