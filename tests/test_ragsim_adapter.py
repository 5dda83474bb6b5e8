"""The C++ ragsim-side adapter (include/rd_ragsim.hpp): RAII index, status -> exception
mapping, choose_retrieval_batch (scheduler.cpp:80-83), the power-law cost fit the
profiler consumes (cost_model.cpp:97-136), and a retrieval worker driven by real
searches with a between-batch reconfiguration (simulator.cpp:328-368). The same
driver links against the oracle (CPU) and the engine (GPU)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(target, *args):
    subprocess.check_call(["make", "-C", ROOT, "-s", target])
    out = subprocess.run([os.path.join(ROOT, target), *map(str, args)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr + out.stdout
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_adapter_on_oracle():
    r = _run("tests/cpp/ragsim_adapter_cpu", 20000, 128, 64, 200)
    assert r["backend"] == "cpu-oracle" and r["failures"] == 0
    assert r["batches"] >= 1 and r["t_ret_fit"]["a"] > 0


@pytest.mark.gpu
def test_adapter_on_engine():
    """The same driver over the engine and over the oracle: identical top-k for every request
    (digest of all ids), whatever batches the worker formed on each."""
    args = (200000, 768, 1024, 400)
    r = _run("tests/cpp/ragsim_adapter_b200", *args)
    assert r["backend"] == "b200-sm100a" and r["failures"] == 0
    o = _run("tests/cpp/ragsim_adapter_cpu", *args)
    assert o["backend"] == "cpu-oracle" and o["failures"] == 0
    assert r["results_digest"] == o["results_digest"]
