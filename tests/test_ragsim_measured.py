"""SURVEY §8(f) row 1 in depth: the reference's own simulator (unmodified simulator.cpp / scheduler.cpp /
cost_model.cpp ..., linked by oracle/build_ref_sim.sh with -Wl,--wrap on retrieval_time and
choose_retrieval_batch) run on the B200 + C2 scenario with its retrieval stage modelled (the
reference's formula) and measured (profiles/round2_measured_tret.json: rd_search on one B200).
Skipped where the harness was not built (it compiles from /root/reference, absent on the GPU box)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "ragsim_measured")
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.json")))


@pytest.fixture(scope="module")
def sim():
    if not os.path.exists(HARNESS):
        if not os.path.isdir("/root/reference/proj/core/src"):
            pytest.skip("reference simulator harness not built (needs /root/reference)")
        subprocess.check_call([os.path.join(ROOT, "oracle", "build_ref_sim.sh")])
    env = dict(os.environ, RAGSIM_TRET=os.path.join(ROOT, "profiles", "round2_measured_tret.json"))
    out = subprocess.run([HARNESS, os.path.join(ROOT, "oracle", "ragsim_b200_c2.json")], capture_output=True,
                         text=True, env=env, timeout=300, check=True)
    return json.loads(out.stdout)


def test_modelled_run_is_the_reference_formula(sim):
    m = sim["modelled"]
    assert m["retrieval_time_calls"] > 0 and m["requests"] > 0
    # every modelled retrieval batch lasts retrieval_time(P, db) for one of the policy's residencies
    db_search, db_load, parts = 0.055878, 0.614655, 32
    allowed = {round(P * db_search + (parts - P) * (db_load + db_search), 9)
               for P in {e["resident_partitions"] for e in m["policy"]}}
    assert round(m["retrieval_stage"]["max"], 9) in allowed


def test_measured_retrieval_replaces_the_formula(sim):
    m, x = sim["modelled"], sim["measured"]
    assert x["retrieval_time_calls"] > 0
    # a retrieval batch on the B200 engine is milliseconds (the table's range), the modelled CPU
    # search seconds; end-to-end latency cannot get worse
    assert 1e-4 < x["retrieval_stage"]["p50"] < 0.5 < m["retrieval_stage"]["p50"]
    assert x["latency"]["average"] <= m["latency"]["average"]
    assert len(x["fits"]) == 5 and all(f["a"] > 0 for f in x["fits"])
