"""Oracle and engine host arithmetic pinned against golden vectors produced by
the REFERENCE ITSELF (oracle/_ref/ref_harness, built from
/root/reference/proj/core/src by oracle/build_ref.sh; output committed as
tests/golden/ref_golden.json):
  - ragsim::Rng / derive_seed (rng.hpp:12-56): every synthetic input derives from these;
  - ragsim::check_feasible gpu_used (memory_planner.cpp:12-35) and
    queue_capacity (prefetch_timeline.cpp:79-90): the HBM reservation and the
    staging-ring depth of the placement layer.
"""
import json
import os

import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ref_golden.json")))
INT_MAX = 2147483647


@pytest.fixture(params=["oracle", "engine_lib"])
def lib(request):
    return request.getfixturevalue(request.param)


def test_rng_streams_match_reference(lib):
    for row in GOLD["rng"]:
        seed = int(row["seed"])
        for i, v in enumerate(row["outputs"]):
            assert lib.splitmix_at(seed, i) == int(v)


def test_derive_seed_matches_reference(lib):
    for row in GOLD["derive_seed"]:
        assert lib.derive_seed(int(row["master"]), int(row["stream"])) == int(row["seed"])


def test_reservation_matches_check_feasible(lib):
    for row in GOLD["placement"]:
        got = lib.llm_reservation_bytes(weight_total=row["weight_total"],
                                        kv_bytes_per_request=row["kv_bytes_per_request"],
                                        workspace_bytes_per_request=row["workspace_bytes_per_request"],
                                        w_gpu=row["w_gpu"], c_gpu=row["c_gpu"], gen_batch_size=row["batch"],
                                        decode_phase=0)
        assert got == pytest.approx(row["gpu_used"], rel=1e-12)
        assert row["gpu_mem"] - got == pytest.approx(row["gpu_slack"], rel=1e-12, abs=1.0)


@pytest.mark.parametrize("phase", ["prefill", "decode"])
def test_staging_depth_matches_queue_capacity(lib, phase):
    for row in GOLD["placement"]:
        want = row[f"queue_capacity_{phase}"]
        per_layer_off = (1.0 - row["w_gpu"]) * row["weight_total"] / row["num_layers"]
        if per_layer_off <= 0:
            assert want == INT_MAX
            continue
        used = lib.llm_reservation_bytes(weight_total=row["weight_total"],
                                         kv_bytes_per_request=row["kv_bytes_per_request"],
                                         workspace_bytes_per_request=row["workspace_bytes_per_request"],
                                         w_gpu=row["w_gpu"], c_gpu=row["c_gpu"], gen_batch_size=row["batch"],
                                         decode_phase=1 if phase == "decode" else 0, workspace_fraction=0.25)
        assert lib.staging_depth(row["gpu_mem"] - used, per_layer_off) == want


def test_reference_test_vectors(lib):
    # test_prefetch_timeline.cpp:147-167 "queue capacity from free GPU memory": free 6 GiB / 2 GiB -> 3
    GiB = 1 << 30
    used = lib.llm_reservation_bytes(weight_total=32 * GiB, w_gpu=0.5, c_gpu=1.0, gen_batch_size=4)
    assert lib.staging_depth(22 * GiB - used, 0.5 * 32 * GiB / 8) == 3
    # test_prefetch_timeline.cpp:169-189: prefill 4, decode 7
    kw = dict(weight_total=32 * GiB, workspace_bytes_per_request=GiB, w_gpu=0.5, c_gpu=1.0, gen_batch_size=4)
    assert lib.staging_depth(24 * GiB - lib.llm_reservation_bytes(**kw), 1 * GiB) == 4
    assert lib.staging_depth(24 * GiB - lib.llm_reservation_bytes(decode_phase=1, **kw), 1 * GiB) == 7
    # test_memory_planner.cpp:59-66: 8B reference point gpu_used 18 GiB
    got = lib.llm_reservation_bytes(weight_total=16 * GiB, kv_bytes_per_request=128 << 20,
                                    workspace_bytes_per_request=64 << 20, w_gpu=0.75, c_gpu=1.0, gen_batch_size=32)
    assert got == 18 * GiB


@pytest.mark.parametrize("i", range(len(GOLD["fit_power_law"])))
def test_fit_power_law_matches_reference(i):
    """include/rd_ragsim.hpp's fit_power_law / predict against the reference's own (cost_model.cpp:97-136,
    compiled by oracle/build_ref.sh) on the golden sample sets, including measured B200 T_ret rows."""
    import subprocess
    g = GOLD["fit_power_law"][i]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call(["make", "-C", root, "-s", "tests/cpp/fit_pin"])
    out = subprocess.run([os.path.join(root, "tests/cpp/fit_pin")] + [f"{b!r},{t!r}" for b, t in g["samples"]],
                         capture_output=True, text=True, check=True)
    f = json.loads(out.stdout)
    assert f["clamped"] == g["clamped"]
    for key in ("a", "c", "residual", "predict_256"):
        assert f[key] == pytest.approx(g[key], rel=1e-12, abs=1e-15), key
