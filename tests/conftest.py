"""Test configuration. `-m gpu` tests need a B200; everything else runs on CPU.

The CPU oracle (oracle/librd_cpu.so) is loaded here as the CHECKER only.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
ORACLE_SO = os.path.join(ROOT, "oracle", "librd_cpu.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running full-size check")


def _ensure_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle")])
    return ORACLE_SO


@pytest.fixture(scope="session")
def oracle():
    from paper_2504_15302_b200.retriever import Library
    return Library(_ensure_oracle())


@pytest.fixture(scope="session")
def engine_lib():
    """The engine .so loaded for its host-side entry points (no GPU needed)."""
    from paper_2504_15302_b200.retriever import ENGINE_PATH, Library
    if os.environ.get("RD_ENGINE_PATH"):  # A/B against another build of the engine
        return Library(os.environ["RD_ENGINE_PATH"])
    if not os.path.exists(ENGINE_PATH):
        subprocess.check_call(["make", "-C", ROOT, os.path.relpath(ENGINE_PATH, ROOT)])
    return Library(ENGINE_PATH)


@pytest.fixture(scope="session")
def engine(engine_lib):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    torch.cuda.init()
    return engine_lib


def fallbacks_allowed(B, k):
    """Margin failures (queries sent to the exact fallback) a test tolerates on synthetic data. The
    residual store's keys sit up to eps_pair below the exact distances, which rank k + 15 clears at
    k <= 17 (rerank margin 14); for larger k the 32-entry candidate lists cap the margin at 32 - k,
    and a few queries per batch fall back (still exact)."""
    return 0 if k <= 17 else max(2, B // 25)
