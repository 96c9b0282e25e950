import json
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

from paper_2508_06041_b200 import model as M  # noqa: E402
from paper_2508_06041_b200 import quant as Q  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and libdpq_b200.so")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(autouse=True)
def _gpu_guard(request):
    if request.node.get_closest_marker("gpu") and not has_gpu():
        pytest.fail("gpu test selected on a machine without a CUDA device")


# toy config of the reference tests (tests/conftest.py:10)
TOY = M.ModelConfig(n_blocks=2, d_model=32, n_heads=4, d_ff=64, seq_cap=64)


@pytest.fixture(scope="session")
def toy_weights():
    return M.init_model(0, TOY)


@pytest.fixture(scope="session")
def toy_store(toy_weights):
    return Q.quantize_model(toy_weights, 6, 3)


@pytest.fixture(scope="session")
def golden_summary():
    with open(os.path.join(GOLDEN, "toy_summary.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_traces():
    return dict(np.load(os.path.join(GOLDEN, "toy_traces.npz")))


@pytest.fixture(scope="session")
def quant_vectors():
    return dict(np.load(os.path.join(GOLDEN, "quant_vectors.npz")))


@pytest.fixture(scope="session")
def report_setup(golden_summary):
    """The configs/toy.json model (seq_cap 256), its store, corpus tokens and
    eval chunks exactly as the reference CLI builds them."""
    cfg = M.ModelConfig.from_dict(golden_summary["config"])
    weights = M.init_model(golden_summary["seed"], cfg)
    store = Q.quantize_model(weights, golden_summary["n_bits"], golden_summary["b_min"])
    tokens = np.frombuffer(open(os.path.join(GOLDEN, "toy_corpus.txt"), "rb").read(),
                           dtype=np.uint8).astype(np.int64)
    e = golden_summary["eval"]
    chunks = [tokens[e["offset"] + i * e["seq_len"]: e["offset"] + (i + 1) * e["seq_len"]]
              for i in range(e["n_samples"])]
    return SimpleNamespace(cfg=cfg, weights=weights, store=store, tokens=tokens, chunks=chunks,
                           store_hash=golden_summary["store_hash"])


def plan_path(name):
    return os.path.join(GOLDEN, "plans", name + ".json")
