"""Shared test setup: the ``gpu`` marker, repo-root imports, golden fixtures."""

import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt", encoding="utf-8") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_traces():
    return load_golden("traces.json.gz")


@pytest.fixture(scope="session")
def golden_grid():
    return load_golden("decomp_grid.json.gz")


@pytest.fixture(scope="session")
def golden_random_instances():
    return load_golden("random_insts.json.gz")


@pytest.fixture(scope="session")
def golden_loader():
    return load_golden("loader.json.gz")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(params=["fused", "multipass"])
def loader_pipeline(request, monkeypatch):
    """Run a loader test through the single-pass loader and through the multi-pass one
    (CT_JSONL_MULTIPASS, read by ct_jsonl_parse on every call)."""
    if request.param == "multipass":
        monkeypatch.setenv("CT_JSONL_MULTIPASS", "1")
    else:
        monkeypatch.delenv("CT_JSONL_MULTIPASS", raising=False)
    return request.param
