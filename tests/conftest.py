"""Shared pytest setup: the `gpu` marker, repo root on sys.path, golden loaders."""

from __future__ import annotations

import functools
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
TESTS = Path(__file__).resolve().parent
GOLDEN = TESTS / "golden"
for p in (str(ROOT), str(TESTS)):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100) device")


@functools.lru_cache(maxsize=None)
def load_golden(name: str):
    return json.loads((GOLDEN / name).read_text())


def unhex(s: str) -> float:
    return float.fromhex(s)


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def dev():
    if not cuda_available():
        pytest.skip("no CUDA device")
    import torch

    return torch.device("cuda:0")
