"""Shared test setup: repo on sys.path, the ``gpu`` marker, golden-fixture loaders."""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np
import pytest

REPO = pathlib.Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu under gpurun)")


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


def load_npz(name):
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_kernels():
    return load_json("kernels.json")


@pytest.fixture(scope="session")
def golden_runs():
    return load_json("runs.json"), load_npz("runs.npz")


@pytest.fixture(scope="session")
def golden_exchange():
    return load_json("exchange.json"), load_npz("exchange.npz")


@pytest.fixture(scope="session")
def golden_random():
    return load_json("random.json"), load_npz("random.npz")


@pytest.fixture(scope="session")
def golden_kats():
    return load_json("kats.json")
