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


def import_lopec(allow_reference_tree: bool = False):
    """Import the reference package for the Machine drop-in tests.

    The drop-in keeps lopec's frontend and host plan, so its tests need lopec
    itself: the copy installed under baseline/_ref (which travels to the GPU box)
    or, in the build container only, the read-only reference tree.
    """
    try:
        import lopec  # noqa: F401
        return True
    except ImportError:
        pass
    cands = [REPO / "baseline" / "_ref"]
    if allow_reference_tree:
        cands.append(pathlib.Path("/root/reference/pkg/src"))
    for c in cands:
        if (c / "lopec" / "__init__.py").exists():
            sys.path.insert(0, str(c))
            try:
                import lopec  # noqa: F401
                return True
            except ImportError:
                sys.path.remove(str(c))
    return False
