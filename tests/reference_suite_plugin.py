"""pytest plugin: run the reference's own test suite with the GPU Machine swapped in.

Loaded with ``-p reference_suite_plugin`` by tests/test_gpu_reference_suite.py before
the reference's test modules are imported, so their ``from lopec.runtime import
Machine`` (and ``lopec.cli``'s) bind the drop-in: every ``Machine(check, config,
field)`` the unmodified reference tests build runs its launches and halo exchanges
on the GPU (``paper_1502_03504_b200.machine``, fp64 -- the reference's precision).
Each construction is counted and the count is written to ``$LOPE_SUITE_REPORT``
so the runner can prove the swap took effect.
"""

import json
import os

_COUNT = {"machines": 0, "devices": None}


def pytest_configure(config):
    import lopec
    import lopec.cli
    import lopec.runtime

    from paper_1502_03504_b200 import machine as M

    base = M.machine_class()          # subclass of the reference Machine, created first
    devices = os.environ.get("LOPE_SUITE_DEVICES")
    devs = [int(x) for x in devices.split(",")] if devices else None
    _COUNT["devices"] = devs

    class GpuMachineForSuite(base):
        def __init__(self, check, config, input_field=None):
            _COUNT["machines"] += 1
            super().__init__(check, config, input_field, dtype="float64", devices=devs)

    GpuMachineForSuite.__name__ = "Machine"
    lopec.runtime.Machine = GpuMachineForSuite
    lopec.cli.Machine = GpuMachineForSuite
    if hasattr(lopec, "Machine"):
        lopec.Machine = GpuMachineForSuite


def pytest_unconfigure(config):
    path = os.environ.get("LOPE_SUITE_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(_COUNT, f)
