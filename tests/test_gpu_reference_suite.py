"""The reference's own runtime and acceptance suites, unchanged, against the GPU Machine.

``/root/reference/pkg/tests/test_runtime.py`` (snapshot semantics, point sources,
halo exchange of every padded cell, device counters, faults) and
``test_acceptance.py`` (criteria 1-9, e.g. criterion 3's 108 oracle trials with seed
20260823 and criterion 6's twenty shuffle seeds) are staged by ``build()`` under
baseline/_ref/reference_suite (git-ignored; they travel to the GPU box with the
built library) and run in a subprocess with ``reference_suite_plugin`` swapping
``lopec.runtime.Machine`` for ``paper_1502_03504_b200.machine.Machine`` before the
test modules import it.  Every assertion must hold; the only failures tolerated are
the suite's wall-clock budgets ("exceeded N s"), which time this container's CPU
frontend as much as the GPU.
"""

import json
import os
import pathlib
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

SUITE = REPO / "baseline" / "_ref" / "reference_suite"
if not (SUITE / "tests" / "test_runtime.py").exists():
    pytest.skip("reference suite not staged (run build() where /root/reference exists)", allow_module_level=True)


def _run(tmp_path, files, devices=None):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REPO / "baseline" / "_ref"), str(REPO), str(REPO / "tests"),
                                         env.get("PYTHONPATH", "")])
    env["LOPE_SUITE_REPORT"] = str(tmp_path / "report.json")
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    if devices:
        env["LOPE_SUITE_DEVICES"] = devices
    xml = tmp_path / "junit.xml"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "reference_suite_plugin",
           f"--junitxml={xml}", "--rootdir", str(SUITE / "tests")] + [str(SUITE / "tests" / f) for f in files]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env, cwd=str(SUITE / "tests"))
    report = json.loads((tmp_path / "report.json").read_text())
    cases, bad = 0, []
    for tc in ET.parse(xml).getroot().iter("testcase"):
        cases += 1
        for f in list(tc.findall("failure")) + list(tc.findall("error")):
            msg = (f.get("message") or "") + (f.text or "")
            if "exceeded" in msg and "s (" in msg:      # a wall-clock budget, not a result
                continue
            bad.append((tc.get("name"), msg[:600]))
    return r, report, cases, bad


@pytest.mark.parametrize("devices", [None, "0,0"], ids=["one_device", "images_on_two_device_slots"])
def test_reference_runtime_and_acceptance_suites_pass_on_the_gpu_machine(tmp_path, devices):
    r, report, cases, bad = _run(tmp_path, ["test_runtime.py", "test_acceptance.py"], devices)
    assert report["machines"] > 100, (report, r.stdout[-2000:], r.stderr[-2000:])
    assert cases >= 30, r.stdout[-3000:]
    assert not bad, bad
