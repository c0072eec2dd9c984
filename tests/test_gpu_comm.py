"""The C-ABI slab communicator (lope_comm, include/lope_b200.h) on the GPU.

``Machine._halo_exchange`` (runtime.py:643-711) and the fused peer-store step behind
the C boundary: P slab images with their own communicators, streams and flags,
driven (1) from Python (``dist.CommMultiSlab``) and (2) from a pure C host
(``tools/abi_slabs.c``), each checked bit for bit against the undecomposed run /
the oracle.  All images share one GPU inside one process and are driven round by
round, so no kernel waits on another (B200_PROFILING.md: ranks on one GPU must not).
"""

import json
import os
import shutil
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)


def _env():
    e = dict(os.environ)
    e["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
    return e


def test_comm_slabs_in_one_process_match_the_oracle():
    r = subprocess.run([sys.executable, str(REPO / "tests" / "comm_child.py")], capture_output=True, text=True,
                       timeout=600, env=_env(), cwd=str(REPO))
    assert r.returncode == 0, r.stderr[-3000:]
    rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(rows) == 7
    for row in rows:
        name, shape, dt, p, steps = row["case"]
        assert row["equal"], row
        if p > 1:
            # one synchronised operation for HALO_TRANSFER plus one per fused step
            assert row["epochs"] == [steps] * p, row
            assert row["transport"] == "peer"


def _build_c_driver(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    out = tmp_path / "abi_slabs"
    r = subprocess.run([gcc, "-O2", "-o", str(out), str(REPO / "tools" / "abi_slabs.c"), f"-I{REPO / 'include'}",
                        "-I/usr/local/cuda/include", f"-L{REPO / 'paper_1502_03504_b200'}", "-llope_b200",
                        "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{REPO / 'paper_1502_03504_b200'}",
                        "-Wl,-rpath,/usr/local/cuda/lib64"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("p,n,steps", [(2, 128, 8), (4, 64, 6), (3, 96, 1)])
def test_pure_c_host_drives_the_slab_exchange(tmp_path, p, n, steps):
    exe = _build_c_driver(tmp_path)
    env = _env()
    env["LOPE_CACHE_DIR"] = str(REPO / "paper_1502_03504_b200" / "_jit_cache")
    r = subprocess.run([str(exe), "rr", str(p), str(n), str(steps)], capture_output=True, text=True, timeout=300,
                       env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["bitwise_equal_to_undecomposed"] is True and d["images"] == p and d["err"] == "no error", d


def test_pure_c_multi_process_mode_refuses_a_shared_gpu(tmp_path):
    if torch.cuda.device_count() >= 2:
        pytest.skip("several GPUs: the multi-process mode would run")
    exe = _build_c_driver(tmp_path)
    r = subprocess.run([str(exe), "procs", "2", "64", "3"], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "needs 2 GPUs" in r.stderr
