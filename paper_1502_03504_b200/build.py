"""Build liblope_b200.so in-tree (nvcc, sm_100a) and pre-compile the known kernels.

    python -m paper_1502_03504_b200.build          # or __graft_entry__.build()

The shared library holds the C ABI (include/lope_b200.h), the AOT halo-fill /
copy-through / synthetic-input kernels and the NVRTC driver.  Body-specialised
stencil kernels are compiled by NVRTC for sm_100a; this script compiles the
configuration and corpus kernels once so their cubins ship in ``_jit_cache/``
(NVRTC needs no GPU).
"""

from __future__ import annotations

import os
import pathlib
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "liblope_b200.so"
CACHE = PKG / "_jit_cache"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_LIB = "/usr/local/cuda/lib64"

SOURCES = [CSRC / "lope_api.cu", CSRC / "lope_comm.cu", CSRC / "lope_codegen.cpp"]
DEPS = SOURCES + [CSRC / "lope_device.cuh", CSRC / "lope_codegen.h", CSRC / "lope_internal.h",
                  REPO / "include" / "lope_b200.h"]


def _gen_device_inc() -> pathlib.Path:
    src = (CSRC / "lope_device.cuh").read_text()
    if ")LOPESRC\"" in src:
        raise RuntimeError("device source contains the raw-string delimiter")
    inc = CSRC / "lope_device_src.inc"
    text = 'R"LOPESRC(' + src + ')LOPESRC"\n'
    if not inc.exists() or inc.read_text() != text:
        inc.write_text(text)
    return inc


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build_lib(force: bool = False, verbose: bool = False) -> pathlib.Path:
    _gen_device_inc()
    if not force and not _stale():
        return LIB
    cmd = [NVCC, "-shared", "-Xcompiler", "-fPIC", "-std=c++17", "-O3", "-lineinfo",
           "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", str(REPO / "include"), "-I", str(CSRC),
           *[str(s) for s in SOURCES],
           "-o", str(LIB) + ".tmp",
           "-L", CUDA_LIB, "-lnvrtc", "-ldl", "-Xlinker", f"-rpath,{CUDA_LIB}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stdout + res.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


def precompile_kernels() -> list:
    """NVRTC-compile the benchmark/corpus kernels into the shipped cubin cache."""
    sys.path.insert(0, str(REPO))
    from paper_1502_03504_b200 import _lib, stencils
    from paper_1502_03504_b200.ir import serialize

    done = []
    for name, dtypes in (("heat2d", ("f32", "f64")), ("ninept2d", ("f32", "f64")),
                         ("lap3d7", ("f32", "f64")), ("box5x5", ("f64", "f32")),
                         ("laplacian", ("f64", "f32")), ("avg3", ("f64", "f32")),
                         ("drift2", ("f64", "f32"))):
        text = serialize(stencils.by_name(name))
        for dt in dtypes:
            k = _lib.compile_kernel(text, dt)
            if name in ("lap3d7", "ninept2d", "box5x5", "heat2d"):
                _lib.check(_lib.lib().lope_kernel_prepare(k), "lope_kernel_prepare")   # tuning variants
            _lib.destroy_kernel(k)
            done.append(f"{name}:{dt}")
    return done


REFERENCE = pathlib.Path("/root/reference/pkg")
SUITE = REPO / "baseline" / "_ref" / "reference_suite"


def stage_reference_suite() -> bool:
    """Copy the reference's own test suite and corpus next to its installed package
    (baseline/_ref/reference_suite: git-ignored, travels to the GPU box like the .so),
    so tests/test_gpu_reference_suite.py can re-run it against the GPU Machine.  Only
    here, where /root/reference exists; it is test infrastructure, never product."""
    import shutil
    if not (REFERENCE / "tests").is_dir():
        return SUITE.is_dir()
    for sub in ("tests", "corpus"):
        dst = SUITE / sub
        if dst.exists():
            shutil.rmtree(dst)
        shutil.copytree(REFERENCE / sub, dst, ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return True


def main() -> None:
    build_lib(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built", LIB)
    print("precompiled", ", ".join(precompile_kernels()))
    print("reference suite staged:", stage_reference_suite())


if __name__ == "__main__":
    main()
