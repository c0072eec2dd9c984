"""ctypes binding of liblope_b200.so (include/lope_b200.h).

There is no fallback: if the library is missing or a call fails, this module
raises.  Build it with ``python -m paper_1502_03504_b200.build``.
"""

from __future__ import annotations

import ctypes
import os
import pathlib

from .diagnostics import RuntimeFault

PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG / "liblope_b200.so"
CACHE_DIR = PKG / "_jit_cache"

F32, F64 = 1, 2
DTYPES = {"f32": F32, "float32": F32, "f64": F64, "float64": F64}

EXPORTS = ("lope_abi_version", "lope_last_error", "lope_set_cache_dir", "lope_layout_init",
           "lope_kernel_compile", "lope_kernel_destroy", "lope_kernel_describe",
           "lope_kernel_source", "lope_launch", "lope_step", "lope_step_arrays", "lope_step_planes", "lope_halo_fill", "lope_pack",
           "lope_unpack", "lope_pack_padded", "lope_unpack_padded", "lope_copy_box", "lope_copy_boxes", "lope_box_pack", "lope_plan_candidates", "lope_plan_set", "lope_plan_set_tile", "lope_plan_set_variant", "lope_kernel_prepare", "lope_step_multi",
           "lope_step_planes_peer", "lope_ipc_export", "lope_ipc_open", "lope_ipc_close", "lope_copy_bytes",
           "lope_box_unpack", "lope_fill_hash", "lope_face_span", "lope_launch_count",
           "lope_comm_create", "lope_comm_destroy", "lope_comm_record_size", "lope_comm_export",
           "lope_comm_connect", "lope_comm_nccl_unique_id", "lope_comm_nccl_init", "lope_comm_info",
           "lope_halo_exchange", "lope_halo_exchange_begin", "lope_halo_exchange_end",
           "lope_comm_step", "lope_comm_sync", "lope_peer_enable")


class Layout(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("interior", ctypes.c_int64 * 3), ("lo", ctypes.c_int32 * 3),
                ("hi", ctypes.c_int32 * 3), ("padded", ctypes.c_int64 * 3),
                ("stride", ctypes.c_int64 * 3), ("count", ctypes.c_int64),
                ("elem_bytes", ctypes.c_int64), ("base", ctypes.c_int64)]

    def __repr__(self):
        r = self.rank
        return (f"Layout(rank={r}, dtype={'f32' if self.dtype == F32 else 'f64'}, "
                f"interior={tuple(self.interior[:r])}, lo={tuple(self.lo[:r])}, "
                f"hi={tuple(self.hi[:r])}, stride={tuple(self.stride[:3])}, count={self.count})")


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          f"`python -m paper_1502_03504_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(str(LIB_PATH))
    P, I32, I64, SZ, VP = (ctypes.POINTER, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t,
                           ctypes.c_void_p)
    L.lope_abi_version.restype = ctypes.c_int
    L.lope_last_error.restype = ctypes.c_char_p
    L.lope_set_cache_dir.argtypes = [ctypes.c_char_p]
    L.lope_layout_init.argtypes = [P(Layout), I32, I32, P(I64), P(I32), P(I32)]
    L.lope_kernel_compile.argtypes = [ctypes.c_char_p, SZ, I32, P(VP)]
    L.lope_kernel_destroy.argtypes = [VP]
    L.lope_kernel_describe.argtypes = [VP, ctypes.c_char_p, SZ]
    L.lope_kernel_source.argtypes = [VP, ctypes.c_char_p, SZ]
    L.lope_launch.argtypes = [VP, P(Layout), P(I64), P(VP), P(VP), P(ctypes.c_double), P(I64), VP]
    L.lope_step.argtypes = [VP, P(Layout), VP, VP, P(ctypes.c_double), P(I64), I32, VP]
    L.lope_step_arrays.argtypes = [VP, P(Layout), P(VP), P(VP), P(ctypes.c_double), P(I64), I32, VP]
    L.lope_step_planes.argtypes = [VP, P(Layout), VP, VP, I64, I64, P(ctypes.c_double), P(I64), I32, VP]
    L.lope_halo_fill.argtypes = [P(Layout), VP, I32, VP]
    L.lope_pack.argtypes = [P(Layout), VP, VP, VP]
    L.lope_unpack.argtypes = [P(Layout), VP, VP, VP]
    L.lope_pack_padded.argtypes = [P(Layout), VP, VP, VP]
    L.lope_unpack_padded.argtypes = [P(Layout), VP, VP, VP]
    L.lope_copy_box.argtypes = [P(Layout), VP, VP, P(I64), P(I64), P(I64), VP]
    L.lope_copy_boxes.argtypes = [P(Layout), I32, P(VP), P(VP), P(I64), P(I64), P(I64), VP]
    L.lope_kernel_prepare.argtypes = [VP]
    L.lope_step_planes_peer.argtypes = [VP, P(Layout), VP, VP, I64, I64, P(ctypes.c_double), P(I64), I32, VP, VP, VP]
    L.lope_ipc_export.argtypes = [VP, ctypes.c_char_p, P(I64)]
    L.lope_ipc_open.argtypes = [ctypes.c_char_p, I64, P(VP)]
    L.lope_ipc_close.argtypes = [VP]
    L.lope_copy_bytes.argtypes = [VP, VP, I64, VP]
    L.lope_step_multi.argtypes = [VP, P(Layout), VP, VP, I64, P(ctypes.c_double), P(I64), VP, P(I32)]
    L.lope_comm_create.argtypes = [I32, I32, P(VP)]
    L.lope_comm_destroy.argtypes = [VP]
    L.lope_comm_record_size.restype = ctypes.c_int
    L.lope_comm_export.argtypes = [VP, P(Layout), VP, VP, ctypes.c_char_p]
    L.lope_comm_connect.argtypes = [VP, ctypes.c_char_p]
    L.lope_comm_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.lope_comm_nccl_init.argtypes = [VP, ctypes.c_char_p]
    L.lope_comm_info.argtypes = [VP, P(I32), P(I32), P(ctypes.c_uint32), P(I32)]
    L.lope_halo_exchange.argtypes = [VP, I32, I32, VP]
    L.lope_halo_exchange_begin.argtypes = [VP, I32, I32, VP]
    L.lope_halo_exchange_end.argtypes = [VP, VP]
    L.lope_comm_step.argtypes = [VP, VP, I32, P(ctypes.c_double), P(I64), VP]
    L.lope_comm_sync.argtypes = [VP, VP]
    L.lope_peer_enable.argtypes = [I32]
    L.lope_plan_candidates.argtypes = [VP, P(I32), P(I32), P(I32), I32, P(I32)]
    L.lope_plan_set.argtypes = [VP, P(Layout), I32, I32, I32, I32]
    L.lope_plan_set_tile.argtypes = [VP, P(Layout), I32, P(I32), I32, I32, P(I32)]
    L.lope_plan_set_variant.argtypes = [VP, P(Layout), I32, P(I32), I32, I32, P(I32)]
    L.lope_box_pack.argtypes = [P(Layout), VP, P(I64), P(I64), VP, VP]
    L.lope_box_unpack.argtypes = [P(Layout), VP, P(I64), P(I64), VP, VP]
    L.lope_fill_hash.argtypes = [P(Layout), VP, ctypes.c_uint64, P(I64), P(I64), VP]
    L.lope_face_span.argtypes = [P(Layout), I32, P(I64), P(I64)]
    L.lope_launch_count.restype = I64
    for name in EXPORTS:
        if not hasattr(L, name):
            raise ImportError(f"{LIB_PATH} does not export {name}")
    if L.lope_abi_version() != 1:
        raise ImportError("liblope_b200.so ABI version mismatch")
    CACHE_DIR.mkdir(exist_ok=True)
    L.lope_set_cache_dir(str(CACHE_DIR).encode())
    _lib = L
    return L


def _code(code: int) -> str:
    if code > 0:
        return f"E{code:03d}"
    return "E000"


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().lope_last_error().decode(errors="replace")
        if rc > 0:
            raise RuntimeFault(_code(rc), f"{what}: {msg}")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


def dtype_code(dtype) -> int:
    import numpy as np
    if isinstance(dtype, int) and dtype in (F32, F64):
        return dtype
    if isinstance(dtype, str) and dtype in DTYPES:
        return DTYPES[dtype]
    dt = np.dtype(str(dtype).replace("torch.", ""))
    if dt == np.float32:
        return F32
    if dt == np.float64:
        return F64
    raise TypeError(f"unsupported element type {dtype}; the hot path computes in float32 or float64")


def make_layout(rank, dtype, interior, lo, hi) -> Layout:
    L = Layout()
    ext = (ctypes.c_int64 * 3)(*(list(interior) + [1] * (3 - len(interior))))
    lo_ = (ctypes.c_int32 * 3)(*(list(lo) + [0] * (3 - len(lo))))
    hi_ = (ctypes.c_int32 * 3)(*(list(hi) + [0] * (3 - len(hi))))
    check(lib().lope_layout_init(ctypes.byref(L), rank, dtype_code(dtype), ext, lo_, hi_),
          "lope_layout_init")
    return L


def compile_kernel(text: str, dtype) -> int:
    h = ctypes.c_void_p()
    b = text.encode()
    check(lib().lope_kernel_compile(b, len(b), dtype_code(dtype), ctypes.byref(h)),
          "lope_kernel_compile")
    return h.value


def destroy_kernel(h) -> None:
    if h:
        lib().lope_kernel_destroy(h)


def describe(h) -> str:
    buf = ctypes.create_string_buffer(1 << 16)
    check(lib().lope_kernel_describe(h, buf, len(buf)), "lope_kernel_describe")
    return buf.value.decode()


def source(h) -> str:
    buf = ctypes.create_string_buffer(1 << 22)
    check(lib().lope_kernel_source(h, buf, len(buf)), "lope_kernel_source")
    return buf.value.decode()


def face_span(layout: Layout, which: int):
    off, cnt = ctypes.c_int64(), ctypes.c_int64()
    check(lib().lope_face_span(ctypes.byref(layout), which, ctypes.byref(off), ctypes.byref(cnt)),
          "lope_face_span")
    return off.value, cnt.value


def launch_count() -> int:
    return int(lib().lope_launch_count())


def exported_symbols():
    L = lib()
    return [n for n in EXPORTS if hasattr(L, n)]


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")
