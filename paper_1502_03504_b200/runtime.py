"""Host runtime: GPU-resident halo arrays, kernel launches and halo transfers.

This is the reference's hot path (lopec/runtime.py) re-expressed over
liblope_b200.so.  Vocabulary and semantics follow the reference:

* ``HaloArray`` — one image's block of a halo-padded array
  (``DistributedArray`` blocks, runtime.py:73-94; layout ir.py:189-230), kept in
  HBM.  It owns two buffers: the live one and a spare that becomes the next
  launch's output (the double buffering of ``_launch``: the reference copies a
  snapshot, runtime.py:596; here the live buffer *is* the snapshot and the
  spare receives the stores, so no copy is made).
* ``launch``   — ``Machine._launch`` + ``_launch_vector`` (runtime.py:541-618):
  1-based inclusive ranges, E108 outside the interior, empty ranges allowed.
* ``halo_transfer`` — ``Machine._halo_exchange`` (runtime.py:643-711) for an
  image that is its own neighbour in every dimension (P = 1).  Partitioned
  arrays use ``paper_1502_03504_b200.dist``.
* ``iterate``  — ``do it = 1, nsteps; HALO_TRANSFER(U); do concurrent ... end
  do`` (corpus/*.lope).  Steps 1..K-1 run as one fused kernel each (launch of
  step t + the periodic fill of step t+1); the last launch copies the halo
  through, so the final state equals the reference's.

Buffers are torch CUDA tensors (torch is used for allocation, streams and
copies only); every computation is a liblope_b200.so kernel.
"""

from __future__ import annotations

import ctypes
import json
from typing import Dict, Iterable, Optional, Sequence

import numpy as np

from . import _lib
from .diagnostics import ALLOC_SHAPE, RuntimeFault
from .ir import KernelIR, deserialize, serialize


def _torch():
    import torch
    return torch


def _stream_handle(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _torch_dtype(code):
    torch = _torch()
    return torch.float32 if code == _lib.F32 else torch.float64


def _np_dtype(code):
    return np.float32 if code == _lib.F32 else np.float64


class HaloArray:
    """A halo-padded array block resident in HBM (``real, dimension(...), HALO(lo:*:hi, ...)``).

    ``interior``: extents m_d; ``lo``/``hi``: halo widths per dim (0..8).
    """

    def __init__(self, interior: Sequence[int], lo: Sequence[int], hi: Sequence[int],
                 dtype="float32", device=None, name: str = "u"):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("HaloArray needs a CUDA device (there is no CPU path)")
        interior = tuple(int(m) for m in interior)
        rank = len(interior)
        if len(lo) != rank or len(hi) != rank:
            raise RuntimeFault(ALLOC_SHAPE, "halo widths must have one entry per dimension")
        self.name = name
        self.rank = rank
        self.interior = interior
        self.lo = tuple(int(w) for w in lo)
        self.hi = tuple(int(w) for w in hi)
        self.layout = _lib.make_layout(rank, dtype, interior, self.lo, self.hi)
        self.dtype_code = self.layout.dtype
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self._bufs = [torch.zeros(self.layout.count, dtype=_torch_dtype(self.dtype_code),
                                  device=self.device), None]
        self._live = 0

    # -- buffers -----------------------------------------------------------

    @property
    def data(self):
        """The live buffer (flat, ``layout.count`` elements)."""
        return self._bufs[self._live]

    def spare(self, stream=None):
        """The other buffer of the ping-pong pair (allocated on first use).

        The zero fill is enqueued on ``stream`` (default: the current stream), the
        stream the caller is about to write the buffer on, so it can never land after
        those writes."""
        torch = _torch()
        j = 1 - self._live
        if self._bufs[j] is None:
            if stream is None:
                self._bufs[j] = torch.zeros_like(self._bufs[self._live])
            else:
                # the live buffer was filled on another stream: order against it first
                stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(stream):
                    self._bufs[j] = torch.zeros_like(self._bufs[self._live])
        return self._bufs[j]

    def swap(self) -> None:
        self._live = 1 - self._live

    def padded_view(self):
        """Device view of the padded block as a torch tensor indexed [c2, c1, c0]."""
        L = self.layout
        p = [int(L.padded[d]) for d in range(3)]
        v = self.data.view(p[2], p[1], int(L.stride[1]))
        return v[:, :, int(L.base):int(L.base) + p[0]]

    def interior_view(self):
        L = self.layout
        v = self.padded_view()
        return v[L.lo[2]:L.lo[2] + L.interior[2], L.lo[1]:L.lo[1] + L.interior[1],
                 L.lo[0]:L.lo[0] + L.interior[0]]

    # -- host transfers (scatter / gather) ----------------------------------

    def set_interior(self, field: np.ndarray, stream=None) -> None:
        """``_scatter_block`` (runtime.py:477-486): host field -> interior."""
        field = np.asarray(field, dtype=_np_dtype(self.dtype_code))
        if field.shape != self.interior:
            raise RuntimeFault(ALLOC_SHAPE, f"field shape {field.shape} does not match the "
                                            f"interior {self.interior}")
        host = np.asfortranarray(field)
        _lib.check(_lib.lib().lope_pack(ctypes.byref(self.layout), host.ctypes.data_as(ctypes.c_void_p),
                                        ctypes.c_void_p(self.data.data_ptr()),
                                        ctypes.c_void_p(_stream_handle(stream))), "lope_pack")
        _torch().cuda.current_stream().synchronize() if stream is None else stream.synchronize()

    def upload(self, host_ptr: int, stream=None) -> None:
        """Interior <- host column-major buffer at ``host_ptr`` (pinned for async copies)."""
        _lib.check(_lib.lib().lope_pack(ctypes.byref(self.layout), ctypes.c_void_p(host_ptr),
                                        ctypes.c_void_p(self.data.data_ptr()),
                                        ctypes.c_void_p(_stream_handle(stream))), "lope_pack")

    def download(self, host_ptr: int, stream=None) -> None:
        """Host column-major buffer at ``host_ptr`` <- interior (asynchronous on the stream)."""
        _lib.check(_lib.lib().lope_unpack(ctypes.byref(self.layout), ctypes.c_void_p(self.data.data_ptr()),
                                          ctypes.c_void_p(host_ptr),
                                          ctypes.c_void_p(_stream_handle(stream))), "lope_unpack")

    def get_interior(self, stream=None) -> np.ndarray:
        """Gather the interior to the host (numpy, reference index order)."""
        out = np.empty(self.interior, dtype=_np_dtype(self.dtype_code), order="F")
        _lib.check(_lib.lib().lope_unpack(ctypes.byref(self.layout),
                                          ctypes.c_void_p(self.data.data_ptr()),
                                          out.ctypes.data_as(ctypes.c_void_p),
                                          ctypes.c_void_p(_stream_handle(stream))), "lope_unpack")
        _torch().cuda.current_stream().synchronize() if stream is None else stream.synchronize()
        return np.ascontiguousarray(out) if out.ndim == 1 else out

    def get_padded(self) -> np.ndarray:
        """The whole padded block on the host, numpy index order (c0, c1, ...)."""
        v = self.padded_view().cpu().numpy()          # [c2, c1, c0]
        v = np.transpose(v, (2, 1, 0))
        return np.ascontiguousarray(v.reshape(v.shape[:self.rank]))

    def fill_hash(self, seed: int, global_extent=None, global_origin=None, stream=None) -> None:
        """Synthetic U(-1,1) field generated on the device (oracle: hash_values)."""
        ge = list(global_extent or self.interior) + [1] * (3 - len(global_extent or self.interior))
        go = list(global_origin or [0] * self.rank) + [0] * (3 - len(global_origin or [0] * self.rank))
        _lib.check(_lib.lib().lope_fill_hash(ctypes.byref(self.layout),
                                             ctypes.c_void_p(self.data.data_ptr()),
                                             ctypes.c_uint64(seed), (ctypes.c_int64 * 3)(*ge),
                                             (ctypes.c_int64 * 3)(*go),
                                             ctypes.c_void_p(_stream_handle(stream))),
                   "lope_fill_hash")

    def nbytes_interior(self) -> int:
        return int(np.prod(self.interior)) * int(self.layout.elem_bytes)


_L2_RESIDENT_BYTES = 64 << 20      # fields this small are launch-bound, not HBM-bound
_AUTOTUNE_MIN_CELLS = 1 << 25      # ~128 MB fp32: below this the defaults are within noise


def _autotune_enabled() -> bool:
    import os
    return os.environ.get("LOPE_AUTOTUNE", "1") not in ("0", "")


def _tune_key(arr, mask):
    L = arr.layout
    return (tuple(L.interior[:3]), tuple(L.lo[:3]), tuple(L.hi[:3]), int(mask))


class PlanTuner:
    """Online choice of the tiled kernel's execution plan for one geometry.

    The candidates (compiled tile variants x z-chunks, ``lope_plan_candidates``)
    compute identical bits, so real steps double as measurements: each candidate
    runs ``STEPS`` consecutive steps (both ping-pong directions, as in steady
    state), timed with CUDA events on the launching stream, in ``PASSES``
    round-robin passes (forward, then reverse order); the lowest mean wins and
    becomes the plan (``lope_plan_set``).  Timing a candidate on repeated launches in one direction
    ranks the plans differently (measured on B200), hence real alternating steps.

    Watchdog: the short-z-chunk plans have a slow mode (same plan, same buffers, 25-30%
    slower for hundreds of steps, entered and left unpredictably -- see DESIGN §9).
    When the winner is such a plan, the tuner keeps timing every step (events queried
    without blocking) and falls back to the best long-chunk plan once the median of
    the last ``WATCH`` steps is ``SLOW`` times the winner's fastest observed step time
    (its fast mode; the slow mode is >= 1.25x; the 1000 W power cap alone costs up to
    1.21x on config 3: 1.42 -> 1.70 ms).
    """

    STEPS = 6
    PASSES = 2
    WARM = 12       # untimed steps first: an idle GPU's clocks ramp up over the first ~ms
    WATCH = 12      # steps in the watchdog's window
    SLOW = 1.25     # watchdog threshold relative to the winner's fastest step (the power cap alone: <= 1.21x)
    SAFE_ZCHUNK = 16  # plans with at least this many planes per unit have no slow mode
    SAFE_MARGIN = 1.05  # fall back only if the slow mode is this much slower than the safe plan

    def __init__(self, kernel: "CompiledKernel", layout, wrap_mask: int):
        self.kernel = kernel
        self.layout = layout
        self.mask = int(wrap_mask)
        cap = 64
        v, z, y, n = (ctypes.c_int32 * cap)(), (ctypes.c_int32 * cap)(), (ctypes.c_int32 * cap)(), ctypes.c_int32()
        _lib.check(_lib.lib().lope_plan_candidates(kernel.handle, v, z, y, cap, ctypes.byref(n)),
                   "lope_plan_candidates")
        self.cands = [(int(v[i]), int(z[i]), int(y[i])) for i in range(min(n.value, cap))]
        # passes alternate forward / reverse and scores are the mean over passes: the
        # board's clocks drift during tuning (power ramp), a linear drift then cancels
        order = list(range(len(self.cands)))
        self.trials = [c for p in range(self.PASSES) for c in (order if p % 2 == 0 else order[::-1])]
        self.pos = 0
        self.sub = 0
        self.warm = self.WARM
        self.timed = []              # (candidate index, start event, end event)
        self._start = None
        self.report = {"candidates": [], "best": None}
        self.done = len(self.cands) <= 1
        self.monitoring = False
        self._watch = []             # (start, end) events of recent steps, oldest first
        self._durations = []
        self._safe = None            # (long-chunk candidate, the winner's fastest step ms)
        self._safe_ms = 0.0          # the long-chunk candidate's own tuned ms

    @property
    def steps_needed(self) -> int:
        return self.WARM + len(self.trials) * self.STEPS

    def _set(self, variant: int, zchunk: int, yband: int) -> None:
        _lib.check(_lib.lib().lope_plan_set(self.kernel.handle, ctypes.byref(self.layout), self.mask,
                                            variant, zchunk, yband), "lope_plan_set")

    @property
    def active(self) -> bool:
        return not self.done or self.monitoring

    def before(self, stream=None) -> None:
        if self.done:
            if self.monitoring:
                self._start = _torch().cuda.Event(enable_timing=True)
                self._start.record(stream)
            return
        if self.warm > 0:
            return
        if self.sub == 0:
            self._set(*self.cands[self.trials[self.pos]])
            self._start = _torch().cuda.Event(enable_timing=True)
            self._start.record(stream)

    def after(self, stream=None) -> None:
        if self.done:
            if self.monitoring:
                self._watch_step(stream)
            return
        if self.warm > 0:
            self.warm -= 1
            return
        self.sub += 1
        if self.sub < self.STEPS:
            return
        end = _torch().cuda.Event(enable_timing=True)
        end.record(stream)
        self.timed.append((self.trials[self.pos], self._start, end))
        self.sub = 0
        self.pos += 1
        if self.pos == len(self.trials):
            self._finish()

    def _finish(self) -> None:
        self.timed[-1][2].synchronize()
        acc = {}
        for c, a, b in self.timed:
            acc.setdefault(c, []).append(a.elapsed_time(b) / self.STEPS)
        best = {c: sum(v) / len(v) for c, v in acc.items()}
        ci = min(best, key=best.get)
        self._set(*self.cands[ci])
        safe = [c for c in best if self.cands[c][1] >= self.SAFE_ZCHUNK]
        if self.layout.rank == 3 and self.cands[ci][1] < self.SAFE_ZCHUNK and safe:
            cs = min(safe, key=best.get)
            self._safe = (cs, min(acc[ci]))     # the winner's fastest trial: its fast mode
            self._safe_ms = best[cs]            # what the long-chunk plan itself costs
            self.monitoring = True
        desc = json.loads(self.kernel.describe())
        self.report = {"candidates": [list(self.cands[c]) + [round(best[c], 5)] for c in sorted(best)],
                       "best": {"variant": self.cands[ci][0], "zchunk": self.cands[ci][1],
                                "yband": self.cands[ci][2], "ms_per_step": round(best[ci], 5)},
                       "plans": desc.get("plans"), "fallback": None}
        self.timed = []
        self.done = True

    def _watch_step(self, stream) -> None:
        end = _torch().cuda.Event(enable_timing=True)
        end.record(stream)
        self._watch.append((self._start, end))
        while self._watch and self._watch[0][1].query():      # completed: no host stall
            a, b = self._watch.pop(0)
            self._durations.append(a.elapsed_time(b))
        self._check_window()

    def _check_window(self) -> None:
        """Fall back to the long-chunk plan if the recent steps are in the slow mode."""
        self._durations = self._durations[-self.WATCH:]
        if self._durations:
            cs, fast_ms = self._safe
            self._safe = (cs, min(fast_ms, min(self._durations)))
        if len(self._durations) == self.WATCH:
            med = sorted(self._durations)[self.WATCH // 2]
            cs, tuned_ms = self._safe
            # switch only when the long-chunk plan is expected to be faster than the slow
            # mode itself (on some boxes every long-chunk plan runs at slow-mode speed)
            if med > self.SLOW * tuned_ms and med > self.SAFE_MARGIN * self._safe_ms:
                self._set(*self.cands[cs])
                self.monitoring = False
                self._watch = []
                self.report["fallback"] = {"to": list(self.cands[cs]), "median_ms": round(med, 5),
                                           "tuned_ms": round(tuned_ms, 5)}


class CompiledKernel:
    """A locally-oriented kernel compiled for sm_100a (``lope_kernel_compile``)."""

    def __init__(self, kernel, dtype="float32"):
        if isinstance(kernel, KernelIR):
            self.ir = kernel
            text = serialize(kernel)
        elif isinstance(kernel, str):
            text = kernel
            self.ir = deserialize(text)
        else:      # a lopec.ir.KernelIR (duck-typed)
            from .ir import from_lopec
            self.ir = from_lopec(kernel)
            text = serialize(self.ir)
        self.text = text
        self.dtype_code = _lib.dtype_code(dtype)
        self.handle = _lib.compile_kernel(text, self.dtype_code)
        self._tuners = {}

    def __del__(self):
        try:
            _lib.destroy_kernel(getattr(self, "handle", None))
        except Exception:
            pass

    def describe(self) -> str:
        return _lib.describe(self.handle)

    def source(self) -> str:
        return _lib.source(self.handle)

    def tuner(self, arr: "HaloArray", wrap_mask: int) -> Optional["PlanTuner"]:
        """The online plan tuner for ``arr``'s geometry while it is still measuring
        (None once a plan is chosen, for small blocks, with ``LOPE_AUTOTUNE=0`` and
        during CUDA-graph capture).  There is deliberately no offline plan table: the
        short-z-chunk plans' speed depends on where the buffers sit in HBM (the plan
        that ran 1.49 ms sustained on one allocation ran 1.88 ms on another), so the
        plan is measured on the live buffers."""
        key = _tune_key(arr, wrap_mask)
        t = self._tuners.get(key)
        if t is None:
            if not _autotune_enabled() or arr.layout.count < _AUTOTUNE_MIN_CELLS:
                return None
            t = self._tuners[key] = PlanTuner(self, arr.layout, wrap_mask)
        if not t.active or _torch().cuda.is_current_stream_capturing():
            return None
        return t

    def tuning(self, arr: "HaloArray", wrap_mask: int) -> bool:
        """True while the plan for ``arr``'s geometry is still being measured (the
        watchdog that may follow does not count)."""
        t = self.tuner(arr, wrap_mask)
        return t is not None and not t.done

    def tune(self, arr: "HaloArray", scalars=None, wrap_mask: Optional[int] = None, stream=None) -> dict:
        """Choose the plan for ``arr``'s geometry now by running real fused steps under
        each candidate (this advances the field by ``PlanTuner.steps_needed`` steps --
        the bits are the same whichever plan runs them).  Returns the tuning report."""
        mask = (1 << arr.rank) - 1 if wrap_mask is None else wrap_mask
        key = _tune_key(arr, mask)
        t = self._tuners.get(key)
        if t is None:
            t = self._tuners[key] = PlanTuner(self, arr.layout, mask)
        while not t.done:
            step(self, arr, scalars, mask, stream)
        return t.report

    def scalar_args(self, scalars: Optional[Dict[str, float]]):
        scalars = scalars or {}
        n = max(1, len(self.ir.scalar_params))
        rs = (ctypes.c_double * n)()
        is_ = (ctypes.c_int64 * n)()
        for i, name in enumerate(self.ir.scalar_params):
            if name not in scalars:
                raise RuntimeFault("E202", f"scalar parameter '{name}' has no value")
            v = scalars[name]
            if self.ir.param_types.get(name) == "integer":
                is_[i] = int(v)
            else:
                rs[i] = float(v)
        return rs, is_


_NVTX = None


def _nvtx(name):
    """NVTX range around a hot-path call when ``LOPE_NVTX=1`` (Nsight timelines: one
    range per launch / step / exchange, the reference's event log as a trace)."""
    global _NVTX
    if _NVTX is None:
        import os
        _NVTX = os.environ.get("LOPE_NVTX", "0") not in ("0", "")
    if not _NVTX:
        return _NullRange()
    return _torch().cuda.nvtx.range(name)


class _NullRange:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def launch(kernel: CompiledKernel, arrays: Sequence[HaloArray], ranges=None,
           scalars: Optional[Dict[str, float]] = None, stream=None) -> None:
    """One ``do concurrent`` launch (runtime.py:541-618) over 1-based inclusive ``ranges``.

    ``arrays`` binds the kernel's array parameters in order.  Stored arrays are
    written into their spare buffer (the reference's live buffer) and become
    live; everything outside the range is copied through.
    """
    ir = kernel.ir
    if len(arrays) != len(ir.array_params):
        raise RuntimeFault(ALLOC_SHAPE, f"kernel '{ir.name}' takes {len(ir.array_params)} arrays")
    if len({id(a) for a in arrays}) != len(arrays):
        raise RuntimeFault(ALLOC_SHAPE, "the same array is bound to two kernel parameters")
    rank = ir.rank
    if ranges is None:
        ranges = [(1, m) for m in arrays[0].interior]
    if len(ranges) != rank:
        raise RuntimeFault(ALLOC_SHAPE, f"launch needs {rank} ranges")
    na = len(arrays)
    layouts = (_lib.Layout * na)(*[a.layout for a in arrays])
    rng = (ctypes.c_int64 * (2 * rank))(*[int(v) for r in ranges for v in r])
    ins = (ctypes.c_void_p * na)(*[a.data.data_ptr() for a in arrays])
    stored = set(ir.stored_arrays)
    outs = (ctypes.c_void_p * na)(*[(a.spare(stream).data_ptr() if p in stored else None)
                                    for p, a in zip(ir.array_params, arrays)])
    rs, is_ = kernel.scalar_args(scalars)
    _lib.check(_lib.lib().lope_launch(kernel.handle, layouts, rng, ins, outs, rs, is_,
                                      ctypes.c_void_p(_stream_handle(stream))), "lope_launch")
    for p, a in zip(ir.array_params, arrays):
        if p in stored:
            a.swap()


def halo_transfer(arr: HaloArray, dims_mask: Optional[int] = None, stream=None) -> None:
    with _nvtx(f"lope.halo_transfer {arr.name or ''}"):
        _halo_transfer(arr, dims_mask, stream)


def _halo_transfer(arr: HaloArray, dims_mask: Optional[int] = None, stream=None) -> None:
    """``HALO_TRANSFER(U, BC=CYCLIC)`` for one image (every neighbour is self)."""
    mask = (1 << arr.rank) - 1 if dims_mask is None else dims_mask
    _lib.check(_lib.lib().lope_halo_fill(ctypes.byref(arr.layout), ctypes.c_void_p(arr.data.data_ptr()),
                                         mask, ctypes.c_void_p(_stream_handle(stream))),
               "lope_halo_fill")


def step(kernel: CompiledKernel, arr: HaloArray, scalars=None, wrap_mask: Optional[int] = None,
         stream=None) -> None:
    with _nvtx(f"lope.step {kernel.ir.name}"):
        _step(kernel, arr, scalars, wrap_mask, stream)


def _step(kernel: CompiledKernel, arr: HaloArray, scalars=None, wrap_mask: Optional[int] = None,
          stream=None) -> None:
    """Fused launch (full interior) + the following HALO_TRANSFER's local fill."""
    mask = (1 << arr.rank) - 1 if wrap_mask is None else wrap_mask
    tuner = kernel.tuner(arr, mask)
    if tuner is not None:
        tuner.before(stream)
    rs, is_ = kernel.scalar_args(scalars)
    _lib.check(_lib.lib().lope_step(kernel.handle, ctypes.byref(arr.layout),
                                    ctypes.c_void_p(arr.data.data_ptr()),
                                    ctypes.c_void_p(arr.spare(stream).data_ptr()), rs, is_, mask,
                                    ctypes.c_void_p(_stream_handle(stream))), "lope_step")
    arr.swap()
    if tuner is not None:
        tuner.after(stream)


def step_arrays(kernel: CompiledKernel, arrays: Sequence[HaloArray], scalars=None,
                wrap_mask: Optional[int] = None, stream=None) -> None:
    """``step`` for kernels over several arrays: one fused full-interior launch whose
    stored arrays also receive their periodic images (``lope_step_arrays``) -- the state
    after the launch (runtime.py:541-618) and the next ``HALO_TRANSFER`` of every stored
    array (runtime.py:643-697)."""
    ir = kernel.ir
    if len(arrays) != len(ir.array_params):
        raise RuntimeFault(ALLOC_SHAPE, f"kernel '{ir.name}' takes {len(ir.array_params)} arrays")
    if len({id(a) for a in arrays}) != len(arrays):
        raise RuntimeFault(ALLOC_SHAPE, "the same array is bound to two kernel parameters")
    mask = (1 << ir.rank) - 1 if wrap_mask is None else wrap_mask
    na = len(arrays)
    layouts = (_lib.Layout * na)(*[a.layout for a in arrays])
    ins = (ctypes.c_void_p * na)(*[a.data.data_ptr() for a in arrays])
    stored = set(ir.stored_arrays)
    outs = (ctypes.c_void_p * na)(*[(a.spare(stream).data_ptr() if p in stored else None)
                                    for p, a in zip(ir.array_params, arrays)])
    rs, is_ = kernel.scalar_args(scalars)
    with _nvtx(f"lope.step_arrays {ir.name}"):
        _lib.check(_lib.lib().lope_step_arrays(kernel.handle, layouts, ins, outs, rs, is_, mask,
                                               ctypes.c_void_p(_stream_handle(stream))), "lope_step_arrays")
    for p, a in zip(ir.array_params, arrays):
        if p in stored:
            a.swap()


def iterate_arrays(kernel: CompiledKernel, arrays: Sequence[HaloArray], steps: int, scalars=None,
                   stream=None) -> None:
    """``do it = 1, steps; HALO_TRANSFER(every array); do concurrent call K(arrays); end do``
    for kernels over several arrays: fused steps, then a plain final launch."""
    if steps <= 0:
        return
    for a in arrays:
        halo_transfer(a, stream=stream)
    for _ in range(steps - 1):
        step_arrays(kernel, arrays, scalars, stream=stream)
    launch(kernel, arrays, None, scalars, stream=stream)


def multi_step(kernel: CompiledKernel, arr: HaloArray, nsteps: int, scalars=None, stream=None) -> None:
    with _nvtx(f"lope.multi_step {kernel.ir.name} x{nsteps}"):
        _multi_step(kernel, arr, nsteps, scalars, stream)


def _multi_step(kernel: CompiledKernel, arr: HaloArray, nsteps: int, scalars=None, stream=None) -> None:
    """``nsteps`` fused steps (every dim periodic) in as few launches as the kernel
    allows: rank-2 kernels on fields of at least a tile plus four halos advance four
    steps per launch in shared memory (``lope_step_multi``), bit-identical to
    ``nsteps`` calls of ``step``."""
    if nsteps <= 0:
        return
    rs, is_ = kernel.scalar_args(scalars)
    live = ctypes.c_int32()
    a, b = arr.data, arr.spare(stream)
    _lib.check(_lib.lib().lope_step_multi(kernel.handle, ctypes.byref(arr.layout), ctypes.c_void_p(a.data_ptr()),
                                          ctypes.c_void_p(b.data_ptr()), int(nsteps), rs, is_,
                                          ctypes.c_void_p(_stream_handle(stream)), ctypes.byref(live)),
               "lope_step_multi")
    if live.value == 1:
        arr.swap()


def iterate(kernel: CompiledKernel, arr: HaloArray, steps: int, scalars=None, stream=None) -> None:
    """``do it = 1, steps; HALO_TRANSFER(U); do concurrent (full interior) call K(U); end do``."""
    if steps <= 0:
        return
    halo_transfer(arr, stream=stream)
    if arr.layout.count * arr.layout.elem_bytes <= _L2_RESIDENT_BYTES:
        multi_step(kernel, arr, steps - 1, scalars, stream=stream)   # launch-bound: temporal blocking
    else:
        for _ in range(steps - 1):
            step(kernel, arr, scalars, stream=stream)
    launch(kernel, [arr], None, scalars, stream=stream)


def run(kernel, field: np.ndarray, steps: int, scalars=None, halo=None, dtype=None) -> np.ndarray:
    """End-to-end: host field in, ``steps`` iterations on the GPU, host field out."""
    if not isinstance(kernel, CompiledKernel):
        kernel = CompiledKernel(kernel, dtype or "float32")
    ir = kernel.ir
    fp = ir.footprints[ir.array_params[0]].dims
    lo = [n for n, _ in fp] if halo is None else [h[0] for h in halo]
    hi = [p for _, p in fp] if halo is None else [h[1] for h in halo]
    field = np.asarray(field)
    arr = HaloArray(field.shape, lo, hi, dtype="float32" if kernel.dtype_code == _lib.F32 else "float64")
    arr.set_interior(field)
    iterate(kernel, arr, steps, scalars)
    return arr.get_interior()


def run_pinned(kernel: CompiledKernel, shape, lo, hi, dtype, host_in, host_out, steps: int,
               scalars=None, stream=None) -> None:
    """End-to-end through the public API with caller-provided (pinned) host buffers.

    ``host_in`` / ``host_out``: torch CPU tensors holding the interior in
    column-major order (numpy ``order='F'``).  Returns after the download
    has completed.
    """
    torch = _torch()
    if stream is None:
        arr = HaloArray(shape, lo, hi, dtype)
        arr.spare()
    else:
        # both ping-pong buffers are zero-filled on `stream` itself, before the upload
        # and the steps enqueued there (a fill left on another stream could land later)
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            arr = HaloArray(shape, lo, hi, dtype)
            arr.spare()
    arr.upload(host_in.data_ptr(), stream)
    iterate(kernel, arr, steps, scalars, stream)
    arr.download(host_out.data_ptr(), stream)
    (stream or _torch().cuda.current_stream()).synchronize()


def run_pinned_batch(kernel: CompiledKernel, shape, lo, hi, dtype, host_ins, host_outs, steps: int,
                     scalars=None, slots: int = 3) -> None:
    """``run_pinned`` over a sequence of independent fields with the PCIe copies hidden
    behind the stencil work: field i is uploaded on a copy stream while field i-1 iterates
    on the compute stream and field i-2 downloads on a third stream (H2D and D2H run in
    both PCIe directions at once).  ``slots`` device blocks rotate; an upload waits until
    its slot's previous field has been downloaded.  ``host_ins`` / ``host_outs``: pinned
    torch CPU tensors (column-major interiors), one per field (the same tensor may repeat).
    Returns after the last download has completed."""
    torch = _torch()
    n = len(host_ins)
    if len(host_outs) != n:
        raise ValueError("one output buffer per input field")
    if n == 0:
        return
    cur = torch.cuda.current_stream()
    h2d, comp, d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for st in (h2d, comp, d2h):
        st.wait_stream(cur)
    nslot = max(1, min(slots, n))
    L = _lib.make_layout(len(shape), dtype, tuple(shape), tuple(lo), tuple(hi))
    per_slot = 2 * L.count * L.elem_bytes        # one ping-pong pair
    free_b, _ = torch.cuda.mem_get_info()
    # blocks torch's caching allocator holds but does not use count as free too
    free_b += torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
    nslot = max(1, min(nslot, int(0.9 * free_b) // max(1, per_slot)))
    blocks = []
    with torch.cuda.stream(comp):
        for _ in range(nslot):
            b = HaloArray(shape, lo, hi, dtype)
            b.spare()               # both ping-pong buffers, zero-filled on `comp`
            blocks.append(b)
    h2d.wait_stream(comp)
    free = [None] * nslot           # event: the slot's last download has been issued/done
    for i in range(n):
        k = i % nslot
        b = blocks[k]
        if free[k] is not None:
            h2d.wait_event(free[k])
        b.upload(host_ins[i].data_ptr(), h2d)
        up = torch.cuda.Event()
        up.record(h2d)
        comp.wait_event(up)
        iterate(kernel, b, steps, scalars, comp)
        done = torch.cuda.Event()
        done.record(comp)
        d2h.wait_event(done)
        b.download(host_outs[i].data_ptr(), d2h)
        fr = torch.cuda.Event()
        fr.record(d2h)
        free[k] = fr
    d2h.synchronize()               # every download (and so every iteration) has completed
    cur.wait_stream(d2h)


class StepGraph:
    """``steps`` fused steps captured once as a CUDA graph and replayed.

    Construction does not advance the field (the warm-up runs on a scratch block);
    each ``replay()`` advances it by ``steps`` fused steps.

    For small (L2-resident) fields the per-launch host cost dominates (config 1:
    1024^2 in ~3 us of GPU time); a graph replays the whole chain with one
    submission.  The array must not be reallocated between capture and replay;
    ``steps`` should be even so the live buffer is the same after every replay.
    """

    def __init__(self, kernel: CompiledKernel, arr: HaloArray, steps: int, scalars=None, multi: bool = True):
        torch = _torch()
        if steps <= 0:
            raise ValueError("capture a positive number of steps")
        self.arr = arr
        self.steps = steps
        self.multi = multi                # temporal blocking where the kernel allows it
        arr.spare()                       # both ping-pong buffers exist before capture
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            # warm the module / launch caches off-graph on a scratch block of the same
            # geometry: the caller's field is not advanced by the warm-up
            scratch = HaloArray(arr.interior, arr.lo, arr.hi,
                                "float32" if arr.dtype_code == _lib.F32 else "float64", device=arr.device)
            scratch.spare(s)
            if multi:
                multi_step(kernel, scratch, 4, scalars, stream=s)
            step(kernel, scratch, scalars, stream=s)
            step(kernel, scratch, scalars, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        s.synchronize()
        del scratch
        self.graph = torch.cuda.CUDAGraph()
        l0 = _lib.launch_count()
        with torch.cuda.graph(self.graph):
            if multi:
                multi_step(kernel, arr, steps, scalars)
            else:
                for _ in range(steps):
                    step(kernel, arr, scalars)
        self.launches = _lib.launch_count() - l0     # kernels per replay
        # capture recorded the launches without running them; the host-side live buffer
        # flipped `steps` times, which is where the data is after one replay (repeated
        # replays with an odd `steps` re-read the captured input buffer)

    def replay(self) -> None:
        self.graph.replay()
