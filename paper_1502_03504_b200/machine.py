"""Drop-in ``Machine`` for lopec programs with the hot path on the B200.

``lopec`` (the reference) keeps its frontend, checks and host plan; this module
subclasses ``lopec.runtime.Machine`` (runtime.py:97-737) and moves the hot path
to liblope_b200.so:

* ``_launch`` (runtime.py:541-603) -> ``lope_launch``: the launch's array
  blocks live in HBM as ``HaloArray`` twins of the reference's numpy blocks; the
  snapshot is the twin's live buffer, the stores go to its spare (no copy).
* ``_halo_exchange`` (runtime.py:643-711) -> ``lope_copy_box`` slab copies
  between the twins of all images (every image finishes dim d before any starts
  d+1; device mirrors are pulled and pushed with the same counters and events).
* everything else (allocation, scalar assignments, coindexed section copies,
  mirror copies, gather) runs in the reference code on the numpy blocks; the
  twins are synchronised lazily at those points, so a
  ``do it=1,nsteps; HALO_TRANSFER; do concurrent`` loop never leaves the GPU.

Usage mirrors the reference exactly::

    from lopec import parse_source, check_program, RunConfig
    from paper_1502_03504_b200.machine import Machine
    m = Machine(check_program(program), RunConfig(images=4, grid_rows=2), field)
    m.run(); out = m.gather()

Images are spread over the node's GPUs the way the reference spreads them over
its images (runtime.py:97-131): image k's blocks (and device mirrors) live on GPU
``devices[(k - 1) % len(devices)]`` (default: every visible GPU; ``devices=`` or
``LOPE_MACHINE_DEVICES=0,1,...`` override it, repeats allowed so the mapping can be
forced on one GPU).  A launch runs on its image's GPU; a halo slab between images on
different GPUs is one ``lope_copy_box`` on the destination GPU reading the source
through peer access, ordered by CUDA events between the GPUs' streams.

``dtype="float64"`` (default) reproduces the reference bit for bit; ``"float32"``
runs the fp32 restatement.  The per-element orders
(``RunConfig.order``) evaluate the same per-point expression, so they give the
same bits on the GPU; the launch is order-independent by construction.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .ir import from_lopec


def _lopec():
    try:
        import lopec  # noqa: F401
        from lopec import ast as last
        from lopec import plan as lplan
        from lopec import runtime as lrt
        from lopec.diagnostics import ALLOC_SHAPE, UNALLOCATED, RuntimeFault
    except ImportError as e:  # pragma: no cover - depends on the environment
        raise ImportError("paper_1502_03504_b200.machine needs the reference package `lopec` "
                          "(its frontend and host plan); install it or add it to sys.path") from e
    return last, lplan, lrt, ALLOC_SHAPE, UNALLOCATED, RuntimeFault


class _Twin:
    """Device copy of one numpy block (``arr.blocks[k]`` or ``arr.mirrors[k]``)."""

    __slots__ = ("host", "dev", "state")

    def __init__(self, host, dev):
        self.host = host           # the reference's flat float64 ndarray
        self.dev = dev             # HaloArray
        self.state = "host"        # "host": numpy newer; "device": GPU newer; "both": in sync


def _make_machine_class():
    last, lplan, lrt, ALLOC_SHAPE, UNALLOCATED, RuntimeFault = _lopec()
    from . import runtime as R

    class GpuMachine(lrt.Machine):
        """``lopec.runtime.Machine`` with launches and halo exchanges on the GPU."""

        def __init__(self, check, config, input_field=None, dtype="float64", devices=None):
            super().__init__(check, config, input_field)
            torch = R._torch()
            self.dtype = dtype
            self._np_dtype = np.float64 if dtype in ("float64", "f64") else np.float32
            if devices is None:
                env = os.environ.get("LOPE_MACHINE_DEVICES")
                devices = ([int(x) for x in env.split(",") if x.strip()] if env
                           else list(range(torch.cuda.device_count())))
            self.devices = [int(d) for d in devices] or [torch.cuda.current_device()]
            self._gk = {}
            for name, kir in self.kernels.items():
                self._gk[name] = R.CompiledKernel(from_lopec(kir), dtype)
            for a in set(self.devices):
                with torch.cuda.device(a):
                    for b in set(self.devices):
                        if a != b:
                            _lib.check(_lib.lib().lope_peer_enable(b), "lope_peer_enable")
            self._twins = {}

        def device_of(self, k):
            """GPU of image k (1-based): images round-robin over the devices."""
            return self.devices[(k - 1) % len(self.devices)]

        # -- twins -----------------------------------------------------------

        def _twin(self, arr, host, k):
            torch = R._torch()
            key = id(host)
            t = self._twins.get(key)
            if t is None or t.host is not host:
                lay = arr.layout
                with torch.cuda.device(self.device_of(k)):
                    dev = R.HaloArray(lay.interior, lay.lo, lay.hi, self.dtype, name=arr.entity.name)
                t = _Twin(host, dev)
                self._twins[key] = t
            if t.state == "host":
                src = np.ascontiguousarray(host, dtype=self._np_dtype)
                with torch.cuda.device(t.dev.device):
                    _lib.check(_lib.lib().lope_pack_padded(ctypes.byref(t.dev.layout),
                                                           src.ctypes.data_as(ctypes.c_void_p),
                                                           ctypes.c_void_p(t.dev.data.data_ptr()),
                                                           ctypes.c_void_p(R._stream_handle())),
                               "lope_pack_padded")
                    torch.cuda.current_stream().synchronize()
                t.state = "both"
            return t

        def _sync_host(self):
            """Download every twin the GPU changed into its numpy block."""
            torch = R._torch()
            pend = [t for t in self._twins.values() if t.state == "device"]
            for t in pend:
                buf = np.empty(t.host.shape, dtype=self._np_dtype)
                with torch.cuda.device(t.dev.device):
                    _lib.check(_lib.lib().lope_unpack_padded(ctypes.byref(t.dev.layout),
                                                             ctypes.c_void_p(t.dev.data.data_ptr()),
                                                             buf.ctypes.data_as(ctypes.c_void_p),
                                                             ctypes.c_void_p(R._stream_handle())),
                               "lope_unpack_padded")
                    torch.cuda.current_stream().synchronize()
                t.host[:] = buf
                t.state = "both"

        def _fence(self):
            """Order every used GPU's current stream after every other's (the BSP barrier
            between exchange phases when images sit on several GPUs)."""
            torch = R._torch()
            devs = sorted(set(self.devices))
            if len(devs) < 2:
                return
            evs = []
            for d in devs:
                e = torch.cuda.Event()
                e.record(torch.cuda.current_stream(d))
                evs.append(e)
            for d in devs:
                s = torch.cuda.current_stream(d)
                for e in evs:
                    s.wait_event(e)

        def _host_changed(self):
            """The reference code may have written any numpy block: device copies are stale."""
            for t in self._twins.values():
                if t.state == "both":
                    t.state = "host"
            live = {id(b) for a in self.arrays.values() for b in list(a.blocks.values()) + list(a.mirrors.values())}
            for key in [k for k in self._twins if k not in live]:
                del self._twins[key]

        # -- host actions run in the reference code ---------------------------

        def _do(self, a, k):
            if isinstance(a, lplan.LaunchConcurrent):
                self._launch(a, k)
                return
            if isinstance(a, (lplan.GridSetup, lplan.GetSubimage, lplan.ScalarAssign)):
                super()._do(a, k)
                return
            self._sync_host()
            super()._do(a, k)
            self._host_changed()

        def _alloc_host(self, a, k):
            self._sync_host()
            super()._alloc_host(a, k)
            self._host_changed()

        def _dealloc(self, a, k):
            self._sync_host()
            super()._dealloc(a, k)
            self._host_changed()

        def _read_element(self, e, k):
            self._sync_host()
            return super()._read_element(e, k)

        def run(self):
            super().run()
            self._sync_host()

        def gather(self, name=None):
            self._sync_host()
            return super().gather(name)

        # -- the hot path ---------------------------------------------------------

        def _launch(self, a, k):
            """runtime.py:541-603 with the vector evaluation on the GPU."""
            gk = self._gk[a.kernel]
            kir = self.kernels[a.kernel]
            handle = self._device_handle(a.target, k, a.pos)
            on_device = handle != k
            ranges = [(self._int(r.lo, k, "launch range"), self._int(r.hi, k, "launch range"))
                      for r in a.ranges]
            bound = []
            scalars = {}
            interior = None
            for p, arg in zip(self.check.kernels[a.kernel].kernel.params, a.args):
                if isinstance(arg, last.ElementArg):
                    arr = self._live_array(arg.array, k, a.pos)
                    self._require_allocated(arr, k, a.pos)
                    if on_device:
                        if k not in arr.mirrors:
                            raise RuntimeFault(UNALLOCATED, f"'{arg.array}' is not allocated on the device",
                                               a.pos)
                        host = arr.mirrors[k]
                    else:
                        host = arr.blocks[k]
                    bound.append((arr, host))
                    if interior is None:
                        interior = arr.layout.interior
                else:
                    v = self.eval(arg, k)
                    scalars[p] = float(v) if kir.param_types[p] == "real" else int(v)
            if interior is None:
                raise RuntimeFault(ALLOC_SHAPE, f"kernel '{a.kernel}' was launched without an array argument",
                                   a.pos)
            for d, (lo, hi) in enumerate(ranges):
                if lo < 1 or hi > interior[d]:
                    raise RuntimeFault(ALLOC_SHAPE, f"launch range {lo}:{hi} lies outside the interior "
                                                    f"1:{interior[d]} in dim {d + 1}", a.pos)
            self.counters[k]["launches"] += 1
            if on_device:
                self.counters[k]["device_launches"] += 1
            self.events.append(("launch", k, a.kernel, on_device))
            if any(lo > hi for lo, hi in ranges):
                return
            twins = [self._twin(arr, host, k) for arr, host in bound]
            with R._torch().cuda.device(self.device_of(k)):
                R.launch(gk, [t.dev for t in twins], ranges, scalars)
            stored = set(kir.stored_arrays)
            for (p, t) in zip([q for q in gk.ir.array_params], twins):
                if p in stored:
                    t.state = "device"

        def _halo_exchange(self, name, pos):
            """runtime.py:643-711 on the twins: per dim, pull mirrors, fill, push."""
            arr = self.arrays.get(name)
            if arr is None:
                raise RuntimeFault(UNALLOCATED, f"halo_transfer of '{name}' before it is allocated", pos)
            for k in self.images:
                self._require_allocated(arr, k, pos)
            lay = arr.layout
            self.events.append(("halo_transfer", name))
            rank = lay.rank
            padded = lay.padded()
            blocks = {k: self._twin(arr, arr.blocks[k], k) for k in self.images}
            mirrors = {k: self._twin(arr, arr.mirrors[k], k) for k in self.images if k in arr.mirrors}
            torch = R._torch()
            cur_dev = torch.device("cuda", torch.cuda.current_device())
            cur_stream = ctypes.c_void_p(R._stream_handle())
            self._fence()
            for d in range(rank):
                w_lo, w_hi = lay.lo[d], lay.hi[d]
                if w_lo == 0 and w_hi == 0:
                    continue
                m_d = lay.interior[d]

                def box(start, width):
                    lo3 = [0, 0, 0]
                    ext = [int(padded[i]) if i < rank else 1 for i in range(3)]
                    lo3[d] = start
                    ext[d] = width
                    return lo3, ext

                pending = {}      # destination device -> [(dst ptr, src ptr, dlo, slo, ext)]

                def copy(dst, src, dstart, sstart, width):
                    # queued; flush() issues each phase's slabs as one lope_copy_boxes per
                    # destination GPU (a source on another GPU is read over NVLink, peer
                    # access enabled at construction).  Within a phase no slab written
                    # is read by another, so one launch per phase keeps the semantics.
                    dlo, ext = box(dstart, width)
                    slo, _ = box(sstart, width)
                    pending.setdefault(dst.dev.device, []).append(
                        (dst.dev.data.data_ptr(), src.dev.data.data_ptr(), dlo, slo, ext))

                def flush():
                    L = blocks[self.images[0]].dev.layout
                    for dev, items in pending.items():
                        n = len(items)
                        args = (ctypes.byref(L), n, (ctypes.c_void_p * n)(*[it[0] for it in items]),
                                (ctypes.c_void_p * n)(*[it[1] for it in items]),
                                (ctypes.c_int64 * (3 * n))(*[v for it in items for v in it[2]]),
                                (ctypes.c_int64 * (3 * n))(*[v for it in items for v in it[3]]),
                                (ctypes.c_int64 * (3 * n))(*[v for it in items for v in it[4]]))
                        if dev == cur_dev:      # the common case: no device switch, cached stream
                            _lib.check(_lib.lib().lope_copy_boxes(*args, cur_stream), "lope_copy_boxes")
                        else:
                            with torch.cuda.device(dev):
                                _lib.check(_lib.lib().lope_copy_boxes(
                                    *args, ctypes.c_void_p(R._stream_handle())), "lope_copy_boxes")
                    pending.clear()

                low_halo, high_halo = 0, w_lo + m_d
                low_int, high_int = w_lo, m_d
                # phase 1: refresh the blocks' border slabs from the device mirrors
                for k in self.images:
                    if k not in mirrors:
                        continue
                    if w_hi:
                        copy(blocks[k], mirrors[k], low_int, low_int, w_hi)
                        self.counters[k]["d2h"] += 1
                        self.events.append(("d2h", k, name, d))
                    if w_lo:
                        copy(blocks[k], mirrors[k], high_int, high_int, w_lo)
                        self.counters[k]["d2h"] += 1
                        self.events.append(("d2h", k, name, d))
                    blocks[k].state = "device"
                flush()
                self._fence()
                # phase 2: neighbour fills (interior slabs are never written here, so
                # the image order does not matter)
                for k in self.images:
                    if w_lo:
                        nb = self.grid.neighbor(k, 0 if d == 0 else 1, -1)
                        copy(blocks[k], blocks[nb], low_halo, high_int, w_lo)
                        self.events.append(("halo_fill", k, name, d, "low"))
                    if w_hi:
                        nb = self.grid.neighbor(k, 0 if d == 0 else 1, +1)
                        copy(blocks[k], blocks[nb], high_halo, low_int, w_hi)
                        self.events.append(("halo_fill", k, name, d, "high"))
                    blocks[k].state = "device"
                flush()
                self._fence()
                # phase 3: push the received halo slabs down to the mirrors
                for k in self.images:
                    if k not in mirrors:
                        continue
                    if w_lo:
                        copy(mirrors[k], blocks[k], low_halo, low_halo, w_lo)
                        self.counters[k]["h2d"] += 1
                        self.events.append(("h2d", k, name, d))
                    if w_hi:
                        copy(mirrors[k], blocks[k], high_halo, high_halo, w_hi)
                        self.counters[k]["h2d"] += 1
                        self.events.append(("h2d", k, name, d))
                    mirrors[k].state = "device"
                flush()
                self._fence()

    return GpuMachine


_CLS = None


def Machine(check, config, input_field=None, dtype="float64", devices=None):
    """Construct the GPU-backed drop-in for ``lopec.runtime.Machine``."""
    global _CLS
    if _CLS is None:
        _CLS = _make_machine_class()
    return _CLS(check, config, input_field, dtype, devices)


def machine_class():
    global _CLS
    if _CLS is None:
        _CLS = _make_machine_class()
    return _CLS
