"""B200-native LOPe stencil hot path (arXiv 1502.03504, reference package ``lopec``).

Python host API over ``liblope_b200.so`` (hand-written sm_100a CUDA, C ABI in
``include/lope_b200.h``):

* kernel definition: :class:`KernelBuilder` / :func:`from_lopec` -> ``KernelIR``
* halo-array declaration: :class:`HaloArray`
* apply / iterate: :func:`launch`, :func:`step`, :func:`iterate`, :func:`run`
* exchange: :func:`halo_transfer` (one image), :mod:`.dist` (slab partitions over GPUs)
* drop-in for the reference ``Machine``: :mod:`.machine`
"""

from .diagnostics import RuntimeFault
from .ir import (Footprint, IRAssign, KernelBuilder, KernelIR, deserialize, fabs, fmax, fmin,
                 from_lopec, fsqrt, serialize)

__all__ = ["RuntimeFault", "Footprint", "IRAssign", "KernelBuilder", "KernelIR", "deserialize",
           "serialize", "from_lopec", "fabs", "fmax", "fmin", "fsqrt",
           "HaloArray", "CompiledKernel", "launch", "halo_transfer", "step", "iterate", "run"]


def __getattr__(name):
    # the runtime needs torch + the CUDA library; import it on first use
    if name in ("HaloArray", "CompiledKernel", "launch", "halo_transfer", "step", "iterate", "run"):
        from . import runtime
        return getattr(runtime, name)
    raise AttributeError(name)
