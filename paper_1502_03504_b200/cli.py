"""``lopec`` command line with ``run`` on the B200.

The reference CLI (``lopec/cli.py``) is reused unchanged -- same subcommands,
options, exit codes, diagnostics and ``%.17g`` field output -- except that
``cmd_run`` (cli.py:111-142) constructs the GPU ``Machine`` from
``paper_1502_03504_b200.machine`` instead of ``lopec.runtime.Machine``::

    python -m paper_1502_03504_b200.cli run prog.lope --images 4 --grid-rows 2 --steps 100

``LOPE_DTYPE=float32`` selects the fp32 restatement; the default (float64)
reproduces the reference bit for bit.
"""

from __future__ import annotations

import os
import sys
from typing import Optional


def main(argv: Optional[list] = None) -> int:
    from .machine import _lopec, Machine
    _lopec()                                   # loud ImportError without the reference package
    import lopec.cli as C

    dtype = os.environ.get("LOPE_DTYPE", "float64")

    def gpu_machine(check, config, input_field=None):
        return Machine(check, config, input_field, dtype=dtype)

    saved = C.Machine
    C.Machine = gpu_machine
    try:
        return C.main(argv)
    finally:
        C.Machine = saved


if __name__ == "__main__":
    sys.exit(main())
