"""Error convention of the reference (lopec/diagnostics.py:18-41, 105-121), restated.

The C ABI returns the numeric part of the E-code; the host side raises
``RuntimeFault`` with the same code strings the reference uses, so callers that
match on ``fault.code == "E108"`` keep working.
"""

from __future__ import annotations

HALO_BOUNDS = "E102"
IMPURE_KERNEL = "E104"
ALLOC_SHAPE = "E108"
GRID_FACTOR = "E201"
UNALLOCATED = "E202"


class RuntimeFault(Exception):
    """Execution-time failure, rendered ``[pos: ]error[E###]: message``."""

    def __init__(self, code: str, message: str, pos=None):
        self.code = code
        self.message = message
        self.pos = pos
        super().__init__(self.render())

    def render(self) -> str:
        if self.pos is not None:
            return f"{self.pos}: error[{self.code}]: {self.message}"
        return f"error[{self.code}]: {self.message}"
