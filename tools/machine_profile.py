"""cProfile of the drop-in GPU Machine on config 2's program (4096^2 fp64, 20 steps):
where the host time of Machine.run() goes.  python tools/machine_profile.py"""
import cProfile
import pathlib
import pstats
import sys

REPO = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "baseline" / "_ref"))
import numpy as np  # noqa: E402
import lopec  # noqa: E402
from lopec.runtime import RunConfig  # noqa: E402

from oracle import lope_oracle as O  # noqa: E402
from oracle.lope_programs import program_text  # noqa: E402
from paper_1502_03504_b200.machine import Machine  # noqa: E402

prog, _ = lopec.parse_source(program_text("ninept2d"), "ninept2d.lope")
chk = lopec.check_program(prog)
field = np.asfortranarray(O.hash_field((4096, 4096), 3, np.float64))
Machine(chk, RunConfig(steps=2), field.copy()).run()
m = Machine(chk, RunConfig(steps=20), field.copy())
pr = cProfile.Profile()
pr.enable()
m.run()
m.gather()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
