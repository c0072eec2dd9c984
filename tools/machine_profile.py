"""cProfile of the drop-in GPU Machine: where the host time of Machine.run() goes.
    python tools/machine_profile.py [program] [n] [steps]   (default ninept2d 4096 20)"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "ninept2d"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
prog, _ = lopec.parse_source(program_text(name), f"{name}.lope")
chk = lopec.check_program(prog)
field = np.asfortranarray(O.hash_field((n, n), 3, np.float64))
Machine(chk, RunConfig(steps=2), field.copy()).run()
m = Machine(chk, RunConfig(steps=steps), field.copy())
pr = cProfile.Profile()
pr.enable()
m.run()
m.gather()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
