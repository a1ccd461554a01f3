"""Repeats the c1 free-running simulate and reports steps whose L-BFGS iteration
counts differ from the first run's (race hunting)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P  # noqa: E402
from paper_2409_03807_b200 import configs  # noqa: E402

reps_n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
pr = configs.build("c1")
ref = None
bad = 0
for rep in range(reps_n):
    sysm = pr.system("fp64")
    sysm.set_state(pr.initial_state())
    sysm.set_external_force(P.gravity_force(pr.mesh, sysm.mass, configs.GRAVITY))
    reps, zt = sysm.simulate(steps, configs.solver_config())
    it = np.array([r.iterations for r in reps])
    if ref is None:
        ref = it
        print("ref", it.tolist())
    elif not np.array_equal(it, ref):
        bad += 1
        print("rep", rep, "MISMATCH", it.tolist())
    sysm.close()
print("exp", os.environ.get("LSB_SOLVE_EXP", "0"), "bad", bad, "of", reps_n - 1)
