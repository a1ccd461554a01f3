"""Runs a few evaluations + solver steps of one config (for ncu launch lists)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402
import paper_2409_03807_b200 as P  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pr = configs.build(name)
sysm = pr.system()
sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
z = 0.5 * np.random.default_rng(0).standard_normal(pr.model.r)
print(sysm.profile_eval(z, reps=5))
sysm.set_state(pr.initial_state())
sysm.set_external_force(P.gravity_force(pr.mesh, sysm.mass, configs.GRAVITY))
reps, _ = sysm.simulate(steps, configs.solver_config())
print([(r.code, r.iterations, r.value_evals, round(r.wall_time_ms, 3)) for r in reps])
