"""Repeated single evaluations of one config (target for ncu captures)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pr = configs.build(name)
sysm = pr.system()
sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
rng = np.random.default_rng(0)
for _ in range(reps):
    E, g = sysm.eval(0.5 * rng.standard_normal(pr.model.r))
print(name, sysm.solve_kernel_info(), E)
