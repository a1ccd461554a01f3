"""Determinism stress: repeated E+grad evaluations at fixed z must be bitwise
identical (every reduction has a fixed order).  Reports mismatching reps."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P  # noqa: E402
from paper_2409_03807_b200 import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
names = sys.argv[2:] or ["c1", "c2", "c2f"]
systems = {}
for name in names:
    pr = configs.build(name)
    s = pr.system()
    s.set_inertia(configs.timestep0_qbar(pr, s.mass), configs.DT)
    systems[name] = (pr, s)
rng = np.random.default_rng(5)
for name, (pr, s) in systems.items():
    zs = [0.5 * rng.standard_normal(pr.model.r) for _ in range(3)]
    ref = [s.eval(z) for z in zs]
    bad_e = bad_g = 0
    for rep in range(reps):
        for k, z in enumerate(zs):
            E, g = s.eval(z)
            if E != ref[k][0]:
                bad_e += 1
                if bad_e <= 3:
                    print(name, "rep", rep, "z", k, "E", E, "ref", ref[k][0], flush=True)
            if not np.array_equal(g, ref[k][1]):
                bad_g += 1
                if bad_g <= 3:
                    d = np.abs(g - ref[k][1])
                    print(name, "rep", rep, "z", k, "grad maxdiff", d.max(), "at", int(d.argmax()), flush=True)
    print(name, s.solve_kernel_info()["in_use"], "E mismatches", bad_e, "grad mismatches", bad_g, "of", 3 * reps, flush=True)
