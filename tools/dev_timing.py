"""Developer timing probe (not the bench): per-kernel eval times and a few
device-resident steps per config.  Usage: python tools/dev_timing.py c1 c2 c2f c3"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402
import paper_2409_03807_b200 as P  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2", "c2f"]:
    t0 = time.time()
    pr = configs.build(name)
    sysm = pr.system()
    t1 = time.time()
    qbar = configs.timestep0_qbar(pr, sysm.mass)
    sysm.set_inertia(qbar, configs.DT)
    z = 0.5 * np.random.default_rng(0).standard_normal(pr.model.r)
    prof = sysm.profile_eval(z, reps=20)
    st = pr.initial_state()
    sysm.set_state(st)
    sysm.set_external_force(P.gravity_force(pr.mesh, sysm.mass, configs.GRAVITY))
    cfg = configs.solver_config()
    steps = 10
    t2 = time.time()
    reps, zt = sysm.simulate(steps, cfg)
    t3 = time.time()
    ve = sum(r.value_evals for r in reps)
    ge = sum(r.grad_evals for r in reps)
    it = [r.iterations for r in reps]
    print(f"{name}: setup {t1-t0:.1f}s  profile(ms) " + " ".join(f"{k}={v:.4f}" for k, v in prof.items()))
    print(f"   {steps} steps {1e3*(t3-t2)/steps:.3f} ms/step  value_evals={ve} grad_evals={ge} iters={it} "
          f"codes={[r.code for r in reps]} dev_ms={[round(r.wall_time_ms,3) for r in reps]}")
    sysm.close()
