"""Config-4 timing probe: E+grad for 4096 z on the config-2 problem (fp32)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pr = configs.build("c2")
sysm = pr.system("fp32")
sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
Z = configs.latent_batch_c4(pr.model.r, B)
sysm.eval_batched(Z[:128])
for _ in range(reps):
    t0 = time.perf_counter()
    E, G = sysm.eval_batched(Z)
    dt = time.perf_counter() - t0
    print(f"B={B}: {dt*1e3:.2f} ms  {B/dt:.0f} evals/s  E[0]={E[0]:.8e}")
