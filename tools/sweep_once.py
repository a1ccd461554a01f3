"""A few config-3 E+grad evaluations on the default device path (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
pr = configs.build(name)
sysm = pr.system()
sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
z = configs.gaussian_latents(5, 1, pr.model.r)[0]
for _ in range(3):
    print(sysm.eval(z)[0])
