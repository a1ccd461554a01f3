"""Cycle-level stamps of the control-cluster forward (LSB_SOLVE_EXP=32, LSB_TRACE=1)."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["LSB_TRACE"] = "1"
os.environ["LSB_SOLVE_EXP"] = "32"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P  # noqa: E402
from paper_2409_03807_b200 import configs  # noqa: E402

pr = configs.build(sys.argv[1] if len(sys.argv) > 1 else "c2")
sysm = pr.system()
sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
z = 0.5 * np.random.default_rng(0).standard_normal(pr.model.r)
for _ in range(3):
    sysm.eval(z)
buf = (C.c_ulonglong * 512)()
cnt = C.c_int()
P.check(P.lib().lsb_get_trace(sysm.handle, buf, 512, C.byref(cnt)))
prev = None
for i in range(cnt.value):
    tag, t = buf[2 * i], buf[2 * i + 1]
    if tag >= 300 and tag < 1000 and (len(sys.argv) < 3 or str(tag)[0] in sys.argv[2]):
        print(f"{tag}: +{t - prev if prev else 0} cyc")
        prev = t
