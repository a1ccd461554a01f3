"""Per-eval device time of the solve kernel under different L2-flush strategies (experiment)."""
import os
import subprocess
import sys

code = r'''
import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_2409_03807_b200 as P
from paper_2409_03807_b200 import configs
pr = configs.build("c2"); s = pr.system()
s.set_inertia(configs.timestep0_qbar(pr, s.mass), configs.DT)
Z = configs.gaussian_latents(5, 40, pr.model.r)
L = P.lib()
for fb in ([512 << 20, 0] if os.environ.get("LSB_FLUSH_MODE") != "kernel" else [512 << 20]):
    ev = np.zeros(40); of = np.zeros(40); E = np.zeros(40)
    P.check(L.lsb_bench_evals(s.handle, 40, P.dptr(Z), fb, P.dptr(ev), P.dptr(of), P.dptr(E)))
    print(os.environ.get("LSB_FLUSH_MODE", "memset"), "flush" if fb else "noflush",
          "eval us %.1f (median %.1f)" % (ev[5:].mean() * 1e3, np.median(ev[5:]) * 1e3))
'''
for mode in ["memset", "kernel"]:
    env = dict(os.environ)
    if mode == "kernel":
        env["LSB_FLUSH_MODE"] = "kernel"
    subprocess.run([sys.executable, "-c", code], env=env)
