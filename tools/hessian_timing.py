"""Config-5 timing probe: order-2 Lipschitz loss over 1024 pairs on config 2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pr = configs.build("c2")
sysm = pr.system("fp32")
Z1, Z2 = configs.latent_pairs_c5(pr.model.r, P)
sysm.lipschitz_loss(Z1[:8], Z2[:8])
for _ in range(2):
    t0 = time.perf_counter()
    loss = sysm.lipschitz_loss(Z1, Z2)
    dt = time.perf_counter() - t0
    print(f"P={P}: {dt*1e3:.1f} ms  {2*P/dt:.0f} Hessians/s  loss={loss:.10e}")
