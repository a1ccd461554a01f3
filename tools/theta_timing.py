"""Config-5 training-side timing: order-2 Lipschitz loss + dL/dtheta over P pairs on config 2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pr = configs.build("c2")
sysm = pr.system("fp32")
Z1, Z2 = configs.latent_pairs_c5(pr.model.r, P)
sysm.lipschitz_loss_grad(Z1[:8], Z2[:8])
for _ in range(2):
    t0 = time.perf_counter()
    loss = sysm.lipschitz_loss(Z1, Z2)
    t1 = time.perf_counter()
    loss2, grads = sysm.lipschitz_loss_grad(Z1, Z2)
    t2 = time.perf_counter()
    gn = sum(float((gW * gW).sum() + (gb * gb).sum()) for gW, gb in grads) ** 0.5
    print(f"P={P}: loss {1e3*(t1-t0):.1f} ms  loss+grad {1e3*(t2-t1):.1f} ms  loss={loss:.10e} "
          f"same={loss == loss2} |grad|={gn:.6e}")
