"""Run one solve-kernel evaluation on a bar mesh with a chosen decoder shape
(developer probe for new instantiations).  Usage: probe_shapes.py nx ny nz r width prec"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P  # noqa: E402
from paper_2409_03807_b200 import configs  # noqa: E402

nx, ny, nz, r, width = (int(a) for a in sys.argv[1:6])
prec = sys.argv[6] if len(sys.argv) > 6 else "fp32"
mesh = P.make_bar_mesh(nx, ny, nz, 0.25, 0.25, 1.0, pin_left=True)
mu, lam = P.lame_from_young(mesh.num_elements(), 1e5, 1e5, 0.35, seed=1)
model = P.make_bar_decoder(mesh, r, 5, width, P.Activation.Elu, seed=1)
sysm = P.ReducedSystem(mesh, mu, lam, 1000.0, model, prec)
print(sysm.solve_kernel_info(), flush=True)
sysm.set_inertia(configs.timestep0_qbar(type("pr", (), {"mesh": mesh})(), sysm.mass) if False else None, configs.DT)
E, g = sysm.eval(0.3 * np.ones(r))
print("E", E, "g0", g[0], flush=True)
