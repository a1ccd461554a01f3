"""Order-2 Lipschitz loss and its theta-gradient on a smooth-output-layer decoder (27,648 tets, r = 16)
against the oracle (one pair)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P  # noqa: E402
from oracle import pyoracle as oracle  # noqa: E402

mesh = P.make_bar_mesh(12, 12, 32, 1.0, 0.4, 0.4, jitter_frac=0.05, seed=11)
rng = np.random.default_rng(12)
n, r, h = mesh.num_dofs(), 16, 32
layers = []
dims = [r, h, h]
for i in range(2):
    layers.append(P.Layer(rng.standard_normal((dims[i + 1], dims[i])) * 0.4, 0.1 * rng.standard_normal(dims[i + 1]),
                          P.Activation.Silu))
X = mesh.vertices[mesh.free_vertices]
k = rng.uniform(-4.0, 4.0, (h, 3))
ph = rng.uniform(0, 2 * np.pi, h)
B = rng.standard_normal((3, h))
basis = 1.0 + 0.5 * np.sin(X @ k.T + ph)
layers.append(P.Layer(0.02 * (basis[:, None, :] * B[None, :, :]).reshape(n, h), np.zeros(n), P.Activation.Identity))
shift = P.dof_pack(mesh, mesh.vertices)
scale = np.ones(n)
model = P.SubspaceModel(r, n, layers, shift, scale)
mu = 2.0e4 + 1.0e3 * rng.random(mesh.num_elements())
lam = 8.0e4 + 1.0e3 * rng.random(mesh.num_elements())
o = oracle.Oracle.from_mesh(mesh.vertices, mesh.elements, mesh.pinned)
o.set_material(mu, lam, 1000.0)
o.set_decoder([(l.W, l.b, int(l.act)) for l in layers], shift, scale, r)
sysm = P.ReducedSystem(mesh, mu, lam, 1000.0, model, "fp32")
Z1 = 0.5 * rng.standard_normal((1, r))
Z2 = 0.5 * rng.standard_normal((1, r))
lt, gt = sysm.lipschitz_loss_grad(Z1, Z2)
t0 = time.time()
lo, go = o.lipschitz_loss2_grad(Z1, Z2, threads=16)
print(f"oracle {time.time() - t0:.1f} s; loss rel err {abs(lt - lo) / abs(lo):.2e}")
for li, ((a, b), (c, d)) in enumerate(zip(gt, go)):
    print(f"layer {li}: dW rel err {np.linalg.norm(a - c) / np.linalg.norm(c):.2e}  db rel err "
          f"{np.linalg.norm(b - d) / max(np.linalg.norm(d), 1e-300):.2e}")
