"""Accuracy of the evaluation paths (batched fp32 and single-instance) on a decoder whose output layer varies
smoothly over the mesh, against the oracle (the Hessian path has its own GPU test of this case)."""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_03807_b200 as P
from oracle import pyoracle as oracle
def rel_err(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
mesh = P.make_bar_mesh(12, 12, 32, 1.0, 0.4, 0.4, jitter_frac=0.05, seed=11)
rng = np.random.default_rng(12)
n, r, h = mesh.num_dofs(), 16, 32
layers = []
dims = [r, h, h]
for i in range(2):
    layers.append(P.Layer(rng.standard_normal((dims[i + 1], dims[i])) * 0.4, 0.1 * rng.standard_normal(dims[i + 1]), P.Activation.Silu))
X = mesh.vertices[mesh.free_vertices]
k = rng.uniform(-4.0, 4.0, (h, 3)); ph = rng.uniform(0, 2 * np.pi, h); B = rng.standard_normal((3, h))
basis = 1.0 + 0.5 * np.sin(X @ k.T + ph)
Wout = 0.02 * (basis[:, None, :] * B[None, :, :]).reshape(n, h)
layers.append(P.Layer(Wout, np.zeros(n), P.Activation.Identity))
shift = P.dof_pack(mesh, mesh.vertices); scale = np.ones(n)
model = P.SubspaceModel(r, n, layers, shift, scale)
mu = 2.0e4 + 1.0e3 * rng.random(mesh.num_elements()); lam = 8.0e4 + 1.0e3 * rng.random(mesh.num_elements())
o = oracle.Oracle.from_mesh(mesh.vertices, mesh.elements, mesh.pinned)
o.set_material(mu, lam, 1000.0)
o.set_decoder([(l.W, l.b, int(l.act)) for l in layers], shift, scale, r)
Z = 0.5 * rng.standard_normal((256, r))
for prec in ("fp32", "fp64"):
    sysm = P.ReducedSystem(mesh, mu, lam, 1000.0, model, prec)
    E, G = sysm.eval_batched(Z)
    Eo, Go = o.eval_batch(Z[:4], qbar=None)
    print(prec, "batched E err", rel_err(E[:4], Eo), "G err", max(rel_err(G[i], Go[i]) for i in range(4)))
    e1, g1 = sysm.eval(Z[0])
    print(prec, "single E err", abs(e1 - Eo[0]) / abs(Eo[0]), "G err", rel_err(g1, Go[0]))
    sysm.close()
