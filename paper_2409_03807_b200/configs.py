"""The BASELINE.json workloads as concrete problems.

Every mesh, material and decoder is synthetic and seeded; no dataset is read.

  c1  4x4x16 Kuhn bar (1,536 tets, 425 verts), d=8, 5x64 ELU, seed 0, fp64, 100 steps
  c2  16x16x64 (98,304 tets, 18,785 verts), d=16, 5x128 ELU, seed 1, fp64/fp32, 200 steps
  c3  32x32x128 (786,432 tets, 140,481 verts), jitter 0.1 cell (seed 2), per-tet
      E ~ U[5e4, 5e5] (seed 2), d=32, 5x256 ELU, seed 2, fp32, 100 steps, 5 m/s
      impulse on the free (i = nx) face along +y at t = 0
  c4  c2 problem, 4,096 z ~ N(0, 0.5^2 I) from substream(3, 0), objective of
      timestep 0 (qbar = X + h^2 g)
  c5  c2 problem, 1,024 pairs (z1, z2) ~ N(0, 0.5^2 I) from substream(4, 0),
      drawn z1 then z2 per pair; Hessians of the elastic potential only.

Bar: 0.25 x 0.25 x 1.0 m, pinned on the x = 0 (i = 0) face, gravity -9.8 along z,
E = 1e5 Pa, nu = 0.35, rho = 1000 kg/m^3, h = 1/60 s, L-BFGS memory 5,
max line search 128, max iterations 1024, eps 1e-5.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

from . import lipsub as L

GRAVITY = (0.0, 0.0, -9.8)
DT = 1.0 / 60.0
BAR = (0.25, 0.25, 1.0)


@dataclass
class ConfigSpec:
    name: str
    grid: Tuple[int, int, int]
    latent: int
    hidden_layers: int
    width: int
    seed: int
    steps: int
    precision: str
    jitter: float = 0.0
    young: Tuple[float, float] = (1e5, 1e5)
    impulse: Optional[Tuple[float, float, float]] = None
    nu: float = 0.35
    density: float = 1000.0


SPECS = {
    "c1": ConfigSpec("c1", (4, 4, 16), 8, 5, 64, 0, 100, "fp64"),
    "c2": ConfigSpec("c2", (16, 16, 64), 16, 5, 128, 1, 200, "fp64"),
    "c2f": ConfigSpec("c2f", (16, 16, 64), 16, 5, 128, 1, 200, "fp32"),
    "c3": ConfigSpec("c3", (32, 32, 128), 32, 5, 256, 2, 100, "fp32", jitter=0.1, young=(5e4, 5e5),
                     impulse=(0.0, 5.0, 0.0)),
}


def solver_config(spec: ConfigSpec | None = None) -> L.SolverConfig:
    return L.SolverConfig(epsilon=1e-5, max_iters=1024, max_linesearch=128, lbfgs_history=5, dt=DT)


@dataclass
class Problem:
    spec: ConfigSpec
    mesh: L.Mesh
    mu: np.ndarray
    lam: np.ndarray
    model: L.SubspaceModel

    def system(self, precision: Optional[str] = None, device: int = 0) -> L.ReducedSystem:
        return L.ReducedSystem(self.mesh, self.mu, self.lam, self.spec.density, self.model,
                               precision or self.spec.precision, device)

    def initial_state(self) -> L.SimState:
        st = L.rest_state(self.mesh, self.model.r)
        if self.spec.impulse is not None:
            nx = self.spec.grid[0]
            ny, nz = self.spec.grid[1], self.spec.grid[2]
            # free end = grid face i == nx (ids (nx*vy + j)*vz + k)
            ids = np.arange(nx * (ny + 1) * (nz + 1), (nx + 1) * (ny + 1) * (nz + 1))
            st.velocities[ids] = np.asarray(self.spec.impulse)
        return st


def build(name: str) -> Problem:
    spec = SPECS[name]
    nx, ny, nz = spec.grid
    mesh = L.make_bar_mesh(nx, ny, nz, *BAR, jitter_frac=spec.jitter, seed=spec.seed, pin_left=True)
    mu, lam = L.lame_from_young(mesh.num_elements(), spec.young[0], spec.young[1], spec.nu, seed=spec.seed)
    model = L.make_bar_decoder(mesh, spec.latent, spec.hidden_layers, spec.width, L.Activation.Elu,
                               seed=spec.seed, out_scale=1e-2)
    return Problem(spec, mesh, mu, lam, model)


def gaussian_latents(seed: int, count: int, r: int, std: float = 0.5) -> np.ndarray:
    """count x r draws of std * randn from substream(seed, 0) in row order
    (reference rng.hpp:23-51 semantics, via the library's bit-stable generator)."""
    out = np.zeros(count * r)
    L.check(L.lib().lsb_gaussian_stream(seed, 0, count * r, std, L.dptr(out)))
    return out.reshape(count, r)


def latent_batch_c4(r: int, count: int = 4096) -> np.ndarray:
    return gaussian_latents(3, count, r)


def latent_pairs_c5(r: int, pairs: int = 1024) -> Tuple[np.ndarray, np.ndarray]:
    Z = gaussian_latents(4, 2 * pairs, r)
    Z1, Z2 = Z[0::2].copy(), Z[1::2].copy()
    for p in range(pairs):  # resample coincident pairs (losses.cpp:279-283); never hit in practice
        if np.linalg.norm(Z1[p] - Z2[p]) < 1e-12:
            raise RuntimeError("coincident latent pair")
    return Z1, Z2


def timestep0_qbar(problem: Problem, mass: np.ndarray) -> np.ndarray:
    """qbar of reduced_step from rest: q + h v + h^2 f/m = X_free + h^2 g."""
    q0 = L.dof_pack(problem.mesh, problem.mesh.vertices)
    g = np.tile(np.asarray(GRAVITY), problem.mesh.num_free_vertices())
    return q0 + DT * DT * g
