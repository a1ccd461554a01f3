"""Python mirror of the reference `lipsub` interface for the hot path.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/lipsub/*.hpp); every compute call goes through
the C ABI of the sm_100a library (include/lipsub_b200.h).  There is no CPU
fallback anywhere in this module.

  reference (C++)                               here
  -------------------------------------------   -------------------------------------
  Mesh / build_mesh / make_bar_3d (mesh.hpp)    Mesh, build_mesh, make_bar_mesh (6-tet)
  lump_mass, dof_pack / dof_unpack              Mesh.lump_mass, dof_pack, dof_unpack
  Activation, Layer, SubspaceModel (net.hpp)    Activation, Layer, SubspaceModel
  make_mlp_model                                make_bar_decoder (Xavier-normal variant)
  SolverConfig, ExitReport, SimState,           SolverConfig, ExitReport, SimState,
  FrameInput (reduced_solver.hpp)               FrameInput
  PotentialContext + MassMatrix + model         ReducedSystem (one GPU context)
  ReducedObjective::eval / as_objective         ReducedObjective.eval / as_objective
  lbfgs_minimize                                lbfgs_minimize (device-resident for a
                                                ReducedObjective, host loop otherwise)
  reduced_step                                  reduced_step
  reduced_potential_hessian (losses.hpp)        ReducedSystem.hessian_batched
  lipschitz_loss(model, pairs, 2, pot)          lipschitz_loss
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import check, dptr, iptr, lib  # noqa: F401


# --------------------------------------------------------------------------- net.hpp
class Activation(enum.IntEnum):
    Identity = 0
    Silu = 1
    Tanh = 2
    Elu = 3  # BASELINE.json extension (C^1; x <= 0 branch owns x == 0)


def activation_from_string(name: str) -> Activation:
    """reference net.cpp:16-23 (+ 'elu')."""
    table = {"identity": Activation.Identity, "silu": Activation.Silu, "tanh": Activation.Tanh,
             "elu": Activation.Elu}
    if name == "relu":
        raise ValueError("activation: relu is not C^2; use silu or tanh")
    if name not in table:
        raise ValueError(f"activation: unknown tag '{name}'")
    return table[name]


@dataclass
class Layer:
    W: np.ndarray  # rows x cols
    b: np.ndarray  # rows
    act: Activation = Activation.Identity


@dataclass
class SubspaceModel:
    r: int
    n: int
    decoder: List[Layer]
    norm_shift: np.ndarray
    norm_scale: np.ndarray

    def validate(self):
        """reference SubspaceModel::validate (net.cpp:66-88)."""
        if self.r <= 0 or self.n <= 0:
            raise ValueError("model: r and n must be positive")
        width = self.r
        for l in self.decoder:
            if l.W.shape[1] != width or l.b.shape[0] != l.W.shape[0]:
                raise ValueError("model: decoder layer shapes do not chain")
            width = l.W.shape[0]
        if width != self.n:
            raise ValueError("model: decoder output width != n")
        if self.norm_shift.shape[0] != self.n or self.norm_scale.shape[0] != self.n:
            raise ValueError("model: normalization vectors must have length n")
        if np.any(self.norm_scale <= 0):
            raise ValueError("model: norm_scale entries must be positive")


# --------------------------------------------------------------------------- mesh.hpp
@dataclass
class Mesh:
    vertices: np.ndarray           # V x 3 rest positions
    elements: np.ndarray           # E x 4 int32
    pinned: np.ndarray             # sorted unique int32

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64)
        self.elements = np.ascontiguousarray(self.elements, dtype=np.int32)
        self.pinned = np.ascontiguousarray(np.unique(np.asarray(self.pinned, dtype=np.int32)), dtype=np.int32)
        V = self.num_vertices()
        if self.pinned.size and (self.pinned.min() < 0 or self.pinned.max() >= V):
            raise RuntimeError("mesh: pinned vertex out of range")
        self.vertex_pinned = np.zeros(V, dtype=bool)
        self.vertex_pinned[self.pinned] = True
        self.free_index = np.full(V, -1, dtype=np.int64)
        free = np.nonzero(~self.vertex_pinned)[0]
        self.free_index[free] = np.arange(free.size)
        self.free_vertices = free

    def num_vertices(self) -> int:
        return int(self.vertices.shape[0])

    def num_elements(self) -> int:
        return int(self.elements.shape[0])

    def num_free_vertices(self) -> int:
        return int(self.free_vertices.size)

    def num_dofs(self) -> int:
        return 3 * self.num_free_vertices()


def build_mesh(vertices, elements, pinned=()) -> Mesh:
    """reference build_mesh (mesh.cpp:90-145); rest-shape validation runs in lsb_create."""
    return Mesh(np.asarray(vertices, np.float64).reshape(-1, 3), np.asarray(elements, np.int32).reshape(-1, 4),
                np.asarray(pinned, np.int32))


def make_bar_mesh(nx: int, ny: int, nz: int, width: float, height: float, depth: float,
                  jitter_frac: float = 0.0, seed: int = 0, pin_left: bool = True) -> Mesh:
    """Six-tet (Kuhn) bar on the make_bar_3d grid (mesh.cpp:357-397); pins the i == 0 face."""
    L = lib()
    V, E, P = C.c_int(), C.c_int(), C.c_int()
    check(L.lsb_bar_mesh_size(nx, ny, nz, int(pin_left), C.byref(V), C.byref(E), C.byref(P)))
    X = np.zeros((V.value, 3), np.float64)
    T = np.zeros((E.value, 4), np.int32)
    pins = np.zeros(max(P.value, 1), np.int32)
    check(L.lsb_make_bar_mesh(nx, ny, nz, width, height, depth, jitter_frac, seed, int(pin_left), dptr(X),
                              iptr(T), iptr(pins)))
    return Mesh(X, T, pins[:P.value])


def lame_from_young(num_tets: int, E_lo: float, E_hi: float, nu: float, seed: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    mu = np.zeros(num_tets)
    lam = np.zeros(num_tets)
    check(lib().lsb_lame_from_young(num_tets, E_lo, E_hi, nu, seed, dptr(mu), dptr(lam)))
    return mu, lam


def make_bar_decoder(mesh: Mesh, r: int, hidden_layers: int, width: int, act: Activation = Activation.Elu,
                     seed: int = 0, out_scale: float = 1e-2) -> SubspaceModel:
    """Xavier-normal MLP decoder (make_mlp_model structure, net.cpp:90-123)."""
    n = mesh.num_dofs()
    dims = [r] + [width] * hidden_layers + [n]
    total = sum(dims[i + 1] * dims[i] for i in range(len(dims) - 1))
    Wp = np.zeros(total)
    shift = np.zeros(n)
    scale = np.zeros(n)
    pins = mesh.pinned if mesh.pinned.size else np.zeros(1, np.int32)
    check(lib().lsb_make_bar_decoder(mesh.num_vertices(), dptr(mesh.vertices), int(mesh.pinned.size), iptr(pins),
                                     r, hidden_layers, width, int(act), seed, out_scale, dptr(Wp), dptr(shift),
                                     dptr(scale)))
    layers = []
    off = 0
    for i in range(len(dims) - 1):
        rows, cols = dims[i + 1], dims[i]
        W = Wp[off:off + rows * cols].reshape(rows, cols).copy()
        off += rows * cols
        a = act if i < len(dims) - 2 else Activation.Identity
        layers.append(Layer(W, np.zeros(rows), a))
    m = SubspaceModel(r, n, layers, shift, scale)
    m.validate()
    return m


def dof_pack(mesh: Mesh, full_positions: np.ndarray) -> np.ndarray:
    """reference dof_pack (mesh.cpp:436-446)."""
    return np.ascontiguousarray(full_positions[mesh.free_vertices].reshape(-1))


def dof_unpack(mesh: Mesh, q: np.ndarray, pin_values: np.ndarray) -> np.ndarray:
    """reference dof_unpack (mesh.cpp:448-461)."""
    if q.shape[0] != mesh.num_dofs():
        raise ValueError("dof_unpack: q has wrong length")
    full = np.array(pin_values, dtype=np.float64, copy=True).reshape(-1, 3)
    full[mesh.free_vertices] = q.reshape(-1, 3)
    return full


# --------------------------------------------------------------------------- reduced_solver.hpp
@dataclass
class SolverConfig:
    epsilon: float = 1e-5
    max_iters: int = 1024
    max_linesearch: int = 128
    lbfgs_history: int = 8
    dt: float = 0.05

    def validate(self):
        """reference SolverConfig::validate (reduced_solver.cpp:14-20)."""
        if not (self.epsilon > 0.0):
            raise ValueError("solver: epsilon must be > 0")
        if self.max_iters < 1 or self.max_linesearch < 1:
            raise ValueError("solver: iteration caps must be >= 1")
        if not (self.dt > 0.0):
            raise ValueError("solver: dt must be > 0")
        if self.lbfgs_history < 1:
            raise ValueError("solver: lbfgs history must be >= 1")

    def _c(self):
        return _capi.lsb_solver_config(self.epsilon, self.max_iters, self.max_linesearch, self.lbfgs_history, self.dt)


class ExitCode(enum.IntEnum):
    Converged = 1
    Saddle = 2
    LinesearchCap = 3
    IterationCap = 4


def exit_code_name(code: int) -> str:
    """reference exit_code_name (reduced_solver.cpp:22-30)."""
    return {1: "I", 2: "II", 3: "III", 4: "IV"}.get(int(code), "?")


@dataclass
class ExitReport:
    code: int = ExitCode.IterationCap
    iterations: int = 0
    final_grad_inf_norm: float = 0.0
    wall_time_ms: float = 0.0
    value_evals: int = 0
    grad_evals: int = 0

    @staticmethod
    def _from(c: _capi.lsb_exit_report) -> "ExitReport":
        return ExitReport(c.code, c.iterations, c.final_grad_inf_norm, c.wall_time_ms, c.value_evals, c.grad_evals)


@dataclass
class SimState:
    positions: np.ndarray   # V x 3
    velocities: np.ndarray  # V x 3
    z: np.ndarray           # r
    t: float = 0.0


@dataclass
class FrameInput:
    pin_positions: np.ndarray   # V x 3
    external_force: np.ndarray  # n


def rest_state(mesh: Mesh, subspace_dim: int) -> SimState:
    """reference rest_state (scenario.cpp:251-258)."""
    return SimState(mesh.vertices.copy(), np.zeros_like(mesh.vertices), np.zeros(subspace_dim), 0.0)


class ReducedSystem:
    """One device context: mesh + material + lumped mass + decoder resident in HBM
    (the reference's PotentialContext + MassMatrix + SubspaceModel)."""

    def __init__(self, mesh: Mesh, mu, lam, density: float, model: SubspaceModel, precision: str = "fp64",
                 device: int = 0):
        model.validate()
        if model.n != mesh.num_dofs():
            raise ValueError("model: decoder output width != n")
        E = mesh.num_elements()
        mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, np.float64), (E,)))
        lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lam, np.float64), (E,)))
        self.mesh, self.model, self.precision = mesh, model, precision
        self._keep = []
        pins = mesh.pinned if mesh.pinned.size else np.zeros(1, np.int32)
        md = _capi.lsb_mesh_desc(mesh.num_vertices(), dptr(mesh.vertices), E, iptr(mesh.elements),
                                 int(mesh.pinned.size), iptr(pins), dptr(mu), dptr(lam), float(density))
        L = len(model.decoder)
        rows = (C.c_int * L)(*[l.W.shape[0] for l in model.decoder])
        cols = (C.c_int * L)(*[l.W.shape[1] for l in model.decoder])
        acts = (C.c_int * L)(*[int(l.act) for l in model.decoder])
        Ws = [np.ascontiguousarray(l.W, np.float64) for l in model.decoder]
        bs = [np.ascontiguousarray(l.b, np.float64) for l in model.decoder]
        self._keep += [Ws, bs, mu, lam, pins]
        wp = (C.POINTER(C.c_double) * L)(*[dptr(w) for w in Ws])
        bp = (C.POINTER(C.c_double) * L)(*[dptr(b) for b in bs])
        shift = np.ascontiguousarray(model.norm_shift, np.float64)
        scale = np.ascontiguousarray(model.norm_scale, np.float64)
        self._keep += [shift, scale]
        dd = _capi.lsb_decoder_desc(model.r, L, rows, cols, acts, wp, bp, dptr(shift), dptr(scale))
        prec = {"fp64": _capi.LSB_FP64, "fp32": _capi.LSB_FP32}.get(precision)
        if prec is None:
            raise ValueError("precision must be 'fp64' or 'fp32'")
        h = C.c_void_p()
        check(lib().lsb_create(C.byref(md), C.byref(dd), prec, device, C.byref(h)))
        self._h = h
        self.r, self.n = model.r, model.n
        self.mass = np.zeros(self.n)
        tot = C.c_double()
        check(lib().lsb_get_mass(self._h, dptr(self.mass), C.byref(tot)))
        self.total_mass = tot.value
        self._inertia_key = None

    def close(self):
        if getattr(self, "_h", None):
            lib().lsb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # --- objective configuration
    def set_pin_positions(self, pin_positions: np.ndarray):
        check(lib().lsb_set_pin_positions(self._h, dptr(np.ascontiguousarray(pin_positions, np.float64))))

    def set_inertia(self, qbar: Optional[np.ndarray], dt: float):
        q = None if qbar is None else np.ascontiguousarray(qbar, np.float64)
        check(lib().lsb_set_inertia(self._h, dptr(q), float(dt)))

    # --- evaluation
    def eval(self, z: np.ndarray, want_grad: bool = True):
        z = np.ascontiguousarray(z, np.float64)
        if z.shape[0] != self.r:
            raise ValueError("decode: z has wrong length")
        v = C.c_double()
        g = np.zeros(self.r) if want_grad else None
        check(lib().lsb_eval(self._h, dptr(z), C.byref(v), dptr(g)))
        return (v.value, g) if want_grad else v.value

    def decode(self, z: np.ndarray) -> np.ndarray:
        z = np.ascontiguousarray(z, np.float64)
        if z.shape[0] != self.r:
            raise ValueError("decode: z has wrong length")
        q = np.zeros(self.n)
        check(lib().lsb_decode(self._h, dptr(z), dptr(q)))
        return q

    # --- the reference's secondary primitives (device; energy.hpp:71-112, net.hpp:52-59)
    def decode_jacobian(self, z: np.ndarray) -> np.ndarray:
        """decode_jacobian (net.cpp:159-190): n x r."""
        z = np.ascontiguousarray(z, np.float64)
        if z.shape[0] != self.r:
            raise ValueError("decode: z has wrong length")
        J = np.zeros((self.n, self.r))
        check(lib().lsb_decode_jacobian(self._h, dptr(z), dptr(J)))
        return J

    def decode_second_directional(self, z: np.ndarray, u: np.ndarray, v: np.ndarray) -> np.ndarray:
        """decode_second_directional (net.cpp:192-240)."""
        z, u, v = (np.ascontiguousarray(a, np.float64) for a in (z, u, v))
        if not (z.shape[0] == u.shape[0] == v.shape[0] == self.r):
            raise ValueError("decode: z has wrong length")
        out = np.zeros(self.n)
        check(lib().lsb_decode_second_directional(self._h, dptr(z), dptr(u), dptr(v), dptr(out)))
        return out

    def assemble(self, q: np.ndarray, want_grad: bool = True):
        """assemble (energy.cpp:404-437), elastic branch: (value, free-DOF gradient)."""
        q = np.ascontiguousarray(q, np.float64)
        if q.shape[0] != self.n:
            raise ValueError("assemble: q has wrong length")
        v = C.c_double()
        g = np.zeros(self.n) if want_grad else None
        check(lib().lsb_assemble(self._h, dptr(q), C.byref(v), dptr(g)))
        return (v.value, g) if want_grad else v.value

    def element_snh(self, ids, positions: np.ndarray, want_hessian: bool = True):
        """element_snh (energy.cpp:280-298) for element ids at full-space positions (V x 3):
        (energy[k], grad[k, 12], hess[k, 12, 12] or None), each element with its own mu, lambda."""
        ids = np.ascontiguousarray(np.atleast_1d(ids), np.int32)
        pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
        if pos.shape[0] != self.mesh.num_vertices():
            raise ValueError("element_snh: positions must be V x 3")
        k = ids.size
        e, g = np.zeros(k), np.zeros((k, 12))
        H = np.zeros((k, 12, 12)) if want_hessian else None
        check(lib().lsb_element_snh(self._h, k, ids.ctypes.data_as(C.POINTER(C.c_int)), dptr(pos), dptr(e), dptr(g),
                                    dptr(H)))
        return e, g, H

    def elastic_hessian_apply(self, q: np.ndarray, Y: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """elastic_hessian_apply (energy.cpp:481-493): out += H(q) Y, Y n x k."""
        q = np.ascontiguousarray(q, np.float64)
        Y = np.ascontiguousarray(Y, np.float64).reshape(self.n, -1)
        res = np.zeros_like(Y) if out is None else np.ascontiguousarray(out, np.float64).copy()
        check(lib().lsb_elastic_hessian_apply(self._h, dptr(q), Y.shape[1], dptr(Y), dptr(res)))
        return res

    def lbfgs(self, z: np.ndarray, cfg: SolverConfig) -> Tuple[np.ndarray, ExitReport]:
        cfg.validate()
        z = np.array(z, dtype=np.float64, copy=True)
        rep = _capi.lsb_exit_report()
        c = cfg._c()
        check(lib().lsb_lbfgs(self._h, dptr(z), C.byref(c), C.byref(rep)))
        return z, ExitReport._from(rep)

    def projective_newton(self, z: np.ndarray, cfg: SolverConfig) -> Tuple[np.ndarray, ExitReport]:
        """Device objective + device objective Hessians, host d x d projection / LDL^T."""
        cfg.validate()
        z = np.array(z, dtype=np.float64, copy=True)
        rep = _capi.lsb_exit_report()
        c = cfg._c()
        check(lib().lsb_projective_newton(self._h, dptr(z), C.byref(c), C.byref(rep)))
        return z, ExitReport._from(rep)

    # --- dynamics
    def set_state(self, state: SimState):
        check(lib().lsb_set_state(self._h, dptr(np.ascontiguousarray(state.positions, np.float64)),
                                  dptr(np.ascontiguousarray(state.velocities, np.float64)),
                                  dptr(np.ascontiguousarray(state.z, np.float64))))

    def get_state(self) -> SimState:
        V = self.mesh.num_vertices()
        x = np.zeros((V, 3))
        v = np.zeros((V, 3))
        z = np.zeros(self.r)
        t = C.c_double()
        check(lib().lsb_get_state(self._h, dptr(x), dptr(v), dptr(z), C.byref(t)))
        return SimState(x, v, z, t.value)

    def set_external_force(self, force: np.ndarray):
        check(lib().lsb_set_external_force(self._h, dptr(np.ascontiguousarray(force, np.float64))))

    def step(self, cfg: SolverConfig, quasi_static: bool = False) -> ExitReport:
        cfg.validate()
        rep = _capi.lsb_exit_report()
        c = cfg._c()
        check(lib().lsb_step(self._h, C.byref(c), int(quasi_static), C.byref(rep)))
        return ExitReport._from(rep)

    def simulate(self, steps: int, cfg: SolverConfig, quasi_static: bool = False, want_z: bool = True):
        cfg.validate()
        reps = (_capi.lsb_exit_report * max(steps, 1))()
        zt = np.zeros((max(steps, 1), self.r)) if want_z else None
        c = cfg._c()
        check(lib().lsb_simulate(self._h, steps, C.byref(c), int(quasi_static), reps, dptr(zt)))
        out = [ExitReport._from(reps[i]) for i in range(steps)]
        return out, (zt[:steps] if want_z else None)

    # --- batched / second order
    def eval_batched(self, Z: np.ndarray, want_grad: bool = True):
        Z = np.ascontiguousarray(Z, np.float64).reshape(-1, self.r)
        B = Z.shape[0]
        E = np.zeros(B)
        G = np.zeros((B, self.r)) if want_grad else None
        check(lib().lsb_eval_batched(self._h, B, dptr(Z), dptr(E), dptr(G)))
        return (E, G) if want_grad else E

    def hessian_batched(self, Z: np.ndarray) -> np.ndarray:
        Z = np.ascontiguousarray(Z, np.float64).reshape(-1, self.r)
        H = np.zeros((Z.shape[0], self.r, self.r))
        check(lib().lsb_hessian_batched(self._h, Z.shape[0], dptr(Z), dptr(H)))
        return H

    def set_cubature(self, ids: Optional[np.ndarray] = None, weights: Optional[np.ndarray] = None):
        """Runtime cubature (ElementSubset: elastic term = sum_k w_k E_{ids_k}); None restores
        the full element set."""
        if ids is None:
            check(lib().lsb_set_cubature(self._h, 0, None, None))
            return
        ids = np.ascontiguousarray(ids, np.int32)
        w = np.ascontiguousarray(weights, np.float64)
        if ids.shape != w.shape:
            raise ValueError("cubature: ids and weights differ in length")
        check(lib().lsb_set_cubature(self._h, int(ids.size), ids.ctypes.data_as(C.POINTER(C.c_int)), dptr(w)))

    def objective_hessian_batched(self, Z: np.ndarray) -> np.ndarray:
        """ReducedObjective::hessian at each row of Z (inertia included when set)."""
        Z = np.ascontiguousarray(Z, np.float64).reshape(-1, self.r)
        H = np.zeros((Z.shape[0], self.r, self.r))
        check(lib().lsb_objective_hessian(self._h, Z.shape[0], dptr(Z), dptr(H)))
        return H

    def lipschitz_loss(self, Z1: np.ndarray, Z2: np.ndarray) -> float:
        Z1 = np.ascontiguousarray(Z1, np.float64).reshape(-1, self.r)
        Z2 = np.ascontiguousarray(Z2, np.float64).reshape(-1, self.r)
        if Z1.shape != Z2.shape:
            raise ValueError("lipschitz loss: pair arrays differ in shape")
        out = C.c_double()
        check(lib().lsb_lipschitz_loss(self._h, Z1.shape[0], dptr(Z1), dptr(Z2), C.byref(out)))
        return out.value

    def lipschitz_loss_grad(self, Z1: np.ndarray, Z2: np.ndarray):
        """(loss, [(dL/dW, dL/db) per decoder layer]): the order-2 Lipschitz loss and its
        parameter gradient, i.e. build_lipschitz_loss + Tape::backward + param_gradient
        (losses.cpp:196-213, tape.cpp:46-79)."""
        Z1 = np.ascontiguousarray(Z1, np.float64).reshape(-1, self.r)
        Z2 = np.ascontiguousarray(Z2, np.float64).reshape(-1, self.r)
        if Z1.shape != Z2.shape:
            raise ValueError("lipschitz loss: pair arrays differ in shape")
        shapes = [l.W.shape for l in self.model.decoder]
        flat = np.zeros(sum(r * (c + 1) for r, c in shapes))
        out = C.c_double()
        check(lib().lsb_lipschitz_loss_grad(self._h, Z1.shape[0], dptr(Z1), dptr(Z2), C.byref(out), dptr(flat)))
        grads, o = [], 0
        for r, c in shapes:
            gW = flat[o:o + r * c].reshape(r, c)
            o += r * c
            grads.append((gW, flat[o:o + r].copy()))
            o += r
        return out.value, grads

    # --- execution path
    def solve_kernel_info(self):
        g, u = C.c_int(), C.c_int()
        check(lib().lsb_get_solve_info(self._h, C.byref(g), C.byref(u)))
        return {"grid": g.value, "in_use": bool(u.value), "reason": lib().lsb_last_error().decode()}

    def use_solve_kernel(self, enable: bool):
        check(lib().lsb_set_solve_kernel(self._h, int(enable)))

    def dev_flags(self) -> str:
        """Developer switches (LSB_* environment, read once at creation) active on this context."""
        buf = C.create_string_buffer(1024)
        check(lib().lsb_get_dev_flags(self._h, buf, 1024))
        return buf.value.decode()

    # --- measurement hooks
    def launch_count(self) -> int:
        v = C.c_longlong()
        check(lib().lsb_get_launch_count(self._h, C.byref(v)))
        return v.value

    def profile_eval(self, z: np.ndarray, reps: int = 20):
        z = np.ascontiguousarray(z, np.float64)
        a, b, c, d = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        check(lib().lsb_profile_eval(self._h, dptr(z), reps, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return {"out_fwd": a.value, "elem": b.value, "vjp": c.value, "total": d.value}


class ReducedObjective:
    """reference ReducedObjective (reduced_solver.hpp:59-72):
    E(z) = |f(z) - qbar|_M^2 / (2 dt^2) + P(f(z)); without qbar the inertia term is dropped."""

    def __init__(self, system: ReducedSystem, qbar: Optional[np.ndarray] = None, dt: float = 0.05):
        self.system, self.qbar, self.dt = system, qbar, dt

    def _bind(self):
        key = (id(self), self.dt)
        if self.system._inertia_key != key:
            self.system.set_inertia(self.qbar, self.dt)
            self.system._inertia_key = key

    def eval(self, z: np.ndarray, grad: Optional[np.ndarray] = None) -> float:
        """Value; the gradient is written into `grad` when it is not None (the
        reference's nullable out-pointer)."""
        self._bind()
        if grad is None:
            return self.system.eval(z, want_grad=False)
        v, g = self.system.eval(z, want_grad=True)
        grad[:] = g
        return v

    def hessian(self, z: np.ndarray) -> np.ndarray:
        """reference ReducedObjective::hessian (reduced_solver.cpp:204-229)."""
        self._bind()
        return self.system.objective_hessian_batched(np.asarray(z, np.float64).reshape(1, -1))[0]

    def as_objective(self) -> Callable:
        return lambda z, g=None: self.eval(z, g)


def lbfgs_minimize(objective, x: np.ndarray, cfg: SolverConfig) -> ExitReport:
    """reference lbfgs_minimize (reduced_solver.cpp:58-131); x is updated in place.

    For a ReducedObjective the whole loop (two-loop recursion, Armijo search,
    convergence test) runs on the device inside one CUDA graph; for any other
    callable objective(x, grad_or_None) -> value the same algorithm runs on the
    host (it is O(r) work per iteration)."""
    cfg.validate()
    if isinstance(objective, ReducedObjective):
        objective._bind()
        z, rep = objective.system.lbfgs(x, cfg)
        x[:] = z
        return rep
    return _host_lbfgs(objective, x, cfg)


def _host_lbfgs(objective, x, cfg):
    import time
    t0 = time.perf_counter()
    rep = ExitReport()
    n = x.shape[0]
    g = np.zeros(n)
    f = objective(x, g)
    rep.grad_evals += 1
    rep.value_evals += 1
    hist: List[Tuple[np.ndarray, np.ndarray]] = []

    def finish(r):
        r.wall_time_ms = (time.perf_counter() - t0) * 1e3
        return r

    for it in range(cfg.max_iters):
        rep.iterations = it
        rep.final_grad_inf_norm = float(np.max(np.abs(g))) if n else 0.0
        if rep.final_grad_inf_norm < cfg.epsilon:
            rep.code = ExitCode.Converged
            return finish(rep)
        d = -g.copy()
        alpha = [0.0] * len(hist)
        for i in range(len(hist) - 1, -1, -1):
            s, y = hist[i]
            alpha[i] = s.dot(d) / y.dot(s)
            d -= alpha[i] * y
        if hist:
            s, y = hist[-1]
            d *= s.dot(y) / y.dot(y)
        for i, (s, y) in enumerate(hist):
            beta = y.dot(d) / y.dot(s)
            d += (alpha[i] - beta) * s
        gtd = g.dot(d)
        if not (gtd < 0.0):
            rep.code = ExitCode.Saddle
            return finish(rep)
        a = 1.0
        ok = False
        for _ in range(cfg.max_linesearch):
            trial = x + a * d
            ft = objective(trial, None)
            rep.value_evals += 1
            if math.isfinite(ft) and ft <= f + 1e-4 * a * gtd:
                ok = True
                break
            a *= 0.5
        if not ok:
            rep.code = ExitCode.LinesearchCap
            return finish(rep)
        g_new = np.zeros(n)
        f_new = objective(trial, g_new)
        rep.grad_evals += 1
        s = trial - x
        y = g_new - g
        if s.dot(y) > 1e-12 * np.linalg.norm(s) * np.linalg.norm(y):
            hist.append((s, y))
            if len(hist) > cfg.lbfgs_history:
                hist.pop(0)
        x[:] = trial
        f, g = f_new, g_new
    rep.iterations = cfg.max_iters
    rep.final_grad_inf_norm = float(np.max(np.abs(g)))
    rep.code = ExitCode.Converged if rep.final_grad_inf_norm < cfg.epsilon else ExitCode.IterationCap
    return finish(rep)


def project_spd(H: np.ndarray) -> np.ndarray:
    """reference project_spd (energy.cpp:370-380): unchanged when PSD, else negative
    eigenvalues clamp to 1e-10 * max(lambda_max, 0)."""
    H = np.asarray(H, np.float64)
    w, V = np.linalg.eigh(H)
    if w.min() >= 0.0:
        return H
    w = np.where(w < 0.0, 1e-10 * max(w.max(), 0.0), w)
    return (V * w) @ V.T


def projective_newton_minimize(objective, hessian, x: np.ndarray, cfg: SolverConfig) -> ExitReport:
    """reference projective_newton_minimize (reduced_solver.cpp:133-182); x is updated in place.

    For a ReducedObjective (hessian None or its own .hessian) the evaluations and the
    objective Hessians run on the device (lsb_projective_newton); for other callables
    objective(x, grad_or_None) / hessian(x) the same algorithm runs on the host."""
    cfg.validate()
    if isinstance(objective, ReducedObjective) and (hessian is None or getattr(hessian, "__self__", None) is objective):
        objective._bind()
        z, rep = objective.system.projective_newton(x, cfg)
        x[:] = z
        return rep
    import time
    t0 = time.perf_counter()
    rep = ExitReport()
    n = x.shape[0]
    g = np.zeros(n)
    f = objective(x, g)
    rep.grad_evals += 1

    def finish(r):
        r.wall_time_ms = (time.perf_counter() - t0) * 1e3
        return r

    for it in range(cfg.max_iters):
        rep.iterations = it
        rep.final_grad_inf_norm = float(np.max(np.abs(g))) if n else 0.0
        if rep.final_grad_inf_norm < cfg.epsilon:
            rep.code = ExitCode.Converged
            return finish(rep)
        H = project_spd(hessian(x))
        d = np.linalg.solve(H, -g)
        if not np.all(np.isfinite(d)):
            raise RuntimeError("projective newton: singular system")
        gtd = g.dot(d)
        if not (gtd < 0.0):
            rep.code = ExitCode.Saddle
            return finish(rep)
        a, ok = 1.0, False
        for _ in range(cfg.max_linesearch):
            trial = x + a * d
            ft = objective(trial, None)
            rep.value_evals += 1
            if math.isfinite(ft) and ft <= f + 1e-4 * a * gtd:
                ok = True
                break
            a *= 0.5
        if not ok:
            rep.code = ExitCode.LinesearchCap
            return finish(rep)
        x[:] = trial
        f = objective(x, g)
        rep.grad_evals += 1
    rep.iterations = cfg.max_iters
    rep.final_grad_inf_norm = float(np.max(np.abs(g)))
    rep.code = ExitCode.Converged if rep.final_grad_inf_norm < cfg.epsilon else ExitCode.IterationCap
    return finish(rep)


def reduced_step(state: SimState, frame: FrameInput, system: ReducedSystem, cfg: SolverConfig,
                 quasi_static: bool = False) -> ExitReport:
    """reference reduced_step (reduced_solver.cpp:235-277), L-BFGS method.
    The step runs as one CUDA graph (qbar, warm-started device L-BFGS, decode,
    velocity update); `state` is updated in place."""
    system.set_pin_positions(frame.pin_positions)
    system.set_external_force(frame.external_force)
    system.set_state(state)
    rep = system.step(cfg, quasi_static)
    new = system.get_state()
    state.positions[:] = new.positions
    state.velocities[:] = new.velocities
    state.z[:] = new.z
    state.t += cfg.dt
    system._inertia_key = None
    return rep


def gravity_force(mesh: Mesh, mass: np.ndarray, g: Sequence[float]) -> np.ndarray:
    """reference frame_at external force (scenario.cpp:193-199): f = m_i g_c on free DOFs."""
    return mass * np.tile(np.asarray(g, np.float64), mesh.num_free_vertices())


def lipschitz_loss(system: ReducedSystem, pairs: Sequence[Tuple[np.ndarray, np.ndarray]], order: int = 2) -> float:
    """reference lipschitz_loss(model, pairs, order, pot) (losses.cpp:237-244) for
    order 2 on the full elastic potential."""
    if order != 2:
        raise ValueError("lipschitz loss: the device path implements order 2")
    if len(pairs) == 0:
        raise ValueError("lipschitz loss: no pairs")
    Z1 = np.stack([p[0] for p in pairs])
    Z2 = np.stack([p[1] for p in pairs])
    return system.lipschitz_loss(Z1, Z2)


def lipschitz_loss_grad(system: ReducedSystem, pairs: Sequence[Tuple[np.ndarray, np.ndarray]], order: int = 2):
    """build_lipschitz_loss(..., order, pot) + Tape::backward + param_gradient
    (losses.cpp:196-213, tape.cpp:46-79) for order 2: (loss, [(dW, db) per decoder layer])."""
    if order != 2:
        raise ValueError("lipschitz loss: the device path implements order 2")
    if len(pairs) == 0:
        raise ValueError("lipschitz loss: no pairs")
    Z1 = np.stack([p[0] for p in pairs])
    Z2 = np.stack([p[1] for p in pairs])
    return system.lipschitz_loss_grad(Z1, Z2)
