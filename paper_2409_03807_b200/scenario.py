"""Scenario compatibility: the reference's scenario JSON, its meshes,
pin motion and random interaction replays, so a reference scenario (plus a LIPSUBCKPT1
checkpoint, `checkpoint.py`) drives the device solver.

Restates, host side:
* rng.hpp:10-52                 -- std::mt19937_64 streams: randu, randn, randint, substream
* scenario.cpp:48-121           -- scenario_from_json / load_scenario (tet meshes)
* mesh.cpp:175-232              -- load_node_ele (TetGen .node / .ele, 3-D)
* mesh.cpp:357-395              -- make_bar_3d (five tets per cube, alternating parity)
* scenario.cpp:135-205          -- pin_positions_at, sample_interaction, replay_interactions, frame_at

Out of scope (2-D, cloth, bending and contact terms): the bar2d / cloth generators,
OBJ triangle meshes and colliders are rejected with ValueError.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import lipsub as L

_M64 = (1 << 64) - 1


class Rng:
    """std::mt19937_64 (rng.hpp:12), bit-exact."""

    _N, _M = 312, 156

    def __init__(self, seed: int):
        mt = [0] * self._N
        mt[0] = seed & _M64
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self._mt = mt
        self._i = self._N

    def _twist(self):
        mt, N, M = self._mt, self._N, self._M
        upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for i in range(N):
            x = (mt[i] & upper) | (mt[(i + 1) % N] & lower)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + M) % N] ^ xa
        self._i = 0

    def __call__(self) -> int:
        if self._i >= self._N:
            self._twist()
        y = self._mt[self._i]
        self._i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


def randu(rng: Rng, lo: Optional[float] = None, hi: Optional[float] = None) -> float:
    """rng.hpp:15-21."""
    u = float(rng() >> 11) * 2.0 ** -53
    return u if lo is None else lo + (hi - lo) * u


def randn(rng: Rng) -> float:
    """rng.hpp:24-31 (Box-Muller, one value per call)."""
    u1 = 0.0
    while u1 <= 0.0:
        u1 = randu(rng)
    u2 = randu(rng)
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586476925286766559 * u2)


def randint(rng: Rng, n: int) -> int:
    """rng.hpp:33-39 (rejection sampling)."""
    limit = _M64 - _M64 % n
    x = rng()
    while x >= limit:
        x = rng()
    return x % n


def substream(seed: int, tag: int) -> Rng:
    """rng.hpp:43-51 (splitmix64 finalizer)."""
    x = (seed + 0x9E3779B97F4A7C15 * (tag + 1)) & _M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _M64
    x ^= x >> 31
    return Rng(x)


# --------------------------------------------------------------------------- meshes
def make_bar_3d(nx: int, ny: int, nz: int, width: float = 1.0, height: float = 0.25, depth: float = 0.25,
                pin_left: bool = True) -> L.Mesh:
    """The reference's five-tet bar (mesh.cpp:357-395): vertex id (i*vy + j)*vz + k, coordinates
    (w i/nx, h j/ny, d k/nz), alternating-parity split, orientation fixed by swapping corners 2
    and 3 where the signed volume is negative, the i == 0 face pinned."""
    vx, vy, vz = nx + 1, ny + 1, nz + 1
    ii, jj, kk = np.meshgrid(np.arange(vx), np.arange(vy), np.arange(vz), indexing="ij")
    verts = np.stack([width * ii / nx, height * jj / ny, depth * kk / nz], axis=-1).reshape(-1, 3)

    def vid(i, j, k):
        return (i * vy + j) * vz + k

    elems = []
    for i in range(nx):
        for j in range(ny):
            for k in range(nz):
                c = [vid(i, j, k), vid(i + 1, j, k), vid(i, j + 1, k), vid(i + 1, j + 1, k),
                     vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i, j + 1, k + 1), vid(i + 1, j + 1, k + 1)]
                if (i + j + k) % 2 == 1:
                    c[0], c[1] = c[1], c[0]
                    c[2], c[3] = c[3], c[2]
                    c[4], c[5] = c[5], c[4]
                    c[6], c[7] = c[7], c[6]
                elems += [[c[0], c[1], c[2], c[4]], [c[1], c[3], c[2], c[7]], [c[1], c[5], c[4], c[7]],
                          [c[2], c[4], c[6], c[7]], [c[1], c[2], c[4], c[7]]]
    T = np.array(elems, np.int32).reshape(-1, 4)
    d = verts[T[:, 1:]] - verts[T[:, :1]]
    neg = np.linalg.det(np.transpose(d, (0, 2, 1))) < 0
    T[neg, 2], T[neg, 3] = T[neg, 3].copy(), T[neg, 2].copy()
    pins = [vid(0, j, k) for j in range(vy) for k in range(vz)] if pin_left else []
    return L.build_mesh(verts, T, pins)


def _content_lines(path: str):
    try:
        with open(path) as f:
            lines = f.read().splitlines()
    except OSError:
        raise RuntimeError(f"mesh: cannot open '{path}'")
    # blank lines and '#' comments are skipped (mesh.cpp:162-168)
    return [(i, ln) for i, ln in enumerate(lines) if ln.strip() and not ln.lstrip().startswith("#")]


def load_node_ele(node_path: str, pinned=()) -> L.Mesh:
    """TetGen .node / .ele reader (mesh.cpp:175-232): index base taken from the first vertex
    id; vertices may come in any order; 3-D tets only here."""
    if ".node" not in node_path:
        raise RuntimeError(f"mesh: node/ele format expects a .node path, got '{node_path}'")
    dot = node_path.rfind(".node")
    ele_path = node_path[:dot] + ".ele" + node_path[dot + 5:]

    def fail(path, line_no, what):
        raise RuntimeError(f"mesh: parse error in '{path}' line {line_no + 1}: {what}")

    nl = _content_lines(node_path)
    if not nl:
        fail(node_path, 0, "missing header")
    hdr = nl[0][1].split()
    try:
        nv, dim = int(hdr[0]), int(hdr[1])
    except (IndexError, ValueError):
        fail(node_path, nl[0][0], "expected '<V> <dim>' header")
    if dim not in (2, 3):
        fail(node_path, nl[0][0], "dim must be 2 or 3")
    if dim == 2:
        raise ValueError("scenario: 2-D meshes are out of scope for the device solver")
    verts = np.zeros((nv, 3))
    seen = np.zeros(nv, bool)
    base = None
    if len(nl) - 1 < nv:
        fail(node_path, nl[-1][0], "unexpected end of vertex list")
    for (ln, s) in nl[1:1 + nv]:
        tok = s.split()
        try:
            vid = int(tok[0])
        except (IndexError, ValueError):
            fail(node_path, ln, "expected vertex id")
        if base is None:
            base = vid
        vid -= base
        if vid < 0 or vid >= nv:
            fail(node_path, ln, "vertex id out of range")
        if len(tok) < 4:
            fail(node_path, ln, "expected coordinate")
        try:
            verts[vid] = [float(x) for x in tok[1:4]]
        except ValueError:
            fail(node_path, ln, "expected coordinate")
        seen[vid] = True
    missing = np.nonzero(~seen)[0]
    if missing.size:
        raise RuntimeError(f"mesh: vertex {int(missing[0])} missing in '{node_path}'")
    el = _content_lines(ele_path)
    if not el:
        fail(ele_path, 0, "missing header")
    eh = el[0][1].split()
    try:
        ne, nper = int(eh[0]), int(eh[1])
    except (IndexError, ValueError):
        fail(ele_path, el[0][0], "expected '<E> <nodes-per-element>' header")
    if nper != dim + 1:
        fail(ele_path, el[0][0], f"expected {dim + 1} nodes per element")
    if len(el) - 1 < ne:
        fail(ele_path, el[-1][0], "unexpected end of element list")
    T = np.zeros((ne, 4), np.int64)
    for k, (ln, s) in enumerate(el[1:1 + ne]):
        tok = s.split()
        if len(tok) < 1 + nper:
            fail(ele_path, ln, "expected vertex index")
        T[k] = [int(x) - base for x in tok[1:1 + nper]]
    if T.size and (T.min() < 0 or T.max() >= nv):
        raise RuntimeError("mesh: element vertex id out of range")
    return L.build_mesh(verts, T.astype(np.int32), pinned)


# --------------------------------------------------------------------------- scenario
@dataclass
class Material:
    mu: float = 1e4
    lam: float = 1e4
    density: float = 1e3
    bend_stiffness: float = 0.0
    contact_stiffness: float = 1e5
    contact_margin: float = 1e-3

    def validate(self):
        """MaterialParams::validate (mesh.cpp:13-19)."""
        if not self.mu > 0.0:
            raise ValueError("material: mu must be > 0")
        if not self.lam >= 0.0:
            raise ValueError("material: lambda must be >= 0")
        if not self.density > 0.0:
            raise ValueError("material: density must be > 0")
        if self.bend_stiffness < 0.0 or self.contact_stiffness < 0.0:
            raise ValueError("material: stiffnesses must be >= 0")


@dataclass
class InteractionParams:
    force_min: float = 0.0
    force_max: float = 0.0
    patch_radius: float = 0.0
    steps_min: int = 1
    steps_max: int = 1


@dataclass
class PinMotion:
    kind: str = "none"  # "none" | "oscillate"
    axis: np.ndarray = field(default_factory=lambda: np.zeros(3))
    amplitude: float = 0.0
    period: float = 1.0


@dataclass
class Interaction:
    patch: List[int]
    force_per_vertex: np.ndarray
    start: int = 0
    duration: int = 0


@dataclass
class Scenario:
    name: str
    mesh: L.Mesh
    material: Material
    gravity: np.ndarray
    dt: float = 0.05
    quasi_static: bool = False
    interact: InteractionParams = field(default_factory=InteractionParams)
    pin_motion: PinMotion = field(default_factory=PinMotion)
    episodes: int = 10
    steps_per_episode: int = 100
    test_fraction: float = 0.2

    def system(self, model: L.SubspaceModel, precision: str = "fp64", device: int = 0) -> L.ReducedSystem:
        """The device context for this scenario's mesh and material (PotentialContext +
        MassMatrix, scenario.hpp:57-61) with the given decoder."""
        E = self.mesh.num_elements()
        return L.ReducedSystem(self.mesh, np.full(E, self.material.mu), np.full(E, self.material.lam),
                               self.material.density, model, precision, device)


def _vec(j) -> np.ndarray:
    return np.asarray([float(x) for x in j], np.float64)


def _mesh_from_json(j: dict, base_dir: str, pins) -> L.Mesh:
    if "generator" in j:
        g = j["generator"]
        typ = g["type"]
        if typ == "bar3d":
            return make_bar_3d(int(g["nx"]), int(g["ny"]), int(g["nz"]), float(g.get("width", 1.0)),
                               float(g.get("height", 0.25)), float(g.get("depth", 0.25)),
                               bool(g.get("pin_left", True)))
        if typ in ("bar2d", "cloth"):
            raise ValueError(f"scenario: mesh generator '{typ}' (2-D / cloth) is out of scope for the device solver")
        raise ValueError(f"scenario: unknown mesh generator '{typ}'")
    path = os.path.join(base_dir, j["path"])
    fmt = j.get("format", "node_ele")
    if fmt == "node_ele":
        return load_node_ele(path, pins)
    if fmt == "obj":
        raise ValueError("scenario: OBJ triangle meshes (cloth) are out of scope for the device solver")
    raise ValueError(f"scenario: unknown mesh format '{fmt}'")


def scenario_from_json(j: dict, base_dir: str = ".") -> Scenario:
    """scenario_from_json (scenario.cpp:48-121)."""
    name = j.get("name", "scenario")
    pins = []
    if "pins" in j and "vertices" in j["pins"]:
        pins = [int(v) for v in j["pins"]["vertices"]]
    mesh = _mesh_from_json(j["mesh"], base_dir, pins)
    if pins:  # an explicit vertex list overrides the generator's pins (with_pins, mesh.cpp:147-149)
        mesh = L.build_mesh(mesh.vertices, mesh.elements, pins)
    mat = Material()
    if "material" in j:
        m = j["material"]
        mat.mu = float(m.get("mu", mat.mu))
        mat.lam = float(m.get("lambda", mat.lam))
        mat.density = float(m.get("density", mat.density))
        mat.bend_stiffness = float(m.get("bend_stiffness", mat.bend_stiffness))
        mat.contact_stiffness = float(m.get("contact_stiffness", mat.contact_stiffness))
        mat.contact_margin = float(m.get("contact_margin", mat.contact_margin))
    mat.validate()
    gravity = _vec(j["gravity"]) if "gravity" in j else np.zeros(3)
    if gravity.size != 3:
        raise ValueError("scenario: gravity dimension mismatch")
    s = Scenario(name, mesh, mat, gravity)
    s.dt = float(j.get("dt", 0.05))
    s.quasi_static = bool(j.get("quasi_static", False))
    s.episodes = int(j.get("episodes", 10))
    s.steps_per_episode = int(j.get("steps_per_episode", 100))
    s.test_fraction = float(j.get("test_fraction", 0.2))
    if j.get("colliders"):
        raise ValueError("scenario: colliders (contact terms) are out of scope for the device solver")
    if "interactions" in j:
        it = j["interactions"]
        s.interact = InteractionParams(float(it.get("force_min", 0.0)), float(it.get("force_max", 0.0)),
                                       float(it.get("patch_radius", 0.0)), int(it.get("steps_min", 1)),
                                       int(it.get("steps_max", 1)))
    if "pin_motion" in j:
        pm = j["pin_motion"]
        typ = pm.get("type", "none")
        if typ == "oscillate":
            axis = _vec(pm["axis"])
            if axis.size != 3:
                raise ValueError("scenario: pin_motion axis dimension mismatch")
            s.pin_motion = PinMotion("oscillate", axis, float(pm.get("amplitude", 0.0)), float(pm.get("period", 1.0)))
        elif typ != "none":
            raise ValueError(f"scenario: unknown pin_motion '{typ}'")
    return s


def load_scenario(path: str) -> Scenario:
    """load_scenario (scenario.cpp:123-133)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"scenario: cannot open '{path}'")
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise RuntimeError(f"scenario: invalid JSON in '{path}': {e}")
    return scenario_from_json(j, os.path.dirname(path))


def pin_positions_at(s: Scenario, t: float) -> np.ndarray:
    """pin_positions_at (scenario.cpp:135-144): rest positions, pinned rows offset by the
    oscillation amplitude * sin(2 pi t / period) * axis."""
    pins = s.mesh.vertices.copy()
    if s.pin_motion.kind == "oscillate":
        off = s.pin_motion.amplitude * math.sin(2.0 * math.pi * t / s.pin_motion.period) * s.pin_motion.axis
        pins[s.mesh.pinned] += off
    return pins


def sample_interaction(s: Scenario, episode_steps: int, rng: Rng) -> Interaction:
    """sample_interaction (scenario.cpp:146-171), same draw order."""
    X = s.mesh.vertices
    center = randint(rng, s.mesh.num_vertices())
    d = X - X[center]
    patch = [int(v) for v in np.nonzero(np.sqrt((d * d).sum(axis=1)) <= s.interact.patch_radius)[0]]
    if not patch:
        patch = [center]
    while True:
        dvec = np.array([randn(rng) for _ in range(3)])
        norm = float(np.linalg.norm(dvec))
        if norm >= 1e-12:
            break
    mag = randu(rng, s.interact.force_min, s.interact.force_max)
    force = (mag / norm / len(patch)) * dvec
    span = max(s.interact.steps_max - s.interact.steps_min, 0)
    duration = s.interact.steps_min + (randint(rng, span + 1) if span > 0 else 0)
    duration = min(duration, episode_steps)
    latest = max(episode_steps - duration, 0)
    start = randint(rng, latest + 1) if latest > 0 else 0
    return Interaction(patch, force, start, duration)


def replay_interactions(s: Scenario, steps: int, rng: Rng) -> List[Interaction]:
    """replay_interactions (scenario.cpp:173-185): back-to-back interactions covering steps."""
    seq, cursor = [], 0
    while cursor < steps:
        it = sample_interaction(s, s.steps_per_episode, rng)
        it.start = cursor
        it.duration = max(it.duration, 1)
        cursor += it.duration
        seq.append(it)
    return seq


def frame_at(s: Scenario, mass: np.ndarray, interactions: List[Interaction], step: int, t: float) -> L.FrameInput:
    """frame_at (scenario.cpp:187-205): pin positions at t; m_i g on free DOFs plus the active
    interactions' per-vertex forces."""
    mesh = s.mesh
    f = L.gravity_force(mesh, mass, s.gravity)
    for it in interactions:
        if step < it.start or step >= it.start + it.duration:
            continue
        for v in it.patch:
            fi = mesh.free_index[v]
            if fi >= 0:
                f[3 * fi:3 * fi + 3] += it.force_per_vertex
    return L.FrameInput(pin_positions_at(s, t), f)
