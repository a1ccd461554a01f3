"""Scenario compatibility, host side: the reference's RNG streams,
its five-tet bar generator and node/ele reader (restating test_mesh.cpp:63-67, 151-159,
178-188), scenario JSON parsing (scenario.cpp:48-121) and the replay machinery
(scenario.cpp:135-205)."""
import json
import math
import os

import numpy as np
import pytest

from conftest import rel_err


@pytest.fixture(scope="module")
def S():
    from paper_2409_03807_b200 import scenario
    return scenario


def test_rng_streams_match_the_reference_generator(S, oracle):
    """std::mt19937_64 + Box-Muller bit-exact against the oracle's C++ streams."""
    for seed, tag in [(0, 0), (1, 7), (3, 0), (4, 0), (12345, 99)]:
        rng = S.substream(seed, tag)
        got = np.array([S.randn(rng) for _ in range(50)])
        assert np.array_equal(got, oracle.randn_seq(seed, tag, 50))
    rng = S.substream(5, 2)
    got = np.array([S.randu(rng) for _ in range(40)])
    assert np.array_equal(got, oracle._randu_seq(5, 2, 40))
    # randint: rejection sampling over the raw 64-bit stream
    r1, r2 = S.substream(9, 1), S.substream(9, 1)
    vals = [S.randint(r1, 17) for _ in range(100)]
    assert vals == [r2() % 17 for _ in range(100)]  # the rejection limit is never hit for n = 17
    assert min(vals) >= 0 and max(vals) < 17


def test_bar3d_five_tets(S):
    m = S.make_bar_3d(4, 2, 3, 0.4, 0.2, 0.3)
    assert m.num_elements() == 5 * 4 * 2 * 3
    assert m.num_vertices() == 5 * 3 * 4
    X, T = m.vertices, m.elements
    d = X[T[:, 1:]] - X[T[:, :1]]
    vol = np.linalg.det(np.transpose(d, (0, 2, 1))) / 6.0
    assert np.all(vol > 0)
    assert abs(vol.sum() - 0.4 * 0.2 * 0.3) < 1e-12
    # conforming: every triangular face is shared by at most two tets
    faces = {}
    for t in T:
        for f in ([t[0], t[1], t[2]], [t[0], t[1], t[3]], [t[0], t[2], t[3]], [t[1], t[2], t[3]]):
            key = tuple(sorted(f))
            faces[key] = faces.get(key, 0) + 1
    assert max(faces.values()) == 2
    # boundary faces exactly tile the box surface: 2 triangles per boundary quad
    nb = sum(1 for c in faces.values() if c == 1)
    assert nb == 2 * 2 * (4 * 2 + 4 * 3 + 2 * 3)
    # i == 0 face pinned; vertex ids (i*vy + j)*vz + k, coordinates w i/nx, h j/ny, d k/nz
    assert list(m.pinned) == list(range(3 * 4))
    assert np.allclose(X[(2 * 3 + 1) * 4 + 2], [0.2, 0.2 / 2, 0.3 * 2 / 3])
    assert S.make_bar_3d(2, 1, 1, pin_left=False).pinned.size == 0


def test_bar3d_rest_state_is_stress_free(S, oracle):
    """test_mesh.cpp:63-67: F = I at rest on make_bar_3d(2, 1, 1, 0.4, 0.2, 0.2)."""
    m = S.make_bar_3d(2, 1, 1, 0.4, 0.2, 0.2)
    o = oracle.Oracle.from_mesh(m.vertices, m.elements, m.pinned)
    for e in range(m.num_elements()):
        en, g, _ = o.element_snh(e, 2.0, 3.0, m.vertices)
        assert abs(en) < 1e-14 and np.max(np.abs(g)) < 1e-12


def _write_node_ele(mesh, node_path, base=0, comments=False):
    with open(node_path, "w") as f:
        if comments:
            f.write("# written by the test\n\n")
        f.write(f"{mesh.num_vertices()} 3 0 0\n")
        for v in range(mesh.num_vertices()):
            x = mesh.vertices[v]
            f.write(f"{v + base} {float(x[0])!r} {float(x[1])!r} {float(x[2])!r}\n")
    with open(node_path[:-5] + ".ele", "w") as f:
        f.write(f"{mesh.num_elements()} 4 0\n")
        for e in range(mesh.num_elements()):
            t = mesh.elements[e] + base
            f.write(f"{e + base} {t[0]} {t[1]} {t[2]} {t[3]}\n")


@pytest.mark.parametrize("base,comments", [(0, False), (1, True)])
def test_node_ele_round_trip(S, tmp_path, base, comments):
    """test_mesh.cpp:151-159 (exact vertices), plus 1-based ids and comment lines."""
    m = S.make_bar_3d(2, 1, 1, 0.4, 0.2, 0.2, False)
    node = str(tmp_path / "bar.node")
    _write_node_ele(m, node, base, comments)
    got = S.load_node_ele(node, [0, 3])
    assert got.num_vertices() == m.num_vertices() and got.num_elements() == m.num_elements()
    assert np.array_equal(got.vertices, m.vertices)
    assert np.array_equal(got.elements, m.elements)
    assert list(got.pinned) == [0, 3]


def test_node_ele_errors(S, tmp_path):
    """test_mesh.cpp:178-188 (3-D variant): a parse error carries its line number."""
    bad = tmp_path / "bad.node"
    bad.write_text("2 3 0 0\n0 0.0 0.0 0.0\n1 nope 0.0 0.0\n")
    (tmp_path / "bad.ele").write_text("0 4 0\n")
    with pytest.raises(RuntimeError, match="line 3"):
        S.load_node_ele(str(bad))
    miss = tmp_path / "miss.node"
    miss.write_text("3 3\n0 0 0 0\n1 1 0 0\n1 1 1 0\n")
    (tmp_path / "miss.ele").write_text("0 4\n")
    with pytest.raises(RuntimeError, match="vertex 2 missing"):
        S.load_node_ele(str(miss))
    twod = tmp_path / "flat.node"
    twod.write_text("3 2\n0 0 0\n1 1 0\n2 0 1\n")
    with pytest.raises(ValueError, match="out of scope"):
        S.load_node_ele(str(twod))
    with pytest.raises(RuntimeError, match="cannot open"):
        S.load_node_ele(str(tmp_path / "none.node"))


def _bar_json(**over):
    j = {
        "name": "bar3",
        "mesh": {"generator": {"type": "bar3d", "nx": 4, "ny": 2, "nz": 2, "width": 0.8, "height": 0.2,
                               "depth": 0.2, "pin_left": True}},
        "material": {"mu": 2e4, "lambda": 3e4, "density": 900.0},
        "gravity": [0.0, -9.8, 0.0],
        "dt": 0.04,
        "interactions": {"force_min": 5.0, "force_max": 20.0, "patch_radius": 0.12, "steps_min": 3, "steps_max": 7},
        "pin_motion": {"type": "oscillate", "axis": [0.0, 1.0, 0.0], "amplitude": 0.01, "period": 0.5},
        "episodes": 4,
        "steps_per_episode": 30,
    }
    j.update(over)
    return j


def test_scenario_from_json(S, tmp_path):
    p = tmp_path / "scen.json"
    p.write_text(json.dumps(_bar_json()))
    s = S.load_scenario(str(p))
    assert s.name == "bar3" and s.mesh.num_elements() == 5 * 16
    assert (s.material.mu, s.material.lam, s.material.density) == (2e4, 3e4, 900.0)
    assert np.array_equal(s.gravity, [0.0, -9.8, 0.0]) and s.dt == 0.04 and not s.quasi_static
    assert (s.interact.steps_min, s.interact.steps_max) == (3, 7)
    assert s.pin_motion.kind == "oscillate" and s.episodes == 4 and s.steps_per_episode == 30
    # defaults (scenario.cpp: dt 0.05, zero gravity, 10 episodes of 100 steps)
    d = S.scenario_from_json({"mesh": {"generator": {"type": "bar3d", "nx": 1, "ny": 1, "nz": 1}}})
    assert d.dt == 0.05 and np.array_equal(d.gravity, np.zeros(3)) and d.episodes == 10
    assert d.steps_per_episode == 100 and d.material.mu == 1e4
    # an explicit pin list overrides the generator's pins
    o = S.scenario_from_json(_bar_json(pins={"vertices": [5, 1]}))
    assert list(o.mesh.pinned) == [1, 5]
    # a node/ele mesh relative to the scenario file
    m = S.make_bar_3d(2, 1, 1, 0.4, 0.2, 0.2, False)
    _write_node_ele(m, str(tmp_path / "m.node"))
    (tmp_path / "s2.json").write_text(json.dumps({"mesh": {"path": "m.node"}, "pins": {"vertices": [0]}}))
    s2 = S.load_scenario(str(tmp_path / "s2.json"))
    assert s2.mesh.num_elements() == 10 and list(s2.mesh.pinned) == [0]


@pytest.mark.parametrize("over,err,msg", [
    ({"mesh": {"generator": {"type": "wedge", "nx": 1, "ny": 1, "nz": 1}}}, ValueError, "unknown mesh generator"),
    ({"mesh": {"generator": {"type": "bar2d", "nx": 2, "ny": 1}}}, ValueError, "out of scope"),
    ({"mesh": {"path": "x.obj", "format": "obj"}}, ValueError, "out of scope"),
    ({"mesh": {"path": "x.msh", "format": "gmsh"}}, ValueError, "unknown mesh format"),
    ({"material": {"mu": 0.0}}, ValueError, "mu must be > 0"),
    ({"material": {"lambda": -1.0}}, ValueError, "lambda must be >= 0"),
    ({"material": {"density": 0.0}}, ValueError, "density must be > 0"),
    ({"gravity": [0.0, -9.8]}, ValueError, "gravity dimension mismatch"),
    ({"colliders": [{"type": "sphere", "center": [0, 0, 0], "radius": 1.0}]}, ValueError, "out of scope"),
    ({"pin_motion": {"type": "spin"}}, ValueError, "unknown pin_motion"),
    ({"pin_motion": {"type": "oscillate", "axis": [1.0, 0.0]}}, ValueError, "axis dimension mismatch"),
])
def test_scenario_errors(S, over, err, msg):
    with pytest.raises(err, match=msg):
        S.scenario_from_json(_bar_json(**over))


def test_load_scenario_io_errors(S, tmp_path):
    with pytest.raises(RuntimeError, match="cannot open"):
        S.load_scenario(str(tmp_path / "nope.json"))
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(RuntimeError, match="invalid JSON"):
        S.load_scenario(str(tmp_path / "bad.json"))


def test_pin_motion_and_frames(S):
    from paper_2409_03807_b200 import lipsub as L
    s = S.scenario_from_json(_bar_json())
    t = 0.1
    pins = S.pin_positions_at(s, t)
    off = 0.01 * math.sin(2.0 * math.pi * t / 0.5)
    assert np.allclose(pins[s.mesh.pinned, 1] - s.mesh.vertices[s.mesh.pinned, 1], off, atol=1e-15)
    assert np.array_equal(np.delete(pins, s.mesh.pinned, 0), np.delete(s.mesh.vertices, s.mesh.pinned, 0))
    mass = np.linspace(1.0, 2.0, s.mesh.num_dofs())
    it = S.Interaction([20, 0, 25], np.array([1.0, -2.0, 0.5]), start=2, duration=3)
    f2 = S.frame_at(s, mass, [it], 2, t).external_force
    f5 = S.frame_at(s, mass, [it], 5, t).external_force
    g = L.gravity_force(s.mesh, mass, s.gravity)
    assert np.array_equal(f5, g)  # outside [start, start + duration)
    assert s.mesh.free_index[0] < 0
    for v in (20, 25):  # vertex 0 is pinned and receives nothing
        fi = s.mesh.free_index[v]
        assert np.allclose(f2[3 * fi:3 * fi + 3], g[3 * fi:3 * fi + 3] + it.force_per_vertex)
    assert np.count_nonzero(f2 - g) == 6


def test_interaction_sampling(S):
    s = S.scenario_from_json(_bar_json())
    a = S.sample_interaction(s, 30, S.substream(11, 7))
    b = S.sample_interaction(s, 30, S.substream(11, 7))
    assert a.patch == b.patch and np.array_equal(a.force_per_vertex, b.force_per_vertex)
    assert (a.start, a.duration) == (b.start, b.duration)
    X = s.mesh.vertices
    c = a.patch
    assert 3 <= a.duration <= 7 and 0 <= a.start <= 30 - a.duration
    mag = np.linalg.norm(a.force_per_vertex) * len(a.patch)
    assert 5.0 <= mag <= 20.0
    seq = S.replay_interactions(s, 100, S.substream(3, 7))
    assert seq[0].start == 0
    for x, y in zip(seq, seq[1:]):
        assert y.start == x.start + x.duration and x.duration >= 1
    assert seq[-1].start + seq[-1].duration >= 100
    # patch = vertices within patch_radius of a centre vertex
    for it in seq[:5]:
        d = np.linalg.norm(X[it.patch][:, None, :] - X[None, it.patch, :], axis=-1)
        assert d.max() <= 2 * 0.12 + 1e-12
