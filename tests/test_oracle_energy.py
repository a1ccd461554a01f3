"""Oracle self-tests: stable neo-Hookean element + assembly.

Restates the reference's own known-answer / property tests for the hot path
(proj/tests/test_energy.cpp) against the CPU oracle, which pins the oracle
(the reference ships no golden files and cannot be built here)."""
import numpy as np
import pytest

from conftest import rel_err

TET = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


def _single_tet(oracle):
    return oracle.Oracle.from_mesh(TET, np.array([[0, 1, 2, 3]], np.int32), np.zeros(0, np.int32))


def density_oracle(F, mu, lam):
    """test_energy.cpp:43-54 (independent density)."""
    de = F.shape[1]
    c = de / (de + 1.0)
    I = np.sum(F * F)
    J = np.linalg.det(F)
    return (0.5 * mu * (I - de) - 0.5 * mu * (np.log(I + 1.0) - np.log(de + 1.0)) + 0.5 * lam * (J - 1) ** 2
            - c * mu * (J - 1))


def test_rest_is_critical_point(oracle):
    """test_energy.cpp:123-132."""
    o = _single_tet(oracle)
    e, g, H = o.element_snh(0, 2.0, 3.0, TET)
    assert abs(e) < 1e-14
    assert np.max(np.abs(g)) < 1e-12


def test_uniform_scaling_known_answer(oracle):
    """test_energy.cpp:134-147: F = 2I, mu = lambda = 1 -> vol * psi = 3.860112083638196."""
    o = _single_tet(oracle)
    e, _, _ = o.element_snh(0, 1.0, 1.0, 2.0 * TET)
    expected = (1.0 / 6.0) * density_oracle(2.0 * np.eye(3), 1.0, 1.0)
    assert rel_err(e, expected) < 1e-12
    assert abs(e - 3.860112083638196) < 1e-15


def test_inverted_element_finite(oracle):
    """test_energy.cpp:149-161 (tet variant)."""
    o = _single_tet(oracle)
    X = TET.copy()
    X[3, 2] = -1.0
    e, g, H = o.element_snh(0, 1.0, 1.0, X)
    assert np.isfinite(e) and np.all(np.isfinite(g)) and np.all(np.isfinite(H))


@pytest.mark.parametrize("seed", range(8))
def test_element_fd(oracle, seed):
    """test_energy.cpp:58-81/163-169: FD gradient 1e-6, Hessian 1e-4, exact symmetry."""
    o = _single_tet(oracle)
    rng = np.random.default_rng(100 + seed)
    x0 = TET.reshape(-1) + 0.15 * rng.standard_normal(12)
    mu, lam = 1.3, 0.7

    def energy(x):
        return o.element_snh(0, mu, lam, x.reshape(4, 3), False)[0]

    def grad(x):
        return o.element_snh(0, mu, lam, x.reshape(4, 3), False)[1]

    e, g, H = o.element_snh(0, mu, lam, x0.reshape(4, 3), True)
    h = 1e-6
    fd = np.array([(energy(x0 + h * np.eye(12)[i]) - energy(x0 - h * np.eye(12)[i])) / (2 * h) for i in range(12)])
    assert rel_err(g, fd) < 1e-6
    hh = 1e-5
    fdH = np.stack([(grad(x0 + hh * np.eye(12)[i]) - grad(x0 - hh * np.eye(12)[i])) / (2 * hh) for i in range(12)],
                   axis=1)
    assert rel_err(H, fdH) < 1e-4
    assert rel_err(H, H.T, 1e-30) < 1e-10


@pytest.fixture(scope="module")
def bar(oracle):
    o = oracle.Oracle.bar(3, 2, 2, 1.0, 0.4, 0.5, 0.0, 0, True)
    o.set_material(2.0, 1.5, 1.0)
    X = o.mesh_arrays()[0]
    fi = o.mesh_arrays()[4]
    q0 = X[fi >= 0].reshape(-1)
    return o, q0


def test_assembly_subsets(bar):
    """test_energy.cpp:285-312: full subset bit-identical, empty -> 0, singleton sum."""
    o, q0 = bar
    rng = np.random.default_rng(31)
    q = q0 + 0.05 * rng.standard_normal(q0.size)
    v, g = o.assemble(q)
    vf, gf = o.assemble(q, np.arange(o.E), np.ones(o.E))
    assert v == vf and np.array_equal(g, gf)
    ve, ge = o.assemble(q, np.zeros(0, np.int32), np.zeros(0))
    assert ve == 0.0 and np.linalg.norm(ge) == 0.0
    total = sum(o.assemble(q, np.array([e], np.int32), np.ones(1))[0] for e in range(o.E))
    assert rel_err(total, v) < 1e-14


def test_assembly_fd_and_rest(bar):
    """test_energy.cpp:313-333: FD gradient 1e-6; rest force-free < 1e-8."""
    o, q0 = bar
    rng = np.random.default_rng(32)
    q = q0 + 0.05 * rng.standard_normal(q0.size)
    v, g = o.assemble(q)
    h = 1e-6
    fd = np.array([(o.assemble(q + h * np.eye(q.size)[i])[0] - o.assemble(q - h * np.eye(q.size)[i])[0]) / (2 * h)
                   for i in range(q.size)])
    assert rel_err(g, fd) < 1e-6
    assert np.max(np.abs(o.assemble(q0)[1])) < 1e-8


def test_hessian_apply_matches_fd(bar):
    """test_energy.cpp:334-343 (apply vs the Hessian, here vs FD of the gradient)."""
    o, q0 = bar
    rng = np.random.default_rng(33)
    q = q0 + 0.05 * rng.standard_normal(q0.size)
    Y = rng.standard_normal((q.size, 3))
    HY = o.hessian_apply(q, Y)
    h = 1e-5
    fdH = np.stack([(o.assemble(q + h * np.eye(q.size)[i])[1] - o.assemble(q - h * np.eye(q.size)[i])[1]) / (2 * h)
                    for i in range(q.size)], axis=1)
    assert rel_err(HY, fdH @ Y) < 1e-4


def test_lumped_mass_conserves(oracle):
    """test_mesh.cpp:70-107: total lumped mass = density * volume."""
    o = oracle.Oracle.bar(4, 4, 16, 0.25, 0.25, 1.0, 0.0, 0, True)
    o.set_material(1.0, 1.0, 1000.0)
    assert abs(o.total_mass - 1000.0 * 0.25 * 0.25 * 1.0) < 1e-9
    _, _, Dm, vol, _ = o.mesh_arrays()
    assert abs(vol.sum() - 0.0625) < 1e-12
    assert np.all(vol > 0)


def test_runtime_cubature_full_unit_set_is_plain_assembly(oracle):
    """ElementSubset::full with unit weights shares the plain-assembly code path (energy.hpp:22-24):
    bit-identical; all weights 2 doubles the elastic energy exactly."""
    ob = oracle.problem("c1")
    z = 0.3 * np.random.default_rng(3).standard_normal(ob.r)
    E0, g0 = ob.eval(z)
    ids = np.arange(ob.E, dtype=np.int32)
    ob.set_cubature(ids, np.ones(ob.E))
    E1, g1 = ob.eval(z)
    assert E1 == E0 and np.array_equal(g1, g0)
    ob.set_cubature(ids, 2.0 * np.ones(ob.E))
    E2, g2 = ob.eval(z)
    assert E2 == 2.0 * E0 and np.array_equal(g2, 2.0 * g0)
    ob.set_cubature(None)
    assert ob.eval(z)[0] == E0
