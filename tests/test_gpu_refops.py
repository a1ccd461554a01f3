"""GPU parity of the reference's secondary hot-path primitives exported through the C ABI
(SURVEY §8(b) "Other ★ entry points") against the CPU oracle on identical inputs:

* lsb_assemble               <- assemble, elastic branch      (energy.hpp:99-101, energy.cpp:404-437)
* lsb_element_snh            <- element_snh with its Hessian  (energy.hpp:71-72, energy.cpp:280-298)
* lsb_elastic_hessian_apply  <- elastic_hessian_apply         (energy.hpp:109-112, energy.cpp:481-493)
* lsb_decode_jacobian        <- decode_jacobian               (net.hpp:52-53, net.cpp:159-190)
* lsb_decode_second_directional <- decode_second_directional  (net.hpp:57-59, net.cpp:192-240)

Tolerances: 1e-10 relative (norm-wise rel_err, tests/helpers.hpp:16-18) on fp64 contexts,
1e-4 on fp32-storage contexts (element records and W_out in fp32)."""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-10, "fp32": 1e-4}


def _problem(name, precision, oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build(name)
    return pr, pr.system(precision), oracle.problem(name)


@pytest.mark.parametrize("name,precision", [("c1", "fp64"), ("c1", "fp32"), ("c2", "fp64")])
def test_assemble_and_hessian_apply(name, precision, oracle, product):
    pr, sysm, ob = _problem(name, precision, oracle, product)
    rng = np.random.default_rng(3)
    q = sysm.decode(0.5 * rng.standard_normal(pr.model.r)) + 1e-3 * rng.standard_normal(pr.model.n)
    v, g = sysm.assemble(q)
    vo, go = ob.assemble(q)
    assert rel_err(v, vo) < TOL[precision], (v, vo)
    assert rel_err(g, go) < TOL[precision]
    assert sysm.assemble(q, want_grad=False) == v
    v2, g2 = sysm.assemble(q)
    assert v2 == v and np.array_equal(g2, g)  # fixed-order sums: bitwise repeatable
    Y = rng.standard_normal((pr.model.n, 3))
    HY = sysm.elastic_hessian_apply(q, Y)
    HYo = ob.hessian_apply(q, Y)
    assert rel_err(HY, HYo) < TOL[precision]
    acc = sysm.elastic_hessian_apply(q, Y, out=HY)  # out += H Y
    assert rel_err(acc, 2 * HYo) < TOL[precision]


def test_assemble_displaced_pins(oracle, product):
    pr, sysm, ob = _problem("c1", "fp64", oracle, product)
    pins = pr.mesh.vertices.copy()
    pins[pr.mesh.pinned] += np.array([1e-3, -2e-3, 5e-4])
    sysm.set_pin_positions(pins)
    ob.set_pins(pins)
    q = product.dof_pack(pr.mesh, pr.mesh.vertices)
    v, g = sysm.assemble(q)
    vo, go = ob.assemble(q)
    assert vo > 0 and rel_err(v, vo) < 1e-10 and rel_err(g, go) < 1e-10


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_element_snh_with_hessian(precision, oracle, product):
    pr, sysm, ob = _problem("c1", precision, oracle, product)
    rng = np.random.default_rng(9)
    X = pr.mesh.vertices
    pos = X + 0.05 * rng.standard_normal(X.shape) * 0.0625
    ids = np.array([0, 1, 17, 500, pr.mesh.num_elements() - 1])
    e, g, H = sysm.element_snh(ids, pos)
    for k, el in enumerate(ids):
        eo, go, Ho = ob.element_snh(int(el), float(pr.mu[el]), float(pr.lam[el]), pos)
        assert rel_err(e[k], eo) < TOL[precision]
        assert rel_err(g[k], go) < TOL[precision]
        assert rel_err(H[k], Ho) < TOL[precision]
        assert np.allclose(H[k], H[k].T, rtol=0, atol=1e-12 * np.abs(H[k]).max())
    e2, g2, H2 = sysm.element_snh(ids, pos, want_hessian=False)
    assert H2 is None and np.array_equal(e2, e) and np.array_equal(g2, g)
    with pytest.raises(ValueError):
        sysm.element_snh([pr.mesh.num_elements()], pos)


def test_element_snh_closed_form(oracle, product):
    """F = 2I on every element of a scaled mesh: energy = vol psi(2I) with the closed-form
    density of test_energy.cpp:134-147 (mu = lambda = 1: psi = 23.160672501829175)."""
    P = product
    mesh = P.make_bar_mesh(2, 1, 1, 1.0, 0.5, 0.5, pin_left=False)
    model = P.make_bar_decoder(mesh, 2, 1, 8, P.Activation.Elu, seed=0, out_scale=1e-2)
    sysm = P.ReducedSystem(mesh, 1.0, 1.0, 1.0, model, "fp64")
    vols = []
    X, T = mesh.vertices, mesh.elements
    for t in T:
        D = np.stack([X[t[1]] - X[t[0]], X[t[2]] - X[t[0]], X[t[3]] - X[t[0]]], axis=1)
        vols.append(abs(np.linalg.det(D)) / 6)
    e, g, H = sysm.element_snh(np.arange(len(T)), 2.0 * X)
    assert np.allclose(e, 23.160672501829175 * np.asarray(vols), rtol=1e-13, atol=0)


@pytest.mark.parametrize("name,precision", [("c1", "fp64"), ("c2", "fp64"), ("c2", "fp32")])
def test_decode_jacobian_and_second_directional(name, precision, oracle, product):
    pr, sysm, ob = _problem(name, precision, oracle, product)
    rng = np.random.default_rng(21)
    r = pr.model.r
    z, u, v = (0.5 * rng.standard_normal(r) for _ in range(3))
    J = sysm.decode_jacobian(z)
    Jo = ob.decode_jacobian(z)
    assert rel_err(J, Jo) < TOL[precision]
    s2 = sysm.decode_second_directional(z, u, v)
    s2o = ob.decode_second_directional(z, u, v)
    assert rel_err(s2, s2o) < TOL[precision]
    assert np.array_equal(s2, sysm.decode_second_directional(z, v, u)) or \
        rel_err(s2, sysm.decode_second_directional(z, v, u)) < 1e-14


@pytest.mark.parametrize("act", [1, 2, 3])
def test_primitives_general_decoder(act, oracle, product):
    """SiLU / tanh / ELU hidden layers with biases, non-unit scales, two hidden layers."""
    from test_gpu_eval import _tiny_problem
    P = product
    mesh, model, mu, lam, o = _tiny_problem(oracle, product, P.Activation(act))
    sysm = P.ReducedSystem(mesh, mu, lam, 5.0, model, "fp64")
    rng = np.random.default_rng(4)
    z, u, v = (0.4 * rng.standard_normal(model.r) for _ in range(3))
    assert rel_err(sysm.decode_jacobian(z), o.decode_jacobian(z)) < 1e-10
    assert rel_err(sysm.decode_second_directional(z, u, v), o.decode_second_directional(z, u, v)) < 1e-10
    q = sysm.decode(z)
    v_, g_ = sysm.assemble(q)
    vo, go = o.assemble(q)
    assert rel_err(v_, vo) < 1e-10 and rel_err(g_, go) < 1e-10


def test_primitives_config3_scale(oracle, product):
    """The largest config (786,432 tets, n = 408,672, d = 32, fp32 storage): assemble at a
    decoded configuration and decode_jacobian against the oracle."""
    pr, sysm, ob = _problem("c3", "fp32", oracle, product)
    rng = np.random.default_rng(5)
    z = 0.5 * rng.standard_normal(pr.model.r)
    q = sysm.decode(z)
    v, g = sysm.assemble(q)
    vo, go = ob.assemble(q)
    assert rel_err(v, vo) < 1e-4 and rel_err(g, go) < 1e-4
    J = sysm.decode_jacobian(z)
    assert J.shape == (pr.model.n, pr.model.r)
    Jo = ob.decode_jacobian(z)
    assert rel_err(J, Jo) < 1e-4
