"""Independent-route pins of the oracle, restated from the reference's own tests.

* acceptance.cpp:397-506 (criterion 2, "oracle equivalence"): lipschitz_loss(model, pairs,
  order, pot) for orders 0, 1, 2 against a PLAIN route -- a plain-loop decoder forward, a
  plain-loop Jacobian, the assembled Hessian applied to it and plain-loop second directional
  derivatives (plain_reduced_hessian, acceptance.cpp:397-444) -- at 1e-8 relative over 50
  batches of 3 pairs drawn 0.4 randn.  The reference runs it on a 2-D 5x2 bar with a SiLU
  r = 3, 2 x 8 decoder, scale 0.4, mu = 2, lambda = 1.5; the oracle is 3-D only, so the
  same decoder shape and material sit on a 3x2x1 tet bar (30 tets).
* test_solvers.cpp:196-225 ("no elasticity: least-squares projection onto the span"): with
  the elastic term removed by runtime cubature, one reduced_step of a linear-span decoder
  minimises the pure inertia term, so z* equals the closed-form weighted least-squares
  solution (B^T M B)^-1 B^T M (qbar - q_prev) at 1e-8 (max-norm), eps = 1e-12, dt = 0.05.
  The reference's empty ElementSubset is expressed as a one-element subset of weight 0
  (vol * 0: no energy, no forces).  The same step runs through the device in
  tests/test_gpu_eval.py::test_wls_step_device.

The plain route uses only the oracle's assemble / elastic_hessian_apply (energy.cpp) and
activation_eval (net.cpp:34-64) -- not its decode, decode_jacobian, tape or loss code."""
import numpy as np
import pytest

from conftest import rel_err


def _act(oracle, act, a, order):
    return np.array([oracle.activation_eval(act, float(x), order) for x in a])


def plain_decode(oracle, layers, shift, scale, z):
    """plain_decode_fn (acceptance.cpp:383-395)."""
    y = np.asarray(z, np.float64)
    for W, b, act in layers:
        y = _act(oracle, act, W @ y + b, 0)
    return scale * y + shift


def plain_jacobian(oracle, layers, scale, z):
    y = np.asarray(z, np.float64)
    G = np.eye(len(z))
    for W, b, act in layers:
        a = W @ y + b
        G = _act(oracle, act, a, 1)[:, None] * (W @ G)
        y = _act(oracle, act, a, 0)
    return scale[:, None] * G


def plain_reduced_hessian(oracle, o, layers, shift, scale, z):
    """plain_reduced_hessian (acceptance.cpp:397-444): J^T (K J) + sum_ab g . s * d2f(e_a, e_b)."""
    r = len(z)
    q = plain_decode(oracle, layers, shift, scale, z)
    J = plain_jacobian(oracle, layers, scale, z)
    _, g = o.assemble(q)
    H = J.T @ o.hessian_apply(q, J)
    for a in range(r):
        for b in range(a, r):
            yy = np.asarray(z, np.float64)
            p, t, s = np.eye(r)[a], np.eye(r)[b], np.zeros(r)
            for W, bb, act in layers:
                av = W @ yy + bb
                d1, d2 = _act(oracle, act, av, 1), _act(oracle, act, av, 2)
                ap, at, as_ = W @ p, W @ t, W @ s
                yy = _act(oracle, act, av, 0)
                p, t, s = d1 * ap, d1 * at, d2 * ap * at + d1 * as_
            v = g @ (scale * s)
            H[a, b] += v
            if a != b:
                H[b, a] += v
    return H


@pytest.fixture(scope="module")
def criterion2(oracle):
    o = oracle.Oracle.bar(3, 2, 1, 1.0, 0.4, 0.3, 0.0, 0, False)
    o.set_material(2.0, 1.5, 1.0)
    n = o.n
    rng = np.random.default_rng(99)
    dims = [3, 8, 8, n]
    layers = []
    for i in range(3):  # Glorot-scaled weights, non-zero biases
        sd = np.sqrt(2.0 / (dims[i] + dims[i + 1]))
        layers.append((sd * rng.standard_normal((dims[i + 1], dims[i])), 0.1 * rng.standard_normal(dims[i + 1]),
                       1 if i < 2 else 0))
    X, _, _, _, fi = o.mesh_arrays()
    shift = X[fi >= 0].reshape(-1)
    scale = np.full(n, 0.4)
    o.set_decoder(layers, shift, scale, 3)
    return o, layers, shift, scale


def test_lipschitz_loss_order2_vs_plain_route(oracle, criterion2):
    """acceptance.cpp:449-506, order 2 (the hot-path loss): 1e-8."""
    o, layers, shift, scale = criterion2
    rng = np.random.default_rng(993)
    worst = 0.0
    for batch in range(50):
        Z1 = 0.4 * rng.standard_normal((3, 3))
        Z2 = 0.4 * rng.standard_normal((3, 3))
        produced = o.lipschitz_loss2(Z1, Z2)
        ref = np.mean([np.sum((plain_reduced_hessian(oracle, o, layers, shift, scale, a) -
                               plain_reduced_hessian(oracle, o, layers, shift, scale, b)) ** 2) /
                       np.sum((a - b) ** 2) for a, b in zip(Z1, Z2)])
        worst = max(worst, abs(produced - ref) / max(abs(ref), 1e-300))
    assert worst < 1e-8, worst


def test_reduced_hessian_vs_plain_route(oracle, criterion2):
    """reduced_potential_hessian (losses.cpp:301-316) against the plain route, entrywise."""
    o, layers, shift, scale = criterion2
    rng = np.random.default_rng(5)
    for _ in range(4):
        z = 0.4 * rng.standard_normal(3)
        H = o.reduced_potential_hessian(z)
        Hp = plain_reduced_hessian(oracle, o, layers, shift, scale, z)
        assert rel_err(H, Hp) < 1e-10, rel_err(H, Hp)


def test_potential_value_and_gradient_vs_plain_route(oracle, criterion2):
    """The order-0 / order-1 plain routes of acceptance.cpp:470-484 (assembled energy of the
    plain decode; dense plain Jacobian times the assembled gradient) against the oracle's
    quasi-static ReducedObjective::eval (reduced_solver.cpp:184-202)."""
    o, layers, shift, scale = criterion2
    rng = np.random.default_rng(6)
    for _ in range(3):
        z = 0.4 * rng.standard_normal(3)
        q = plain_decode(oracle, layers, shift, scale, z)
        assert rel_err(q, o.decode(z)) < 1e-12
        P, g = o.assemble(q)
        E, gz = o.eval(z)  # quasi-static objective = elastic potential only
        assert rel_err(E, P) < 1e-12
        assert rel_err(gz, plain_jacobian(oracle, layers, scale, z).T @ g) < 1e-10


def test_elasticity_free_step_is_weighted_least_squares(oracle):
    """test_solvers.cpp:196-225 at 1e-8."""
    o = oracle.Oracle.bar(3, 2, 2, 1.0, 0.4, 0.5, 0.05, 3, True)
    o.set_material(2.0, 1.5, 3.0)
    n, r = o.n, 3
    rng = np.random.default_rng(407)
    basis = 0.1 * rng.standard_normal((n, r))
    X, _, _, _, fi = o.mesh_arrays()
    shift = X[fi >= 0].reshape(-1)
    o.set_decoder([(basis, np.zeros(n), 0)], shift, np.ones(n), r)  # linear_span_model
    force = np.zeros(n)
    force[1::3] = -0.5 * o.mass[1::3]
    o.set_cubature([0], [0.0])  # the elastic term vanishes (reference: empty ElementSubset)
    from types import SimpleNamespace
    cfg = SimpleNamespace(epsilon=1e-12, max_iters=1024, max_linesearch=128, lbfgs_history=8, dt=0.05)
    pos, vel, z, code, iters = o.reduced_step(X, np.zeros_like(X), np.zeros(r), X, force, cfg)
    q_prev = shift
    qbar = q_prev + cfg.dt ** 2 * force / o.mass
    JtMJ = basis.T @ (o.mass[:, None] * basis)
    z_star = np.linalg.solve(JtMJ, basis.T @ (o.mass * (qbar - q_prev)))
    assert code == 1
    assert np.abs(z - z_star).max() < 1e-8, np.abs(z - z_star).max()
    o.set_cubature(None)
