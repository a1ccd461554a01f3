"""Oracle self-tests: decoder derivatives, L-BFGS, reduced objective, Lipschitz loss.

Restates proj/tests/test_net.cpp, test_solvers.cpp, test_losses.cpp checks for the
hot path against the CPU oracle."""
import numpy as np
import pytest

from conftest import rel_err


def _tiny(oracle, act=1, r=3, hidden=2, width=6, seed=5, scale=0.4):
    o = oracle.Oracle.bar(3, 2, 1, 1.0, 0.4, 0.3, 0.0, 0, True)
    o.set_material(2.0, 1.0, 5.0)
    rng = np.random.default_rng(seed)
    n = o.n
    dims = [r] + [width] * hidden + [n]
    layers = []
    for i in range(len(dims) - 1):
        W = rng.standard_normal((dims[i + 1], dims[i])) * 0.5
        b = rng.standard_normal(dims[i + 1]) * 0.1
        layers.append((W, b, act if i < len(dims) - 2 else 0))
    X, _, _, _, fi = o.mesh_arrays()
    shift = X[fi >= 0].reshape(-1)
    o.set_decoder(layers, shift, np.full(n, scale), r)
    return o, layers, shift


@pytest.mark.parametrize("act", [1, 2, 3])
def test_activation_fd(oracle, act):
    """test_net.cpp:39-53 (+ ELU away from its kink)."""
    # the reference test's own inputs: x = 3 randn(substream(7, 0)), one stream
    # shared by Silu (draws 0-19) then Tanh (20-39) (test_net.cpp:40-43); ELU continues.
    block = {1: 0, 2: 1, 3: 2}[act]
    for x in 3.0 * oracle.randn_seq(7, 0, 60)[20 * block:20 * block + 20]:
        if act == 3 and abs(x) < 1e-3:
            continue
        h = 1e-6
        for order in range(3):
            if act == 3 and order >= 1 and x > 0:
                continue
            fd = (oracle.activation_eval(act, x + h, order) - oracle.activation_eval(act, x - h, order)) / (2 * h)
            assert rel_err(oracle.activation_eval(act, x, order + 1), fd, 1e-8) < 1e-6


def test_elu_kink_convention(oracle):
    """ELU^(k)(0) takes the x <= 0 branch."""
    assert oracle.activation_eval(3, 0.0, 0) == 0.0
    assert oracle.activation_eval(3, 0.0, 1) == 1.0
    assert oracle.activation_eval(3, 0.0, 2) == 1.0
    assert oracle.activation_eval(3, 1e-300, 2) == 0.0


def test_decode_matches_plain_forward(oracle):
    """test_net.cpp:72-81 (plain_decode, helpers.hpp:68-82) at 1e-12."""
    o, layers, shift = _tiny(oracle)
    rng = np.random.default_rng(11)
    for _ in range(5):
        z = rng.standard_normal(3)
        y = z
        for W, b, a in layers:
            y = np.array([oracle.activation_eval(a, v, 0) for v in W @ y + b])
        assert rel_err(o.decode(z), 0.4 * y + shift) < 1e-12


def test_decode_jacobian_fd(oracle):
    """test_net.cpp:107-117: FD at h = 1e-5, tol 1e-6."""
    o, _, _ = _tiny(oracle)
    rng = np.random.default_rng(15)
    for _ in range(5):
        z = rng.standard_normal(3)
        J = o.decode_jacobian(z)
        h = 1e-5
        fd = np.stack([(o.decode(z + h * e) - o.decode(z - h * e)) / (2 * h) for e in np.eye(3)], axis=1)
        assert rel_err(J, fd) < 1e-6


def test_second_directional(oracle):
    """test_net.cpp:141-162: exact symmetry, FD-of-Jacobian at 1e-5."""
    o, _, _ = _tiny(oracle)
    rng = np.random.default_rng(21)
    z, u, v = rng.standard_normal(3), rng.standard_normal(3), rng.standard_normal(3)
    a = o.decode_second_directional(z, u, v)
    b = o.decode_second_directional(z, v, u)
    assert np.array_equal(a, b)
    h = 1e-5
    fd = ((o.decode_jacobian(z + h * v) - o.decode_jacobian(z - h * v)) / (2 * h)) @ u
    assert rel_err(a, fd, 1e-10) < 1e-5


def test_second_directional_linear_is_zero(oracle):
    o = oracle.Oracle.bar(2, 1, 1, 1.0, 0.4, 0.3, 0.0, 0, True)
    o.set_material(2.0, 1.0, 5.0)
    rng = np.random.default_rng(1)
    W = rng.standard_normal((o.n, 2))
    o.set_decoder([(W, np.zeros(o.n), 0)], np.zeros(o.n), np.ones(o.n), 2)
    assert np.linalg.norm(o.decode_second_directional(rng.standard_normal(2), rng.standard_normal(2),
                                                      rng.standard_normal(2))) == 0.0


# ----------------------------------------------------------------- L-BFGS (test_solvers.cpp:30-93, 369-386)
def test_lbfgs_already_converged(oracle):
    x, code, it, gn = oracle.lbfgs_minimize(lambda x, g: _quad_small(x, g), np.ones(2) * 0.1, epsilon=1e-3)
    assert code == 1 and it == 0


def _quad_small(x, g):
    if g is not None:
        g[:] = 2e-6 * x
    return 1e-6 * x.dot(x)


def test_lbfgs_quadratic_closed_form(oracle):
    A = np.array([[3.0, 0.5], [0.5, 1.0]])
    b = np.array([1.0, -2.0])

    def f(x, g):
        if g is not None:
            g[:] = A @ x - b
        return 0.5 * x @ A @ x - b @ x

    x, code, it, gn = oracle.lbfgs_minimize(f, np.zeros(2), epsilon=1e-10)
    assert code == 1
    assert np.max(np.abs(x - np.linalg.solve(A, b))) < 1e-8
    assert gn < 1e-10


def test_lbfgs_rosenbrock(oracle):
    def f(x, g):
        a = 1.0 - x[0]
        b = x[1] - x[0] * x[0]
        if g is not None:
            g[0] = -2.0 * a - 400.0 * x[0] * b
            g[1] = 200.0 * b
        return a * a + 100.0 * b * b

    x, code, it, gn = oracle.lbfgs_minimize(f, np.array([-1.2, 1.0]), epsilon=1e-8)
    assert code == 1 and it < 1024
    assert np.max(np.abs(x - 1.0)) < 1e-5


def test_lbfgs_monotone_and_exit_sweep(oracle):
    rng = np.random.default_rng(413)
    for _ in range(10):
        M = rng.standard_normal((4, 4))
        A = M @ M.T + 0.5 * np.eye(4)
        b = rng.standard_normal(4)
        accepted = []

        def f(x, g):
            v = 0.5 * x @ A @ x - b @ x
            if g is not None:
                g[:] = A @ x - b
                accepted.append(v)
            return v

        x, code, it, gn = oracle.lbfgs_minimize(f, rng.standard_normal(4), epsilon=1e-9, max_iters=40)
        if code == 1:
            assert gn < 1e-9
        assert all(accepted[i] <= accepted[i - 1] + 1e-15 for i in range(1, len(accepted)))


# ----------------------------------------------------------------- reduced objective (test_solvers.cpp:114-169)
def test_reduced_objective_derivatives(oracle):
    o, _, shift = _tiny(oracle, r=3)
    rng = np.random.default_rng(403)
    qbar = shift + 0.02 * rng.standard_normal(o.n)
    for _ in range(3):
        z = 0.3 * rng.standard_normal(3)
        v, g = o.eval(z, qbar=qbar, dt=0.05)
        h = 1e-6
        fd = np.array([(o.eval(z + h * e, qbar=qbar, dt=0.05, want_grad=False)
                        - o.eval(z - h * e, qbar=qbar, dt=0.05, want_grad=False)) / (2 * h) for e in np.eye(3)])
        assert rel_err(g, fd) < 1e-6
        H = o.hessian(z, qbar=qbar, dt=0.05)
        hh = 1e-5
        fdH = np.stack([(o.eval(z + hh * e, qbar=qbar, dt=0.05)[1] - o.eval(z - hh * e, qbar=qbar, dt=0.05)[1])
                        / (2 * hh) for e in np.eye(3)], axis=1)
        assert rel_err(H, fdH) < 1e-4
        # grad = J^T (grad P + M (q - qbar) / dt^2) at 1e-10
        q = o.decode(z)
        _, gP = o.assemble(q)
        full = gP + o.mass * (q - qbar) / 0.05 ** 2
        assert rel_err(g, o.decode_jacobian(z).T @ full) < 1e-10


# ----------------------------------------------------------------- Lipschitz loss (test_losses.cpp:197-267)
def test_lipschitz_order2_vs_fd(oracle):
    o, _, _ = _tiny(oracle, r=2, hidden=1, width=6, seed=81)
    rng = np.random.default_rng(75)
    Z1, Z2 = rng.standard_normal((2, 2)), rng.standard_normal((2, 2))
    loss = o.lipschitz_loss2(Z1, Z2)

    def hess_fd(z):
        h = 1e-5
        return np.stack([(o.eval(z + h * e, qbar=None)[1] - o.eval(z - h * e, qbar=None)[1]) / (2 * h)
                         for e in np.eye(2)], axis=1)

    exp = np.mean([np.sum((hess_fd(a) - hess_fd(b)) ** 2) / np.sum((a - b) ** 2) for a, b in zip(Z1, Z2)])
    assert rel_err(loss, exp, 1e-10) < 1e-4
    assert o.lipschitz_loss2(Z2, Z1) == loss  # swap symmetry
    assert loss >= 0.0


def test_lipschitz_constant_decoder_and_coincident(oracle):
    o = oracle.Oracle.bar(3, 2, 1, 1.0, 0.4, 0.3, 0.0, 0, True)
    o.set_material(2.0, 1.0, 5.0)
    X, _, _, _, fi = o.mesh_arrays()
    shift = X[fi >= 0].reshape(-1)
    o.set_decoder([(np.zeros((4, 3)), np.zeros(4), 1), (np.zeros((o.n, 4)), np.zeros(o.n), 0)], shift,
                  np.ones(o.n), 3)
    rng = np.random.default_rng(0)
    assert o.lipschitz_loss2(rng.standard_normal((3, 3)), rng.standard_normal((3, 3))) == 0.0
    z = rng.standard_normal((1, 3))
    with pytest.raises(ValueError, match="coincident"):
        o.lipschitz_loss2(z, z.copy())


# ---- project_spd (test_energy.cpp:344-370) and projective Newton (test_solvers.cpp:94-113) ----
def test_project_spd_reference_cases(oracle):
    A = np.array([[2.0, 1.0], [1.0, 2.0]])
    assert np.array_equal(oracle.project_spd(A), A)  # PSD input returned unchanged
    P = oracle.project_spd(np.diag([1.0, -1.0]))
    assert abs(P[0, 0] - 1.0) < 1e-12 and abs(P[1, 1] - 1e-10) < 1e-20
    rng = np.random.default_rng(41)
    for _ in range(12):
        A = rng.standard_normal((5, 5))
        A = 0.5 * (A + A.T)
        P = oracle.project_spd(A)
        assert np.linalg.eigvalsh(P).min() >= -1e-12
        assert np.abs(P - P.T).max() <= 1e-12 * np.abs(P).max()


def test_projective_newton_quadratic_one_step(oracle):
    A = np.array([[4.0, 1.0, 0.0], [1.0, 3.0, 0.5], [0.0, 0.5, 2.0]])
    b = np.array([1.0, 0.0, -1.0])

    def fn(x, g):
        if g is not None:
            g[:] = A @ x - b
        return 0.5 * x @ A @ x - b @ x

    x, rep = oracle.projective_newton_minimize(fn, lambda x: A, np.zeros(3), epsilon=1e-10)
    assert rep["code"] == 1 and rep["iterations"] == 1
    assert np.abs(x - np.linalg.solve(A, b)).max() < 1e-10


def test_projective_newton_reduced_objective_matches_lbfgs_minimizer(oracle):
    from paper_2409_03807_b200 import configs
    ob = oracle.problem("c1")
    # timestep-0 objective: qbar = X_free + h^2 g
    X = ob.mesh_arrays()[0]
    free = np.nonzero(ob.mesh_arrays()[4] >= 0)[0]
    qbar = X[free].reshape(-1) + configs.DT ** 2 * np.tile(configs.GRAVITY, free.size)
    res = ob.projective_newton(np.zeros(ob.r), qbar=qbar, dt=configs.DT, epsilon=1e-8)
    assert res["code"] == 1 and res["iterations"] < 20
    E, g = ob.eval(res["z"], qbar=qbar, dt=configs.DT)
    assert np.abs(g).max() < 1e-8
    xl, code, _, _ = oracle.lbfgs_minimize(lambda z, gg: _obj(ob, z, gg, qbar), np.zeros(ob.r), epsilon=1e-8)
    assert code == 1
    assert np.abs(xl - res["z"]).max() < 1e-6


def _obj(ob, z, g, qbar):
    from paper_2409_03807_b200 import configs
    if g is None:
        return ob.eval(z, qbar=qbar, dt=configs.DT, want_grad=False)
    E, gg = ob.eval(z, qbar=qbar, dt=configs.DT)
    g[:] = gg
    return E
