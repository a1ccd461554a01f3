"""Oracle self-tests for the training-side theta-gradient of the order-2 Lipschitz loss
(SURVEY §8(f) rank 3).

Restates the reference's own checks:
* test_energy.cpp:93-118 -- the third-derivative contraction equals the FD gradient of
  x -> <A, H(x) B> (rel < 2e-5, h = 1e-5, single unpinned tet, mu = 1.1, lambda = 0.9);
* test_losses.cpp:47-78, 293-305 -- every parameter gradient of build_lipschitz_loss
  (order 2) equals central differences of the loss (h = 1e-4, rel < 1e-4) on a tiny mesh
  with a SiLU decoder, norm_scale 0.5 and norm_shift = rest.
The loss value itself is pinned by test_oracle_net_solver.py (lipschitz_loss2)."""
import numpy as np
import pytest

from conftest import rel_err

TET = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)


@pytest.mark.parametrize("seed", range(6))
def test_third_contraction_matches_fd(oracle, seed):
    o = oracle.Oracle.from_mesh(TET, np.array([[0, 1, 2, 3]], np.int32), np.zeros(0, np.int32))
    o.set_material(1.1, 0.9, 1.0)
    rng = np.random.default_rng(50 + seed)
    x0 = TET.reshape(-1) + 0.1 * rng.standard_normal(12)
    A = rng.standard_normal((12, 2))
    B = rng.standard_normal((12, 2))

    def inner(x):
        return float(np.sum(A * o.hessian_apply(x, B)))

    qbar = o.third_contraction(x0, A, B)
    h = 1e-5
    fd = np.array([(inner(x0 + h * np.eye(12)[i]) - inner(x0 - h * np.eye(12)[i])) / (2 * h) for i in range(12)])
    assert rel_err(qbar, fd) < 2e-5, rel_err(qbar, fd)
    # the contraction uses sym(A B^T): swapping A and B changes nothing
    assert rel_err(o.third_contraction(x0, B, A), qbar) < 1e-13


def _model(oracle, r, hidden, width, seed, act=1, nx=3, ny=2, nz=1):
    o = oracle.Oracle.bar(nx, ny, nz, 0.6, 0.3, 0.3, 0.0, 0, True)
    o.set_material(1.5, 1.0, 2.0)
    rng = np.random.default_rng(seed)
    dims = [r] + [width] * hidden + [o.n]
    layers = []
    for i in range(len(dims) - 1):
        W = rng.standard_normal((dims[i + 1], dims[i])) * np.sqrt(2.0 / (dims[i] + dims[i + 1]))
        b = 0.1 * rng.standard_normal(dims[i + 1])
        layers.append((W, b, act if i < len(dims) - 2 else 0))
    X, _, _, _, fi = o.mesh_arrays()
    shift = X[fi >= 0].reshape(-1)
    scale = np.full(o.n, 0.5)
    o.set_decoder(layers, shift, scale, r)
    return o, layers, shift, scale


def _fd_check(o, layers, shift, scale, r, Z1, Z2, h=1e-4, tol=1e-4):
    loss, grads = o.lipschitz_loss2_grad(Z1, Z2)
    assert rel_err(loss, o.lipschitz_loss2(Z1, Z2)) < 1e-13
    for l, (W, b, act) in enumerate(layers):
        for which, P in (("W", W), ("b", b)):
            fd = np.zeros(P.size)
            flat = P.reshape(-1)
            for k in range(P.size):
                saved = flat[k]
                flat[k] = saved + h
                o.set_decoder(layers, shift, scale, r)
                fp = o.lipschitz_loss2(Z1, Z2)
                flat[k] = saved - h
                o.set_decoder(layers, shift, scale, r)
                fm = o.lipschitz_loss2(Z1, Z2)
                flat[k] = saved
                fd[k] = (fp - fm) / (2 * h)
            o.set_decoder(layers, shift, scale, r)
            g = grads[l][0] if which == "W" else grads[l][1]
            err = rel_err(g.reshape(-1), fd, 1e-8)
            assert err < tol, (l, which, err)


def test_theta_gradient_matches_fd_one_hidden_layer(oracle):
    """test_losses.cpp:293-305 shape: r = 2, one SiLU hidden layer of width 5, one pair."""
    o, layers, shift, scale = _model(oracle, 2, 1, 5, 99)
    rng = np.random.default_rng(91)
    Z1 = 0.5 * rng.standard_normal((1, 2))
    Z2 = 0.5 * rng.standard_normal((1, 2))
    _fd_check(o, layers, shift, scale, 2, Z1, Z2)


def test_theta_gradient_matches_fd_two_hidden_layers_two_pairs(oracle):
    """test_losses.cpp:306-320 shape (two hidden layers), here with r = 3 and two pairs."""
    o, layers, shift, scale = _model(oracle, 3, 2, 4, 103)
    rng = np.random.default_rng(92)
    Z1 = 0.5 * rng.standard_normal((2, 3))
    Z2 = 0.5 * rng.standard_normal((2, 3))
    _fd_check(o, layers, shift, scale, 3, Z1, Z2)


def test_theta_gradient_tanh_hidden(oracle):
    o, layers, shift, scale = _model(oracle, 2, 2, 3, 7, act=2)
    rng = np.random.default_rng(93)
    _fd_check(o, layers, shift, scale, 2, 0.5 * rng.standard_normal((1, 2)), 0.5 * rng.standard_normal((1, 2)))


def test_theta_gradient_thread_split_and_pair_swap(oracle):
    o, layers, shift, scale = _model(oracle, 3, 2, 4, 11)
    rng = np.random.default_rng(94)
    Z1 = 0.5 * rng.standard_normal((5, 3))
    Z2 = 0.5 * rng.standard_normal((5, 3))
    l1, g1 = o.lipschitz_loss2_grad(Z1, Z2, threads=1)
    l3, g3 = o.lipschitz_loss2_grad(Z1, Z2, threads=3)
    ls, gs = o.lipschitz_loss2_grad(Z2, Z1)
    assert l1 == pytest.approx(l3, rel=1e-13) and l1 == pytest.approx(ls, rel=1e-13)
    for (a, b), (c, d), (e, f) in zip(g1, g3, gs):
        assert rel_err(c, a) < 1e-12 and rel_err(d, b) < 1e-12
        assert rel_err(e, a) < 1e-12 and rel_err(f, b) < 1e-12


def test_theta_gradient_coincident_pair_rejected(oracle):
    o, _, _, _ = _model(oracle, 2, 1, 3, 5)
    z = np.array([[0.1, 0.2]])
    with pytest.raises(ValueError):  # std::invalid_argument (losses.cpp:203-204)
        o.lipschitz_loss2_grad(z, z.copy())
