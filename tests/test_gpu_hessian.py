"""GPU parity of the subspace Hessian of the elastic potential
(reference reduced_potential_hessian, losses.cpp:301-316) and of the order-2
Lipschitz loss (lipschitz_loss(model, pairs, 2, pot), losses.cpp:196-213,237-244)
against the CPU oracle.  Device path: fp32 with fp64 reductions; tolerance
1e-4 relative (north star, config 5)."""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_hessian_matches_oracle_c1(precision, oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system(precision)
    ob = oracle.problem("c1")
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 12)
    Z = np.concatenate([Z1, Z2])
    H = sysm.hessian_batched(Z)
    for k in range(0, Z.shape[0], 5):
        Ho = ob.reduced_potential_hessian(Z[k])
        assert rel_err(H[k], Ho) < 1e-4, (k, rel_err(H[k], Ho))
        assert np.array_equal(H[k], H[k].T)


def test_lipschitz_loss_matches_oracle_c1(oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp64")
    ob = oracle.problem("c1")
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 24)
    loss = product.lipschitz_loss(sysm, list(zip(Z1, Z2)))
    ref = ob.lipschitz_loss2(Z1, Z2, threads=8)
    assert rel_err(loss, ref) < 1e-4, (loss, ref)
    assert product.lipschitz_loss(sysm, list(zip(Z2, Z1))) == pytest.approx(loss, rel=1e-12)
    with pytest.raises(ValueError, match="coincident"):
        sysm.lipschitz_loss(Z1[:1], Z1[:1].copy())


def test_hessian_general_decoder(oracle, product):
    """Non-ELU activation, biases, scale != 1, pinned-vertex mesh (r = 8)."""
    P = product
    mesh = P.make_bar_mesh(3, 2, 2, 1.0, 0.4, 0.5, jitter_frac=0.05, seed=3)
    rng = np.random.default_rng(4)
    n = mesh.num_dofs()
    dims = [8, 16, 16, n]
    layers = []
    for i in range(3):
        W = rng.standard_normal((dims[i + 1], dims[i])) * (0.4 if i < 2 else 0.05)
        b = 0.1 * rng.standard_normal(dims[i + 1])
        layers.append(P.Layer(W, b, P.Activation.Silu if i < 2 else P.Activation.Identity))
    shift = P.dof_pack(mesh, mesh.vertices)
    scale = 0.3 + 0.1 * rng.random(n)
    model = P.SubspaceModel(8, n, layers, shift, scale)
    mu = 2.0 + rng.random(mesh.num_elements())
    lam = 1.0 + rng.random(mesh.num_elements())
    sysm = P.ReducedSystem(mesh, mu, lam, 3.0, model, "fp64")
    o = oracle.Oracle.from_mesh(mesh.vertices, mesh.elements, mesh.pinned)
    o.set_material(mu, lam, 3.0)
    o.set_decoder([(l.W, l.b, int(l.act)) for l in layers], shift, scale, 8)
    Z = 0.5 * rng.standard_normal((5, 8))
    H = sysm.hessian_batched(Z)
    for k in range(5):
        assert rel_err(H[k], o.reduced_potential_hessian(Z[k])) < 1e-4


@pytest.mark.parametrize("inertia", [True, False])
def test_objective_hessian_matches_oracle(inertia, oracle, product):
    """lsb_objective_hessian == ReducedObjective::hessian (reduced_solver.cpp:204-229), with the
    M/h^2 block and the inertia residual's curvature when qbar is set (1e-4, fp32 path)."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp32")
    ob = oracle.problem("c1")
    qbar = configs.timestep0_qbar(pr, ob.mass) if inertia else None
    obj = product.ReducedObjective(sysm, qbar, configs.DT)
    rng = np.random.default_rng(21)
    Z = 0.5 * rng.standard_normal((5, pr.model.r))
    for z in Z:
        Hg = obj.hessian(z)
        Ho = ob.hessian(z, qbar=qbar, dt=configs.DT)
        assert rel_err(Hg, Ho) < 1e-4, rel_err(Hg, Ho)
        assert np.abs(Hg - Hg.T).max() == 0.0


@pytest.mark.parametrize("inertia", [True, False])
def test_projective_newton_matches_oracle(inertia, oracle, product):
    """Device projective Newton (projective_newton_minimize, reduced_solver.cpp:133-182) against
    the oracle's on config 1: same exit code, the same minimiser."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp64")
    ob = oracle.problem("c1")
    qbar = configs.timestep0_qbar(pr, ob.mass) if inertia else None
    obj = product.ReducedObjective(sysm, qbar, configs.DT)
    cfg = configs.solver_config()
    cfg.epsilon = 1e-8
    z = np.zeros(pr.model.r)
    rep = product.projective_newton_minimize(obj, obj.hessian, z, cfg)
    res = ob.projective_newton(np.zeros(pr.model.r), qbar=qbar, dt=configs.DT, epsilon=1e-8)
    assert rep.code == res["code"] == 1, (rep.code, res["code"])
    assert abs(rep.iterations - res["iterations"]) <= 1, (rep.iterations, res["iterations"])
    assert np.abs(z - res["z"]).max() < 1e-7 * max(1.0, np.abs(res["z"]).max())
    g = np.zeros(pr.model.r)
    obj.eval(z, g)
    assert np.abs(g).max() < 1e-8


def test_hessian_chunk_width_changes_are_transparent(oracle, product):
    """The Hessian path sizes its chunks by the call (16-point multiples up to 256): the same z gives the
    same Hessian whether it is computed alone, inside a 300-point call, or alone again afterwards (the
    pinned rows of the chunk buffers are re-laid when the width changes), and matches the oracle."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp64")
    ob = oracle.problem("c1")
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 150)
    Z = np.concatenate([Z1, Z2])
    H_small = sysm.hessian_batched(Z[:3])
    H_big = sysm.hessian_batched(Z)
    H_again = sysm.hessian_batched(Z[:3])
    assert np.array_equal(H_small, H_again)
    for k in range(3):
        assert rel_err(H_big[k], H_small[k]) < 1e-6
    for k in (0, 150, 299):
        assert rel_err(H_big[k], ob.reduced_potential_hessian(Z[k])) < 1e-4


@pytest.mark.parametrize("r", [8, 16, 32])
def test_edge_space_hessian_kernel_small_mesh(oracle, product, monkeypatch, r):
    """The edge-space chained-MMA element Hessian kernel at every supported latent dimension (r = 8: one
    half-empty m tile; 16; 32: two m tiles, four n tiles) on a 216-tet mesh against the oracle's
    reduced_potential_hessian (losses.cpp:301-316) at the 1e-4 bar."""
    P = product
    monkeypatch.setenv("LSB_HESS3", "1")
    mesh = P.make_bar_mesh(4, 3, 3, 1.0, 0.4, 0.5, jitter_frac=0.05, seed=9)
    rng = np.random.default_rng(6)
    n = mesh.num_dofs()
    dims = [r, 16, 16, n]
    layers = []
    for i in range(3):
        W = rng.standard_normal((dims[i + 1], dims[i])) * (0.4 if i < 2 else 0.05)
        b = 0.1 * rng.standard_normal(dims[i + 1])
        layers.append(P.Layer(W, b, P.Activation.Silu if i < 2 else P.Activation.Identity))
    shift = P.dof_pack(mesh, mesh.vertices)
    scale = 0.3 + 0.1 * rng.random(n)
    model = P.SubspaceModel(r, n, layers, shift, scale)
    mu = 2.0 + rng.random(mesh.num_elements())
    lam = 1.0 + rng.random(mesh.num_elements())
    sysm = P.ReducedSystem(mesh, mu, lam, 3.0, model, "fp64")
    o = oracle.Oracle.from_mesh(mesh.vertices, mesh.elements, mesh.pinned)
    o.set_material(mu, lam, 3.0)
    o.set_decoder([(l.W, l.b, int(l.act)) for l in layers], shift, scale, r)
    Z = 0.5 * rng.standard_normal((5, r))
    H = sysm.hessian_batched(Z)
    worst = max(rel_err(H[k], o.reduced_potential_hessian(Z[k])) for k in range(5))
    assert worst < 1e-4, worst
    sysm.close()


def test_edge_space_hessian_smooth_decoder(oracle, product):
    """A decoder whose output layer varies smoothly over the mesh (as a trained subspace does, unlike the
    Xavier-random one of the configs): neighbouring vertices' Jacobian rows nearly coincide, so the
    element Hessian kernel must split the EDGE DIFFERENCES of the rows, not the rows, into TF32 parts, and a
    single TF32 pass would leave correlated rounding errors (7.5e-4 here).  27,648 tets, r = 16, against
    reduced_potential_hessian
    (losses.cpp:301-316) at the 1e-4 bar."""
    P = product
    mesh = P.make_bar_mesh(12, 12, 32, 1.0, 0.4, 0.4, jitter_frac=0.05, seed=11)
    rng = np.random.default_rng(12)
    n, r, h = mesh.num_dofs(), 16, 32
    layers = []
    dims = [r, h, h]
    for i in range(2):
        layers.append(P.Layer(rng.standard_normal((dims[i + 1], dims[i])) * 0.4, 0.1 * rng.standard_normal(dims[i + 1]),
                              P.Activation.Silu))
    X = mesh.vertices[mesh.free_vertices]                      # free vertices x 3
    k = rng.uniform(-4.0, 4.0, (h, 3))                         # long wavelengths against the 1/32 cell size
    ph = rng.uniform(0, 2 * np.pi, h)
    B = rng.standard_normal((3, h))
    basis = 1.0 + 0.5 * np.sin(X @ k.T + ph)                   # free vertices x h, smooth, O(1) offset
    Wout = 0.02 * (basis[:, None, :] * B[None, :, :]).reshape(n, h)
    layers.append(P.Layer(Wout, np.zeros(n), P.Activation.Identity))
    shift = P.dof_pack(mesh, mesh.vertices)
    scale = np.ones(n)
    model = P.SubspaceModel(r, n, layers, shift, scale)
    mu = 2.0e4 + 1.0e3 * rng.random(mesh.num_elements())
    lam = 8.0e4 + 1.0e3 * rng.random(mesh.num_elements())
    sysm = P.ReducedSystem(mesh, mu, lam, 1000.0, model, "fp32")
    o = oracle.Oracle.from_mesh(mesh.vertices, mesh.elements, mesh.pinned)
    o.set_material(mu, lam, 1000.0)
    o.set_decoder([(l.W, l.b, int(l.act)) for l in layers], shift, scale, r)
    Z = 0.5 * rng.standard_normal((3, r))
    H = sysm.hessian_batched(Z)
    worst = max(rel_err(H[i], o.reduced_potential_hessian(Z[i])) for i in range(3))
    assert worst < 1e-4, worst
    sysm.close()
