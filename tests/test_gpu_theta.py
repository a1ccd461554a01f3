"""GPU parity of the training-side theta-gradient of the order-2 Lipschitz loss
(reference build_lipschitz_loss + Tape::backward,
losses.cpp:196-213, tape.cpp:46-79, 245-279) against the CPU oracle, whose own
gradient is pinned by central differences (tests/test_oracle_theta.py, the
reference's test_losses.cpp:47-78 check).  Device path: fp32 arithmetic, fp64
accumulation; tolerance 1e-4 relative (norm-wise per parameter block), as the loss
in config 5."""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-4


def _compare(sysm, o, Z1, Z2, threads=8):
    loss, grads = sysm.lipschitz_loss_grad(Z1, Z2)
    ref_loss, ref = o.lipschitz_loss2_grad(Z1, Z2, threads=threads)
    assert rel_err(loss, ref_loss) < 1e-4, (loss, ref_loss)
    errs = []
    for l, ((gW, gb), (rW, rb)) in enumerate(zip(grads, ref)):
        eW, eb = rel_err(gW, rW), rel_err(gb, rb)
        errs.append((l, eW, eb))
    print("theta-gradient rel errors per layer (W, b):", errs)
    for l, eW, eb in errs:
        assert eW < GRAD_TOL and eb < GRAD_TOL, (l, eW, eb)
    return loss, grads


def test_theta_grad_matches_oracle_c1(oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp32")
    ob = oracle.problem("c1")
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 6)
    loss, grads = _compare(sysm, ob, Z1, Z2)
    # the value is the device Lipschitz loss (same Hessian chunks, bit-identical)
    assert loss == sysm.lipschitz_loss(Z1, Z2)
    # pair order is irrelevant (losses.cpp:205-209 is symmetric in z1, z2)
    loss2, grads2 = sysm.lipschitz_loss_grad(Z2, Z1)
    assert loss2 == pytest.approx(loss, rel=1e-12)
    for (a, b), (c, d) in zip(grads, grads2):
        assert rel_err(c, a) < 1e-5 and rel_err(d, b) < 1e-5
    with pytest.raises(ValueError, match="coincident"):
        sysm.lipschitz_loss_grad(Z1[:1], Z1[:1].copy())


def test_theta_grad_two_chunks_c1(oracle, product):
    """40 pairs = 80 points: one full 64-point chunk and a partial one."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp32")
    ob = oracle.problem("c1")
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 40)
    _compare(sysm, ob, Z1, Z2)


@pytest.mark.parametrize("r", [16, 32])
def test_theta_grad_general_decoder(oracle, product, r):
    """SiLU hidden layers with biases, per-row scale, jittered mesh with pins, r = 16 / 32."""
    P = product
    mesh = P.make_bar_mesh(3, 2, 2, 1.0, 0.4, 0.5, jitter_frac=0.05, seed=3)
    rng = np.random.default_rng(40 + r)
    n = mesh.num_dofs()
    dims = [r, 24, 20, n]
    layers = []
    for i in range(3):
        W = rng.standard_normal((dims[i + 1], dims[i])) * (0.3 if i < 2 else 0.05)
        b = 0.1 * rng.standard_normal(dims[i + 1])
        layers.append(P.Layer(W, b, P.Activation.Silu if i < 2 else P.Activation.Identity))
    shift = P.dof_pack(mesh, mesh.vertices)
    scale = 0.3 + 0.1 * rng.random(n)
    model = P.SubspaceModel(r, n, layers, shift, scale)
    mu = 2.0 + rng.random(mesh.num_elements())
    lam = 1.0 + rng.random(mesh.num_elements())
    sysm = P.ReducedSystem(mesh, mu, lam, 3.0, model, "fp32")
    o = oracle.Oracle.from_mesh(mesh.vertices, mesh.elements, mesh.pinned)
    o.set_material(mu, lam, 3.0)
    o.set_decoder([(l.W, l.b, int(l.act)) for l in layers], shift, scale, r)
    Z1 = 0.5 * rng.standard_normal((3, r))
    Z2 = 0.5 * rng.standard_normal((3, r))
    _compare(sysm, o, Z1, Z2)
