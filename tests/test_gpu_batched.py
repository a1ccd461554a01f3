"""GPU parity of the batched path (config 4 shape: many z on one mesh/decoder)
against the oracle's ReducedObjective::eval loop (reference reduced_solver.cpp:184-202).
The batched path computes in fp32 (storage and arithmetic) with fp64 reductions:
tolerance 1e-4 relative (north-star fp32 bar)."""
import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,precision", [("c1", "fp64"), ("c2", "fp32")])
def test_batched_eval_matches_oracle(name, precision, oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build(name)
    sysm = pr.system(precision)
    ob = oracle.problem(name)
    qbar = configs.timestep0_qbar(pr, ob.mass)
    sysm.set_inertia(qbar, configs.DT)
    Z = configs.latent_batch_c4(pr.model.r, 300 if name == "c1" else 150)
    E, G = sysm.eval_batched(Z)
    idx = np.arange(0, Z.shape[0], 7 if name == "c1" else 25)
    Eo, Go = ob.eval_batch(Z[idx], qbar=qbar, dt=configs.DT, threads=8)
    assert rel_err(E[idx], Eo) < 1e-4
    worst = max(rel_err(G[i], Go[k]) for k, i in enumerate(idx))
    assert worst < 1e-4, worst
    # value-only path agrees with the gradient path
    E2 = sysm.eval_batched(Z[:40], want_grad=False)
    assert np.allclose(E2, E[:40], rtol=1e-12, atol=0)


def test_batched_matches_single_instance(product):
    """Batched (fp32) vs single-instance (fp64) device evaluations on the same z."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp64")
    sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
    Z = configs.latent_batch_c4(pr.model.r, 20)
    E, G = sysm.eval_batched(Z)
    for b in range(0, 20, 5):
        e, g = sysm.eval(Z[b])
        assert rel_err(E[b], e) < 1e-5 and rel_err(G[b], g) < 1e-4


def test_batched_tcgen05_matches_cuda_core_sgemm(product, monkeypatch):
    """The tcgen05 3xTF32 GEMMs (default) against the CUDA-core SGEMM fallback (LSB_TC=0)
    on the same batch: E and dE/dz agree to fp32 accuracy."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    Z = configs.latent_batch_c4(pr.model.r, 96)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("LSB_TC", flag)
        sysm = pr.system("fp32")
        sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
        out[flag] = sysm.eval_batched(Z)
        sysm.close()
    E1, G1 = out["1"]
    E0, G0 = out["0"]
    assert rel_err(E1, E0) < 1e-6
    assert rel_err(G1, G0) < 1e-5


def test_pin_positions_set_after_batched_use(oracle, product):
    """lsb_set_pin_positions after the batched and Hessian engines were built: their pinned rows of u
    follow the new pins (the pins enter the energy through u, energy.cpp:155-157)."""
    from paper_2409_03807_b200 import configs
    pr = configs.build("c1")
    sysm = pr.system("fp64")
    ob = oracle.problem("c1")
    Z = configs.latent_batch_c4(pr.model.r, 12)
    E0, _ = sysm.eval_batched(Z)          # engines built with the rest-position pins
    sysm.hessian_batched(Z[:3])
    pins = pr.mesh.vertices.copy()
    pins[pr.mesh.pinned] += np.array([0.002, -0.001, 0.0015])
    sysm.set_pin_positions(pins)
    ob.set_pins(pins)
    E, G = sysm.eval_batched(Z)
    Eo, Go = ob.eval_batch(Z[:4], qbar=None)
    assert rel_err(E[:4], Eo) < 1e-4 and rel_err(E0[:4], Eo) > 1e-3  # the pins moved the energy
    assert max(rel_err(G[i], Go[i]) for i in range(4)) < 1e-4
    H = sysm.hessian_batched(Z[:3])
    for k in range(3):
        assert rel_err(H[k], ob.reduced_potential_hessian(Z[k])) < 1e-4
    e1, g1 = sysm.eval(Z[0])              # single-instance path on the same pins
    assert rel_err(E[0], e1) < 1e-5
