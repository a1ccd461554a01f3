"""GPU parity at the BASELINE.json configs' own stated shapes (not reduced stand-ins).

* config 3 (32x32x128 jittered Kuhn bar, 786,432 tets, per-tet E ~ U[5e4, 5e5], d = 32,
  5x256 ELU, n = 408,672 > 262,144 so the default device path is the multi-kernel CUDA-graph
  path): E and grad E at seeded z against the oracle (ReducedObjective::eval,
  reduced_solver.cpp:184-202) at fp32 1e-4 and fp64 1e-10; a teacher-forced reduced_step
  (reduced_solver.cpp:235-277) at t = 0 with the 5 m/s impulse and at t = 1.
* config 4 (4,096 z from substream(3, 0) on the config-2 problem, fp32): the whole batch in
  one call, every 128th column against the oracle at 1e-4.
* config 5 (config-2 mesh and decoder, d = 16, pairs from substream(4, 0)): the subspace
  Hessians of the elastic potential (reduced_potential_hessian, losses.cpp:301-316) of 8
  pairs at 1e-4, the same Hessians sliced out of the full 1,024-pair batch, and the order-2
  loss (lipschitz_loss(model, pairs, 2, pot), losses.cpp:196-213, 237-244) over those 8
  pairs at 1e-4.

Tolerances: the north star's (1e-10 relative in fp64 mode, 1e-4 in fp32 mode, norm-wise
rel_err of reference tests/helpers.hpp:16-18).  For the fp32 c3 step: the exit code is
exact, the iteration count within 1 of the oracle's, and z* within 1e-4 relative (max-norm
over ||z*||_inf) -- fp32 storage of W_out and the element records perturbs the line search
by ~1e-7 relative in E."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3(oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build("c3")
    ob = oracle.problem("c3")
    return pr, ob


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_c3_eval_matches_oracle(precision, c3, product):
    from paper_2409_03807_b200 import configs
    pr, ob = c3
    assert pr.model.n == 408672 and pr.mesh.num_elements() == 786432
    sysm = pr.system(precision)
    try:
        assert np.allclose(sysm.mass, ob.mass, rtol=1e-12, atol=0)  # jittered volumes: last-bit differences
        qbar = configs.timestep0_qbar(pr, ob.mass)
        obj = product.ReducedObjective(sysm, qbar, configs.DT)
        tol = 1e-4 if precision == "fp32" else 1e-10
        for z in configs.gaussian_latents(31, 3, pr.model.r):
            g = np.zeros(pr.model.r)
            E = obj.eval(z, g)
            Eo, go = ob.eval(z, qbar=qbar, dt=configs.DT)
            assert rel_err(E, Eo) < tol, (precision, rel_err(E, Eo))
            assert rel_err(g, go) < tol, (precision, rel_err(g, go))
            assert obj.eval(z) == E
    finally:
        sysm.close()


def test_c3_teacher_forced_steps(c3, product):
    """Steps t = 0 (impulse) and t = 1, each from the oracle's start-of-step state."""
    from paper_2409_03807_b200 import configs
    P = product
    pr, ob = c3
    cfg = configs.solver_config()
    st0 = pr.initial_state()
    sysm = pr.system("fp32")
    try:
        f = P.gravity_force(pr.mesh, sysm.mass, configs.GRAVITY)
        start = (st0.positions.copy(), st0.velocities.copy(), np.zeros(pr.model.r))
        for t in range(2):
            res = ob.simulate(1, cfg, gravity=configs.GRAVITY, positions=start[0], velocities=start[1], z=start[2])
            state = P.SimState(start[0].copy(), start[1].copy(), start[2].copy(), 0.0)
            frame = P.FrameInput(pr.mesh.vertices.copy(), f)
            rep = P.reduced_step(state, frame, sysm, cfg)
            assert rep.code == res["codes"][0], (t, rep.code, res["codes"][0])
            assert abs(rep.iterations - res["iterations"][0]) <= 1, (t, rep.iterations, res["iterations"][0])
            zs = max(np.abs(res["z"]).max(), 1e-30)
            assert np.abs(state.z - res["z"]).max() / zs < 1e-4, (t, np.abs(state.z - res["z"]).max(), zs)
            assert rel_err(state.positions, res["positions"]) < 1e-9
            if t == 0:
                assert res["iterations"][0] > 0  # the impulse makes step 0 non-trivial
            start = (res["positions"], res["velocities"], res["z"])
    finally:
        sysm.close()


def test_c4_full_batch_matches_oracle(oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build("c2")
    sysm = pr.system("fp32")
    ob = oracle.problem("c2")
    qbar = configs.timestep0_qbar(pr, ob.mass)
    sysm.set_inertia(qbar, configs.DT)
    Z = configs.latent_batch_c4(pr.model.r, 4096)
    E, G = sysm.eval_batched(Z)
    idx = np.arange(0, 4096, 128)
    Eo, Go = ob.eval_batch(Z[idx], qbar=qbar, dt=configs.DT, threads=16)
    assert rel_err(E[idx], Eo) < 1e-4
    worst = max(rel_err(G[i], Go[k]) for k, i in enumerate(idx))
    assert worst < 1e-4, worst
    assert np.all(np.isfinite(E)) and np.all(np.isfinite(G))
    sysm.close()


def test_c5_hessians_and_loss_match_oracle(oracle, product):
    from paper_2409_03807_b200 import configs
    pr = configs.build("c2")
    sysm = pr.system("fp32")
    ob = oracle.problem("c2")
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 1024)
    k = 8
    pts = np.concatenate([Z1[:k], Z2[:k]])
    with ThreadPoolExecutor(8) as ex:  # ctypes releases the GIL: one oracle Hessian per thread
        Ho = list(ex.map(ob.reduced_potential_hessian, pts))
    Hs = sysm.hessian_batched(pts)
    for i in range(2 * k):
        assert rel_err(Hs[i], Ho[i]) < 1e-4, (i, rel_err(Hs[i], Ho[i]))
        assert np.array_equal(Hs[i], Hs[i].T)
    # the same points inside the full config-5 batch (2,048 Hessians in one call)
    Hall = sysm.hessian_batched(np.concatenate([Z1, Z2]))
    for i in range(k):
        assert rel_err(Hall[i], Ho[i]) < 1e-4
        assert rel_err(Hall[1024 + i], Ho[k + i]) < 1e-4
    # order-2 loss over those pairs, against the oracle's lipschitz_loss and the Hessians above
    loss = sysm.lipschitz_loss(Z1[:k], Z2[:k])
    ref = ob.lipschitz_loss2(Z1[:k], Z2[:k], threads=8)
    assert rel_err(loss, ref) < 1e-4, (loss, ref)
    manual = np.mean([np.sum((Ho[i] - Ho[k + i]) ** 2) / np.sum((Z1[i] - Z2[i]) ** 2) for i in range(k)])
    assert rel_err(ref, manual) < 1e-10
    full = sysm.lipschitz_loss(Z1, Z2)
    manual_full = np.mean([np.sum((Hall[i] - Hall[1024 + i]) ** 2) / np.sum((Z1[i] - Z2[i]) ** 2)
                           for i in range(1024)])
    assert rel_err(full, manual_full) < 1e-5, (full, manual_full)
    sysm.close()
