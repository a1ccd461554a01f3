"""A reference scenario (JSON) plus a LIPSUBCKPT1 checkpoint drive the device solver
(SURVEY §8(f) rank 4): the acceptance replay loop (proj/tests/acceptance.cpp:517-540)
-- replay_interactions, frame_at with oscillating pins, reduced_step -- on the device,
checked step by step against the oracle's reduced_step under the same frames."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scenario_json():
    return {
        "name": "replay_bar",
        "mesh": {"generator": {"type": "bar3d", "nx": 6, "ny": 2, "nz": 2, "width": 0.9, "height": 0.2,
                               "depth": 0.2, "pin_left": True}},
        "material": {"mu": 2e4, "lambda": 3e4, "density": 900.0},
        "gravity": [0.0, -9.8, 0.0],
        "dt": 0.04,
        "interactions": {"force_min": 5.0, "force_max": 40.0, "patch_radius": 0.1, "steps_min": 3,
                         "steps_max": 9},
        "pin_motion": {"type": "oscillate", "axis": [0.0, 0.0, 1.0], "amplitude": 0.02, "period": 0.6},
        "steps_per_episode": 30,
    }


@pytest.mark.parametrize("path", ["solve", "graph"])
def test_scenario_replay_matches_oracle(oracle, product, tmp_path, path):
    from paper_2409_03807_b200 import checkpoint, scenario as S
    P = product
    s = S.scenario_from_json(_scenario_json())
    model = P.make_bar_decoder(s.mesh, 8, 2, 24, P.Activation.Silu, seed=5, out_scale=1e-2)
    ck = str(tmp_path / "model.ckpt")
    checkpoint.save_checkpoint(model, ck)
    model = checkpoint.load_checkpoint(ck)
    sysm = s.system(model, "fp64")
    sysm.use_solve_kernel(path == "solve")
    o = oracle.Oracle.from_mesh(s.mesh.vertices, s.mesh.elements, s.mesh.pinned)
    o.set_material(s.material.mu, s.material.lam, s.material.density)
    o.set_decoder([(l.W, l.b, int(l.act)) for l in model.decoder], model.norm_shift, model.norm_scale, model.r)
    cfg = P.SolverConfig(epsilon=1e-7, max_iters=1024, max_linesearch=128, lbfgs_history=5, dt=s.dt)
    steps = 40
    its = S.replay_interactions(s, steps, S.substream(1, 7))
    state = P.rest_state(s.mesh, model.r)
    opos, ovel, oz = state.positions.copy(), state.velocities.copy(), state.z.copy()
    moved = 0.0
    for step in range(steps):
        frame = S.frame_at(s, sysm.mass, its, step, state.t + s.dt)
        rep = P.reduced_step(state, frame, sysm, cfg, s.quasi_static)
        opos, ovel, oz, code, iters = o.reduced_step(opos, ovel, oz, frame.pin_positions, frame.external_force, cfg)
        assert rep.code == code, (step, rep.code, code)
        assert abs(rep.iterations - iters) <= 1, (step, rep.iterations, iters)
        assert np.max(np.abs(state.z - oz)) < 1e-6 * max(1.0, np.max(np.abs(oz))), step
        assert np.max(np.abs(state.positions - opos)) < 1e-9, step
        moved = max(moved, float(np.max(np.abs(state.z))))
    assert moved > 1e-3  # the interactions and the moving pins actually drive the subspace
    # the pinned rows follow the oscillation
    assert np.allclose(state.positions[s.mesh.pinned], S.pin_positions_at(s, state.t)[s.mesh.pinned])
