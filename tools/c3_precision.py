"""Diagnose config-3 step 1 in fp64 vs fp32 (device-resident solver)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402
import paper_2409_03807_b200 as P  # noqa: E402

pr = configs.build("c3")
for prec in sys.argv[1:] or ["fp64", "fp32"]:
    sysm = pr.system(prec)
    st = pr.initial_state()
    sysm.set_state(st)
    sysm.set_external_force(P.gravity_force(pr.mesh, sysm.mass, configs.GRAVITY))
    cfg = configs.solver_config()
    cfg.max_iters = 200
    reps, zt = sysm.simulate(2, cfg)
    print(prec, [(r.code, r.iterations, r.value_evals, r.grad_evals, r.final_grad_inf_norm, round(r.wall_time_ms, 2)) for r in reps])
    print("  z1", np.round(zt[0][:6], 6))
    # energy along the first step's path
    q0 = P.dof_pack(pr.mesh, st.positions)
    v0 = P.dof_pack(pr.mesh, st.velocities)
    qbar = q0 + configs.DT * v0 + configs.DT ** 2 * np.tile(configs.GRAVITY, pr.mesh.num_free_vertices())
    sysm.set_inertia(qbar, configs.DT)
    E0, g0 = sysm.eval(np.zeros(pr.model.r))
    E1, g1 = sysm.eval(zt[0])
    print(f"  E(0)={E0:.12e} |g0|inf={np.abs(g0).max():.3e}  E(z1)={E1:.12e} |g1|inf={np.abs(g1).max():.3e}")
    sysm.close()
