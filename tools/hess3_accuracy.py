"""Accuracy of the element Hessian kernels against the oracle: relative Frobenius error of the reduced
potential Hessian on config 1 (1,536 tets, r = 8) and the config-5 problem (98,304 tets, r = 16).
Run with LSB_HESS3=0 for the D^T M' kernel."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_03807_b200 import configs  # noqa: E402
from oracle import pyoracle  # noqa: E402

for name, npts in (("c1", 12), ("c2", 3)):
    pr = configs.build(name)
    sysm = pr.system("fp32" if name == "c2" else "fp64")
    ob = pyoracle.problem(name)
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, npts)
    Z = np.concatenate([Z1, Z2])[:npts]
    H = sysm.hessian_batched(Z)
    errs = [np.linalg.norm(H[k] - ob.reduced_potential_hessian(Z[k])) / np.linalg.norm(H[k]) for k in range(npts)]
    print(f"{name}: LSB_HESS3={os.environ.get('LSB_HESS3', '1')} max rel err {max(errs):.2e} mean {np.mean(errs):.2e}")
