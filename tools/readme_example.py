"""The README usage example, runnable (python tools/readme_example.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1605_08021_b200 import Context
from workloads import get_config, atom_positions, sketch_draws
cfg = get_config("c1_1d_insulator"); R = atom_positions(cfg)
ctx = Context.from_config(cfg)
gs = ctx.ground_state(R, scf_tol=cfg.scf_tol)                       # Psi, eps, V, rho, G on the GPU
dr = [sketch_draws(cfg.seed, k, cfg.n_pert, cfg.sketch_r) for k in range(cfg.n_outer)]
th, nu = np.stack([d[0] for d in dr]), np.stack([d[1] for d in dr])  # SRFT draws per outer iteration
U, info = ctx.dyson(gs["Psi"], gs["eps"], gs["V"], gs["G"], cfg.n_cheb, cfg.n_outer, th, nu,
                    id_eps=cfg.id_eps, cg_tol=cfg.cg_tol)
D, lam = ctx.dynamical_matrix(R, gs["rho"], gs["G"], U)             # D and omega^2
print("N_mu", info["n_mu"], "lambda[:4]", lam[:4])
