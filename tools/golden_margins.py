"""Print the parity margins of a full-size golden run (tests/test_gpu_golden.py's loop, no asserts):
rel(W sample) per outer iteration, rel(D), lambda error.   python tools/golden_margins.py <config>"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_golden as tg  # noqa: E402
from workloads import atom_positions, get_config, sketch_draws  # noqa: E402
from oracle.model import Model  # noqa: E402
from paper_1605_08021_b200 import Context  # noqa: E402

name = sys.argv[1]
gold, gs = tg._load(name)
cfg = get_config(name)
R = atom_positions(cfg)
G = Model(cfg, R).G_matrix()
ctx = Context.from_config(cfg)
T = tg.T
Psi_t, eps_t, V_t, rho_t, G_t = T(gs["Psi"].T), T(gs["eps"]), T(gs["V"]), T(gs["rho"]), T(G.T)
n = G.shape[1]
Gp = G_t.clone()
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("ACP_")}, "W": []}
for k in range(cfg.n_outer):
    th, nu = sketch_draws(cfg.seed, k, n, cfg.sketch_r)
    S, Xi, nk = ctx.compress(Psi_t, Gp, th, nu, id_eps=cfg.id_eps)
    W, info = ctx.apply_chi0(Psi_t, eps_t, V_t, S, Xi, cfg.n_cheb, cg_tol=cfg.cg_tol)
    Ws = W[torch.as_tensor(gold[f"W{k}_idx"], device="cuda")].cpu().numpy().T
    out["W"].append(float(tg.rel(Ws, gold[f"W{k}"])))
    U, Gp = ctx.smw_update(G_t, S, W)
D, lam = ctx.dynamical_matrix(R, rho_t, G_t, U)
out["D"] = float(tg.rel(D, gold["D"]))
out["lam"] = float(np.abs(lam - gold["lam"]).max() / np.abs(gold["lam"]).max())
print(out)
