"""Per-phase clock64 profile of the cluster QRCP on a config (ACP_QR_PROFILE), for tuning."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import atom_positions, get_config, sketch_draws  # noqa: E402
from paper_1605_08021_b200 import Context  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "c1_1d_insulator")
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/qr_prof.txt"
ctx = Context.from_config(cfg)
R = atom_positions(cfg)
gs = ctx.ground_state(R, scf_tol=cfg.scf_tol)
th, nu = sketch_draws(cfg.seed, 0, cfg.n_pert, cfg.sketch_r)
ctx.compress(gs["Psi"], gs["G"], th, nu, id_eps=cfg.id_eps)
if os.path.exists(out):
    os.unlink(out)
os.environ["ACP_QR_PROFILE"] = out
torch.cuda.synchronize()
S, Xi, n = ctx.compress(gs["Psi"], gs["G"], th, nu, id_eps=cfg.id_eps)
t = np.loadtxt(out)
t = t[(t > 0).all(axis=1)]  # drop the exit step (unfinished phases)
d = np.diff(t, axis=1)
step = np.diff(t[:, 0])
print("N_mu", n, "steps", len(t))
print("mean cycles per phase [local argmax+push | syncthreads | publish | cl.sync | winner+exit test | v from DSMEM | update]:", d.mean(0).round(0))
print("mean cycles per step:", step.mean().round(0), " -> us per step at 1.9 GHz:", (step.mean() / 1.9e3).round(2))
