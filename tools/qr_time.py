"""Time acp_compress (Alg. 2) on a config's GPU ground state: the structured Kronecker QRCP
(default) vs the formed-sketch persistent kernel (ACP_QRCP_DENSE=1 in the environment).
  python tools/qr_time.py <config> [reps]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import atom_positions, get_config, sketch_draws  # noqa: E402
from paper_1605_08021_b200 import Context  # noqa: E402

cfg = get_config(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = Context.from_config(cfg)
R = atom_positions(cfg)
gs = ctx.ground_state(R, scf_tol=max(cfg.scf_tol, 1e-10))
th, nu = sketch_draws(cfg.seed, 0, cfg.n_pert, cfg.sketch_r)
S, Xi, n = ctx.compress(gs["Psi"], gs["G"], th, nu, id_eps=cfg.id_eps)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    S, Xi, n = ctx.compress(gs["Psi"], gs["G"], th, nu, id_eps=cfg.id_eps)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(json.dumps({"config": cfg.name, "n_mu": n, "ms": 1e3 * min(ts), "dense": bool(os.environ.get("ACP_QRCP_DENSE")),
                  "S_head": [int(x) for x in S[:8].cpu()], "S_sum": int(S.sum().item())}))
