"""Launch one hot kernel of the CUDA path on synthetic inputs (for ncu captures).

  python profiles/kernel_probe.py --which 0|1|2 [--config c1_1d_insulator] [--ncols 928] [--reps 3]

which: 0 = K1 Fourier operator (H apply), 1 = K2 DMMA projection Psi^T Y, 2 = K3 fused update.
Inputs are seeded random arrays of the workload's shapes (no oracle, no ground state).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import get_config  # noqa: E402
from paper_1605_08021_b200 import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", type=int, default=0)
ap.add_argument("--config", default="c1_1d_insulator")
ap.add_argument("--ncols", type=int, default=928)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = get_config(a.config)
ctx = Context.from_config(cfg)
g = torch.Generator(device="cuda").manual_seed(0)
Psi = torch.randn(cfg.n_occ, cfg.n_grid, dtype=torch.float64, device="cuda", generator=g) * 0.1
V = torch.randn(cfg.n_grid, dtype=torch.float64, device="cuda", generator=g) * 0.01
X = torch.randn(a.ncols, cfg.n_grid, dtype=torch.float64, device="cuda", generator=g)
Y = torch.zeros_like(X)
ctx.kernel_bench(a.which, Psi, V, X, Y, a.reps)
torch.cuda.synchronize()
print("ok", a.which, cfg.name, a.ncols, float(Y.abs().sum()))
