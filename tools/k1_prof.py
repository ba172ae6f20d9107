"""Debug: one K1 launch through acp_fourier_apply (not graph-captured), for ACP_F2C_PROF."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import get_config  # noqa: E402
from paper_1605_08021_b200 import Context  # noqa: E402

cfg = get_config(sys.argv[1])
ncols = int(sys.argv[2])
ctx = Context.from_config(cfg)
X = torch.randn(ncols, cfg.n_grid, dtype=torch.float64, device="cuda")
V = torch.randn(cfg.n_grid, dtype=torch.float64, device="cuda") * 0.01
for _ in range(3):
    ctx.fourier_apply(X, 0, diag=V)
torch.cuda.synchronize()
print("ok")
