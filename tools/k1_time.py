"""Time K1 (the Fourier operator, H apply with V) -- or K2 / K3 with which = 1 / 2 -- through
acp_kernel_bench at a config's production batch width, CUDA events on the library stream; prints
one JSON line.  Also the target of the ncu --set full captures (profiles/traffic.json).
  python tools/k1_time.py <config> <ncols> [reps] [which]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import get_config  # noqa: E402
from paper_1605_08021_b200 import Context  # noqa: E402

cfg = get_config(sys.argv[1])
ncols = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
which = int(sys.argv[4]) if len(sys.argv) > 4 else 0
ctx = Context.from_config(cfg)
st = torch.cuda.Stream()
ctx.set_stream(st)
g = torch.Generator(device="cuda").manual_seed(0)
Psi = torch.randn(cfg.n_occ, cfg.n_grid, dtype=torch.float64, device="cuda", generator=g) * 0.1
V = torch.randn(cfg.n_grid, dtype=torch.float64, device="cuda", generator=g) * 0.01
X = torch.randn(ncols, cfg.n_grid, dtype=torch.float64, device="cuda", generator=g)
Y = torch.zeros_like(X)
ctx.kernel_bench(which, Psi, V, X, Y, reps)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
ctx.kernel_bench(which, Psi, V, X, Y, reps)
e1.record(st)
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / reps
byts = (16.0 if which == 0 else 8.0 if which == 1 else 24.0) * cfg.n_grid * ncols
print(json.dumps({"config": cfg.name, "which": which, "ncols": ncols, "us": us, "GBps": byts / us / 1e3,
                  "frac": byts / us / 1e3 / 6554.9, "env": {k: v for k, v in os.environ.items() if k.startswith("ACP_")}}))
