"""Probe the full-size 2D configs on the GPU: K1 accuracy/timing and the ground state (gap, SCF).

  python tools/probe_2d.py [c3_2d_8x8|c4_2d_16x16] [max_scf_iter] [eps0 override]

Prints one JSON line per config.  The oracle is used only for the cheap FFT-based
operator reference (Model.kinetic), never for the dense solvers.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import atom_positions, get_config  # noqa: E402
from paper_1605_08021_b200 import Context, AcpError  # noqa: E402
from oracle.model import Model  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3_2d_8x8"
    max_it = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    cfg = get_config(name)
    if len(sys.argv) > 3:
        import dataclasses
        cfg = dataclasses.replace(cfg, eps0=float(sys.argv[3]))
    R = atom_positions(cfg)
    ctx = Context.from_config(cfg)
    m = Model(cfg, R)
    out = {"config": name, "eps0": cfg.eps0, "N_g": m.Ng}
    rng = np.random.default_rng(0)
    X = rng.standard_normal((m.Ng, 4))
    Y = ctx.fourier_apply(torch.as_tensor(X.T.copy(), device="cuda"), 0).cpu().numpy().T
    ref = m.kinetic(X)
    out["k1_rel_err"] = float(np.abs(Y - ref).max() / np.abs(ref).max())
    G = ctx.perturbations(R).cpu().numpy().T
    Go = m.G_matrix()
    out["G_rel_err"] = float(np.abs(G - Go).max() / np.abs(Go).max())
    # K1 timing on a PCG-sized batch
    nb = 512
    Xb = torch.randn(nb, m.Ng, dtype=torch.float64, device="cuda")
    ctx.fourier_apply(Xb, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        ctx.fourier_apply(Xb, 0)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    out["k1_batch"] = nb
    out["k1_ms"] = dt * 1e3
    out["k1_GBps"] = 16.0 * m.Ng * nb / dt / 1e9
    t0 = time.perf_counter()
    try:
        gs = ctx.ground_state(R, scf_tol=cfg.scf_tol, max_scf_iter=max_it)
        out.update(scf_iter=gs["n_iter"], scf_res=gs["residual"], gap=gs["gap"],
                   eps_occ_top=float(gs["eps"][cfg.n_occ - 1]), eps=gs["eps"].cpu().numpy().tolist()[-8:])
    except AcpError as e:
        out["scf_error"] = str(e)
    out["scf_s"] = time.perf_counter() - t0
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
