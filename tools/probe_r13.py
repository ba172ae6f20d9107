"""Oracle-side check of DESIGN.md reading R13 (configs[3], [4] as stated, eps0 = 10, are gapless).

  python tools/probe_r13.py [--sizes 3,4] [--max-iter 300] > profiles/R2_r13_oracle_probe.json

Runs the oracle's SCF (oracle.scf with the matrix-free LOBPCG eigensolver of oracle.iterative,
PAPER.md:855) on n x n square lattices with configs[3]'s parameters (spacing 10, Z = 2, sigma = 2,
kappa = 0.01, eps0 = 10, 24 points per atom per axis, doubly occupied, seeded jitter 0.2) and
records the HOMO-LUMO gap and the density residual along the way, and whether the SCF reached
1e-8.  The k-mesh of an n x n supercell contains the zone-boundary points X and M when n is even
(4 x 4, like 8 x 8 and 16 x 16), not when n is odd (3 x 3).  Calls only oracle/ and workloads/.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import atom_positions  # noqa: E402
from workloads.configs import SystemConfig  # noqa: E402
from oracle.model import Model  # noqa: E402
from oracle import iterative as oit  # noqa: E402
import oracle.scf as oscf  # noqa: E402


def run(n, max_iter, eps0):
    cfg = SystemConfig(name=f"r13_{n}x{n}_eps{eps0:g}", dim=2, n_side=n, spacing=10.0, Z=2.0, sigma=2.0, kappa=0.01,
                       eps0=eps0, grid=(24 * n, 24 * n), n_occ=n * n, occ=2.0, n_cheb=8, jitter=0.2, seed=103,
                       sketch_r=16, n_outer=2)
    m = Model(cfg, atom_positions(cfg))
    hist = []

    def ck(it, rho):
        pass

    t0 = time.time()
    # record (iteration, residual, gap) by wrapping the eigensolver (it sees every SCF iteration)
    base = oit.lobpcg_eigensolver(tol=1e-10)

    def eig(model, V, nb, X0, scf_res=0.0):
        w, X = base(model, V, nb, X0, scf_res)
        hist.append(dict(it=len(hist) + 1, prev_residual=None if not np.isfinite(scf_res) else float(scf_res),
                         gap=float(w[cfg.n_occ] - w[cfg.n_occ - 1])))
        return w, X

    converged, res = True, None
    try:
        gs = oscf.scf(m, tol=1e-8, max_iter=max_iter, eigensolver=eig)
        res = gs.residual
    except RuntimeError as e:
        converged = False
        res = float(str(e).split("residual ")[1].split(" ")[0])
    gaps = [h["gap"] for h in hist]
    tail = gaps[-20:]
    return dict(config=cfg.name, supercell=f"{n}x{n}", k_mesh_has_X_and_M=(n % 2 == 0), eps0=eps0,
                scf_converged_to_1e_8=converged, final_residual=res, iterations=len(hist),
                gap_last20_min=float(min(tail)), gap_last20_max=float(max(tail)), gap_first=gaps[0],
                residual_history=[h["prev_residual"] for h in hist][1::10], seconds=round(time.time() - t0, 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="3,4")
    ap.add_argument("--max-iter", type=int, default=300)
    ap.add_argument("--eps0", type=float, default=10.0)
    a = ap.parse_args()
    out = {"what": "DESIGN.md R13: oracle SCF on configs[3]-parameter square lattices (eps0 = %g)" % a.eps0,
           "script": "tools/probe_r13.py", "runs": []}
    for n in [int(x) for x in a.sizes.split(",")]:
        out["runs"].append(run(n, a.max_iter, a.eps0))
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
