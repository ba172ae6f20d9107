"""Write the oracle's end-to-end results for one full-size config (calls only oracle/ + workloads/).

  python tools/make_golden.py <config> [--outer-only 1]

Produces
  tests/golden/<config>_gs.npz     the oracle's ground state (Psi, eps, V, rho) -- the INPUT the GPU
                                   parity test feeds to the CUDA path; committed when Psi is at most
                                   GS_COMMIT_MAX bytes (configs[2], c3g), else tests/cache/ (c4g:
                                   134 MB, git-ignored)
  tests/golden/<config>_acp.npz    the oracle's Alg. 4 + D results on that input (committed):
                                   per-outer N_mu, pivots S, ||U^k - U^{k-1}||, W on a seeded
                                   mu-sample, D, lambda, and a digest of the input arrays

Dense path (oracle.scf dense SCF, dense compressed solves) when N_g <= 6000 (configs[0..2]);
matrix-free path (oracle.iterative: LOBPCG SCF, MINRES Sternheimer) beyond (the 2D configs),
pinned to the dense one in tests/test_oracle_iterative.py.  Nothing here reads the CUDA path.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from workloads import atom_positions, get_config, sketch_draws  # noqa: E402
from oracle.model import Model  # noqa: E402
from oracle.scf import scf  # noqa: E402
from oracle import acp as oacp, iterative as oit, phonon as ophonon  # noqa: E402

DENSE_MAX_NG = 6000
N_W_SAMPLE = 6        # mu-columns of W stored per outer iteration
N_XI = 32             # interpolation vectors of outer 0 kept for bench.py's oracle sample
GS_COMMIT_MAX = 32 << 20   # ground states up to this size go to tests/golden/ (tracked)


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def w_sample(n_mu: int, k: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng([seed, 7000 + k])
    return np.sort(rng.choice(n_mu, size=min(N_W_SAMPLE, n_mu), replace=False))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--minres-tol", type=float, default=1e-12)
    ap.add_argument("--scf-tol", type=float, default=None)
    ap.add_argument("--minres-block", type=int, default=64)
    ap.add_argument("--resume-res", type=float, default=None,
                    help="SCF residual of the checkpointed density: sets the first LOBPCG tolerance on resume "
                         "(otherwise the loose first-iteration one)")
    ap.add_argument("--gs-only", action="store_true",
                    help="(re)build the cached ground state (+ outer 0's interpolation vectors for bench.py) and "
                         "check it against the committed golden file's input digest; no Alg. 4")
    ap.add_argument("--outer-only", type=int, default=0,
                    help="1: outer iteration 0 only -- pivots, N_mu and W on the mu-sample (configs[4]: "
                         "the ~85k MINRES solves of the full Alg. 4 are days of CPU)")
    a = ap.parse_args()
    cfg = get_config(a.config)
    cache = os.path.join(ROOT, "tests", "cache")
    gold = os.path.join(ROOT, "tests", "golden")
    os.makedirs(cache, exist_ok=True)
    t_start = time.time()

    def log(msg):
        print(f"[{time.time() - t_start:8.1f} s] {cfg.name}: {msg}", flush=True)

    R = atom_positions(cfg)
    m = Model(cfg, R)
    dense = m.Ng <= DENSE_MAX_NG
    small = m.Ng * cfg.n_occ * 8 <= GS_COMMIT_MAX
    gs_path = os.path.join(gold if small else cache, f"{cfg.name}_gs.npz")
    if not os.path.exists(gs_path) and os.path.exists(os.path.join(cache, f"{cfg.name}_gs.npz")):
        gs_path = os.path.join(cache, f"{cfg.name}_gs.npz")
    if os.path.exists(gs_path):
        z = np.load(gs_path)
        Psi, eps, V, rho = z["Psi"], z["eps"], z["V"], z["rho"]
        assert np.array_equal(z["R"], R), "cached ground state is for other positions"
        log(f"ground state from cache (residual {float(z['residual']):.2e})")
    else:
        if dense:
            gs = scf(m, tol=a.scf_tol or cfg.scf_tol, verbose=True)
        else:
            # both sides of the parity test consume these same arrays, so the SCF tolerance only
            # sets how close they are to the self-consistent state, not the parity (R16)
            ck = os.path.join(cache, f"{cfg.name}_scf_rho.npy")
            rho0 = np.load(ck) if os.path.exists(ck) else None
            if rho0 is not None:
                log("resuming the SCF from the checkpointed density")
            es = oit.lobpcg_eigensolver(tol=1e-10)
            if rho0 is not None and a.resume_res:
                base = es

                def es(model, V, nb, X0, scf_res=0.0):  # noqa: F811
                    return base(model, V, nb, X0, scf_res if np.isfinite(scf_res) else a.resume_res)
            gs = scf(m, tol=a.scf_tol or 1e-9, eigensolver=es, verbose=True,
                     rho0=rho0, checkpoint=lambda it, rho: np.save(ck, rho) if it % 5 == 0 else None)
        Psi, eps, V, rho = gs.Psi, gs.eps, gs.V, gs.rho
        gs_path = os.path.join(gold if small else cache, f"{cfg.name}_gs.npz")
        np.savez(gs_path, Psi=Psi, eps=eps, V=V, rho=rho, R=R, residual=gs.residual, n_iter=gs.n_iter)
        log(f"ground state: {gs.n_iter} SCF iterations, residual {gs.residual:.2e}, gap {gs.gap:.6f}")
    n_occ = cfg.n_occ
    G = m.G_matrix()
    if a.gs_only:
        dg = digest(Psi, eps, V, rho, R)
        gp = os.path.join(gold, f"{cfg.name}_acp.npz")
        if os.path.exists(gp):
            want = str(np.load(gp)["input_digest"])
            log(f"input digest {dg} vs golden {want}: {'MATCH' if dg == want else 'MISMATCH'}")
        th, nu = sketch_draws(cfg.seed, 0, G.shape[1], cfg.sketch_r)
        S, Xi, _ = oacp.compress(m, Psi, G, th, nu, cfg.id_eps)
        np.savez(os.path.join(cache, f"{cfg.name}_xi0.npz"), Xi=np.ascontiguousarray(Xi[:, :N_XI]),
                 S=np.asarray(S[:N_XI]))
        log(f"outer 0 interpolation vectors cached (N_mu = {len(S)})")
        return
    H = m.hamiltonian_dense(V) if dense else None
    solve = None if dense else oit.SternheimerMinres(m, V, Psi, tol=a.minres_tol, block=a.minres_block)
    samples = {}

    def on_outer(k, S, W, Y, Xi):
        idx = w_sample(len(S), k, cfg.seed)
        samples[k] = (idx, W[:, idx].copy())
        if k == 0:
            # interpolation vectors of outer iteration 0 for the oracle's timed sample in bench.py
            # (cpu_baseline / --impl reference on the grids where the dense oracle cannot run)
            np.savez(os.path.join(cache, f"{cfg.name}_xi0.npz"), Xi=np.ascontiguousarray(Xi[:, :N_XI]),
                     S=np.asarray(S[:N_XI]))

    draws = lambda k, n: sketch_draws(cfg.seed, k, n, cfg.sketch_r)  # noqa: E731
    if a.outer_only:
        # Alg. 2 on G' = G (outer 0), then Eq. eqncompressU + Eq. eqnW for the
        # sampled mu only: W's columns are independent (each solves its own right-hand sides)
        th, nu = draws(0, G.shape[1])
        S, Xi, _ = oacp.compress(m, Psi, G, th, nu, cfg.id_eps)
        log(f"outer 0: N_mu = {len(S)}")
        np.savez(os.path.join(cache, f"{cfg.name}_xi0.npz"), Xi=np.ascontiguousarray(Xi[:, :N_XI]),
                 S=np.asarray(S[:N_XI]))
        idx = w_sample(len(S), 0, cfg.seed)
        W0 = oacp.compressed_W(m, H, Psi, eps[:n_occ], S[idx], np.ascontiguousarray(Xi[:, idx]), cfg.n_cheb,
                               solve=solve)
        out = dict(n_mu=np.asarray([len(S)]), S=np.asarray(S, dtype=np.int64), W0_idx=idx, W0=W0,
                   input_digest=digest(Psi, eps, V, rho, R),
                   meta=json.dumps(dict(config=cfg.name, outer_only=1,
                                        path="dense" if dense else "matrix-free (LOBPCG + MINRES)",
                                        minres_tol=None if dense else a.minres_tol,
                                        seconds=round(time.time() - t_start, 1), script="tools/make_golden.py")))
        np.savez_compressed(os.path.join(gold, f"{cfg.name}_acp.npz"), **out)
        log("written (outer 0 only)")
        return
    res = oacp.acp_dyson(m, H, Psi, eps[:n_occ], G, cfg.n_cheb, cfg.n_outer, cfg.id_eps, draws,
                         solve=solve, keep=False, log=log, on_outer=on_outer)
    D = ophonon.dynamical_matrix(m, rho, G, res.U)
    lam = np.linalg.eigvalsh(D)
    log(f"D done: max|D| {np.abs(D).max():.4e}, lambda [{lam[0]:.3e}, {lam[-1]:.3e}]")
    out = dict(
        D=D, lam=lam, n_mu=np.asarray(res.n_mu), diff=np.asarray(res.diff),
        S=np.concatenate(res.S).astype(np.int64), U_norm=np.linalg.norm(res.U),
        input_digest=digest(Psi, eps, V, rho, R),
        meta=json.dumps(dict(config=cfg.name, path="dense" if dense else "matrix-free (LOBPCG + MINRES)",
                             minres_tol=None if dense else a.minres_tol,
                             minres_iterations=None if dense else [int(x) for x in solve.iterations],
                             seconds=round(time.time() - t_start, 1), script="tools/make_golden.py")))
    for k, (idx, Ws) in samples.items():
        out[f"W{k}_idx"] = idx
        out[f"W{k}"] = Ws
    np.savez_compressed(os.path.join(gold, f"{cfg.name}_acp.npz"), **out)
    log("written")


if __name__ == "__main__":
    main()
