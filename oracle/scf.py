"""Ground state by dense diagonalisation (oracle; test infrastructure only).

PAPER.md:186-207 (Eqs. Hamil, effV): H[rho] = -1/2 Delta + V[rho],
V[rho] = K * (rho + m) (no xc in the model),
rho = f sum_{i<=N_occ} |psi_i|^2 (f = occupation, reading R2).
PAPER.md:855 uses LOBPCG + Anderson mixing; the oracle instead diagonalises
the dense H exactly (SURVEY §7 "dense-H SCF") and mixes densities with
Anderson acceleration of a Kerker-preconditioned residual.  The
mixing scheme only changes the path to the fixed point, not the fixed point.
Forces: PAPER.md:231-243 (Eq. force).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.linalg as sla

from .model import Model


@dataclasses.dataclass
class GroundState:
    Psi: np.ndarray        # (Ng, n_occ), int psi_i psi_j = delta_ij
    eps: np.ndarray        # (n_occ + n_extra,) ascending
    rho: np.ndarray        # (Ng,)  f * sum |psi_i|^2
    V: np.ndarray          # (Ng,)  effective potential of the final H
    n_iter: int
    residual: float

    @property
    def gap(self) -> float:
        n = self.Psi.shape[1]
        return float(self.eps[n] - self.eps[n - 1])


def eigenpairs(model: Model, V: np.ndarray, n: int):
    """Lowest n eigenpairs of H[V], orbitals normalised so int psi^2 = 1."""
    H = model.hamiltonian_dense(V)
    w, X = sla.eigh(H, subset_by_index=[0, n - 1], driver="evr")
    return w, X / np.sqrt(model.dV)


def density(model: Model, Psi: np.ndarray) -> np.ndarray:
    return model.f * np.sum(Psi * Psi, axis=1)


def scf(model: Model, tol: float = 1e-12, max_iter: int = 400, n_extra: int = 4,
        rho0: np.ndarray | None = None, history: int = 12, beta: float = 0.5,
        kerker_k0: float = 0.5, verbose: bool = False, eigensolver=None, checkpoint=None) -> GroundState:
    """Self-consistent field iteration to ||rho_out - rho_in|| / ||rho_in|| <= tol.

    eigensolver(model, V, nb, X0, scf_res) -> (eps, Psi) replaces the dense diagonalisation (the
    matrix-free LOBPCG of oracle.iterative); X0 = the previous orbitals or None,
    scf_res = the previous SCF residual (inf at first), which sets how tightly it must solve.
    checkpoint(it, rho) is called every iteration (long runs save rho to resume from via rho0)."""
    m = model.pseudocharge()
    if rho0 is None:
        rho = np.clip(-m, 0.0, None)
        rho *= model.Ne / model.integrate(rho)
    else:
        rho = rho0.copy()
    k2 = model.k2
    kerker = (k2 / (k2 + kerker_k0 ** 2))
    kerker[(0,) * model.dim] = 0.0  # the k=0 residual is zero (charge conservation)

    def precond(res):
        return model.fourier_multiply(res, kerker)

    X_hist, F_hist = [], []
    nb = model.n_occ + n_extra
    err = np.inf
    for it in range(1, max_iter + 1):
        V = model.yukawa(rho + m)
        if eigensolver is None:
            eps, Psi = eigenpairs(model, V, nb)
        else:
            eps, Psi = eigensolver(model, V, nb, None if it == 1 else Psi * np.sqrt(model.dV), err)
        rho_out = density(model, Psi[:, : model.n_occ])
        res = rho_out - rho
        err = float(np.linalg.norm(res) / np.linalg.norm(rho))
        if verbose:
            print(f"scf {it:4d}  res {err:.3e}  gap {eps[model.n_occ] - eps[model.n_occ - 1]:.6f}", flush=True)
        if checkpoint:
            checkpoint(it, rho)
        if err <= tol:
            return GroundState(Psi=Psi[:, : model.n_occ].copy(), eps=eps, rho=rho_out, V=V,
                               n_iter=it, residual=err)
        f = precond(res)
        X_hist.append(rho.copy())
        F_hist.append(f.copy())
        if len(X_hist) > history + 1:
            X_hist.pop(0)
            F_hist.pop(0)
        if len(X_hist) >= 2:
            dX = np.stack([X_hist[i + 1] - X_hist[i] for i in range(len(X_hist) - 1)], 1)
            dF = np.stack([F_hist[i + 1] - F_hist[i] for i in range(len(F_hist) - 1)], 1)
            gamma, *_ = np.linalg.lstsq(dF, f, rcond=None)
            rho_new = rho + beta * f - (dX + beta * dF) @ gamma
        else:
            rho_new = rho + beta * f
        # keep total charge exact
        rho_new *= model.Ne / model.integrate(rho_new)
        rho = rho_new
    raise RuntimeError(f"SCF did not converge: residual {err:.3e} after {max_iter} iterations")


def forces(model: Model, gs: GroundState) -> np.ndarray:
    """F_{I,a} = -int g_{I,a} rho - dE_II/dR_{I,a} (Eq. force). Shape (N_A, d)."""
    G = model.G_matrix()
    F = -(G.T @ gs.rho) * model.dV
    return F.reshape(model.NA, model.dim) - model.e_ii_gradient()
