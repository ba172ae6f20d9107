"""Linear response of PAPER §2.2 (oracle; test infrastructure only).

* Q = I - sum_i psi_i psi_i^T; on the grid with int psi^2 = 1,
  Q v = v - Psi (dV Psi^T v).
* Sternheimer: Q(eps - H)Q zeta = Q rhs.  Q(eps-H)Q is
  singular on range(I-Q); the oracle solves the nonsingular
  (Q(eps-H)Q - P) zeta = Q rhs, P = I - Q, whose solution lies in range(Q)
  (SPEC.md:350 reading), by dense LU.
* chi0 g = 2 f sum_i psi_i (.) Q(eps_i - H)^{-1} Q(psi_i (.) g) (PAPER.md:410-416,
  Eq. Sternheimer; Alg. 1).  The paper's factor 2 is for
  rho = sum psi^2; with occupation f the prefactor is 2f (reading R2).
* Adler-Wiser: chi0(r,r') = 2f sum_i sum_{a>N}
  psi_i psi_a psi_i' psi_a' / (eps_i - eps_a), from the full eigendecomposition.
* Dyson: chi = (I - chi0 v_hxc)^{-1} chi0, v_hxc = K (no f_xc).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .model import Model


def project_Q(model: Model, Psi: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Q v = v - Psi (dV Psi^T v)."""
    return v - Psi @ (model.dV * (Psi.T @ v))


def projected_operator(model: Model, H: np.ndarray, Psi: np.ndarray, shift: float) -> np.ndarray:
    """Dense (Q(shift - H)Q - P) with P = dV Psi Psi^T (SPEC.md:350 reading)."""
    Ng = model.Ng
    P = model.dV * (Psi @ Psi.T)
    Q = np.eye(Ng) - P
    A = Q @ (shift * np.eye(Ng) - H) @ Q - P
    return A


def sternheimer_solve(model: Model, H: np.ndarray, Psi: np.ndarray, shift: float,
                      rhs: np.ndarray) -> np.ndarray:
    """zeta with Q(shift - H)Q zeta = Q rhs, zeta in range(Q)."""
    A = projected_operator(model, H, Psi, shift)
    return np.linalg.solve(A, project_Q(model, Psi, rhs))


def chi0_apply(model: Model, H: np.ndarray, Psi: np.ndarray, eps: np.ndarray,
               G: np.ndarray) -> np.ndarray:
    """Alg. 1 for every column of G: u = 2f sum_i psi_i (.) zeta_i."""
    G = np.atleast_2d(G.T).T
    U = np.zeros_like(G)
    for i in range(Psi.shape[1]):
        A = projected_operator(model, H, Psi, eps[i])
        lu = sla.lu_factor(A)
        rhs = project_Q(model, Psi, Psi[:, i:i + 1] * G)
        zeta = sla.lu_solve(lu, rhs)
        U += 2.0 * model.f * Psi[:, i:i + 1] * zeta
    return U


def chi0_adler_wiser_matrix(model: Model, H: np.ndarray, n_occ: int) -> np.ndarray:
    """Operator matrix of chi0 from Eq. AdlerWiser, acting on grid vectors.

    (chi0 g)(r) = int chi0(r, r') g(r') dr' = dV * sum_r' chi0(r, r') g(r').
    """
    w, X = sla.eigh(H)
    Phi = X / np.sqrt(model.dV)
    occ, vir = Phi[:, :n_occ], Phi[:, n_occ:]
    C = np.zeros((model.Ng, model.Ng))
    for i in range(n_occ):
        Pij = occ[:, i:i + 1] * vir                      # psi_i psi_a, (Ng, Nvir)
        C += (Pij / (w[i] - w[n_occ:])) @ Pij.T
    return 2.0 * model.f * C * model.dV


def yukawa_matrix(model: Model) -> np.ndarray:
    """Operator matrix of v_hxc = K (Fourier symbol Khat)."""
    Kmat = model.dense_fourier_operator(model.Khat)
    return 0.5 * (Kmat + Kmat.T)


def dyson_dense(model: Model, chi0_mat: np.ndarray, G: np.ndarray) -> np.ndarray:
    """U = chi G = (I - chi0 v_hxc)^{-1} chi0 G (Eq. chi)."""
    Kmat = yukawa_matrix(model)
    A = np.eye(model.Ng) - chi0_mat @ Kmat
    return np.linalg.solve(A, chi0_mat @ G)


def dyson_dfpt(model: Model, H: np.ndarray, Psi: np.ndarray, eps: np.ndarray,
               G: np.ndarray) -> np.ndarray:
    """Exact chi G with chi0 applied by Alg. 1 (direct Sternheimer solves).

    The Dyson fixed point u = chi0 g + chi0 v u is solved
    exactly by assembling chi0 as an operator matrix column-by-column via
    Alg. 1 (N_g applications) and a dense solve; used for tiny systems only.
    """
    C0 = chi0_apply(model, H, Psi, eps, np.eye(model.Ng))
    return dyson_dense(model, C0, G)


def sternheimer_free_electron(model: Model, occ_mask: np.ndarray, shift: float, rhs: np.ndarray) -> np.ndarray:
    """Closed form of Q(shift - H)Q zeta = Q rhs for the free-electron case V = 0
    with the occupied orbitals = the plane waves of a complete shell set (occ_mask over the FFT
    bins, True = occupied).  H = -1/2 Laplacian is diagonal in Fourier space and Q removes the
    occupied bins, so zeta^(k) = rhs^(k) / (shift - |k|^2/2) on unoccupied bins and 0 on
    occupied ones (the solution in range(Q)).  Used as a full-grid pin (no dense matrices)."""
    with np.errstate(divide="ignore"):
        mult = np.where(occ_mask, 0.0, 1.0 / (shift - 0.5 * model.k2))
    return model.fourier_multiply(rhs, mult)
