"""Dynamical matrix and phonon modes (oracle; test infrastructure only).

PAPER.md:258-273: D_{I,J} = (M_I M_J)^{-1/2} d2E_tot/dR_I dR_J, D u_k = omega_k^2 u_k.
PAPER.md:288-300 (Eq. SecDeriv): d2E/dR_I dR_J = int g_I (chi g_J) + delta_IJ int rho d2V_I
+ d2E_II; PAPER.md:309-318 (Eq. chiterm) + 376: first term = g_{I,a}^T chi g_{J,b}.
Frozen phonon: central differences of Hellmann-Feynman forces.
Masses M_I = 1 (reading R6); D is symmetrised (D + D^T)/2.
"""
from __future__ import annotations

import numpy as np

from workloads.configs import SystemConfig
from .model import Model
from .scf import GroundState, forces, scf


def dynamical_matrix(model: Model, rho: np.ndarray, G: np.ndarray, U: np.ndarray,
                     masses: np.ndarray | None = None, parts: bool = False):
    """D from U = chi G (Eq. SecDeriv).  Index (I, a) -> I*d + a."""
    d = model.dim
    n = d * model.NA
    D_chi = model.dV * (G.T @ U)
    D_loc = np.zeros((n, n))
    for I in range(model.NA):
        h = model.d2V(I)                          # (Ng, d, d)
        D_loc[I * d:(I + 1) * d, I * d:(I + 1) * d] = model.dV * np.einsum("r,rab->ab", rho, h)
    D_ii = model.e_ii_hessian()
    D = D_chi + D_loc + D_ii
    if masses is not None:
        mm = np.repeat(np.asarray(masses, dtype=np.float64), d)
        D = D / np.sqrt(np.outer(mm, mm))
    D = 0.5 * (D + D.T)
    if parts:
        return D, (D_chi, D_loc, D_ii)
    return D


def phonon_modes(D: np.ndarray):
    """lambda_k = omega_k^2 ascending, omega_k = sqrt(max(lambda,0))."""
    lam, modes = np.linalg.eigh(D)
    return lam, np.sqrt(np.clip(lam, 0.0, None)), modes


def fd_dynamical_matrix(cfg: SystemConfig, R: np.ndarray, delta: float = 1e-3,
                        gs0: GroundState | None = None, scf_tol: float = 1e-13) -> np.ndarray:
    """Frozen-phonon D_{(I,a),(J,b)} = -(F_{J,b}(R + delta e_{I,a}) - F_{J,b}(R - delta e_{I,a}))/(2 delta)."""
    R = np.asarray(R, dtype=np.float64)
    NA, d = R.shape
    D = np.zeros((d * NA, d * NA))
    rho0 = None if gs0 is None else gs0.rho
    for I in range(NA):
        for a in range(d):
            F = []
            for s in (+1.0, -1.0):
                Rs = R.copy()
                Rs[I, a] += s * delta
                m = Model(cfg, Rs)
                gs = scf(m, tol=scf_tol, rho0=rho0)
                F.append(forces(m, gs).reshape(-1))
            D[I * d + a, :] = -(F[0] - F[1]) / (2.0 * delta)
    return 0.5 * (D + D.T)
