"""Discretised model of PAPER §2.1 and §4.1 (oracle; test infrastructure only).

Conventions (readings R1-R4):
  * Periodic cell of lengths L_a, uniform grid, grid functions
    stored flattened in C order (index alpha = i0*n1 + i1 in 2D).
  * A function f with continuous Fourier coefficients fhat(k) = int_cell f e^{-ikr}
    has grid values f(r_alpha) = (1/Omega) sum_k fhat(k) e^{ik r_alpha}
    (band-limited to the grid frequencies).
  * Yukawa kernel K(x,y) = 2 pi e^{-kappa|x-y|}/(kappa eps0) (PAPER.md:836,
    Eq. yukawa) has symbol Khat(k) = 4 pi / (eps0 (|k|^2 + kappa^2)); the
    same symbol defines the 2D kernel.
  * Gaussian pseudocharge m_I(x) = -Z/(2 pi sigma^2)^{d/2} e^{-|x|^2/(2 sigma^2)}
    (PAPER.md:830 for d=1), so mhat_I(k) = -Z e^{-sigma^2 |k|^2 / 2} and
    int m_I = -Z.
  * V_I = v_c * m_I (Eq. pseudocharge); g_{I,a} = dV_I/dR_{I,a}
     has coefficients -i k_a Khat mhat e^{-ik.R_I}; the second
    derivative d2V_I/dR_a dR_b has (-i k_a)(-i k_b) Khat mhat e^{-ik.R_I}.
    Odd (first-derivative) multipliers use k_a with the Nyquist entry zeroed so
    that real functions stay real.
  * E_II ("also computed using the Yukawa interaction K"): the
    smeared-pseudocharge interaction 1/2 sum_{I!=J} int int m_I K m_J
    (SPEC.md:272), i.e. 1/2 sum_{I!=J} phi(R_I - R_J) with
    phi(d) = (1/Omega) sum_k Khat mhat^2 cos(k.d).
"""
from __future__ import annotations

import numpy as np

from workloads.configs import SystemConfig


class Model:
    """Grid + atoms + kernel for one configuration (all fp64)."""

    def __init__(self, cfg: SystemConfig, R: np.ndarray):
        self.cfg = cfg
        self.dim = cfg.dim
        self.shape = tuple(cfg.grid)
        self.L = np.asarray(cfg.cell, dtype=np.float64)
        self.Ng = int(np.prod(self.shape))
        self.Omega = float(np.prod(self.L))
        self.dV = self.Omega / self.Ng
        self.R = np.asarray(R, dtype=np.float64).reshape(-1, self.dim)
        self.NA = self.R.shape[0]
        self.Z = float(cfg.Z)
        self.f = float(cfg.occ)
        self.n_occ = cfg.n_occ
        self.Ne = self.Z * self.NA
        # Fourier frequencies per axis, broadcast to grid shape (numpy fft order).
        ks = []
        for a in range(self.dim):
            m = np.fft.fftfreq(self.shape[a], d=1.0 / self.shape[a])  # integers
            k1 = 2.0 * np.pi * m / self.L[a]
            shp = [1] * self.dim
            shp[a] = self.shape[a]
            ks.append(np.broadcast_to(k1.reshape(shp), self.shape).copy())
        self.k = ks                                  # list of arrays (grid shape)
        self.k2 = sum(ka * ka for ka in ks)
        kodd = []
        for a in range(self.dim):
            ka = ks[a].copy()
            if self.shape[a] % 2 == 0:
                idx = [slice(None)] * self.dim
                idx[a] = self.shape[a] // 2
                ka[tuple(idx)] = 0.0
            kodd.append(ka)
        self.kodd = kodd
        self.Khat = 4.0 * np.pi / (cfg.eps0 * (self.k2 + cfg.kappa ** 2))
        self.mhat0 = -self.Z * np.exp(-0.5 * cfg.sigma ** 2 * self.k2)
        # real-space coordinates (flattened grid, (Ng, d))
        axes = [np.arange(n) * (self.L[a] / n) for a, n in enumerate(self.shape)]
        mesh = np.meshgrid(*axes, indexing="ij")
        self.r = np.stack([x.reshape(-1) for x in mesh], axis=1)

    # -- Fourier helpers -------------------------------------------------
    def from_fourier(self, fhat: np.ndarray) -> np.ndarray:
        """Grid values of the function with continuous coefficients fhat (flattened)."""
        out = np.fft.ifftn(fhat, axes=tuple(range(self.dim))) * (self.Ng / self.Omega)
        return np.real(out).reshape(-1)

    def phase(self, I: int) -> np.ndarray:
        kr = sum(self.k[a] * self.R[I, a] for a in range(self.dim))
        return np.exp(-1j * kr)

    def fourier_multiply(self, f: np.ndarray, mult: np.ndarray) -> np.ndarray:
        """Apply a Fourier multiplier to grid vector(s) f (Ng,) or (Ng, n)."""
        f = np.asarray(f)
        vec = f.ndim == 1
        F = f.reshape(self.shape + ((1,) if vec else (f.shape[1],)))
        ax = tuple(range(self.dim))
        out = np.fft.ifftn(np.fft.fftn(F, axes=ax) * mult[..., None], axes=ax)
        out = np.real(out).reshape(self.Ng, -1)
        return out[:, 0] if vec else out

    # -- Yukawa kernel (Eq. yukawa) -----
    def yukawa(self, f: np.ndarray) -> np.ndarray:
        """v = K * f, i.e. (K f)(r) = int K(r, r') f(r') dr'."""
        return self.fourier_multiply(f, self.Khat)

    def yukawa_inverse(self, v: np.ndarray) -> np.ndarray:
        """B = v_hxc^{-1} G: inverse symbol, exact for kappa > 0."""
        return self.fourier_multiply(v, 1.0 / self.Khat)

    def kinetic(self, f: np.ndarray) -> np.ndarray:
        """-1/2 Laplacian via the Fourier symbol |k|^2/2 (Eq. Hamil)."""
        return self.fourier_multiply(f, 0.5 * self.k2)

    # -- pseudocharges and potentials ---------
    def pseudocharge(self, I: int | None = None) -> np.ndarray:
        if I is None:
            return sum(self.pseudocharge(J) for J in range(self.NA))
        return self.from_fourier(self.mhat0 * self.phase(I))

    def v_ion(self) -> np.ndarray:
        """V_ion = sum_I V_I(r - R_I), V_I = v_c * m_I (Eq. pseudocharge)."""
        tot = sum(self.mhat0 * self.phase(I) for I in range(self.NA))
        return self.from_fourier(self.Khat * tot)

    def G_matrix(self) -> np.ndarray:
        """G = [g_1 ... g_{dN_A}], g_{I,a} = dV_I/dR_{I,a}.

        Column order: j = I*d + a.
        """
        cols = []
        for I in range(self.NA):
            base = self.Khat * self.mhat0 * self.phase(I)
            for a in range(self.dim):
                cols.append(self.from_fourier(-1j * self.kodd[a] * base))
        return np.stack(cols, axis=1)

    def d2V(self, I: int) -> np.ndarray:
        """d2 V_I(r-R_I)/dR_{I,a} dR_{I,b} as an (Ng, d, d) array (Eq. SecDeriv 2nd term)."""
        base = self.Khat * self.mhat0 * self.phase(I)
        out = np.empty((self.Ng, self.dim, self.dim))
        for a in range(self.dim):
            for b in range(self.dim):
                out[:, a, b] = self.from_fourier(
                    (-1j * self.kodd[a]) * (-1j * self.kodd[b]) * base)
        return out

    # -- ion-ion term (reading R4) ------------------
    def _phi_coeff(self) -> np.ndarray:
        return (self.Khat * self.mhat0 ** 2 / self.Omega).reshape(-1)

    def e_ii(self) -> float:
        c = self._phi_coeff()
        kf = [ka.reshape(-1) for ka in self.k]
        e = 0.0
        for I in range(self.NA):
            for J in range(self.NA):
                if I == J:
                    continue
                d = self.R[I] - self.R[J]
                kd = sum(kf[a] * d[a] for a in range(self.dim))
                e += 0.5 * float(np.sum(c * np.cos(kd)))
        return e

    def e_ii_gradient(self) -> np.ndarray:
        """dE_II/dR_{I,a}, shape (N_A, d)."""
        c = self._phi_coeff()
        kf = [ka.reshape(-1) for ka in self.k]
        out = np.zeros((self.NA, self.dim))
        for I in range(self.NA):
            for J in range(self.NA):
                if I == J:
                    continue
                d = self.R[I] - self.R[J]
                kd = sum(kf[a] * d[a] for a in range(self.dim))
                s = np.sin(kd)
                for a in range(self.dim):
                    out[I, a] += -float(np.sum(c * kf[a] * s))
        return out

    def e_ii_hessian(self) -> np.ndarray:
        """d2E_II/dR_{I,a} dR_{J,b}, shape (dN_A, dN_A), index I*d + a (Eq. SecDeriv 3rd term)."""
        c = self._phi_coeff()
        kf = [ka.reshape(-1) for ka in self.k]
        d_ = self.dim
        H = np.zeros((d_ * self.NA, d_ * self.NA))
        for I in range(self.NA):
            for J in range(self.NA):
                if I == J:
                    continue
                dvec = self.R[I] - self.R[J]
                kd = sum(kf[a] * dvec[a] for a in range(d_))
                cs = np.cos(kd)
                for a in range(d_):
                    for b in range(d_):
                        # phi''_ab(d) = -(1/Omega) sum Khat mhat^2 k_a k_b cos(k.d)
                        h = -float(np.sum(c * kf[a] * kf[b] * cs))
                        H[I * d_ + a, J * d_ + b] -= h
                        H[I * d_ + a, I * d_ + b] += h
        return H

    # -- dense operators (oracle-only) ------------------------------------
    def dense_fourier_operator(self, mult: np.ndarray) -> np.ndarray:
        """Dense N_g x N_g matrix of a Fourier multiplier acting on grid vectors."""
        return self.fourier_multiply(np.eye(self.Ng), mult)

    def hamiltonian_dense(self, V: np.ndarray) -> np.ndarray:
        """H = -1/2 Delta + V as a dense symmetric matrix."""
        H = self.dense_fourier_operator(0.5 * self.k2)
        H = 0.5 * (H + H.T)
        H[np.diag_indices(self.Ng)] += V
        return H

    def integrate(self, f: np.ndarray) -> float:
        return float(np.sum(f) * self.dV)
