"""Matrix-free oracle path for the full-size configs (oracle; test infrastructure only).

The dense oracle (scf.eigenpairs, response.projected_operator + LU) needs N_g x N_g matrices,
which is impossible on the 2D grids of configs[3] (N_g = 36864) and configs[4] (N_g = 65536).
This module replaces ONLY those two dense steps by the solvers the paper itself uses; every
other step (SCF mixing, SRFT sketch, QRCP, interpolation vectors, W assembly, SMW, D) is the
same oracle code (oracle.scf, oracle.acp, oracle.phonon):

* H psi = -1/2 Delta psi + V psi applied through its Fourier symbol |k|^2/2 (PAPER.md:189
  Eq. Hamil; "represented in a plane wave basis set"), by a real FFT library call
  (scipy.fft; the same multiplier convention as Model.fourier_multiply).
* Ground state: the lowest eigenpairs of H[V] by LOBPCG ("the linearized eigenvalue
  problems are solved by using the locally optimal block preconditioned conjugate gradient
  (LOBPCG) solver"; scipy.sparse.linalg.lobpcg as the library step), inside oracle.scf.scf's
  Kerker-Anderson loop.
* Sternheimer equations Q(eps~_c - H)Q zeta = Q xi (Eq. eqncompressU
  PAPER.md:622-628) by MINRES ("the use of the minimal residual method (MINRES)
  gives the best numerical performance"), written out below from Paige & Saunders'
  recurrences, batched over right-hand sides (each column runs its own scalar recurrence; the
  columns share only the operator applications), with the SPD preconditioner
  Q F^{-1} (|k|^2/2 + tau)^{-1} F Q (reading R14: it changes the iteration path only).
  Iterates stay in range(Q), i.e. the solution is the one in range(Q) (reading R3).
  Convergence is declared on the TRUE residual ||Q rhs - A zeta|| <= tol ||Q rhs||.

Pinned against the dense oracle in tests/test_oracle_iterative.py (tiny 1D and 2D systems).
"""
from __future__ import annotations

import os
import warnings

import numpy as np
import scipy.fft as sfft
from scipy.sparse.linalg import LinearOperator, lobpcg

from .model import Model

WORKERS = int(os.environ.get("ORACLE_FFT_WORKERS", os.cpu_count() or 1))


class FourierOps:
    """Real-FFT application of real-even Fourier multipliers on a model's grid."""

    def __init__(self, model: Model):
        self.m = model
        self.shape = model.shape
        self.ax = tuple(range(model.dim))
        h = self.shape[-1] // 2 + 1           # rfft keeps bins 0..n_last/2 of the last axis

        def half(mult):
            return np.ascontiguousarray(mult[..., :h])

        self.kin_h = half(0.5 * model.k2)
        self._half = half

    def multiply(self, mult_half: np.ndarray, X: np.ndarray) -> np.ndarray:
        """F^{-1} diag(mult) F X for real X (Ng,) or (Ng, n); mult given on the rfft half grid."""
        vec = X.ndim == 1
        n = 1 if vec else X.shape[1]
        A = X.reshape(self.shape + (n,))
        ax = self.ax
        F = sfft.rfftn(A, axes=ax, workers=WORKERS)
        F *= mult_half[..., None]
        out = sfft.irfftn(F, s=self.shape, axes=ax, workers=WORKERS).reshape(self.m.Ng, n)
        return out[:, 0] if vec else out

    def half(self, mult: np.ndarray) -> np.ndarray:
        return self._half(mult)

    def hamiltonian(self, V: np.ndarray, X: np.ndarray) -> np.ndarray:
        """H X = -1/2 Delta X + V X."""
        if X.ndim == 1:
            return self.multiply(self.kin_h, X) + V * X
        return self.multiply(self.kin_h, X) + V[:, None] * X


# ---------------------------------------------------------------- ground state (LOBPCG)
def lobpcg_eigensolver(tol: float = 1e-10, maxiter: int = 80, tau: float = 0.5):
    """eigensolver(model, V, nb, X0, scf_res) -> (eps, Psi) for oracle.scf.scf: the lowest nb
    eigenpairs of H[V] by LOBPCG, preconditioned by the kinetic symbol
    (|k|^2/2 + tau)^{-1}, warm-started from the previous SCF iteration's orbitals; Psi normalised
    int psi^2 = 1.  The eigen-residual target follows the SCF residual (1e-2 of it, floor tol --
    LOBPCG in fp64 stalls near 1e-11, so a floor below that only burns maxiter iterations): an
    inexact inner solve early in the SCF only changes the path to the fixed point."""

    def solve(model: Model, V: np.ndarray, nb: int, X0, scf_res=0.0):
        tol_k = max(tol, min(1e-4, 1e-2 * scf_res))
        ops = FourierOps(model)
        Ng = model.Ng
        A = LinearOperator((Ng, Ng), matvec=lambda x: ops.hamiltonian(V, x.reshape(-1)),
                           matmat=lambda X: ops.hamiltonian(V, X), dtype=np.float64)
        pre = ops.half(1.0 / (0.5 * model.k2 + tau))
        M = LinearOperator((Ng, Ng), matvec=lambda x: ops.multiply(pre, x.reshape(-1)),
                           matmat=lambda X: ops.multiply(pre, X), dtype=np.float64)
        if X0 is None:
            # seeded random block, low-pass filtered (a smooth deterministic start)
            rng = np.random.default_rng(12345)
            X0 = ops.multiply(ops.half(np.exp(-model.k2)), rng.standard_normal((Ng, nb)))
        with warnings.catch_warnings():
            # scipy warns when the residuals stall a little above tol (~1e-11 in fp64); the
            # Rayleigh-Ritz below and the SCF residual decide instead
            warnings.simplefilter("ignore", UserWarning)
            w, X = lobpcg(A, X0.copy(), M=M, tol=tol_k, maxiter=maxiter, largest=False)
        idx = np.argsort(w)
        w, X = w[idx], X[:, idx]
        # Rayleigh-Ritz once more in the converged block (orthonormal eigenvector basis)
        Q, _ = np.linalg.qr(X)
        Hs = Q.T @ ops.hamiltonian(V, Q)
        w, Y = np.linalg.eigh(0.5 * (Hs + Hs.T))
        X = Q @ Y
        return w, X / np.sqrt(model.dV)

    return solve


# ---------------------------------------------------------------- Sternheimer (MINRES)
class SternheimerMinres:
    """solve(shift, rhs) for oracle.acp.compressed_W: zeta in range(Q) with
    Q(shift - H)Q zeta = Q rhs, by preconditioned MINRES."""

    def __init__(self, model: Model, V: np.ndarray, Psi: np.ndarray, tol: float = 1e-12,
                 maxiter: int = 3000, tau: float = 0.05, block: int = 512):
        self.m = model
        self.ops = FourierOps(model)
        self.V = V
        self.Psi = Psi
        self.tol = tol
        self.maxiter = maxiter
        self.block = block
        self.pre = self.ops.half(1.0 / (0.5 * model.k2 + tau))
        self.iterations = []          # per block: MINRES steps taken

    def Q(self, X):
        """Q X = X - Psi (dV Psi^T X)."""
        return X - self.Psi @ (self.m.dV * (self.Psi.T @ X))

    def A(self, shift, X):
        """Q(shift - H)Q X for X in range(Q) -- every vector MINRES feeds here is (the right-hand
        side is Q rhs, the preconditioner's outputs are projected), so the inner Q is the identity
        on it and only the outer Q is applied (it also removes any rounding drift)."""
        return self.Q(shift * X - self.ops.hamiltonian(self.V, X))

    def Minv(self, X):
        """Q M^{-1} Q X for X in range(Q) (MINRES applies it to residuals, which are),
        M^{-1} = F^{-1} (|k|^2/2 + tau)^{-1} F: symmetric positive definite on range(Q)."""
        return self.Q(self.ops.multiply(self.pre, X))

    def __call__(self, shift: float, rhs: np.ndarray) -> np.ndarray:
        out = np.empty_like(rhs)
        for j0 in range(0, rhs.shape[1], self.block):
            j1 = min(rhs.shape[1], j0 + self.block)
            out[:, j0:j1] = self._minres(shift, self.Q(rhs[:, j0:j1]))
        return out

    def _minres(self, shift, b):
        """Paige-Saunders MINRES, one scalar recurrence per column (x0 = 0).  The working arrays
        hold the columns still iterating; converged columns leave them at the residual checks."""
        n = b.shape[1]
        eps = np.finfo(np.float64).eps
        xout = np.zeros_like(b)
        bnorm = np.linalg.norm(b, axis=0)
        cols = np.nonzero(bnorm > 0)[0]            # global column index of each working column
        if len(cols) == 0:
            self.iterations.append(0)
            return xout
        bw = b[:, cols].copy()
        x = np.zeros_like(bw)
        r1 = bw.copy()
        y = self.Minv(r1)
        beta1 = np.sqrt(np.maximum(np.einsum("ij,ij->j", r1, y), 0.0))
        oldb = np.zeros(len(cols))
        beta = beta1.copy()
        dbar = np.zeros(len(cols))
        epsln = np.zeros(len(cols))
        phibar = beta1.copy()
        cs = -np.ones(len(cols))
        sn = np.zeros(len(cols))
        w = np.zeros_like(bw)
        w2 = np.zeros_like(bw)
        r2 = r1.copy()
        itn = 0
        check_every = 10
        while len(cols) and itn < self.maxiter:
            itn += 1
            v = y / beta
            ya = self.A(shift, v)
            if itn >= 2:
                ya -= (beta / oldb) * r1
            alfa = np.einsum("ij,ij->j", v, ya)
            ya -= (alfa / beta) * r2
            r1, r2 = r2, ya
            y = self.Minv(ya)
            oldb = beta
            beta = np.sqrt(np.maximum(np.einsum("ij,ij->j", ya, y), 0.0))
            oldeps = epsln
            delta = cs * dbar + sn * alfa
            gbar = sn * dbar - cs * alfa
            epsln = sn * beta
            dbar = -cs * beta
            gamma = np.maximum(np.hypot(gbar, beta), eps)
            cs = gbar / gamma
            sn = beta / gamma
            phi = cs * phibar
            phibar = sn * phibar
            w1 = w2
            w2 = w
            w = (v - oldeps * w1 - delta * w2) / gamma
            x += phi * w
            if itn % check_every == 0 or (phibar <= 0.01 * self.tol * beta1).any():
                # stop on the true residual of the column (the recurrence's estimate is in the
                # M^{-1} norm); converged columns leave the working set
                res = np.linalg.norm(bw - self.A(shift, x), axis=0)
                done = res <= self.tol * bnorm[cols]
                if done.any():
                    xout[:, cols[done]] = x[:, done]
                    keep = ~done
                    cols = cols[keep]
                    bw, x, r1, r2, y, w, w2 = (arr[:, keep] for arr in (bw, x, r1, r2, y, w, w2))
                    beta1, oldb, beta, dbar, epsln, phibar, cs, sn = (
                        arr[keep] for arr in (beta1, oldb, beta, dbar, epsln, phibar, cs, sn))
        if len(cols):
            raise RuntimeError(f"MINRES: {len(cols)} columns not converged after {itn} iterations")
        self.iterations.append(itn)
        return xout
