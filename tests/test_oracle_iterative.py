"""Pins for oracle/iterative.py (the matrix-free path used for the full-size 2D golden runs):
every piece against the dense oracle on systems small enough for dense matrices, 1D and 2D.

The dense oracle is itself pinned (paper values, FD frozen phonon, LAPACK, closed forms), so
agreement here carries those pins over to the matrix-free path."""
import numpy as np
import pytest

from workloads import atom_positions, sketch_draws
from workloads.configs import small_config, small_config_2d
from oracle.model import Model
from oracle.scf import scf
from oracle import acp as oacp, iterative as oit, phonon as ophonon, response as ors


@pytest.fixture(scope="module", params=["tiny4", "tiny2d"])
def dense_system(request):
    cfg = small_config() if request.param == "tiny4" else small_config_2d(grid=(24, 24))
    R = atom_positions(cfg)
    m = Model(cfg, R)
    gs = scf(m, tol=1e-12)
    return cfg, R, m, gs, m.hamiltonian_dense(gs.V)


def test_fft_hamiltonian_matches_dense(dense_system):
    cfg, R, m, gs, H = dense_system
    X = np.random.default_rng(3).standard_normal((m.Ng, 5))
    ops = oit.FourierOps(m)
    assert np.abs(ops.hamiltonian(gs.V, X) - H @ X).max() < 1e-13 * np.abs(H @ X).max()
    assert np.abs(ops.multiply(ops.half(m.Khat), X) - m.yukawa(X)).max() < 1e-13 * np.abs(m.yukawa(X)).max()


def test_lobpcg_scf_matches_dense_scf(dense_system):
    """PAPER.md:855 (LOBPCG inside the SCF) reaches the dense-diagonalisation fixed point."""
    cfg, R, m, gs, H = dense_system
    gi = scf(m, tol=1e-10, eigensolver=oit.lobpcg_eigensolver(tol=1e-11))
    n = cfg.n_occ
    assert np.abs(gi.eps[: n + 1] - gs.eps[: n + 1]).max() < 1e-9
    assert np.abs(gi.rho - gs.rho).max() < 1e-8 * np.abs(gs.rho).max()
    # same occupied subspace (orbitals may rotate inside degenerate groups)
    P1 = m.dV * gi.Psi @ gi.Psi.T
    P0 = m.dV * gs.Psi @ gs.Psi.T
    assert np.abs(P1 - P0).max() < 1e-8
    assert np.abs(m.dV * gi.Psi.T @ gi.Psi - np.eye(n)).max() < 1e-12


def test_minres_sternheimer_matches_dense(dense_system):
    """Q(eps - H)Q zeta = Q rhs by MINRES vs the dense solve, at
    the extreme Chebyshev nodes (the least and most definite shifts)."""
    cfg, R, m, gs, H = dense_system
    rhs = np.random.default_rng(5).standard_normal((m.Ng, 7))
    sol = oit.SternheimerMinres(m, gs.V, gs.Psi, tol=1e-13, block=4)   # two blocks, ragged tail
    for shift in (gs.eps[0], gs.eps[cfg.n_occ - 1]):
        zd = ors.sternheimer_solve(m, H, gs.Psi, shift, rhs)
        zi = sol(shift, rhs)
        assert np.abs(zi - zd).max() < 1e-12 * np.abs(zd).max()
        assert np.abs(ors.project_Q(m, gs.Psi, zi) - zi).max() < 1e-13 * np.abs(zi).max()
    # a zero right-hand side stays zero (no division by ||b|| = 0)
    z0 = sol(gs.eps[0], np.zeros((m.Ng, 2)))
    assert not np.any(z0)


def test_minres_alg4_matches_dense_alg4(dense_system):
    """Alg. 4 + D with the MINRES solves against the dense oracle on the same ground state:
    identical discrete decisions (N_mu, pivots) and W of the first outer iteration to rounding;
    later iterations inherit the SMW core's conditioning (tiny2d: ~1e3 from rounding to Y), so
    U and D are compared at the north-star bar."""
    cfg, R, m, gs, H = dense_system
    G = m.G_matrix()
    draws = lambda k, n: sketch_draws(cfg.seed, k, n, cfg.sketch_r)  # noqa: E731
    eo = gs.eps[: cfg.n_occ]
    r1 = oacp.acp_dyson(m, H, gs.Psi, eo, G, cfg.n_cheb, cfg.n_outer, cfg.id_eps, draws)
    seen = {}
    sol = oit.SternheimerMinres(m, gs.V, gs.Psi, tol=1e-12)
    r2 = oacp.acp_dyson(m, None, gs.Psi, eo, G, cfg.n_cheb, cfg.n_outer, cfg.id_eps, draws, solve=sol,
                        keep=False, on_outer=lambda k, S, W, Y, Xi: seen.setdefault(k, W.copy()))
    assert r1.n_mu == r2.n_mu
    for a, b in zip(r1.S, r2.S):
        assert np.array_equal(a, b)
    assert np.abs(seen[0] - r1.W[0]).max() < 1e-12 * np.abs(r1.W[0]).max()
    D1 = ophonon.dynamical_matrix(m, gs.rho, G, r1.U)
    D2 = ophonon.dynamical_matrix(m, gs.rho, G, r2.U)
    assert np.abs(D2 - D1).max() < 1e-8 * np.abs(D1).max()
    assert np.abs(r2.U - r1.U).max() < 1e-8 * np.abs(r1.U).max()
