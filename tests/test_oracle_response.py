"""Pins for oracle/response.py: Sternheimer vs Adler-Wiser, chi0 invariants, Dyson."""
import numpy as np

from oracle import response as rs


def test_projector(tiny_system):
    cfg, R, m, gs = tiny_system
    v = np.random.default_rng(1).standard_normal(m.Ng)
    Qv = rs.project_Q(m, gs.Psi, v)
    assert np.abs(rs.project_Q(m, gs.Psi, Qv) - Qv).max() < 1e-12
    assert np.abs(m.dV * gs.Psi.T @ Qv).max() < 1e-12
    assert np.abs(rs.project_Q(m, gs.Psi, gs.Psi[:, 0])).max() < 1e-12


def test_sternheimer_vs_adler_wiser(tiny_system):
    """Eq. Sternheimer == Eq. AdlerWiser with full spectrum."""
    cfg, R, m, gs = tiny_system
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    C0 = rs.chi0_adler_wiser_matrix(m, H, cfg.n_occ)
    U1 = rs.chi0_apply(m, H, gs.Psi, gs.eps, G)
    assert np.abs(C0 @ G - U1).max() < 1e-11 * np.abs(U1).max()


def test_sternheimer_single_solve_vs_pseudoinverse(tiny_system):
    cfg, R, m, gs = tiny_system
    H = m.hamiltonian_dense(gs.V)
    rhs = np.random.default_rng(2).standard_normal(m.Ng)
    shift = 0.5 * (gs.eps[0] + gs.eps[cfg.n_occ - 1])
    z = rs.sternheimer_solve(m, H, gs.Psi, shift, rhs)
    Q = np.eye(m.Ng) - m.dV * gs.Psi @ gs.Psi.T
    A = Q @ (shift * np.eye(m.Ng) - H) @ Q
    zp = np.linalg.pinv(A, rcond=1e-10) @ (Q @ rhs)
    assert np.abs(z - zp).max() < 1e-9 * np.abs(zp).max()
    assert np.abs(A @ z - Q @ rhs).max() < 1e-10 * np.abs(rhs).max()


def test_chi0_symmetric_nsd_and_charge_conserving(tiny_system):
    """chi0 symmetric, negative semidefinite, int chi0 g = 0, chi0 const = 0."""
    cfg, R, m, gs = tiny_system
    H = m.hamiltonian_dense(gs.V)
    rng = np.random.default_rng(3)
    F = rng.standard_normal((m.Ng, 3))
    U = rs.chi0_apply(m, H, gs.Psi, gs.eps, F)
    S = m.dV * F.T @ U
    assert np.abs(S - S.T).max() < 1e-10 * np.abs(S).max()
    assert np.linalg.eigvalsh(0.5 * (S + S.T)).max() < 1e-12
    assert np.abs(U.sum(axis=0) * m.dV).max() < 1e-10 * np.abs(U).max()
    Uc = rs.chi0_apply(m, H, gs.Psi, gs.eps, np.ones((m.Ng, 1)))
    assert np.abs(Uc).max() < 1e-10


def test_dyson_dense_residual_and_dfpt(tiny_system):
    """Eq. chi satisfies the Dyson identity u = chi0 g + chi0 v u,
    and agrees with chi0 assembled column-by-column by Alg. 1."""
    cfg, R, m, gs = tiny_system
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    C0 = rs.chi0_adler_wiser_matrix(m, H, cfg.n_occ)
    U = rs.dyson_dense(m, C0, G)
    Kmat = rs.yukawa_matrix(m)
    # residual identity of the Dyson equation
    res = U - C0 @ G - C0 @ (Kmat @ U)
    assert np.abs(res).max() < 1e-10 * np.abs(U).max()
    U2 = rs.dyson_dfpt(m, H, gs.Psi, gs.eps, G)
    assert np.abs(U2 - U).max() < 1e-9 * np.abs(U).max()
