"""Pin of the free-electron closed form (oracle/response.sternheimer_free_electron,
oracle/acp.compressed_W_free_electron) against the dense oracle path on a small grid."""
import numpy as np

from workloads.configs import small_config_2d, small_config
from oracle.model import Model
from oracle import response as rs, acp as oacp
from free_electron import plane_wave_ground_state


def _case(cfg, m2max):
    R = np.zeros((cfg.n_atoms, cfg.dim))
    m = Model(cfg, R)
    Psi, eps, occ = plane_wave_ground_state(cfg.grid, cfg.cell, m2max)
    return m, Psi, eps, occ


def test_plane_waves_are_orthonormal_eigenvectors():
    m, Psi, eps, occ = _case(small_config_2d(grid=(16, 16)), 5)
    assert Psi.shape[1] == 21 and occ.sum() == 21
    assert np.abs(m.dV * Psi.T @ Psi - np.eye(21)).max() < 1e-12
    assert np.abs(m.kinetic(Psi) - Psi * eps[None, :]).max() < 1e-12


def test_free_electron_sternheimer_matches_dense():
    for cfg, m2 in [(small_config_2d(grid=(16, 16)), 5), (small_config(grid=(64,)), 9)]:
        m, Psi, eps, occ = _case(cfg, m2)
        H = m.hamiltonian_dense(np.zeros(m.Ng))
        rhs = np.random.default_rng(3).standard_normal((m.Ng, 3))
        for shift in (eps[0], 0.5 * (eps[0] + eps[-1]), eps[-1]):
            z_dense = rs.sternheimer_solve(m, H, Psi, shift, rhs)
            z_fe = rs.sternheimer_free_electron(m, occ, shift, rhs)
            assert np.abs(z_fe - z_dense).max() < 1e-9 * np.abs(z_dense).max()


def test_free_electron_W_matches_dense():
    cfg = small_config_2d(grid=(16, 16))
    m, Psi, eps, occ = _case(cfg, 5)
    H = m.hamiltonian_dense(np.zeros(m.Ng))
    rng = np.random.default_rng(4)
    S = np.sort(rng.choice(m.Ng, 6, replace=False))
    Xi = rng.standard_normal((m.Ng, 6))
    W_dense = oacp.compressed_W(m, H, Psi, eps, S, Xi, 4)
    W_fe = oacp.compressed_W_free_electron(m, Psi, eps, occ, S, Xi, 4)
    assert np.abs(W_fe - W_dense).max() < 1e-9 * np.abs(W_dense).max()
