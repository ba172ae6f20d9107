"""Pins for oracle/phonon.py: DFPT D vs frozen-phonon FD, sum rule, symmetry, masses."""
import numpy as np
import pytest

from workloads import atom_positions
from workloads.configs import small_config
from oracle.model import Model
from oracle.scf import scf
from oracle import response as rs, phonon


@pytest.fixture(scope="module")
def dfpt_D(tiny_system):
    cfg, R, m, gs = tiny_system
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    C0 = rs.chi0_adler_wiser_matrix(m, H, cfg.n_occ)
    U = rs.dyson_dense(m, C0, G)
    return phonon.dynamical_matrix(m, gs.rho, G, U), (m, gs, G, C0)


def test_dfpt_matches_frozen_phonon(tiny_system, dfpt_D):
    """Eq. SecDeriv/chiterm vs central differences of Eq. force
    (frozen phonon).  Pins the 2f prefactor, signs, local and E_II terms."""
    cfg, R, m, gs = tiny_system
    D, (m, gs, G, C0) = dfpt_D
    Dfd = phonon.fd_dynamical_matrix(cfg, R, delta=1e-3, gs0=gs)
    err = np.abs(Dfd - D).max() / np.abs(D).max()
    assert err < 2e-6
    # a dropped factor (prefactor 2 instead of 2f = 4) is far outside that band
    Uw = rs.dyson_dense(m, 0.5 * C0, G)
    Dw = phonon.dynamical_matrix(m, gs.rho, G, Uw)
    assert np.abs(Dfd - Dw).max() / np.abs(D).max() > 1e-2


def test_sum_rule_and_symmetry(dfpt_D):
    D, _ = dfpt_D
    assert np.abs(D - D.T).max() == 0.0
    assert np.abs(D.sum(axis=1)).max() < 1e-9 * np.abs(D).max()


def test_mass_scaling(tiny_system, dfpt_D):
    cfg, R, m, gs = tiny_system
    D, (m, gs, G, C0) = dfpt_D
    U = rs.dyson_dense(m, C0, G)
    D4 = phonon.dynamical_matrix(m, gs.rho, G, U, masses=4.0 * np.ones(m.NA))
    lam, om, _ = phonon.phonon_modes(D)
    lam4, om4, _ = phonon.phonon_modes(D4)
    assert np.abs(lam4 - lam / 4).max() < 1e-14 * np.abs(lam).max() + 1e-18
    assert np.abs(om4[1:] - om[1:] / 2).max() < 1e-10


def test_periodic_lattice_acoustic_mode():
    """periodic 1D lattice -> exactly d near-zero (acoustic) frequencies."""
    cfg = small_config(jitter=0.0)
    m = Model(cfg, atom_positions(cfg))
    gs = scf(m, tol=1e-13)
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    U = rs.dyson_dense(m, rs.chi0_adler_wiser_matrix(m, H, cfg.n_occ), G)
    lam, om, _ = phonon.phonon_modes(phonon.dynamical_matrix(m, gs.rho, G, U))
    assert np.sum(np.abs(lam) < 1e-9 * np.abs(lam).max()) == 1
    assert lam[1] > 1e-6 * np.abs(lam).max()


# ---------------------------------------------------------------- 2D (configs[3], [4] shape)
@pytest.fixture(scope="module")
def system_2d():
    from workloads.configs import small_config_2d
    cfg = small_config_2d(grid=(24, 24))
    R = atom_positions(cfg)
    m = Model(cfg, R)
    gs = scf(m, tol=1e-13)
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    C0 = rs.chi0_adler_wiser_matrix(m, H, cfg.n_occ)
    U = rs.dyson_dense(m, C0, G)
    D, parts = phonon.dynamical_matrix(m, gs.rho, G, U, parts=True)
    return cfg, R, m, gs, G, C0, D, parts


def test_2d_dfpt_matches_frozen_phonon(system_2d):
    """2D Eq. SecDeriv/chiterm vs central differences of the 2D forces
    (frozen phonon): pins the x/y column order of G, the 2D d2V block (incl. the
    x-y cross terms), the 2D E_II Hessian and the 2f prefactor together."""
    cfg, R, m, gs, G, C0, D, parts = system_2d
    Dfd = phonon.fd_dynamical_matrix(cfg, R, delta=1e-3, gs0=gs)
    err = np.abs(Dfd - D).max() / np.abs(D).max()
    assert err < 2e-6, err
    # the off-diagonal x-y blocks carry weight (a dropped cross term would show)
    xy = np.abs(D[0::2, 1::2]).max() / np.abs(D).max()
    assert xy > 1e-3
    # wrong prefactor 2 instead of 2f = 4 (reading R2) is far outside the band
    Dw = phonon.dynamical_matrix(m, gs.rho, G, rs.dyson_dense(m, 0.5 * C0, G))
    assert np.abs(Dfd - Dw).max() / np.abs(D).max() > 1e-2
    # so is a local term with the x-y cross entries dropped
    D_chi, D_loc, D_ii = parts
    D_loc_diag = D_loc.copy()
    D_loc_diag[0::2, 1::2] = 0.0
    D_loc_diag[1::2, 0::2] = 0.0
    Dd = 0.5 * ((D_chi + D_loc_diag + D_ii) + (D_chi + D_loc_diag + D_ii).T)
    if np.abs(D_loc[0::2, 1::2]).max() > 1e-4 * np.abs(D).max():
        assert np.abs(Dfd - Dd).max() / np.abs(D).max() > 10 * err


def test_2d_sum_rule_and_symmetry(system_2d):
    """Acoustic sum rule in x and in y (a rigid translation along either axis costs nothing)."""
    D = system_2d[6]
    assert np.abs(D - D.T).max() == 0.0
    for b in range(2):
        assert np.abs(D[:, b::2].sum(axis=1)).max() < 1e-8 * np.abs(D).max()
    lam = np.linalg.eigvalsh(D)
    assert np.sum(np.abs(lam) < 1e-7 * np.abs(lam).max()) == 2   # two acoustic modes in 2D
