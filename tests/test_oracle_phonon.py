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
