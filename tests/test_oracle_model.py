"""Pins for oracle/model.py: closed forms, PDE identities, finite differences."""
import numpy as np
import pytest

from workloads import atom_positions
from workloads.configs import small_config
from oracle.model import Model


def _model(**kw):
    cfg = small_config(**kw)
    return Model(cfg, atom_positions(cfg))


def test_grid_metadata():
    m = _model()
    assert m.Ng == 96
    assert abs(m.dV * m.Ng - m.Omega) < 1e-12
    assert np.isclose(m.k[0][1], 2 * np.pi / m.L[0])


def test_pseudocharge_normalisation():
    # int m_I = -Z_I
    m = _model()
    assert abs(m.integrate(m.pseudocharge(0)) + m.Z) < 1e-10
    assert abs(m.integrate(m.pseudocharge()) + m.Z * m.NA) < 1e-10


def test_pseudocharge_gaussian_closed_form():
    # m_I(x) = -Z/sqrt(2 pi sigma^2) exp(-x^2/(2 sigma^2)), periodised
    m = _model()
    x = m.r[:, 0]
    s = m.cfg.sigma
    ref = np.zeros_like(x)
    for n in range(-3, 4):
        d = x - m.R[0, 0] + n * m.L[0]
        ref += -m.Z / np.sqrt(2 * np.pi * s * s) * np.exp(-d * d / (2 * s * s))
    assert np.abs(m.pseudocharge(0) - ref).max() < 1e-12


def test_yukawa_constant_and_cosine():
    # K*c = 4 pi c/(eps0 kappa^2); K*cos(2 pi x/L) = 4pi/eps0/((2pi/L)^2+kappa^2) cos
    m = _model()
    c = 0.7
    v = m.yukawa(np.full(m.Ng, c))
    assert np.allclose(v, 4 * np.pi * c / (m.cfg.eps0 * m.cfg.kappa ** 2), rtol=1e-13)
    x = m.r[:, 0]
    k = 2 * np.pi / m.L[0]
    v = m.yukawa(np.cos(k * x))
    ref = 4 * np.pi / m.cfg.eps0 / (k * k + m.cfg.kappa ** 2) * np.cos(k * x)
    assert np.abs(v - ref).max() < 1e-11 * np.abs(ref).max()


def test_yukawa_solves_screened_poisson_fd():
    # -K'' + kappa^2 K = (4 pi/eps0) delta.  Check with a 4th-order
    # finite-difference Laplacian (independent of the FFT) on a smooth periodic f.
    m = _model(grid=(768,))
    x = m.r[:, 0]
    f = np.exp(np.sin(2 * np.pi * x / m.L[0])) - 1.2 * np.cos(4 * np.pi * x / m.L[0])
    u = m.yukawa(f)
    h = m.L[0] / m.Ng
    lap = (-np.roll(u, 2) + 16 * np.roll(u, 1) - 30 * u + 16 * np.roll(u, -1) - np.roll(u, -2)) / (12 * h * h)
    lhs = -lap + m.cfg.kappa ** 2 * u
    assert np.abs(lhs - 4 * np.pi / m.cfg.eps0 * f).max() < 1e-6 * np.abs(f).max()


def test_yukawa_inverse_roundtrip():
    m = _model()
    f = np.random.default_rng(0).standard_normal(m.Ng)
    assert np.abs(m.yukawa_inverse(m.yukawa(f)) - f).max() < 1e-9  # cond(K) ~ 1e4 on this grid


def test_kinetic_plane_wave():
    # V=0, psi = cos(k x) -> H psi = k^2/2 psi
    m = _model()
    x = m.r[:, 0]
    k = 3 * 2 * np.pi / m.L[0]
    assert np.abs(m.kinetic(np.cos(k * x)) - 0.5 * k * k * np.cos(k * x)).max() < 1e-12


def test_g_is_fd_derivative_of_V():
    # g_{I,a} = dV_I(r - R_I)/dR_{I,a}; central difference h = 1e-4
    cfg = small_config()
    R = atom_positions(cfg)
    m = Model(cfg, R)
    G = m.G_matrix()
    hstep = 1e-4
    for I in range(m.NA):
        Rp, Rm = R.copy(), R.copy()
        Rp[I, 0] += hstep
        Rm[I, 0] -= hstep
        mp, mm = Model(cfg, Rp), Model(cfg, Rm)
        fd = (mp.v_ion() - mm.v_ion()) / (2 * hstep)
        assert np.abs(fd - G[:, I]).max() < 1e-7 * np.abs(G[:, I]).max()
        assert abs(m.integrate(G[:, I])) < 1e-12


def test_d2V_is_fd_derivative_of_g():
    cfg = small_config()
    R = atom_positions(cfg)
    m = Model(cfg, R)
    hstep = 1e-4
    Rp, Rm = R.copy(), R.copy()
    Rp[1, 0] += hstep
    Rm[1, 0] -= hstep
    fd = (Model(cfg, Rp).G_matrix()[:, 1] - Model(cfg, Rm).G_matrix()[:, 1]) / (2 * hstep)
    h = m.d2V(1)[:, 0, 0]
    assert np.abs(fd - h).max() < 1e-7 * np.abs(h).max()


def test_eii_pair_closed_form_gaussians():
    # Two Gaussians in 1D interacting through the (non-periodic) Yukawa kernel:
    # int int m_1 K m_2 = (Z^2 2pi/(kappa eps0)) * E[e^{-kappa|X|}], X ~ N(d, 2 sigma^2).
    # With a large cell the periodic images are negligible (e^{-kappa L}).
    from scipy.special import erfc
    cfg = small_config(n_side=2, spacing=40.0, kappa=0.5, grid=(1024,), jitter=0.0)
    R = np.array([[10.0], [13.7]])
    m = Model(cfg, R)
    d, s2, k = 3.7, 2 * cfg.sigma ** 2, cfg.kappa
    s = np.sqrt(s2)
    # E[e^{-k|X|}] for X ~ N(d, s^2)
    ex = 0.5 * np.exp(k * k * s2 / 2) * (np.exp(-k * d) * erfc((k * s2 - d) / (s * np.sqrt(2)))
                                         + np.exp(k * d) * erfc((k * s2 + d) / (s * np.sqrt(2))))
    ref = cfg.Z ** 2 * 2 * np.pi / (k * cfg.eps0) * ex
    assert abs(m.e_ii() - ref) < 1e-9 * abs(ref)


def test_eii_derivatives_fd():
    cfg = small_config()
    R = atom_positions(cfg)
    m = Model(cfg, R)
    g = m.e_ii_gradient()
    Hs = m.e_ii_hessian()
    hstep = 1e-4
    for I in range(m.NA):
        Rp, Rm = R.copy(), R.copy()
        Rp[I, 0] += hstep
        Rm[I, 0] -= hstep
        mp, mm = Model(cfg, Rp), Model(cfg, Rm)
        # E_II ~ 1e4 (k=0 term), so the energy difference uses a larger step
        Rp2, Rm2 = R.copy(), R.copy()
        Rp2[I, 0] += 1e-2
        Rm2[I, 0] -= 1e-2
        fdg = (Model(cfg, Rp2).e_ii() - Model(cfg, Rm2).e_ii()) / 2e-2
        assert abs(fdg - g[I, 0]) < 1e-5 * abs(g).max()
        fdH = (mp.e_ii_gradient() - mm.e_ii_gradient()).reshape(-1) / (2 * hstep)
        assert np.abs(fdH - Hs[I, :]).max() < 1e-6 * np.abs(Hs).max()
    assert np.abs(Hs.sum(axis=1)).max() < 1e-12 * np.abs(Hs).max() + 1e-14   # translation invariance


def test_2d_model_basics():
    cfg = small_config(dim=2, n_side=2, spacing=6.0, grid=(24, 24), n_occ=4, jitter=0.1)
    m = Model(cfg, atom_positions(cfg))
    assert abs(m.integrate(m.pseudocharge()) + m.Z * m.NA) < 1e-9
    G = m.G_matrix()
    assert G.shape == (576, 8)
    assert np.abs(G.sum(axis=0) * m.dV).max() < 1e-10
