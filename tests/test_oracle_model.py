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


# ---------------------------------------------------------------- 2D branch (configs[3], [4] shape)
def _model_2d(**kw):
    from workloads.configs import small_config_2d
    cfg = small_config_2d(grid=(24, 24), **kw)
    return cfg, atom_positions(cfg)


def test_2d_g_columns_are_fd_derivatives_of_V():
    """Both columns g_{I,x}, g_{I,y} of every atom against central differences of
    V_ion in R_{I,a}; a transposed axis or a wrong k-component fails by O(1)."""
    cfg, R = _model_2d()
    m = Model(cfg, R)
    G = m.G_matrix()
    h = 1e-4
    for I in range(m.NA):
        for a in range(2):
            Rp, Rm = R.copy(), R.copy()
            Rp[I, a] += h
            Rm[I, a] -= h
            fd = (Model(cfg, Rp).v_ion() - Model(cfg, Rm).v_ion()) / (2 * h)
            col = G[:, 2 * I + a]
            assert np.abs(fd - col).max() < 1e-7 * np.abs(col).max()
            assert abs(m.integrate(col)) < 1e-12 * np.abs(col).max() * m.Omega


def test_2d_d2V_all_entries_fd():
    """d2V_I/dR_a dR_b for a, b in {x, y} (incl. the a != b cross terms) against central
    differences of g_{I,b} in R_{I,a}; the 2x2 block is symmetric."""
    cfg, R = _model_2d()
    m = Model(cfg, R)
    h = 1e-4
    I = 2
    H2 = m.d2V(I)
    for a in range(2):
        Rp, Rm = R.copy(), R.copy()
        Rp[I, a] += h
        Rm[I, a] -= h
        dG = (Model(cfg, Rp).G_matrix() - Model(cfg, Rm).G_matrix()) / (2 * h)
        for b in range(2):
            fd = dG[:, 2 * I + b]
            assert np.abs(fd - H2[:, a, b]).max() < 1e-7 * np.abs(H2).max(), (a, b)
    assert np.array_equal(H2[:, 0, 1], H2[:, 1, 0])
    # the cross term is not identically zero for a generic position (else the check is vacuous)
    assert np.abs(H2[:, 0, 1]).max() > 1e-2 * np.abs(H2).max()


def test_2d_eii_gradient_and_hessian_fd():
    """E_II (reading R4) in 2D: gradient vs central differences of the energy, the full Hessian
    (x/y and cross-atom blocks) vs central differences of the gradient, translation invariance."""
    cfg, R = _model_2d()
    m = Model(cfg, R)
    g = m.e_ii_gradient()
    Hs = m.e_ii_hessian()
    for I in range(m.NA):
        for a in range(2):
            Rp, Rm = R.copy(), R.copy()
            Rp[I, a] += 1e-2
            Rm[I, a] -= 1e-2
            fdg = (Model(cfg, Rp).e_ii() - Model(cfg, Rm).e_ii()) / 2e-2
            assert abs(fdg - g[I, a]) < 1e-5 * np.abs(g).max()
            Rp, Rm = R.copy(), R.copy()
            Rp[I, a] += 1e-4
            Rm[I, a] -= 1e-4
            fdH = (Model(cfg, Rp).e_ii_gradient() - Model(cfg, Rm).e_ii_gradient()).reshape(-1) / 2e-4
            assert np.abs(fdH - Hs[2 * I + a, :]).max() < 1e-6 * np.abs(Hs).max()
    assert np.abs(Hs - Hs.T).max() < 1e-12 * np.abs(Hs).max()
    # translation invariance in x and in y separately: sum over J of the (I a, J b) block is 0
    for b in range(2):
        assert np.abs(Hs[:, b::2].sum(axis=1)).max() < 1e-11 * np.abs(Hs).max()
    assert np.abs(g.sum(axis=0)).max() < 1e-11 * np.abs(g).max()


def test_2d_eii_pair_closed_form_gaussians():
    """Two 2D Gaussians through the Yukawa symbol 4pi/(eps0(|k|^2+kappa^2)): in the
    plane this is the kernel (2/eps0) K_0(kappa r) (the 2D Green's function of -Delta + kappa^2
    times 4 pi / eps0), so E_12 = Z^2 (2/eps0) E[K_0(kappa |X|)], X ~ N(d, 2 sigma^2 I_2).  A
    large cell makes the periodic images negligible; the expectation is a 2D quadrature."""
    from scipy.special import k0
    from workloads.configs import small_config_2d
    cfg = small_config_2d(n_side=2, spacing=30.0, kappa=0.4, sigma=1.0, grid=(256, 256), jitter=0.0)
    R = np.array([[20.0, 25.0], [22.9, 26.3]])
    m = Model(cfg, R)
    d = R[1] - R[0]
    s2 = 2 * cfg.sigma ** 2
    # polar quadrature centred on the kernel's log singularity at X = 0, radial variable r = u^2
    # (the integrand ~ u^3 log u is then smooth enough for Gauss-Legendre), uniform in angle
    nu_, nt = 600, 512
    xu, wu = np.polynomial.legendre.leggauss(nu_)
    umax = np.sqrt(np.hypot(*d) + 10.0 * np.sqrt(s2))
    u = 0.5 * umax * (xu + 1)
    wu = 0.5 * umax * wu
    r = u * u
    th = 2 * np.pi * np.arange(nt) / nt
    X = r[:, None] * np.cos(th)[None, :]
    Y = r[:, None] * np.sin(th)[None, :]
    dens = np.exp(-((X - d[0]) ** 2 + (Y - d[1]) ** 2) / (2 * s2)) / (2 * np.pi * s2)
    val = k0(cfg.kappa * r)[:, None]
    ex = float(np.sum((wu * 2 * u * r)[:, None] * dens * val) * (2 * np.pi / nt))
    ref = cfg.Z ** 2 * (2.0 / cfg.eps0) * ex
    assert abs(m.e_ii() - ref) < 1e-9 * abs(ref), (m.e_ii(), ref)
