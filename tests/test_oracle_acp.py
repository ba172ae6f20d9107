"""Pins for oracle/acp.py: Chebyshev/Lagrange closed forms, SRFT vs FFT, QRCP vs LAPACK,
ID exactness, SMW vs dense inverse, ACP -> exact DFPT limit."""
import numpy as np
import pytest
import scipy.linalg as sla

from workloads import sketch_draws
from oracle import acp, response as rs


def test_chebyshev_nodes_closed_forms():
    # SPEC.md:401-403
    assert np.allclose(acp.chebyshev_nodes(-1.0, 3.0, 1), [1.0])
    n2 = acp.chebyshev_nodes(-1.0, 1.0, 2)
    assert np.allclose(sorted(n2), [-np.cos(np.pi / 4), np.cos(np.pi / 4)])
    n = acp.chebyshev_nodes(-0.3, 0.2, 9)
    assert n.min() > -0.3 and n.max() < 0.2
    # zeros of T_Nc on the reference interval
    t = (2 * n - (-0.3 + 0.2)) / (0.2 + 0.3)
    assert np.abs(np.cos(9 * np.arccos(np.clip(t, -1, 1)))).max() < 1e-12
    assert np.allclose(acp.chebyshev_nodes(0.5, 0.5, 4), 0.5)


def test_lagrange_weights():
    # Kronecker at nodes, partition of unity, polynomial reproduction
    nodes = acp.chebyshev_nodes(-0.4, 0.1, 7)
    L = acp.lagrange_weights(nodes, nodes)
    assert np.abs(L - np.eye(7)).max() < 1e-13
    e = np.random.default_rng(0).uniform(-0.4, 0.1, 50)
    L = acp.lagrange_weights(nodes, e)
    assert np.abs(L.sum(axis=1) - 1).max() < 1e-12
    p = lambda x: 3 * x ** 6 - x ** 3 + 0.5
    assert np.abs(L @ p(nodes) - p(e)).max() < 1e-12


def test_srft_matches_fft():
    """Alg. 2 step 1(a) is a DFT of eta-weighted columns: check vs numpy FFT."""
    rng = np.random.default_rng(4)
    G = rng.standard_normal((30, 12))
    theta, nu = sketch_draws(5, 0, 12, 8)
    Gt = acp.srft_sketch(G, theta, nu)
    eta = np.exp(2j * np.pi * theta)
    F = np.fft.fft(G * eta, axis=1)          # sum_{j=0}^{n-1} e^{-2pi i j nu/n} x_j
    for q, v in enumerate(nu):
        ref = np.exp(-2j * np.pi * v / 12) * F[:, v % 12]   # paper's I = j + 1 convention
        assert np.abs(Gt[:, 2 * q] - ref.real).max() < 1e-12
        assert np.abs(Gt[:, 2 * q + 1] - ref.imag).max() < 1e-12


def test_qrcp_matches_lapack_dgeqp3():
    rng = np.random.default_rng(6)
    for shape in [(20, 50), (40, 30), (64, 200)]:
        A = rng.standard_normal(shape) * np.exp(rng.uniform(-3, 0, shape[1]))
        qr = acp.qrcp(A, eps=0.0)
        Qr, Rr, P = sla.qr(A, pivoting=True, mode="economic")
        k = qr.n_mu
        assert np.array_equal(qr.perm[:k], P[:k])
        assert np.abs(qr.rdiag - np.abs(np.diag(Rr))[:k]).max() < 1e-12 * abs(Rr[0, 0])
        assert np.abs(np.abs(qr.R) - np.abs(Rr[:k, :])).max() < 1e-11 * abs(Rr[0, 0])


def test_qrcp_threshold_rule():
    """Alg. 2 step 3: |R_{N+1,N+1}| < eps |R_11| <= |R_{N,N}|."""
    rng = np.random.default_rng(7)
    A = rng.standard_normal((60, 80)) * np.exp(-0.25 * np.arange(80))[None, :]
    for eps in (1e-1, 1e-3, 1e-6):
        qr = acp.qrcp(A, eps)
        full = acp.qrcp(A, 0.0)
        d = full.rdiag
        N = qr.n_mu
        assert d[N - 1] >= eps * d[0]
        assert N == len(d) or d[N] < eps * d[0]


def test_interpolative_decomposition_exact_rank():
    """exact rank-5 matrix -> N_mu = 5 and exact reconstruction; Xi(S,:) = I."""
    rng = np.random.default_rng(8)
    Mfull = rng.standard_normal((100, 5)) @ rng.standard_normal((5, 40))    # Ng x cols
    qr = acp.qrcp(Mfull.T, eps=1e-10)
    S, Xi = acp.interpolation_vectors(qr, 100)
    assert qr.n_mu == 5
    assert np.abs(Xi[S, :] - np.eye(5)).max() < 1e-12
    assert np.abs(Xi @ Mfull[S, :] - Mfull).max() < 1e-10 * np.abs(Mfull).max()


def test_smw_equals_dense_inverse(tiny_system):
    """Eq. dyson4 second equality (Sherman-Morrison-Woodbury)."""
    cfg, R, m, gs = tiny_system
    rng = np.random.default_rng(9)
    G = m.G_matrix()
    S = np.sort(rng.choice(m.Ng, 10, replace=False))
    W = 1e-3 * rng.standard_normal((m.Ng, 10))
    U, Gp, Y = acp.smw_update(m, G, W, S)
    Pi = np.zeros((m.Ng, 10))
    Pi[S, np.arange(10)] = 1.0
    Kmat = rs.yukawa_matrix(m)
    B = m.yukawa_inverse(G)
    Ut = np.linalg.solve(np.eye(m.Ng) - W @ Pi.T @ Kmat, B)
    assert np.abs((Ut - B) - U).max() < 1e-9 * np.abs(U).max()
    assert np.abs(Kmat @ Ut - Gp).max() < 1e-8 * np.abs(Gp).max()


def test_acp_full_selection_is_exact_dyson(tiny_system):
    """With every grid point selected (Xi = I) chi0~ = chi0 up to Chebyshev error, so one SMW
    step solves the Dyson equation -- error falls with N_c."""
    cfg, R, m, gs = tiny_system
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    C0 = rs.chi0_adler_wiser_matrix(m, H, cfg.n_occ)
    Uex = rs.dyson_dense(m, C0, G)
    S = np.arange(m.Ng)
    errs = []
    for Nc in (4, 8, 16):
        W = acp.compressed_W(m, H, gs.Psi, gs.eps[: cfg.n_occ], S, np.eye(m.Ng), Nc)
        U, _, _ = acp.smw_update(m, G, W, S)
        errs.append(np.linalg.norm(U - Uex) / np.linalg.norm(Uex))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-9


def test_acp_converges_to_dfpt(tiny_system):
    """Alg. 4 with a tight ID threshold, many Chebyshev nodes and outer iterations -> exact
    chi G; the error falls monotonically along that path (Table 1 pattern)."""
    cfg, R, m, gs = tiny_system
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    C0 = rs.chi0_adler_wiser_matrix(m, H, cfg.n_occ)
    Uex = rs.dyson_dense(m, C0, G)
    draws = lambda k, n: sketch_draws(cfg.seed, k, n, cfg.sketch_r)
    errs = []
    for eps_id, Nc, nout in [(1e-3, 4, 2), (1e-8, 12, 6), (1e-12, 20, 8)]:
        res = acp.acp_dyson(m, H, gs.Psi, gs.eps[: cfg.n_occ], G, Nc, nout, eps_id, draws)
        errs.append(np.linalg.norm(res.U - Uex) / np.linalg.norm(Uex))
        assert all(res.diff[i + 1] < res.diff[i] for i in range(len(res.diff) - 1))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-7
