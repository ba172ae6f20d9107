"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Tolerances: building blocks 1e-12 relative (pure fp64 rounding);
Sternheimer-derived quantities are limited by the CG tolerance (1e-11 relative
residual) times the conditioning of Q(H - eps)Q on range(Q) -> 1e-9 relative on
W and U; the acceptance bar of BASELINE.json:north_star is 1e-8 relative on D and
1e-7 relative on the phonon eigenvalues.  Integer outputs (QRCP pivots) are bit-exact.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import atom_positions, get_config, sketch_draws  # noqa: E402
from workloads.configs import small_config, small_config_2d  # noqa: E402
from oracle.model import Model  # noqa: E402
from oracle.scf import scf  # noqa: E402
from oracle import acp as oacp, phonon as ophonon, response as ors  # noqa: E402


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def T(x, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda").contiguous()


class Sys:
    """Oracle ground state + everything the GPU calls need, for one config."""

    def __init__(self, cfg):
        from paper_1605_08021_b200 import Context
        self.cfg = cfg
        self.R = atom_positions(cfg)
        self.m = Model(cfg, self.R)
        self.gs = scf(self.m, tol=cfg.scf_tol)
        self.H = self.m.hamiltonian_dense(self.gs.V)
        self.G = self.m.G_matrix()
        self.ctx = Context.from_config(cfg)
        self.Psi_t = T(self.gs.Psi.T)
        self.eps_t = T(self.gs.eps)
        self.V_t = T(self.gs.V)
        self.rho_t = T(self.gs.rho)
        self.G_t = T(self.G.T)

    def draws(self, k, n):
        return sketch_draws(self.cfg.seed, k, n, self.cfg.sketch_r)


_cache = {}


def system(name):
    if name not in _cache:
        cfg = {"tiny4": small_config, "tiny2d": small_config_2d}.get(name, lambda: get_config(name))()
        _cache[name] = Sys(cfg)
    return _cache[name]


@pytest.fixture(scope="module", params=["tiny4", "c0_1d_tiny", "tiny2d"])
def sysx(request):
    return system(request.param)


# ---------------------------------------------------------------- building blocks
def test_fourier_operators(sysx):
    s = sysx
    rng = np.random.default_rng(11)
    for ncol in (1, 2, 5):          # odd counts exercise the unpaired tail column
        X = rng.standard_normal((s.m.Ng, ncol))
        Xt = T(X.T)
        Y = s.ctx.fourier_apply(Xt, 0).cpu().numpy().T
        assert rel(Y, s.m.kinetic(X)) < 1e-12
        Y = s.ctx.fourier_apply(Xt, 1).cpu().numpy().T
        assert rel(Y, s.m.yukawa(X)) < 1e-12
        shifts = rng.uniform(-0.1, 0.1, ncol)
        Y = s.ctx.fourier_apply(Xt, 0, diag=s.V_t, shift=T(shifts)).cpu().numpy().T
        ref = s.m.kinetic(X) + (s.gs.V[:, None] - shifts[None, :]) * X
        assert rel(Y, ref) < 1e-12
        assert rel(Y, (s.H @ X) - shifts[None, :] * X) < 1e-11


@pytest.mark.parametrize("cs", [1, 2, 4, 8])
def test_fourier_operator_2d_cluster_sizes(cs, monkeypatch):
    """2D K1 with the DSMEM transposes of a cs-CTA cluster (ACP_FFT2D_CS; the kernel that also runs
    the ground-state setup transforms) vs the oracle; odd column counts leave a half-empty pair."""
    from paper_1605_08021_b200 import Context
    s = system("tiny2d")
    monkeypatch.setenv("ACP_FFT2D_CLUSTER", "1")
    monkeypatch.setenv("ACP_FFT2D_CS", str(cs))
    ctx = Context.from_config(s.cfg)
    rng = np.random.default_rng(20 + cs)
    for ncol in (1, 4, 7, 13):
        X = rng.standard_normal((s.m.Ng, ncol))
        Xt = T(X.T)
        assert rel(ctx.fourier_apply(Xt, 0).cpu().numpy().T, s.m.kinetic(X)) < 1e-12
        assert rel(ctx.fourier_apply(Xt, 1).cpu().numpy().T, s.m.yukawa(X)) < 1e-12
        shifts = rng.uniform(-0.1, 0.1, ncol)
        Y = ctx.fourier_apply(Xt, 0, diag=s.V_t, shift=T(shifts)).cpu().numpy().T
        assert rel(Y, (s.H @ X) - shifts[None, :] * X) < 1e-11
    assert rel(ctx.perturbations(s.R).cpu().numpy().T, s.G) < 1e-12
    ctx.close()


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("name", ["c0_1d_tiny", "c1_1d_insulator", "c2_1d_semiconductor"])
def test_fourier_operator_compiled_lengths(name, generic, monkeypatch):
    """1D K1 at the configs' grid lengths (256, 1280, 5120): the compiled-length FFT kernels
    (default) and the runtime-plan kernels (ACP_FFT_GENERIC) vs numpy's FFT, odd column count."""
    from paper_1605_08021_b200 import Context
    if generic:
        monkeypatch.setenv("ACP_FFT_GENERIC", "1")
    cfg = get_config(name)
    ctx = Context.from_config(cfg)
    N, L = cfg.grid[0], cfg.cell[0]
    rng = np.random.default_rng(N)
    X = rng.standard_normal((5, N))
    k = 2 * np.pi * np.fft.fftfreq(N, d=L / N)
    ref = np.real(np.fft.ifft(np.fft.fft(X, axis=1) * (0.5 * k * k)[None], axis=1))
    Y = ctx.fourier_apply(T(X), 0).cpu().numpy()
    assert rel(Y, ref) < 1e-12
    V = rng.standard_normal(N)
    sh = rng.standard_normal(5)
    Y2 = ctx.fourier_apply(T(X), 0, diag=T(V), shift=T(sh)).cpu().numpy()
    assert rel(Y2, ref + (V[None, :] - sh[:, None]) * X) < 1e-12
    ctx.close()


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("name", ["c3g_2d_8x8", "c4g_2d_16x16"])
def test_fourier_operator_2d_compiled_lengths(name, generic, monkeypatch):
    """2D K1 (three passes) on the configs' square grids 192^2 / 256^2: compiled-length FFT
    passes (default) and runtime-plan passes (ACP_FFT_GENERIC) vs numpy's fft2."""
    from paper_1605_08021_b200 import Context
    if generic:
        monkeypatch.setenv("ACP_FFT_GENERIC", "1")
    cfg = get_config(name)
    ctx = Context.from_config(cfg)
    n0, n1 = cfg.grid
    L0, L1 = cfg.cell
    rng = np.random.default_rng(n0)
    X = rng.standard_normal((3, n0, n1))
    k0 = 2 * np.pi * np.fft.fftfreq(n0, d=L0 / n0)
    k1 = 2 * np.pi * np.fft.fftfreq(n1, d=L1 / n1)
    k2 = k0[:, None] ** 2 + k1[None, :] ** 2
    ref = np.real(np.fft.ifft2(np.fft.fft2(X) * (0.5 * k2)[None]))
    Y = ctx.fourier_apply(T(X.reshape(3, -1)), 0).cpu().numpy().reshape(3, n0, n1)
    assert rel(Y, ref) < 1e-12
    ctx.close()


def test_fourier_operator_2d_three_pass():
    """Default 2D K1: row pass, column pass (symbol), row pass + epilogue through the HBM
    intermediate, vs the oracle's operators; odd column counts leave a half-empty last pair."""
    s = system("tiny2d")
    rng = np.random.default_rng(31)
    for ncol in (1, 4, 7, 13):
        X = rng.standard_normal((s.m.Ng, ncol))
        Xt = T(X.T)
        assert rel(s.ctx.fourier_apply(Xt, 0).cpu().numpy().T, s.m.kinetic(X)) < 1e-12
        assert rel(s.ctx.fourier_apply(Xt, 1).cpu().numpy().T, s.m.yukawa(X)) < 1e-12
        shifts = rng.uniform(-0.1, 0.1, ncol)
        Y = s.ctx.fourier_apply(Xt, 0, diag=s.V_t, shift=T(shifts)).cpu().numpy().T
        assert rel(Y, (s.H @ X) - shifts[None, :] * X) < 1e-11


@pytest.mark.parametrize("cs", [0, 1, 8])
def test_fourier_operator_rectangular_grid(cs, monkeypatch):
    """Non-square 2D grid and cell (axis bookkeeping): kinetic symbol vs numpy's FFT; cs = 0 is
    the default three-pass path, cs > 0 the cluster kernel with that cluster size."""
    from paper_1605_08021_b200 import Context
    if cs:
        monkeypatch.setenv("ACP_FFT2D_CLUSTER", "1")
        monkeypatch.setenv("ACP_FFT2D_CS", str(cs))
    n0, n1, L0, L1 = 24, 40, 10.0, 16.0
    ctx = Context(2, (n0, n1), (L0, L1), 2, 2, 2.0, 2.0, 1.0, 0.01, 1.0)
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3, n0, n1))
    k0 = 2 * np.pi * np.fft.fftfreq(n0, d=L0 / n0)
    k1 = 2 * np.pi * np.fft.fftfreq(n1, d=L1 / n1)
    k2 = k0[:, None] ** 2 + k1[None, :] ** 2
    ref = np.real(np.fft.ifft2(np.fft.fft2(X) * (0.5 * k2)[None]))
    Y = ctx.fourier_apply(T(X.reshape(3, -1)), 0).cpu().numpy().reshape(3, n0, n1)
    assert rel(Y, ref) < 1e-12
    ctx.close()


def test_gemms(sysx):
    s = sysx
    rng = np.random.default_rng(12)
    for n in (1, 7, 33, 70):
        Y = rng.standard_normal((s.m.Ng, n))
        C = s.ctx.gemm_tn(s.Psi_t, T(Y.T), alpha=s.m.dV).cpu().numpy().T
        assert rel(C, s.m.dV * s.gs.Psi.T @ Y) < 1e-12
        Cm = rng.standard_normal((s.cfg.n_occ, n))
        Z0 = rng.standard_normal((s.m.Ng, n))
        Z = s.ctx.gemm_nn(s.Psi_t, T(Cm.T), C=T(Z0.T), alpha=-1.0, beta=1.0).cpu().numpy().T
        assert rel(Z, Z0 - s.gs.Psi @ Cm) < 1e-12


@pytest.mark.parametrize("M,K,n", [(300, 100, 70), (301, 97, 65), (128, 64, 64)])
def test_gemm_nn_large_k(M, K, n):
    """The 64 x 64 multistage DMMA tile (K >= 64), aligned and unaligned (odd ld) operands."""
    s = system("tiny4")
    rng = np.random.default_rng(M + K + n)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, n))
    C0 = rng.standard_normal((M, n))
    C = s.ctx.gemm_nn(T(A.T), T(B.T), C=T(C0.T), alpha=-0.5, beta=2.0).cpu().numpy().T
    assert rel(C, 2.0 * C0 - 0.5 * A @ B) < 1e-13


@pytest.mark.parametrize("n", [1, 2, 5, 31, 33, 64, 127, 128, 158, 159, 200, 333, 512])
@pytest.mark.parametrize("kind", ["random", "degenerate", "diagonal", "lowrank"])
@pytest.mark.parametrize("method", ["tridiag", "jacobi"])
def test_sym_eigvals(n, kind, method, monkeypatch):
    """Phonon-spectrum eigenvalue step: single-CTA and cooperative-grid Householder
    tridiagonalisation + Sturm multisection (default), one-warp / block Jacobi (knobs), vs LAPACK."""
    if method == "jacobi":
        if n > 160:
            pytest.skip("block Jacobi: smaller sizes suffice")
        monkeypatch.setenv("ACP_EIG_JACOBI" if n <= 32 else "ACP_EIG_BLOCK", "1")
    s = system("tiny4")
    rng = np.random.default_rng(n * 7 + len(kind))
    if kind == "random":
        A = rng.standard_normal((n, n))
        A = A + A.T
    else:
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        if kind == "degenerate":      # clusters of exactly repeated eigenvalues incl. zeros (acoustic modes)
            lam = np.repeat(np.array([0.0, 1.0, -2.5, 3.0]), (n + 3) // 4)[:n]
        elif kind == "diagonal":      # already tridiagonal: every Householder step is the identity
            Q = np.eye(n)
            lam = rng.standard_normal(n)
        else:                         # rank 2: most trailing columns vanish during the reduction
            lam = np.zeros(n)
            lam[:min(2, n)] = [4.0, -1.0][:min(2, n)]
        A = (Q * lam) @ Q.T
        A = 0.5 * (A + A.T)
    w = s.ctx.sym_eigvals(T(A)).cpu().numpy()
    ref = np.linalg.eigvalsh(A)
    scale = max(np.abs(ref).max(), 1e-300)
    assert np.all(np.diff(w) >= -1e-12 * scale)
    assert np.abs(w - ref).max() <= 1e-12 * scale


@pytest.mark.parametrize("n,nrhs", [(1, 1), (31, 3), (32, 8), (33, 5), (100, 64), (290, 128), (513, 7),
                                    (700, 33)])
def test_lu_solve(n, nrhs):
    """Dense SMW core solve (Eq. dyson4): blocked partially pivoted LU vs LAPACK; a row-permuted
    matrix forces non-trivial pivots."""
    s = system("tiny4")
    rng = np.random.default_rng(n + nrhs)
    A = rng.standard_normal((n, n)) + np.eye(n)
    A = A[rng.permutation(n)]
    A[:, 0] *= 1e-3                      # a small leading column: pivoting is required
    B = rng.standard_normal((n, nrhs))
    _, X = s.ctx.lu_solve(T(A.T), T(B.T))
    X = X.cpu().numpy().T
    Xr = np.linalg.solve(A, B)
    cond = np.linalg.cond(A)
    assert rel(X, Xr) < 1e-15 * cond * n


def test_lu_solve_singular():
    from paper_1605_08021_b200 import AcpError
    s = system("tiny4")
    A = np.ones((40, 40))
    with pytest.raises(AcpError):
        s.ctx.lu_solve(T(A), T(np.ones((1, 40))))


def test_perturbation_matrix(sysx):
    s = sysx
    G = s.ctx.perturbations(s.R).cpu().numpy().T
    assert rel(G, s.G) < 1e-12


# ---------------------------------------------------------------- Alg. 2
def test_compress_pivots_bit_exact(sysx):
    s = sysx
    for k in range(2):
        th, nu = s.draws(k, s.G.shape[1])
        S_o, Xi_o, qr = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
        S_g, Xi_g, n = s.ctx.compress(s.Psi_t, s.G_t, th, nu, id_eps=s.cfg.id_eps)
        assert n == len(S_o)
        assert np.array_equal(S_g.cpu().numpy(), S_o)
        assert rel(Xi_g.cpu().numpy().T, Xi_o) < 1e-9
        # fixed-N_mu mode (Table 1 style), odd count
        nf = max(3, (len(S_o) // 2) | 1)
        S_o2, Xi_o2, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, 0.0, n_fixed=nf)
        S_g2, Xi_g2, n2 = s.ctx.compress(s.Psi_t, s.G_t, th, nu, n_mu_fixed=nf)
        assert n2 == nf and np.array_equal(S_g2.cpu().numpy(), S_o2)
        assert rel(Xi_g2.cpu().numpy().T, Xi_o2) < 1e-9


@pytest.mark.parametrize("knob", ["ACP_QRCP_GRID", "ACP_QRCP_SMEM", "ACP_QRCP_GRID+ACP_QRCP_NOSMEM",
                                  "ACP_QRCP_GRID+ACP_QRCP_NOSMEM+ACP_QRCP_GRID16",
                                  "ACP_QRCP_GRID+ACP_QRCP_NOSMEM+ACP_QRCP_CHUNKED"])
def test_compress_alternative_qrcp_kernels_agree(sysx, monkeypatch, knob):
    """The QRCP kernels -- register-resident cluster (default for small problems), shared-memory
    cluster (ACP_QRCP_SMEM) and grid-wide persistent (ACP_QRCP_GRID; columns in shared memory, or
    in global memory with one warp per column (default for large m) or 16 lanes per column) --
    pick the same pivots and agree with the oracle."""
    from paper_1605_08021_b200 import Context
    s = sysx
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    for k in knob.split("+"):
        monkeypatch.setenv(k, "1")
    ctx = Context.from_config(s.cfg)
    S_g, Xi_g, n = ctx.compress(s.Psi_t, s.G_t, th, nu, id_eps=s.cfg.id_eps)
    ctx.close()
    assert np.array_equal(S_g.cpu().numpy(), S_o)
    assert rel(Xi_g.cpu().numpy().T, Xi_o) < 1e-9


# ---------------------------------------------------------------- Alg. 3
def test_apply_chi0_matches_direct_solves(sysx):
    s = sysx
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    W_o = oacp.compressed_W(s.m, s.H, s.gs.Psi, s.gs.eps[: s.cfg.n_occ], S_o, Xi_o, s.cfg.n_cheb)
    W_g, info = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, T(S_o, torch.int32), T(Xi_o.T), s.cfg.n_cheb,
                                 cg_tol=s.cfg.cg_tol)
    assert info["n_solved"] == s.cfg.n_cheb * len(S_o)
    assert info["max_rel_res"] <= s.cfg.cg_tol
    assert rel(W_g.cpu().numpy().T, W_o) < 1e-9


@pytest.mark.parametrize("n_cheb", [1, 3, 5])
def test_apply_chi0_node_counts(n_cheb):
    """N_c = 1, 3, 5 (one node group, uneven node groups over the streams, more groups than the
    default) against the oracle's direct compressed solves."""
    s = system("tiny4")
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    W_o = oacp.compressed_W(s.m, s.H, s.gs.Psi, s.gs.eps[: s.cfg.n_occ], S_o, Xi_o, n_cheb)
    W_g, info = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, T(S_o, torch.int32), T(Xi_o.T), n_cheb,
                                 cg_tol=s.cfg.cg_tol)
    assert info["n_solved"] == n_cheb * len(S_o)
    assert rel(W_g.cpu().numpy().T, W_o) < 1e-9


@pytest.mark.parametrize("sweep,order", [(1, 3), (2, 3), (1, 8), (3, 1)])
def test_apply_chi0_node_sweep_matches_direct_solves(sysx, monkeypatch, sweep, order):
    """The PCG node sweep (DESIGN reading R21: nodes solved group after group, later groups
    warm-started from the Lagrange extrapolation of the solved nodes; the default only for
    N_mu' >= 768) forced on the small systems: W against the oracle's direct compressed solves
    (Eq. eqncompressU / eqnW) at the same bar as the cold batch, every column converged, and fewer
    CG iterations than the cold batch."""
    s = sysx
    if s.cfg.n_cheb <= sweep:
        pytest.skip("needs more Chebyshev nodes than the group size")
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    W_o = oacp.compressed_W(s.m, s.H, s.gs.Psi, s.gs.eps[: s.cfg.n_occ], S_o, Xi_o, s.cfg.n_cheb)
    St, Xt = T(S_o, torch.int32), T(Xi_o.T)
    monkeypatch.setenv("ACP_PCG_SWEEP", "0")
    _, cold = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb, cg_tol=s.cfg.cg_tol)
    monkeypatch.setenv("ACP_PCG_SWEEP", str(sweep))
    monkeypatch.setenv("ACP_PCG_WARM_K", str(order))
    W_g, info = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb, cg_tol=s.cfg.cg_tol)
    assert info["n_solved"] == s.cfg.n_cheb * len(S_o)
    assert info["max_rel_res"] <= s.cfg.cg_tol
    assert rel(W_g.cpu().numpy().T, W_o) < 1e-9
    assert info["total_iter"] < cold["total_iter"], (info["total_iter"], cold["total_iter"])


def test_apply_chi0_node_sweep_sharding_is_bitwise(sysx, monkeypatch):
    """The warm start is per column (a column's guess uses only its own mu at the other nodes), so
    the RHS shards of the multi-GPU path reproduce the unsharded sweep bit for bit."""
    s = sysx
    if s.cfg.n_cheb < 2:
        pytest.skip("one node")
    monkeypatch.setenv("ACP_PCG_SWEEP", "1")
    th, nu = s.draws(1, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    St, Xt = T(S_o, torch.int32), T(Xi_o.T)
    W_full, _ = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    n = len(S_o)
    cut = (n // 2) & ~1
    W_sh = torch.zeros_like(W_full)
    s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb, mu_range=(0, cut), W=W_sh)
    s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb, mu_range=(cut, n), W=W_sh)
    assert torch.equal(W_full, W_sh)


def test_apply_chi0_sharding_is_bitwise(sysx):
    """RHS sharding across GPUs (even shard sizes) reproduces the unsharded W bit for bit."""
    s = sysx
    th, nu = s.draws(1, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    St, Xt = T(S_o, torch.int32), T(Xi_o.T)
    W_full, _ = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    n = len(S_o)
    cut = (n // 2) & ~1
    W_sh = torch.zeros_like(W_full)
    s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb, mu_range=(0, cut), W=W_sh)
    s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb, mu_range=(cut, n), W=W_sh)
    assert torch.equal(W_full, W_sh)


def test_smw_update_vs_oracle(sysx):
    """Eq. dyson4 alone with a random low-rank chi0~ = W Pi^T of rank N (several LU panels)."""
    s = sysx
    rng = np.random.default_rng(31)
    N = min(100, s.m.Ng // 2)
    S = np.sort(rng.choice(s.m.Ng, N, replace=False)).astype(np.int32)
    W = 1e-2 * rng.standard_normal((s.m.Ng, N))
    U_o, Gp_o, _ = oacp.smw_update(s.m, s.G, W, S)
    U_g, Gp_g = s.ctx.smw_update(s.G_t, T(S, torch.int32), T(W.T))
    assert rel(U_g.cpu().numpy().T, U_o) < 1e-11
    assert rel(Gp_g.cpu().numpy().T, Gp_o) < 1e-11


# ---------------------------------------------------------------- Alg. 4 + D
def _dyson_parity(s, n_outer=None):
    cfg = s.cfg
    n_outer = n_outer or cfg.n_outer
    res = oacp.acp_dyson(s.m, s.H, s.gs.Psi, s.gs.eps[: cfg.n_occ], s.G, cfg.n_cheb, n_outer, cfg.id_eps,
                         s.draws)
    D_o = ophonon.dynamical_matrix(s.m, s.gs.rho, s.G, res.U)
    lam_o = np.linalg.eigvalsh(D_o)
    n = s.G.shape[1]
    th = np.stack([s.draws(k, n)[0] for k in range(n_outer)])
    nu = np.stack([s.draws(k, n)[1] for k in range(n_outer)])
    U_g, info = s.ctx.dyson(s.Psi_t, s.eps_t, s.V_t, s.G_t, cfg.n_cheb, n_outer, th, nu, id_eps=cfg.id_eps,
                            cg_tol=cfg.cg_tol)
    assert info["n_mu"] == res.n_mu
    D_g, lam_g = s.ctx.dynamical_matrix(s.R, s.rho_t, s.G_t, U_g)
    return res, D_o, lam_o, U_g.cpu().numpy().T, D_g, lam_g, info


def test_dyson_deferred_checks_equal_synchronous(sysx, monkeypatch):
    """acp_dyson keeps PCG statistics, LU status and iteration differences on the device until the
    end (default) or synchronises after every stage (ACP_DYSON_SYNC): identical U and info."""
    from paper_1605_08021_b200 import Context
    s = sysx
    cfg = s.cfg
    n = s.G.shape[1]
    th = np.stack([s.draws(k, n)[0] for k in range(cfg.n_outer)])
    nu = np.stack([s.draws(k, n)[1] for k in range(cfg.n_outer)])
    args = (s.Psi_t, s.eps_t, s.V_t, s.G_t, cfg.n_cheb, cfg.n_outer, th, nu)
    U1, i1 = s.ctx.dyson(*args, id_eps=cfg.id_eps, cg_tol=cfg.cg_tol)
    monkeypatch.setenv("ACP_DYSON_SYNC", "1")
    ctx = Context.from_config(cfg)
    U2, i2 = ctx.dyson(*args, id_eps=cfg.id_eps, cg_tol=cfg.cg_tol)
    ctx.close()
    assert torch.equal(U1, U2)
    for key in i1:
        assert np.array_equal(np.asarray(i1[key]), np.asarray(i2[key])), key


def test_dyson_and_dynamical_matrix(sysx):
    s = sysx
    res, D_o, lam_o, U_g, D_g, lam_g, info = _dyson_parity(s)
    assert rel(U_g, res.U) < 1e-9
    assert rel(D_g, D_o) < 1e-8                       # north-star bar
    assert np.abs(lam_g - lam_o).max() / np.abs(lam_o).max() < 1e-7
    assert np.allclose(info["diff"], res.diff, rtol=1e-6, atol=1e-12)


def test_dynamical_matrix_terms_exact(sysx):
    """D assembly alone (given the oracle's U): pure rounding."""
    s = sysx
    U = ors.dyson_dense(s.m, ors.chi0_adler_wiser_matrix(s.m, s.H, s.cfg.n_occ), s.G)
    D_o = ophonon.dynamical_matrix(s.m, s.gs.rho, s.G, U)
    D_g, lam_g = s.ctx.dynamical_matrix(s.R, s.rho_t, s.G_t, T(U.T))
    assert rel(D_g, D_o) < 1e-11
    assert np.abs(lam_g - np.linalg.eigvalsh(D_o)).max() < 1e-12 * np.abs(lam_g).max()
    D4, _ = s.ctx.dynamical_matrix(s.R, s.rho_t, s.G_t, T(U.T), masses=4.0 * np.ones(s.m.NA))
    assert rel(D4, D_o / 4) < 1e-11


# ---------------------------------------------------------------- ground state
def test_ground_state(sysx):
    s = sysx
    out = s.ctx.ground_state(s.R, scf_tol=s.cfg.scf_tol)
    n = s.cfg.n_occ
    eps_g = out["eps"].cpu().numpy()
    assert np.abs(eps_g[: n + 1] - s.gs.eps[: n + 1]).max() < 1e-9
    assert rel(out["rho"].cpu().numpy(), s.gs.rho) < 1e-9
    assert rel(out["V"].cpu().numpy(), s.gs.V) < 1e-9
    assert rel(out["G"].cpu().numpy().T, s.G) < 1e-12
    Psi = out["Psi"].cpu().numpy().T
    assert np.abs(s.m.dV * Psi.T @ Psi - np.eye(n)).max() < 1e-10


@pytest.mark.slow
def test_compress_large_nmu_blocked_trsm():
    """configs[1] with a fixed N_mu = 200 > 160: the interpolation vectors go through the blocked
    upper-triangular solve (gathered [R11 | R12], bsub + DMMA GEMM)."""
    s = system("c1_1d_insulator")
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, 0.0, n_fixed=200)
    S_g, Xi_g, n = s.ctx.compress(s.Psi_t, s.G_t, th, nu, n_mu_fixed=200)
    assert n == 200 and np.array_equal(S_g.cpu().numpy(), S_o)
    assert rel(Xi_g.cpu().numpy().T, Xi_o) < 1e-8


def test_apply_chi0_hostloop_equals_while_node(sysx, monkeypatch):
    """The device-side while-node PCG loop and the host-driven replay (ACP_PCG_HOSTLOOP, used for
    ncu launch lists) run the same kernels in the same order: bitwise-identical W."""
    from paper_1605_08021_b200 import Context
    s = sysx
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    St, Xt = T(S_o, torch.int32), T(Xi_o.T)
    W1, i1 = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    monkeypatch.setenv("ACP_PCG_HOSTLOOP", "1")
    ctx = Context.from_config(s.cfg)
    W2, i2 = ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    ctx.close()
    assert torch.equal(W1, W2) and i1["total_iter"] == i2["total_iter"]


def test_apply_chi0_two_stream_groups_equal_one(sysx, monkeypatch):
    """The batch split into node groups on separate streams (default for small batches) and run
    as one group (ACP_PCG_GROUPS=1) give bitwise-identical W and iteration counts."""
    from paper_1605_08021_b200 import Context
    s = sysx
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    St, Xt = T(S_o, torch.int32), T(Xi_o.T)
    W1, i1 = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    monkeypatch.setenv("ACP_PCG_GROUPS", "1")
    ctx = Context.from_config(s.cfg)
    W2, i2 = ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    ctx.close()
    assert torch.equal(W1, W2) and i1["total_iter"] == i2["total_iter"]


def test_apply_chi0_node_parallel_W_equals_sequential(sysx, monkeypatch):
    """W built node-parallel + ordered sum (default for small problems) and node-sequential in one
    kernel (ACP_W_SEQ=1): the same additions in the same order, bitwise-identical W."""
    from paper_1605_08021_b200 import Context
    s = sysx
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    St, Xt = T(S_o, torch.int32), T(Xi_o.T)
    W1, _ = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    monkeypatch.setenv("ACP_W_SEQ", "1")
    ctx = Context.from_config(s.cfg)
    W2, _ = ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, St, Xt, s.cfg.n_cheb)
    ctx.close()
    assert torch.equal(W1, W2)


def test_apply_chi0_empty_shard(sysx):
    """An empty mu-range (a rank with no columns) is a no-op that leaves W untouched."""
    s = sysx
    th, nu = s.draws(0, s.G.shape[1])
    S_o, Xi_o, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    W = torch.full((len(S_o), s.m.Ng), 7.0, dtype=torch.float64, device="cuda")
    _, info = s.ctx.apply_chi0(s.Psi_t, s.eps_t, s.V_t, T(S_o, torch.int32), T(Xi_o.T), s.cfg.n_cheb,
                               mu_range=(1, 1), W=W)
    assert info["n_solved"] == 0 and bool(torch.all(W == 7.0))


def test_compress_capacity_error(sysx):
    """N_mu larger than the caller's capacity is reported (ACP_ERR_INVALID), not truncated."""
    from paper_1605_08021_b200 import AcpError
    s = sysx
    th, nu = s.draws(0, s.G.shape[1])
    S_o, _, _ = oacp.compress(s.m, s.gs.Psi, s.G, th, nu, s.cfg.id_eps)
    if len(S_o) < 2:
        pytest.skip("needs N_mu >= 2")
    with pytest.raises(AcpError):
        s.ctx.compress(s.Psi_t, s.G_t, th, nu, id_eps=s.cfg.id_eps, n_mu_max=len(S_o) - 1)


# ---------------------------------------------------------------- full size (bench config)
@pytest.mark.slow
def test_bench_config_end_to_end():
    """configs[1] at full size in the configuration bench.py times: GPU ground state ->
    GPU Alg. 4 -> GPU D, against the oracle's own pipeline."""
    s = system("c1_1d_insulator")
    res, D_o, lam_o, U_g, D_g, lam_g, info = _dyson_parity(s)
    assert rel(D_g, D_o) < 1e-8
    assert np.abs(lam_g - lam_o).max() / np.abs(lam_o).max() < 1e-7
    out = s.ctx.ground_state(s.R, scf_tol=s.cfg.scf_tol)
    assert rel(out["rho"].cpu().numpy(), s.gs.rho) < 1e-9


@pytest.mark.parametrize("mb", ["1", "2"])
@pytest.mark.parametrize("n", [32, 64, 128, 192, 256])
def test_fourier_operator_2d_fused(n, mb, monkeypatch):
    """Fused 2D K1 (fft2c.cu: persistent work queue of row / column / row items, transposes
    through a ring of L2-resident planes) on every supported square grid, both register budgets
    (ACP_F2C_MB), against numpy's fft2: kinetic and preconditioner symbols, Yukawa table,
    potential + per-column shifts, odd column counts (half-empty last pair); ACP_F2C_SKEW=1
    shrinks the queue skew and the ring (6 slots) so items wait on their producers and 21 pairs
    cycle through the ring slots."""
    from paper_1605_08021_b200 import Context
    monkeypatch.setenv("ACP_F2C_MB", mb)
    monkeypatch.setenv("ACP_F2C", "1")
    L0, L1 = 0.37 * n, 0.37 * n
    for skew in ("", "1"):
        if skew:
            monkeypatch.setenv("ACP_F2C_SKEW", skew)
        ctx = Context(2, (n, n), (L0, L1), 2, 2, 2.0, 2.0, 1.0, 0.01, 1.0)
        rng = np.random.default_rng(n)
        k0 = 2 * np.pi * np.fft.fftfreq(n, d=L0 / n)
        k1 = 2 * np.pi * np.fft.fftfreq(n, d=L1 / n)
        k2 = k0[:, None] ** 2 + k1[None, :] ** 2
        for ncol in ((1, 2, 9) if not skew else (41,)):
            X = rng.standard_normal((ncol, n, n))
            Xt = T(X.reshape(ncol, -1))
            F = np.fft.fft2(X)
            ref = np.real(np.fft.ifft2(F * (0.5 * k2)[None]))
            assert rel(ctx.fourier_apply(Xt, 0).cpu().numpy().reshape(ncol, n, n), ref) < 1e-12
            khat = 4 * np.pi / (1.0 * (k2 + 0.01 ** 2))
            ref = np.real(np.fft.ifft2(F * khat[None]))
            assert rel(ctx.fourier_apply(Xt, 1).cpu().numpy().reshape(ncol, n, n), ref) < 1e-12
            ref = np.real(np.fft.ifft2(F * (1.0 / (0.5 * k2 + 0.05))[None]))
            assert rel(ctx.fourier_apply(Xt, 2, tau=0.05).cpu().numpy().reshape(ncol, n, n), ref) < 1e-12
            V = rng.standard_normal(n * n)
            sh = rng.uniform(-0.2, 0.2, ncol)
            ref = np.real(np.fft.ifft2(F * (0.5 * k2)[None])).reshape(ncol, -1) + (V[None] - sh[:, None]) * X.reshape(ncol, -1)
            Y = ctx.fourier_apply(Xt, 0, diag=T(V), shift=T(sh)).cpu().numpy()
            assert rel(Y, ref) < 1e-12
        ctx.close()


def test_fused_2d_matches_three_pass(monkeypatch):
    """The fused kernel and the three-pass kernels (ACP_F2C=0) agree to rounding on tiny2d's
    full Alg. 4 (PCG masks and dots inside the solves)."""
    from paper_1605_08021_b200 import Context
    s = system("tiny2d")
    cfg = s.cfg
    n = s.G.shape[1]
    th = np.stack([s.draws(k, n)[0] for k in range(cfg.n_outer)])
    nu = np.stack([s.draws(k, n)[1] for k in range(cfg.n_outer)])
    args = (s.Psi_t, s.eps_t, s.V_t, s.G_t, cfg.n_cheb, cfg.n_outer, th, nu)
    U1, i1 = s.ctx.dyson(*args, id_eps=cfg.id_eps, cg_tol=cfg.cg_tol)
    monkeypatch.setenv("ACP_F2C", "0")
    ctx = Context.from_config(cfg)
    U2, i2 = ctx.dyson(*args, id_eps=cfg.id_eps, cg_tol=cfg.cg_tol)
    ctx.close()
    assert i1["n_mu"] == i2["n_mu"]
    assert rel(U1.cpu().numpy(), U2.cpu().numpy()) < 1e-9
