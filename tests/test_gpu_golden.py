"""Full-size end-to-end parity (configs[2], configs[3] as c3g, configs[4] as c4g): the CUDA path,
fed the oracle's ground state, against the oracle's own Alg. 4 + D on that state.

The oracle side is tools/make_golden.py (dense oracle for configs[2]; for the 2D grids the
matrix-free oracle of oracle/iterative.py -- LOBPCG SCF, MINRES Sternheimer -- pinned to the dense
oracle in tests/test_oracle_iterative.py).  Its results are committed under tests/golden/
(<config>_acp.npz: per-outer N_mu, pivots S, ||U^k - U^{k-1}||, W on a seeded mu-sample, D,
lambda, digest of the input arrays); the ground state it ran on (Psi, eps, V, rho: up to 134 MB)
is the INPUT both sides consume: tests/golden/<config>_gs.npz (committed, configs[2] and c3g: 5 and 19
MB, so the round-end GPU run and a fresh container have it) or tests/cache/<config>_gs.npz (c4g: 134
MB, git-ignored; the same script writes it).

Bars: pivots and N_mu bit-exact (discrete decisions, both sides decide in
fp64); W on the mu-sample 1e-9 relative (CG tolerance 1e-11 x conditioning); D 1e-8 relative and
lambda 1e-7 relative to max|lambda| (north_star)."""
import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import atom_positions, get_config, sketch_draws  # noqa: E402
from oracle.model import Model  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def T(x, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda").contiguous()


def _gs_path(name):
    """The oracle ground state a golden run consumed: committed under tests/golden/ when small
    enough, else the git-ignored cache (tools/make_golden.py writes both)."""
    for d in ("golden", "cache"):
        p = os.path.join(ROOT, "tests", d, f"{name}_gs.npz")
        if os.path.exists(p):
            return p
    return os.path.join(ROOT, "tests", "cache", f"{name}_gs.npz")


def _load(name):
    gold_p = os.path.join(ROOT, "tests", "golden", f"{name}_acp.npz")
    gs_p = _gs_path(name)
    if not os.path.exists(gold_p):
        pytest.skip(f"no golden file for {name} (run tools/make_golden.py {name})")
    if not os.path.exists(gs_p):
        pytest.skip(f"no cached oracle ground state for {name} (run tools/make_golden.py {name})")
    gold = np.load(gold_p)
    gs = np.load(gs_p)
    h = hashlib.sha256()
    for k in ("Psi", "eps", "V", "rho", "R"):
        h.update(np.ascontiguousarray(gs[k]).tobytes())
    assert h.hexdigest()[:32] == str(gold["input_digest"]), "cached ground state is not the golden run's input"
    return gold, gs


def _outer_only(gold) -> bool:
    import json
    return bool(json.loads(str(gold["meta"])).get("outer_only", 0))


@pytest.mark.parametrize("name", ["c2_1d_semiconductor", "c3g_2d_8x8"])
def test_full_size_alg4_and_D(name):
    from paper_1605_08021_b200 import Context
    gold, gs = _load(name)
    assert not _outer_only(gold)
    cfg = get_config(name)
    R = atom_positions(cfg)
    assert np.array_equal(R, gs["R"])
    m = Model(cfg, R)
    G = m.G_matrix()
    ctx = Context.from_config(cfg)
    Psi_t, eps_t, V_t, rho_t, G_t = T(gs["Psi"].T), T(gs["eps"]), T(gs["V"]), T(gs["rho"]), T(G.T)
    n = G.shape[1]
    n_mu = [int(x) for x in gold["n_mu"]]
    S_all = gold["S"]
    offs = np.concatenate([[0], np.cumsum(n_mu)])
    draws = [sketch_draws(cfg.seed, k, n, cfg.sketch_r) for k in range(cfg.n_outer)]

    # ---- Alg. 4 step by step through the C ABI: pivots and W of every outer iteration
    Gp = G_t.clone()
    U = None
    for k in range(cfg.n_outer):
        th, nu = draws[k]
        S, Xi, nk = ctx.compress(Psi_t, Gp, th, nu, id_eps=cfg.id_eps)
        assert nk == n_mu[k], (k, nk, n_mu[k])
        assert np.array_equal(S.cpu().numpy(), S_all[offs[k]:offs[k + 1]]), f"pivots differ at outer {k}"
        W, info = ctx.apply_chi0(Psi_t, eps_t, V_t, S, Xi, cfg.n_cheb, cg_tol=cfg.cg_tol)
        idx = gold[f"W{k}_idx"]
        Ws = W[torch.as_tensor(idx, device="cuda")].cpu().numpy().T
        assert rel(Ws, gold[f"W{k}"]) < 1e-9, (k, rel(Ws, gold[f"W{k}"]))
        del Xi
        U, Gp = ctx.smw_update(G_t, S, W)
        del W
    D, lam = ctx.dynamical_matrix(R, rho_t, G_t, U)
    assert rel(D, gold["D"]) < 1e-8, rel(D, gold["D"])
    assert np.abs(lam - gold["lam"]).max() / np.abs(gold["lam"]).max() < 1e-7
    del U, Gp

    # ---- the same through the one-call acp_dyson (the path bench.py times)
    th = np.stack([d[0] for d in draws])
    nu = np.stack([d[1] for d in draws])
    U2, info = ctx.dyson(Psi_t, eps_t, V_t, G_t, cfg.n_cheb, cfg.n_outer, th, nu, id_eps=cfg.id_eps,
                         cg_tol=cfg.cg_tol)
    assert info["n_mu"] == n_mu
    D2, lam2 = ctx.dynamical_matrix(R, rho_t, G_t, U2)
    assert rel(D2, gold["D"]) < 1e-8, rel(D2, gold["D"])
    assert np.abs(lam2 - gold["lam"]).max() / np.abs(gold["lam"]).max() < 1e-7
    assert np.allclose(info["diff"], gold["diff"], rtol=1e-6)
    ctx.close()


def test_full_size_c4g_outer0():
    """configs[4] (as c4g): the oracle's full Alg. 4 needs ~85k MINRES solves on the 256^2 grid
    (days of host CPU), so its golden run (tools/make_golden.py --outer-only 1) holds outer
    iteration 0 only: Alg. 2 on G' = G at m = N_occ r = 4096 (pivots and N_mu bit-exact) and
    Eq. eqncompressU + Eq. eqnW on the seeded mu-sample (W to 1e-9) -- the production path
    bench.py times (structured Kronecker QRCP, fused 2D K1, K2/K3 at N_occ = 256)."""
    from paper_1605_08021_b200 import Context
    name = "c4g_2d_16x16"
    gold, gs = _load(name)
    assert _outer_only(gold)
    cfg = get_config(name)
    R = atom_positions(cfg)
    assert np.array_equal(R, gs["R"])
    G = Model(cfg, R).G_matrix()
    ctx = Context.from_config(cfg)
    Psi_t, eps_t, V_t = T(gs["Psi"].T), T(gs["eps"]), T(gs["V"])
    th, nu = sketch_draws(cfg.seed, 0, G.shape[1], cfg.sketch_r)
    S, Xi, nk = ctx.compress(Psi_t, T(G.T), th, nu, id_eps=cfg.id_eps)
    assert nk == int(gold["n_mu"][0]), (nk, int(gold["n_mu"][0]))
    assert np.array_equal(S.cpu().numpy(), gold["S"]), "pivots differ at outer 0"
    idx = torch.as_tensor(gold["W0_idx"], device="cuda")
    # the sampled mu-columns only (their solves are independent of the other columns')
    W, info = ctx.apply_chi0(Psi_t, eps_t, V_t, S[idx].contiguous(), Xi[idx].contiguous(), cfg.n_cheb,
                             cg_tol=cfg.cg_tol)
    assert rel(W.cpu().numpy().T, gold["W0"]) < 1e-9, rel(W.cpu().numpy().T, gold["W0"])
    ctx.close()


@pytest.mark.parametrize("dense", [False, True])
@pytest.mark.parametrize("n_occ,Ng", [(64, 2400), (256, 3000)])
def test_qrcp_pivots_full_m(n_occ, Ng, dense, monkeypatch):
    """Alg. 2 steps 2-3 at the sketch heights of configs[3] / configs[4],
    m = N_occ r = 1024 and 4096, seeded inputs, 160 pivots -- bit-exact pivots and Xi to 1e-9
    against the oracle's QRCP: the structured Kronecker QRCP (default, qrcp_kron.cu) and the
    formed-sketch persistent kernels (ACP_QRCP_DENSE: rows in registers at m = 1024, eight
    512-row chunks per column at m = 4096)."""
    from paper_1605_08021_b200 import Context
    from oracle import acp as oacp
    monkeypatch.setenv("ACP_QRCP_DENSE" if dense else "ACP_QRCP_KRON", "1")
    rng = np.random.default_rng(n_occ)
    n_pert = 40
    Psi = rng.standard_normal((Ng, n_occ))
    Gp = rng.standard_normal((Ng, n_pert))
    th = rng.random(n_pert)
    nu = (rng.choice(n_pert, size=8, replace=False) + 1).astype(np.int32)
    ctx = Context(1, (Ng,), (0.5 * Ng,), n_pert, n_occ, 2.0, 2.0, 1.0, 0.01, 10.0)
    S_g, Xi_g, nk = ctx.compress(T(Psi.T), T(Gp.T), th, nu, n_mu_fixed=160)
    Gt = oacp.srft_sketch(Gp, th, nu)
    Mt = oacp.sketch_matrix(Psi, Gt)
    assert Mt.shape == (Ng, n_occ * 16)
    qr = oacp.qrcp(Mt.T, 0.0, n_fixed=160)
    S_o, Xi_o = oacp.interpolation_vectors(qr, Ng)
    assert nk == 160
    assert np.array_equal(S_g.cpu().numpy(), S_o)
    assert rel(Xi_g.cpu().numpy().T, Xi_o) < 1e-9
    ctx.close()


@pytest.mark.parametrize("name", ["c2_1d_semiconductor", "c3g_2d_8x8"])
def test_kronecker_qrcp_equals_formed_sketch_qrcp(name, monkeypatch):
    """The structured QRCP (screening by downdated norms, exact verification of the candidates,
    CGS2) and the formed-sketch persistent kernel (exact norms every step) on the configs' own
    ground states: identical pivots and N_mu, Xi to 1e-10."""
    from paper_1605_08021_b200 import Context
    gs_p = _gs_path(name)
    if not os.path.exists(gs_p):
        pytest.skip("no cached oracle ground state")
    gs = np.load(gs_p)
    cfg = get_config(name)
    R = atom_positions(cfg)
    G = Model(cfg, R).G_matrix()
    th, nu = sketch_draws(cfg.seed, 0, G.shape[1], cfg.sketch_r)
    monkeypatch.setenv("ACP_QRCP_KRON", "1")
    ctx = Context.from_config(cfg)
    S1, Xi1, n1 = ctx.compress(T(gs["Psi"].T), T(G.T), th, nu, id_eps=cfg.id_eps)
    monkeypatch.delenv("ACP_QRCP_KRON")
    monkeypatch.setenv("ACP_QRCP_DENSE", "1")
    ctx2 = Context.from_config(cfg)
    S2, Xi2, n2 = ctx2.compress(T(gs["Psi"].T), T(G.T), th, nu, id_eps=cfg.id_eps)
    assert n1 == n2 and torch.equal(S1, S2)
    assert rel(Xi1.cpu().numpy(), Xi2.cpu().numpy()) < 1e-10
    ctx.close()
    ctx2.close()
