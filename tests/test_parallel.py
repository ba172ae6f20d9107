"""Multi-rank host logic of the RHS-sharded Alg. 4 (paper_1605_08021_b200/parallel.py) on CPU.

world_size 2 over gloo; the per-rank compute is the oracle (a CPU stand-in with the
Context method signatures), so this checks the shard bounds, the padded all-gather of W
and the replicated SMW update -- the same host code bench.py runs over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1605_08021_b200.parallel import shard_bounds


def test_shard_bounds_cover_and_even():
    for n in (1, 2, 7, 8, 33, 162):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b, e, chunk = shard_bounds(n, r, world)
                assert chunk % 2 == 0 and e - b <= chunk
                assert e == b or b % 2 == 0  # FFT column pairs never straddle two ranks
                seen.extend(range(b, e))
            assert seen == list(range(n))


class OracleOps:
    """CPU stand-in for paper_1605_08021_b200.acp.Context (tensors are (n, N_g) row-per-column)."""

    def __init__(self, m, H):
        self.m, self.H = m, H

    def compress(self, Psi, Gp, theta, nu, id_eps=1e-3):
        from oracle import acp as oacp
        S, Xi, _ = oacp.compress(self.m, Psi.T.numpy(), Gp.T.numpy(), theta, nu, id_eps)
        return torch.from_numpy(S.astype(np.int32)), torch.from_numpy(np.ascontiguousarray(Xi.T)), len(S)

    def apply_chi0(self, Psi, eps, V, S, Xi, n_cheb, cg_tol=1e-11, mu_range=None, W=None):
        from oracle import acp as oacp
        b, e = mu_range
        Wl = oacp.compressed_W(self.m, self.H, Psi.T.numpy(), eps.numpy(), S.numpy()[b:e],
                               Xi.T.numpy()[:, b:e], n_cheb)
        W[b:e] = torch.from_numpy(np.ascontiguousarray(Wl.T))
        return W, {"n_solved": n_cheb * (e - b)}

    # -- sharded compression: a numpy restatement of the k_qrs_step protocol (qrcp.cu) ----------
    def qrs_begin(self, Psi, Gp, theta, nu, a, b, n_mu_fixed=0):
        from oracle import acp as oacp
        Gt = oacp.srft_sketch(Gp.T.numpy(), theta, nu)
        Mt = oacp.sketch_matrix(Psi.T.numpy(), Gt)            # (N_g, m)
        self.qm = Mt.shape[1]
        self.a, self.b = a, b
        self.A = np.ascontiguousarray(Mt[a:b].T)              # m x n_loc, owned grid points
        self.pos = np.arange(a, b)
        self.dn = np.zeros(b - a, dtype=bool)
        self.n2 = np.einsum("ij,ij->j", self.A, self.A)
        self.kmax = min(self.qm, Mt.shape[0]) if n_mu_fixed <= 0 else min(self.qm, Mt.shape[0], n_mu_fixed)
        self.fixed = n_mu_fixed
        self.stop, self.N, self.r11 = False, 0, 0.0
        self.R11 = np.zeros((self.kmax, self.kmax))
        self.piv = []
        return self.qm

    def qrs_step(self, s, recv, world, id_eps, send):
        if self.stop:
            return
        m = self.qm
        if s > 0:
            j = s - 1
            cands = recv.numpy().reshape(world, m + 3)
            best = None
            for c in cands:
                if c[0] >= 0 and (best is None or c[0] > best[0] or (c[0] == best[0] and c[1] < best[1])):
                    best = c
            rjj = np.sqrt(max(best[0], 0.0)) if best is not None else 0.0
            r11 = rjj if j == 0 else self.r11
            if best is None or rjj == 0.0 or (self.fixed <= 0 and rjj < id_eps * r11):
                self.stop, self.N = True, j
                return
            if j == 0:
                self.r11 = rjj
            bp, cw, x = int(best[1]), int(best[2]), best[3:]
            xn = np.linalg.norm(x[j:])
            alpha = -xn if x[j] >= 0 else xn
            v = x[j:].copy()
            v[0] -= alpha
            tau = 2.0 / (v @ v)
            self.R11[:j, j] = x[:j]
            self.R11[j, j] = alpha
            self.piv.append(cw)
            for lc in range(self.b - self.a):
                g = self.a + lc
                if g == cw:
                    self.pos[lc], self.dn[lc] = j, True
                    self.A[j:, lc] = 0.0
                    self.A[j, lc] = alpha
                elif not self.dn[lc]:
                    if self.pos[lc] == j:
                        self.pos[lc] = bp
                    c = self.A[j:, lc]
                    c -= tau * v * (v @ c)
                    self.n2[lc] = c[1:] @ c[1:]
        if s >= self.kmax:
            self.stop, self.N = True, s
            return
        live = np.nonzero(~self.dn)[0]
        out = np.zeros(m + 3)
        out[0] = -1.0
        if len(live):
            order = sorted(live, key=lambda lc: (-self.n2[lc], self.pos[lc]))
            lc = order[0]
            out[0], out[1], out[2] = self.n2[lc], self.pos[lc], self.a + lc
            out[3:] = self.A[:, lc]
        send.copy_(torch.from_numpy(out))

    def qrs_status(self):
        return self.stop, self.N

    def qrs_finish(self):
        import scipy.linalg as sla
        N = self.N
        T = sla.solve_triangular(self.R11[:N, :N], self.A[:N, :], lower=False) if self.b > self.a else \
            np.zeros((N, 0))
        XiT = T.T.copy()
        for lc in range(self.b - self.a):
            if self.dn[lc] and self.pos[lc] < N:
                XiT[lc] = 0.0
                XiT[lc, self.pos[lc]] = 1.0
        return torch.tensor(self.piv[:N], dtype=torch.int32), torch.from_numpy(XiT), N

    def smw_update(self, G, S, W):
        from oracle import acp as oacp
        U, Gp, _ = oacp.smw_update(self.m, G.T.numpy(), W.T.numpy(), S.numpy())
        return torch.from_numpy(np.ascontiguousarray(U.T)), torch.from_numpy(np.ascontiguousarray(Gp.T))


def _system():
    from workloads import atom_positions
    from workloads.configs import small_config
    from oracle.model import Model
    from oracle.scf import scf
    cfg = small_config()
    m = Model(cfg, atom_positions(cfg))
    gs = scf(m, tol=1e-13)
    return cfg, m, gs


def _worker(rank, world, port, out, shard_compress=None):
    from workloads import sketch_draws
    from paper_1605_08021_b200.parallel import dyson_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg, m, gs = _system()
        H = m.hamiltonian_dense(gs.V)
        G = torch.from_numpy(np.ascontiguousarray(m.G_matrix().T))
        Psi = torch.from_numpy(np.ascontiguousarray(gs.Psi.T))
        eps = torch.from_numpy(gs.eps[: cfg.n_occ].copy())
        V = torch.from_numpy(gs.V.copy())
        U, info = dyson_sharded(OracleOps(m, H), Psi, eps, V, G, cfg.n_cheb, cfg.n_outer,
                                lambda k: sketch_draws(cfg.seed, k, G.shape[0], cfg.sketch_r), cfg.id_eps,
                                shard_compress=shard_compress)
        out[rank] = (U.numpy().copy(), info["shards"], info["local_solves"], info["n_mu"], info["compression"])
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _compress_worker(rank, world, port, out, fixed):
    from workloads import sketch_draws
    from paper_1605_08021_b200.parallel import compress_sharded
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg, m, gs = _system()
        G = torch.from_numpy(np.ascontiguousarray(m.G_matrix().T))
        Psi = torch.from_numpy(np.ascontiguousarray(gs.Psi.T))
        th, nu = sketch_draws(cfg.seed, 0, G.shape[0], cfg.sketch_r)
        S, Xi, n = compress_sharded(OracleOps(m, None), Psi, G, th, nu, cfg.id_eps, n_mu_fixed=fixed)
        out[rank] = (S.numpy().copy(), Xi.numpy().copy(), n)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,fixed", [(2, 0), (3, 0), (2, 10)])
def test_compress_sharded_matches_one_rank(world, fixed):
    """The sharded pivoted QR protocol (parallel.compress_sharded: per-pivot all-gather of the
    ranks' best columns, replicated winner selection, per-rank rows of Xi) over gloo reproduces the
    one-rank factorisation of the oracle: identical pivots and N_mu on every
    rank, Xi to rounding; N_mu by the threshold rule and fixed."""
    from workloads import sketch_draws
    from oracle import acp as oacp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_compress_worker, args=(world, _free_port(), out, fixed), nprocs=world, join=True,
                       start_method="fork")
    cfg, m, gs = _system()
    G = m.G_matrix()
    th, nu = sketch_draws(cfg.seed, 0, G.shape[1], cfg.sketch_r)
    S_o, Xi_o, _ = oacp.compress(m, gs.Psi, G, th, nu, cfg.id_eps, n_fixed=fixed or None)
    for r in range(world):
        S, Xi, n = out[r]
        assert n == len(S_o)
        assert np.array_equal(S, S_o)
        assert np.abs(Xi.T - Xi_o).max() < 1e-10 * np.abs(Xi_o).max()


def test_use_sharded_compress_rule():
    """None = the measured rule (replicated up to one 8-rank NVSwitch node); explicit values win."""
    from paper_1605_08021_b200.parallel import REPLICATED_COMPRESS_MAX_WORLD, use_sharded_compress
    assert REPLICATED_COMPRESS_MAX_WORLD == 8
    assert [use_sharded_compress(w) for w in (1, 2, 8, 9, 16)] == [False, False, False, True, True]
    assert use_sharded_compress(2, True) and not use_sharded_compress(16, False)


@pytest.mark.parametrize("shard_compress,mode", [(True, "sharded"), (False, "replicated"), (None, "replicated")])
def test_dyson_sharded_two_ranks_matches_single_process(shard_compress, mode):
    from workloads import sketch_draws
    from oracle import acp as oacp
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out, shard_compress), nprocs=world, join=True,
                       start_method="fork")
    cfg, m, gs = _system()
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    ref = oacp.acp_dyson(m, H, gs.Psi, gs.eps[: cfg.n_occ], G, cfg.n_cheb, cfg.n_outer, cfg.id_eps,
                         lambda k, n: sketch_draws(cfg.seed, k, n, cfg.sketch_r))
    U0, sh0, ns0, nmu0, mode0 = out[0]
    U1, sh1, ns1, nmu1, mode1 = out[1]
    assert mode0 == mode1 == mode
    assert nmu0 == nmu1 == ref.n_mu
    assert np.array_equal(U0, U1)                      # replicated SMW: identical on every rank
    assert np.abs(U0.T - ref.U).max() <= 1e-12 * np.abs(ref.U).max()
    # the two shards cover every mu of every outer iteration exactly once
    assert ns0 + ns1 == cfg.n_cheb * sum(ref.n_mu)
    for k, n in enumerate(ref.n_mu):
        (b0, e0), (b1, e1) = sh0[k], sh1[k]
        assert b0 == 0 and e0 == b1 and e1 == n
