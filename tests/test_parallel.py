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


def _worker(rank, world, port, out):
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
                                lambda k: sketch_draws(cfg.seed, k, G.shape[0], cfg.sketch_r), cfg.id_eps)
        out[rank] = (U.numpy().copy(), info["shards"], info["local_solves"], info["n_mu"])
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dyson_sharded_two_ranks_matches_single_process():
    from workloads import sketch_draws
    from oracle import acp as oacp
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="fork")
    cfg, m, gs = _system()
    H = m.hamiltonian_dense(gs.V)
    G = m.G_matrix()
    ref = oacp.acp_dyson(m, H, gs.Psi, gs.eps[: cfg.n_occ], G, cfg.n_cheb, cfg.n_outer, cfg.id_eps,
                         lambda k, n: sketch_draws(cfg.seed, k, n, cfg.sketch_r))
    U0, sh0, ns0, nmu0 = out[0]
    U1, sh1, ns1, nmu1 = out[1]
    assert nmu0 == nmu1 == ref.n_mu
    assert np.array_equal(U0, U1)                      # replicated SMW: identical on every rank
    assert np.abs(U0.T - ref.U).max() <= 1e-12 * np.abs(ref.U).max()
    # the two shards cover every mu of every outer iteration exactly once
    assert ns0 + ns1 == cfg.n_cheb * sum(ref.n_mu)
    for k, n in enumerate(ref.n_mu):
        (b0, e0), (b1, e1) = sh0[k], sh1[k]
        assert b0 == 0 and e0 == b1 and e1 == n
