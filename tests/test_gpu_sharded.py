"""GPU checks of the multi-GPU path (paper_1605_08021_b200/parallel.py) on the one GPU available:

* the sharded pivoted QR kernels (acp_qrs_*) with 2 and 3 ranks EMULATED in one process: each
  rank is its own Context (own column block, own workspace); the all-gather between pivot steps
  is a concatenation of the ranks' send buffers.  The ranks' kernels run one after another and
  never wait on each other (B200_PROFILING.md: no inter-launch spinning on one GPU);
* the real NCCL path at world size 1 (process group over NCCL, all_gather_into_tensor): the
  sharded compression and the sharded Alg. 4 against the one-call acp_compress / acp_dyson.
Pivots bit-exact (discrete decisions), Xi to rounding."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import atom_positions, get_config, sketch_draws  # noqa: E402
from workloads.configs import small_config, small_config_2d  # noqa: E402
from oracle.model import Model  # noqa: E402
from oracle.scf import scf  # noqa: E402
from oracle import acp as oacp  # noqa: E402


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def T(x, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda").contiguous()


def _emulated_compress(ctxs, Psi, Gp, th, nu, id_eps, n_mu_fixed=0):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        out = _emulated_loop(ctxs, Psi, Gp, th, nu, id_eps, n_mu_fixed, st)
    torch.cuda.current_stream().wait_stream(st)
    return out


def _emulated_loop(ctxs, Psi, Gp, th, nu, id_eps, n_mu_fixed, st):
    from paper_1605_08021_b200.parallel import grid_bounds
    world = len(ctxs)
    Ng = Psi.shape[1]
    for c in ctxs:
        c.set_stream(st)  # the ranks' kernels and the torch.cat "all-gather" in one stream order
    bounds = [grid_bounds(Ng, r, world) for r in range(world)]
    ms = [c.qrs_begin(Psi, Gp, th, nu, b[0], b[1], n_mu_fixed=n_mu_fixed) for c, b in zip(ctxs, bounds)]
    m = ms[0]
    sends = [torch.zeros(m + 3, dtype=torch.float64, device="cuda") for _ in range(world)]
    recv = torch.zeros(world * (m + 3), dtype=torch.float64, device="cuda")
    s = 0
    while True:
        for c, snd in zip(ctxs, sends):
            c.qrs_step(s, recv, world, id_eps, snd)
        st = [c.qrs_status() for c in ctxs]
        assert len(set(st)) == 1, st          # every rank decides the stop identically
        if st[0][0]:
            break
        recv = torch.cat(sends)
        s += 1
    outs = [c.qrs_finish() for c in ctxs]
    S = outs[0][0]
    for o in outs[1:]:
        assert torch.equal(o[0], S)
    Xi = torch.cat([o[1] for o in outs]).t().contiguous()
    return S, Xi, outs[0][2]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["tiny4", "c0_1d_tiny", "tiny2d", "c1_1d_insulator"])
def test_sharded_qrcp_emulated_ranks(name, world):
    from paper_1605_08021_b200 import Context
    cfg = {"tiny4": small_config, "tiny2d": small_config_2d}.get(name, lambda: get_config(name))()
    R = atom_positions(cfg)
    m = Model(cfg, R)
    gs = scf(m, tol=cfg.scf_tol)
    G = m.G_matrix()
    th, nu = sketch_draws(cfg.seed, 0, G.shape[1], cfg.sketch_r)
    S_o, Xi_o, _ = oacp.compress(m, gs.Psi, G, th, nu, cfg.id_eps)
    ctxs = [Context.from_config(cfg) for _ in range(world)]
    S, Xi, n = _emulated_compress(ctxs, T(gs.Psi.T), T(G.T), th, nu, cfg.id_eps)
    assert n == len(S_o)
    assert np.array_equal(S.cpu().numpy(), S_o)
    assert rel(Xi.cpu().numpy().T, Xi_o) < 1e-9
    # the one-rank kernel path of acp_compress agrees too
    S1, Xi1, n1 = ctxs[0].compress(T(gs.Psi.T), T(G.T), th, nu, id_eps=cfg.id_eps)
    assert n1 == n and torch.equal(S1, S)
    assert rel(Xi.cpu().numpy(), Xi1.cpu().numpy()) < 1e-10
    for c in ctxs:
        c.close()


def test_sharded_qrcp_full_m_emulated():
    """m = 4096 (configs[4]'s sketch height: the chunked update) over 2 emulated ranks, fixed
    N_mu = 96 on seeded inputs, against the oracle's QRCP."""
    from paper_1605_08021_b200 import Context
    rng = np.random.default_rng(4)
    Ng, n_occ, n_pert = 3000, 256, 40
    Psi = rng.standard_normal((Ng, n_occ))
    Gp = rng.standard_normal((Ng, n_pert))
    th = rng.random(n_pert)
    nu = (rng.choice(n_pert, size=8, replace=False) + 1).astype(np.int32)
    ctxs = [Context(1, (Ng,), (0.5 * Ng,), n_pert, n_occ, 2.0, 2.0, 1.0, 0.01, 10.0) for _ in range(2)]
    S, Xi, n = _emulated_compress(ctxs, T(Psi.T), T(Gp.T), th, nu, 0.0, n_mu_fixed=96)
    qr = oacp.qrcp(oacp.sketch_matrix(Psi, oacp.srft_sketch(Gp, th, nu)).T, 0.0, n_fixed=96)
    S_o, Xi_o = oacp.interpolation_vectors(qr, Ng)
    assert n == 96 and np.array_equal(S.cpu().numpy(), S_o)
    assert rel(Xi.cpu().numpy().T, Xi_o) < 1e-9
    for c in ctxs:
        c.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda:0"))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c0_1d_tiny", "tiny2d"])
def test_nccl_world1_sharded_alg4(name, nccl_world1):
    """The production multi-GPU code (NCCL all_gather_into_tensor for the pivot candidates, Xi and
    W) at world size 1: identical N_mu / pivots and U to rounding vs the one-call acp_dyson."""
    from paper_1605_08021_b200 import Context
    from paper_1605_08021_b200.parallel import compress_sharded, dyson_sharded
    cfg = {"tiny2d": small_config_2d}.get(name, lambda: get_config(name))()
    R = atom_positions(cfg)
    m = Model(cfg, R)
    gs = scf(m, tol=cfg.scf_tol)
    G = m.G_matrix()
    ctx = Context.from_config(cfg)
    Psi, eps, V, Gt = T(gs.Psi.T), T(gs.eps), T(gs.V), T(G.T)
    th, nu = sketch_draws(cfg.seed, 0, G.shape[1], cfg.sketch_r)
    S, Xi, n = compress_sharded(ctx, Psi, Gt, th, nu, cfg.id_eps)
    S1, Xi1, n1 = ctx.compress(Psi, Gt, th, nu, id_eps=cfg.id_eps)
    assert n == n1 and torch.equal(S, S1)
    assert rel(Xi.cpu().numpy(), Xi1.cpu().numpy()) < 1e-10
    dr = [sketch_draws(cfg.seed, k, G.shape[1], cfg.sketch_r) for k in range(cfg.n_outer)]
    U, info = dyson_sharded(ctx, Psi, eps, V, Gt, cfg.n_cheb, cfg.n_outer, lambda k: dr[k], cfg.id_eps,
                            cfg.cg_tol, shard_compress=True)
    assert info["compression"] == "sharded"
    Ur, infor = dyson_sharded(ctx, Psi, eps, V, Gt, cfg.n_cheb, cfg.n_outer, lambda k: dr[k], cfg.id_eps,
                              cfg.cg_tol)   # the default rule at world 1: replicated compression
    assert infor["compression"] == "replicated" and infor["n_mu"] == info["n_mu"]
    U1, info1 = ctx.dyson(Psi, eps, V, Gt, cfg.n_cheb, cfg.n_outer, np.stack([d[0] for d in dr]),
                          np.stack([d[1] for d in dr]), id_eps=cfg.id_eps, cg_tol=cfg.cg_tol)
    assert info["n_mu"] == info1["n_mu"]
    assert rel(U.cpu().numpy(), U1.cpu().numpy()) < 1e-9
    assert rel(Ur.cpu().numpy(), U1.cpu().numpy()) < 1e-9
    ctx.close()
