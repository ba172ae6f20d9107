"""Multi-GPU layer: Alg. 4 with the compressed Sternheimer right-hand sides sharded across ranks
(one process per GPU) and the compression either sharded by grid point or replicated
(use_sharded_compress: replicated up to 8 ranks, where the one-GPU Kronecker QRCP beats the
per-pivot protocol); exchanges over NCCL (NVLink).

* Compression (Alg. 2): rank r owns the grid points [a_r, b_r) -- the columns
  of M~^T.  Each pivot step is one kernel on every rank plus ONE all-gather of the ranks' best
  remaining columns (m + 3 doubles each); every rank then selects the same winner (largest norm,
  lowest position on ties), so the pivots and N_mu equal the one-rank factorisation's.  Each rank
  solves for its own rows of Xi; one all-gather assembles Xi (N_g x N_mu).
* Sternheimer solves: the N_c x N_mu equations are independent; rank r solves
  the mu-columns [b_r, e_r) for all Chebyshev nodes and produces those columns of W (Eq. eqnW);
  one all-gather (straight into the gathered buffer) assembles W.
* The SMW update (Eq. dyson4) is an N_mu x N_mu solve: replicated (deterministic, same inputs),
  so every rank holds the same U after each iteration.
Shard boundaries of W are even, so column pairs of the FFT kernel -- and therefore every
per-column result -- are identical to the single-GPU run.
"""
from __future__ import annotations

from typing import Callable, Tuple

import torch
import torch.distributed as dist

CHECK_EVERY = 32   # pivot steps between stop-flag reads (later steps are device no-ops)

# Ranks up to which the compression runs REPLICATED on every rank (the one-GPU Kronecker QRCP /
# cluster QRCP) rather than with the per-pivot sharded protocol.  Measured on one B200 at c4g
# (profiles/R6a_bench_c4g_dist_n1.json vs R6a_bench_c4g.json): the sharded protocol at world 1
# costs 4.1 s per step (575 us per pivot: the rank's slice of the formed sketch is read and written
# every pivot) against 0.77 s for the one-GPU kernel; scaled to 8 ranks the protocol is ~0.9 s
# (slice / 8 + one all-gather per pivot), still not below the replicated 0.77 s.
REPLICATED_COMPRESS_MAX_WORLD = 8


def use_sharded_compress(world: int, shard_compress=None) -> bool:
    """The compression mode of dyson_sharded: an explicit True / False wins; None = the measured
    rule above (replicated up to one NVSwitch node of 8 ranks, sharded beyond)."""
    if shard_compress is None:
        return world > REPLICATED_COMPRESS_MAX_WORLD
    return bool(shard_compress)


def shard_bounds(n: int, rank: int, world: int) -> Tuple[int, int, int]:
    """Even-aligned contiguous shards: returns (begin, end, chunk) with chunk even."""
    chunk = -(-n // world)
    chunk += chunk & 1
    b = min(n, rank * chunk)
    e = min(n, b + chunk)
    return b, e, chunk


def grid_bounds(Ng: int, rank: int, world: int) -> Tuple[int, int, int]:
    """Contiguous split of the N_g grid points (columns of M~^T): (begin, end, chunk)."""
    chunk = -(-Ng // world)
    b = min(Ng, rank * chunk)
    e = min(Ng, b + chunk)
    return b, e, chunk


def allgather_rows(W_local: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """Gather per-rank row blocks (chunk x N_g each, zero padded) straight into one buffer and
    return its first n rows (a view: the blocks are stored back to back)."""
    world = dist.get_world_size(group)
    out = torch.empty((world * W_local.shape[0],) + tuple(W_local.shape[1:]), dtype=W_local.dtype,
                      device=W_local.device)
    dist.all_gather_into_tensor(out, W_local.contiguous(), group=group)
    return out[:n]


def compress_sharded(ops, Psi, Gp, theta, nu, id_eps: float, group=None, n_mu_fixed: int = 0):
    """Alg. 2 with the grid points split across the ranks of `group`.  Returns (S, Xi, N_mu)
    exactly as ops.compress would: S (N_mu,) int32 in pivot order, Xi (N_mu, N_g)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    Ng = Psi.shape[1]
    a, b, chunk = grid_bounds(Ng, rank, world)
    if Psi.is_cuda and hasattr(ops, "set_stream"):
        # the pivot kernels, the torch ops and the NCCL all-gathers are ordered by running on ONE
        # non-default stream (a null-stream handle would send the library to its own stream)
        cur = torch.cuda.current_stream(Psi.device)
        st = cur if cur.cuda_stream != 0 else torch.cuda.Stream(device=Psi.device)
        st.wait_stream(cur)
        prev = ops.stream_handle() if hasattr(ops, "stream_handle") else None
        with torch.cuda.stream(st):
            ops.set_stream(st)
            out = _compress_sharded_loop(ops, Psi, Gp, theta, nu, id_eps, group, n_mu_fixed, a, b, chunk, world)
        cur.wait_stream(st)
        if prev is not None:
            st.synchronize()
            ops.set_stream_handle(prev)   # the caller's stream choice for the library stays in force
        return out
    return _compress_sharded_loop(ops, Psi, Gp, theta, nu, id_eps, group, n_mu_fixed, a, b, chunk, world)


def _compress_sharded_loop(ops, Psi, Gp, theta, nu, id_eps, group, n_mu_fixed, a, b, chunk, world):
    Ng = Psi.shape[1]
    m = ops.qrs_begin(Psi, Gp, theta, nu, a, b, n_mu_fixed=n_mu_fixed)
    stride = m + 3
    send = torch.zeros(stride, dtype=torch.float64, device=Psi.device)
    recv = torch.zeros(world * stride, dtype=torch.float64, device=Psi.device)
    s = 0
    while True:
        ops.qrs_step(s, recv, world, id_eps, send)
        if s % CHECK_EVERY == CHECK_EVERY - 1:
            stopped, _ = ops.qrs_status()
            if stopped:
                break
        dist.all_gather_into_tensor(recv, send, group=group)
        s += 1
    S, XiT, N = ops.qrs_finish()
    # rows of Xi: rank r holds grid points [a_r, b_r); pad to chunk rows, gather, trim, transpose
    pad = torch.zeros(chunk, N, dtype=XiT.dtype, device=XiT.device)
    pad[: b - a] = XiT
    full = allgather_rows(pad, Ng, group)          # (N_g, N_mu)
    return S, full.t().contiguous(), N


def dyson_sharded(ops, Psi, eps, V, G, n_cheb: int, n_outer: int, draws: Callable[[int], tuple],
                  id_eps: float, cg_tol: float = 1e-11, group=None, shard_compress=None):
    """Alg. 4 on `world` ranks.

    `ops` provides qrs_* / compress / apply_chi0 / smw_update with the signatures of
    paper_1605_08021_b200.acp.Context (a GPU Context in production; tests pass a CPU stand-in to
    exercise the sharding and gather logic under gloo).  `shard_compress`: True = Alg. 2 sharded
    by grid point (compress_sharded), False = replicated on every rank (same inputs, deterministic
    kernels: identical S and Xi everywhere), None = use_sharded_compress(world).  Returns (U, info)
    with U identical on every rank.
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    Gp = G.clone()
    U = None
    sharded_c = use_sharded_compress(world, shard_compress)
    info = dict(n_mu=[], local_solves=0, shards=[], compression="sharded" if sharded_c else "replicated")
    for k in range(n_outer):
        theta, nu = draws(k)
        if sharded_c:
            S, Xi, n = compress_sharded(ops, Psi, Gp, theta, nu, id_eps, group)
        else:
            S, Xi, n = ops.compress(Psi, Gp, theta, nu, id_eps=id_eps)
        b, e, chunk = shard_bounds(n, rank, world)
        W_loc = torch.zeros(chunk, Xi.shape[1], dtype=Xi.dtype, device=Xi.device)
        if e > b:
            W_full = torch.zeros_like(Xi)
            _, st = ops.apply_chi0(Psi, eps, V, S, Xi, n_cheb, cg_tol=cg_tol, mu_range=(b, e), W=W_full)
            W_loc[: e - b] = W_full[b:e]
            info["local_solves"] += st["n_solved"]
        W = allgather_rows(W_loc, n, group)
        U, Gp = ops.smw_update(G, S, W)
        info["n_mu"].append(n)
        info["shards"].append((b, e))
    return U, info
