"""Multi-GPU layer: Alg. 4 with the compressed Sternheimer right-hand sides sharded
across ranks (one process per GPU) and W all-gathered over NCCL (NVLink).

PAPER.md:622-628: the N_c x N_mu equations of Eq. eqncompressU are independent,
so rank r solves the mu-columns [b_r, e_r) for all Chebyshev nodes and produces
those columns of W (Eq. eqnW).  The only exchange per outer iteration is the
all-gather of W (N_g x N_mu doubles).  Compression (Alg. 2) and the small SMW
update (Eq. dyson4) are replicated: they are deterministic functions of
identical inputs, so every rank holds the same U after each iteration.
Shard boundaries are even, so column pairs of the FFT kernel -- and therefore
every per-column result -- are identical to the single-GPU run.
"""
from __future__ import annotations

from typing import Callable, List, Tuple

import torch
import torch.distributed as dist


def shard_bounds(n: int, rank: int, world: int) -> Tuple[int, int, int]:
    """Even-aligned contiguous shards: returns (begin, end, chunk) with chunk even."""
    chunk = -(-n // world)
    chunk += chunk & 1
    b = min(n, rank * chunk)
    e = min(n, b + chunk)
    return b, e, chunk


def allgather_rows(W_local: torch.Tensor, n: int, chunk: int, group=None) -> torch.Tensor:
    """Gather per-rank row blocks (chunk x N_g, zero padded) into the first n rows."""
    world = dist.get_world_size(group)
    parts: List[torch.Tensor] = [torch.empty_like(W_local) for _ in range(world)]
    dist.all_gather(parts, W_local, group=group)
    return torch.cat(parts, dim=0)[:n].contiguous()


def dyson_sharded(ops, Psi, eps, V, G, n_cheb: int, n_outer: int, draws: Callable[[int], tuple],
                  id_eps: float, cg_tol: float = 1e-11, group=None):
    """Alg. 4 on `world` ranks.

    `ops` provides compress / apply_chi0 / smw_update with the signatures of
    paper_1605_08021_b200.acp.Context (a GPU Context in production; tests pass
    a CPU stand-in to exercise the sharding and gather logic under gloo).
    Returns (U, info) with U identical on every rank.
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    Gp = G.clone()
    U = None
    info = dict(n_mu=[], local_solves=0, shards=[])
    for k in range(n_outer):
        theta, nu = draws(k)
        S, Xi, n = ops.compress(Psi, Gp, theta, nu, id_eps=id_eps)
        b, e, chunk = shard_bounds(n, rank, world)
        W_loc = torch.zeros(chunk, Xi.shape[1], dtype=Xi.dtype, device=Xi.device)
        if e > b:
            W_full = torch.zeros_like(Xi)
            _, st = ops.apply_chi0(Psi, eps, V, S, Xi, n_cheb, cg_tol=cg_tol, mu_range=(b, e), W=W_full)
            W_loc[: e - b] = W_full[b:e]
            info["local_solves"] += st["n_solved"]
        W = allgather_rows(W_loc, n, chunk, group)
        U, Gp = ops.smw_update(G, S, W)
        info["n_mu"].append(n)
        info["shards"].append((b, e))
    return U, info
