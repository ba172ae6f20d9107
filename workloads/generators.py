"""Seeded raw random draws (no method arithmetic lives here).

* ``atom_positions``: perfect lattice + seeded uniform jitter, the recipe
  BASELINE.json states for every config ("positions = perfect lattice plus
  seeded uniform jitter +-0.2 bohr").
* ``sketch_draws``: the randomness Alg. 2 step 1 draws:
  one random unit-modulus phase eta_I = exp(2 pi i theta_I) per stacked
  column I, and the subsampled frequency indices nu.  Only the raw theta
  (fraction of a turn, in [0,1)) and the integer nu (1-based, as in the
  paper's sum over I,nu = 1..n) are produced here; each side builds the
  SRFT from them itself.
"""
from __future__ import annotations

import numpy as np

from .configs import SystemConfig


def atom_positions(cfg: SystemConfig) -> np.ndarray:
    """(N_A, d) positions in bohr, wrapped into the periodic cell."""
    rng = np.random.default_rng([cfg.seed, 1])
    if cfg.lattice == "triangular":
        # rectangular cells a x a sqrt(3) with atoms at (0, 0) and (a/2, a sqrt(3)/2) (R19)
        a, h = cfg.spacing, cfg.spacing * np.sqrt(3.0)
        idx = np.indices((cfg.n_side, cfg.n_side)).reshape(2, -1).T.astype(np.float64)
        base = idx * np.array([a, h])
        R = np.stack([base, base + np.array([a / 2, h / 2])], axis=1).reshape(-1, 2)
    else:
        idx = np.indices((cfg.n_side,) * cfg.dim).reshape(cfg.dim, -1).T  # (N_A, d), C order
        R = idx.astype(np.float64) * cfg.spacing
    if cfg.jitter > 0:
        R = R + rng.uniform(-cfg.jitter, cfg.jitter, size=R.shape)
    L = np.asarray(cfg.cell)
    return np.mod(R, L)


def sketch_draws(seed: int, outer_k: int, n_cols: int, r: int):
    """Raw draws for one SRFT sketch of an n_cols-column matrix.

    Returns (theta, nu): theta float64[n_cols] in [0,1); nu int32[r_half]
    distinct values in 1..n_cols with r_half = min(r // 2, n_cols).
    """
    rng = np.random.default_rng([seed, 1000 + outer_k])
    theta = rng.random(n_cols)
    r_half = min(max(r // 2, 1), n_cols)
    nu = rng.choice(n_cols, size=r_half, replace=False).astype(np.int32) + 1
    return theta.astype(np.float64), nu
