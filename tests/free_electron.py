"""Synthetic free-electron ground state for full-grid pins (test helper, no method arithmetic
beyond plane waves): V = 0, orbitals = the real plane waves of every shell |m|^2 <= m2max
(complete shells, so the occupied span is exactly a set of Fourier bins), eps_i = |k_i|^2/2."""
import numpy as np


def plane_wave_ground_state(grid, cell, m2max):
    grid = tuple(grid)
    dim = len(grid)
    L = np.asarray(cell, dtype=np.float64)
    Ng = int(np.prod(grid))
    Omega = float(np.prod(L))
    axes = [np.arange(n) / n for n in grid]                      # r_a / L_a
    mesh = np.meshgrid(*axes, indexing="ij")
    frac = np.stack([x.reshape(-1) for x in mesh], axis=1)      # (Ng, d)
    ms = []
    rng = range(-int(np.sqrt(m2max)) - 1, int(np.sqrt(m2max)) + 2)
    for m in np.array(np.meshgrid(*([list(rng)] * dim), indexing="ij")).reshape(dim, -1).T:
        if np.sum(m * m) <= m2max:
            ms.append(tuple(int(v) for v in m))
    cols, eps = [], []
    for m in sorted(ms, key=lambda t: (sum(v * v for v in t), t)):
        e = 0.5 * sum((2 * np.pi * m[a] / L[a]) ** 2 for a in range(dim))
        phase = 2 * np.pi * (frac @ np.asarray(m, dtype=np.float64))
        if all(v == 0 for v in m):
            cols.append(np.full(Ng, 1.0 / np.sqrt(Omega)))
            eps.append(e)
            continue
        # one (cos, sin) pair per +-m: keep m with its first nonzero component positive
        first = next(v for v in m if v != 0)
        if first < 0:
            continue
        cols.append(np.sqrt(2.0 / Omega) * np.cos(phase))
        cols.append(np.sqrt(2.0 / Omega) * np.sin(phase))
        eps += [e, e]
    Psi = np.stack(cols, axis=1)
    eps = np.asarray(eps)
    order = np.argsort(eps, kind="stable")
    Psi, eps = Psi[:, order], eps[order]
    # occupied FFT bins (numpy fft order)
    occ = np.zeros(grid, dtype=bool)
    for m in ms:
        occ[tuple(mi % n for mi, n in zip(m, grid))] = True
    return Psi, eps, occ.reshape(grid)
