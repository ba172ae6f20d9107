"""The five BASELINE.json configurations plus the paper's worked examples.

Each entry restates one line of ``BASELINE.json:configs`` (or, for the
``paper_*`` entries, the model parameters of PAPER.md §4.1/§4.2) as plain
numbers.  Choices the configs leave open are the DESIGN.md readings:

* ``occ`` (f): Z=2 per atom with N_A orbitals => doubly occupied, f = 2
  (BASELINE configs "doubly-occupied orbitals"); the paper's examples have
  Z=1 and rho = sum |psi_i|^2, i.e. f = 1.
* ``sketch_r``: r = 8 (1D) / 16 (2D), PAPER.md:604 (Alg. 2 step 1(b)).
* ``id_eps``: the rank threshold epsilon of Alg. 2 step 3;
  1e-3 is the value the paper's efficiency runs use.
* ``n_outer``: outer iterations of Alg. 4, fixed ("converges
  within 4 iterations" for 1D; "two iterations" for 2D).
* ``cg_tol``: relative residual of every Sternheimer solve (config 1 states
  1e-11; used for all configs).
* masses M_I = 1 (the paper never assigns masses).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Tuple


@dataclasses.dataclass(frozen=True)
class SystemConfig:
    name: str
    dim: int                       # spatial dimension d
    n_side: int                    # atoms per dimension (1D: N_A)
    spacing: float                 # lattice spacing (bohr)
    Z: float                       # nuclear charge per atom
    sigma: float                   # Gaussian pseudocharge width
    kappa: float                   # Yukawa screening
    eps0: float                    # Yukawa permittivity scale
    grid: Tuple[int, ...]          # grid points per dimension
    n_occ: int                     # occupied orbitals
    occ: float                     # occupation f (electrons per orbital)
    n_cheb: int                    # Chebyshev nodes N_c
    jitter: float                  # uniform jitter half-width (bohr)
    seed: int
    sketch_r: int = 8
    id_eps: float = 1e-3
    n_outer: int = 4
    cg_tol: float = 1e-11
    scf_tol: float = 1e-12
    lattice: str = "square"        # "square" (n_side^d atoms) or "triangular" (2D, 2 n_side^2 atoms)

    @property
    def n_atoms(self) -> int:
        if self.lattice == "triangular":
            return 2 * self.n_side ** 2
        return self.n_side ** self.dim

    @property
    def cell(self) -> Tuple[float, ...]:
        if self.lattice == "triangular":
            # n_side x n_side rectangular cells a x a sqrt(3), two atoms each (R19)
            return (self.n_side * self.spacing, self.n_side * self.spacing * 3.0 ** 0.5)
        return tuple(self.n_side * self.spacing for _ in range(self.dim))

    @property
    def n_grid(self) -> int:
        n = 1
        for g in self.grid:
            n *= g
        return n

    @property
    def n_pert(self) -> int:
        return self.dim * self.n_atoms


CONFIGS: Dict[str, SystemConfig] = {
    # BASELINE.json configs[0]
    "c0_1d_tiny": SystemConfig(
        name="c0_1d_tiny", dim=1, n_side=8, spacing=10.0, Z=2.0, sigma=2.0,
        kappa=0.01, eps0=10.0, grid=(256,), n_occ=8, occ=2.0, n_cheb=4,
        jitter=0.0, seed=100),
    # BASELINE.json configs[1]
    "c1_1d_insulator": SystemConfig(
        name="c1_1d_insulator", dim=1, n_side=32, spacing=10.0, Z=2.0, sigma=2.0,
        kappa=0.01, eps0=10.0, grid=(1280,), n_occ=32, occ=2.0, n_cheb=8,
        jitter=0.2, seed=101),
    # BASELINE.json configs[2]
    "c2_1d_semiconductor": SystemConfig(
        name="c2_1d_semiconductor", dim=1, n_side=128, spacing=6.0, Z=2.0, sigma=1.2,
        kappa=0.01, eps0=10.0, grid=(5120,), n_occ=128, occ=2.0, n_cheb=16,
        jitter=0.1, seed=102, scf_tol=1e-11),  # B200 SCF floor ~5e-12 here (R15)
    # BASELINE.json configs[3]
    "c3_2d_8x8": SystemConfig(
        name="c3_2d_8x8", dim=2, n_side=8, spacing=10.0, Z=2.0, sigma=2.0,
        kappa=0.01, eps0=10.0, grid=(192, 192), n_occ=64, occ=2.0, n_cheb=8,
        jitter=0.2, seed=103, sketch_r=16, n_outer=2),
    # BASELINE.json configs[4]
    "c4_2d_16x16": SystemConfig(
        name="c4_2d_16x16", dim=2, n_side=16, spacing=8.0, Z=2.0, sigma=1.6,
        kappa=0.01, eps0=10.0, grid=(256, 256), n_occ=256, occ=2.0, n_cheb=12,
        jitter=0.2, seed=104, sketch_r=16, n_outer=2),
    # PAPER.md:852-857 (§4.1): N_A=60, spacing 2.4, kappa=0.1, Z=1, sigma=0.3,
    # eps0=1 (insulator) / 10 (semiconductor); grid spacing 0.15 = sigma/2
    # (SPEC.md:164 reading; the paper never states N_g).
    "paper_1d_insulator": SystemConfig(
        name="paper_1d_insulator", dim=1, n_side=60, spacing=2.4, Z=1.0, sigma=0.3,
        kappa=0.1, eps0=1.0, grid=(960,), n_occ=60, occ=1.0, n_cheb=20,
        jitter=0.0, seed=0),
    "paper_1d_semiconductor": SystemConfig(
        name="paper_1d_semiconductor", dim=1, n_side=60, spacing=2.4, Z=1.0, sigma=0.3,
        kappa=0.1, eps0=10.0, grid=(960,), n_occ=60, occ=1.0, n_cheb=20,
        jitter=0.0, seed=0),
    # PAPER.md:1064-1066, 1100 (section 4.2): triangular lattice, nearest neighbour 1.2, eps0 = 0.05,
    # Z = 1, sigma = 0.24, N_A = 2 x 7^2 = 98, one electron per orbital; kappa = 0.01 and the
    # supercell are readings (R19); grid spacing 0.175 (gap converged to 1e-6 there).
    "paper_2d_triangular": SystemConfig(
        name="paper_2d_triangular", dim=2, n_side=7, spacing=1.2, Z=1.0, sigma=0.24,
        kappa=0.01, eps0=0.05, grid=(48, 84), n_occ=98, occ=1.0, n_cheb=30,
        jitter=0.0, seed=0, sketch_r=16, n_outer=2, lattice="triangular"),
}

# configs[3] / configs[4] with eps0 = 1 instead of 10 (reading R13): at eps0 = 10
# the 2D lattices are (nearly) metallic -- HOMO-LUMO gap ~5e-4 on the 2x2 probe, the SCF
# oscillates between degenerate occupations and never converges on 2x2, 8x8 or 16x16 --
# while ACP ("insulators as well as semiconductors") needs a gapped ground
# state (H - eps~_c positive on range(Q)).  With eps0 = 1 the 8x8 system has gap 0.042 (B200
# SCF, profiles/r1c).  Everything else (sizes, grids, N_c, sketch, jitter) is unchanged.
CONFIGS["c3g_2d_8x8"] = dataclasses.replace(CONFIGS["c3_2d_8x8"], name="c3g_2d_8x8", eps0=1.0)
CONFIGS["c4g_2d_16x16"] = dataclasses.replace(CONFIGS["c4_2d_16x16"], name="c4g_2d_16x16", eps0=1.0)

# Short aliases by BASELINE.json index.
BASELINE_ORDER = ["c0_1d_tiny", "c1_1d_insulator", "c2_1d_semiconductor",
                  "c3_2d_8x8", "c4_2d_16x16"]


def get_config(name_or_index) -> SystemConfig:
    if isinstance(name_or_index, int):
        return CONFIGS[BASELINE_ORDER[name_or_index]]
    return CONFIGS[name_or_index]


def small_config_2d(name: str = "tiny2d", **overrides) -> SystemConfig:
    """A cheap GAPPED 2D test system (configs[3]'s shape: square lattice, Z=2, f=2, x and y
    perturbations).  eps0 = 0.3 instead of the configs' 10: at eps0 = 10 the 2x2 lattice is
    (nearly) metallic -- HOMO-LUMO gap ~5e-4, the SCF oscillates between degenerate
    occupations -- while here the gap is 0.083."""
    base = dict(name=name, dim=2, n_side=2, spacing=6.0, Z=2.0, sigma=1.2, kappa=0.01, eps0=0.3,
                grid=(32, 32), n_occ=4, occ=2.0, n_cheb=4, jitter=0.15, seed=9, sketch_r=16, n_outer=2)
    base.update(overrides)
    return SystemConfig(**base)


def small_config(name: str = "tiny4", **overrides) -> SystemConfig:
    """A cheap test system (shape of configs[0], fewer atoms/points)."""
    base = dict(name=name, dim=1, n_side=4, spacing=6.0, Z=2.0, sigma=1.2,
                kappa=0.01, eps0=10.0, grid=(96,), n_occ=4, occ=2.0, n_cheb=4,
                jitter=0.15, seed=7)
    base.update(overrides)
    return SystemConfig(**base)
