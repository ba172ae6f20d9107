"""Pins for oracle/scf.py: the paper's printed ground states and closed forms."""
import json
import os

import numpy as np
import pytest

from workloads import atom_positions, get_config
from workloads.configs import small_config
from oracle.model import Model
from oracle.scf import scf, eigenpairs, forces

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_ground_state.json")))


@pytest.mark.parametrize("name", ["paper_1d_insulator", "paper_1d_semiconductor"])
def test_paper_section_4_1_ground_state(name):
    """gap and density range of the N_A=60 chain, printed to 4 decimals."""
    cfg = get_config(name)
    m = Model(cfg, atom_positions(cfg))
    gs = scf(m, tol=1e-10)
    ref = GOLD[name]
    assert abs(gs.gap - ref["gap"]) <= 5e-5
    assert abs(gs.rho.min() - ref["rho_min"]) <= 5e-5
    assert abs(gs.rho.max() - ref["rho_max"]) <= 5e-5


@pytest.mark.slow
def test_paper_section_4_2_triangular_gap():
    """eps_99 - eps_98 = 1.2637 for the 98-atom triangular lattice of PAPER.md:1064-1066
    (printed to 4 decimals; readings R19: kappa = 0.01, 7 x 7 rectangular two-atom cells).  Pins the
    oracle's 2D conventions (Yukawa symbol, 2D Gaussian pseudocharge, non-square cell).  The SCF
    restarts from the density tools/probe_paper_2d.py (oracle only) converged on this grid, so it must
    hold it as a fixed point within a few iterations instead of running ~30 from scratch."""
    cfg = get_config("paper_2d_triangular")
    m = Model(cfg, atom_positions(cfg))
    rho0 = np.load(os.path.join(os.path.dirname(__file__), "golden", "paper_2d_tri98_rho.npy"))
    gs = scf(m, tol=1e-9, rho0=rho0, max_iter=4)
    assert gs.n_iter <= 3
    assert abs(m.integrate(gs.rho) - 98.0) < 1e-9
    assert abs(gs.gap - GOLD["paper_2d_triangular"]["gap"]) <= 5e-5


def test_free_particle_spectrum():
    """V = 0 -> eigenvalues {0, 1/2 (2pi/L)^2 (x2), 1/2 (4pi/L)^2 (x2), ...}."""
    cfg = small_config()
    m = Model(cfg, atom_positions(cfg))
    w, X = eigenpairs(m, np.zeros(m.Ng), 5)
    k = 2 * np.pi / m.L[0]
    ref = 0.5 * np.array([0, k * k, k * k, 4 * k * k, 4 * k * k])
    assert np.abs(w - ref).max() < 1e-12
    assert np.abs(m.dV * X.T @ X - np.eye(5)).max() < 1e-12


def test_ground_state_invariants(tiny_system):
    cfg, R, m, gs = tiny_system
    assert gs.residual <= 1e-13
    assert abs(m.integrate(gs.rho) - m.Ne) < 1e-10
    assert np.abs(m.dV * gs.Psi.T @ gs.Psi - np.eye(cfg.n_occ)).max() < 1e-12
    H = m.hamiltonian_dense(gs.V)
    res = H @ gs.Psi - gs.Psi * gs.eps[: cfg.n_occ]
    assert np.abs(res).max() < 1e-10
    assert gs.gap > 0
    F = forces(m, gs)
    assert abs(F.sum()) < 1e-9          # Newton's third law / translation invariance


def test_perfect_lattice_has_zero_forces():
    cfg = small_config(jitter=0.0)
    m = Model(cfg, atom_positions(cfg))
    gs = scf(m, tol=1e-13)
    assert np.abs(forces(m, gs)).max() < 1e-9
