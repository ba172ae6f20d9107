import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: oracle cases taking more than ~20 s on CPU")


@pytest.fixture(scope="session")
def tiny_system():
    """Small 1D system (configs[0] shape, 4 atoms, 96 points) with its exact ground state."""
    from workloads import atom_positions
    from workloads.configs import small_config
    from oracle.model import Model
    from oracle.scf import scf
    cfg = small_config()
    R = atom_positions(cfg)
    m = Model(cfg, R)
    gs = scf(m, tol=1e-13)
    return cfg, R, m, gs
