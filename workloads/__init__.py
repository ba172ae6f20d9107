"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This package holds ONLY problem descriptions (BASELINE.json configs) and
seeded random draws (atomic jitter, SRFT phases and frequency picks).  It
contains none of the ACP method's arithmetic: both the oracle (``oracle/``)
and the CUDA library turn these raw draws into model quantities themselves.
"""
from .configs import CONFIGS, SystemConfig, get_config
from .generators import atom_positions, sketch_draws

__all__ = ["CONFIGS", "SystemConfig", "get_config", "atom_positions", "sketch_draws"]
