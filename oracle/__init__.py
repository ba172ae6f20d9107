"""CPU fp64 ORACLE for the ACP hot path (Lin, Xu, Ying, arXiv 1605.08021).

TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct NumPy/SciPy code
that restates PAPER.md (cited per function as PAPER.md:<line>, section /
equation / algorithm).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
It shares no code with the CUDA path (``paper_1605_08021_b200``); the only
shared module is ``workloads`` (seeded raw draws, no method arithmetic).

Modules
  model     -- grid, Yukawa kernel, pseudocharges, g_{I,a}, d2V, E_II (PAPER §2.1, §4.1)
  scf       -- dense-diagonalisation SCF, forces (PAPER §2.1, Eqs. Hamil/effV/force)
  response  -- Q, Sternheimer, chi0 (Alg. 1), Adler-Wiser, Dyson (PAPER §2.2)
  acp       -- Chebyshev/Lagrange, SRFT sketch, QRCP/ID (Alg. 2), W (Alg. 3), SMW (Alg. 4)
  phonon    -- dynamical matrix (Eq. SecDeriv), frozen-phonon FD, modes

Pins (tests/test_oracle_*.py) tie every function to something other than
itself: printed paper values, closed forms, LAPACK, brute force, FD.
"""
