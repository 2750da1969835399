"""CPU oracle for the TT-IGA hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference algorithms of
arXiv 2509.13224's `ttiga` package (reference tree `pkg/src/ttiga/`), written
from the algorithm descriptions, with every function citing the reference
file:line it follows. It exists to *check* the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
  (``cpu_baseline`` and ``--impl reference``) may import it;
* the product package ``paper_2509_13224_b200`` never imports it and has no
  CPU fallback.

Parity pin: the oracle is checked against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` imports ``/root/reference``
in the build container and commits ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Extensions beyond the reference (the BASELINE.json configs name geometries
and boundary data the reference does not ship: quarter cylinder, deformed
cube, seeded random cube, Dirichlet data from a manufactured solution on
adjacent faces, exact basis count per direction) are marked ``EXTENSION`` in
their docstrings; their parity is anchored on oracle-vs-CUDA agreement and on
manufactured-solution convergence, not on reference golden vectors.
"""
