"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the FaVeST VSHT hot path.

This package restates, in numpy, the reference algorithm of
``/root/reference/pkg/src/favest`` for the forward / adjoint vector spherical
harmonic transforms (``forward_favest`` / ``adjoint_favest``) so that the
CUDA path in ``paper_1908_00041_b200`` can be checked against it.

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` (as the checker) and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs.  The product path
never imports it; there is no CPU fallback.

Parity pin: the restatement is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src`` and writes ``tests/golden/*.npz``), see
``tests/test_oracle.py``.
"""

from .favest_oracle import *  # noqa: F401,F403
