"""CPU oracle for the geometry-stage hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1805_08893_b200`` never does (tests/test_no_oracle_in_product.py
checks that).  Parity status: pinned against the reference's own KATs and
against fixtures generated from the unmodified reference
(tests/golden/make_golden.py).
"""
from .oracle import *  # noqa: F401,F403
