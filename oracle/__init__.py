"""CPU oracle for stochastic GCP-Adam (arXiv 2605.20353) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product (``paper_2605_20353_b200``) never imports it and shares no code with
it.  The arithmetic lives in ``gcp_oracle.c`` (plain fp64 C, single thread);
this module only marshals arguments and strings the per-rank C calls into the
paper's multi-rank algorithms (Alg. 2-4) in plain Python loops.

Parity status per function is listed in DESIGN.md §5; the pins are in
``tests/test_oracle_*.py``.
"""
from .oracle import *  # noqa: F401,F403
