"""CPU oracle for the tensor-collective hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1801_03855_b200``) never imports it and shares no code with it.
"""
from .tc_oracle import *  # noqa: F401,F403
