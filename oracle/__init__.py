"""TEST INFRASTRUCTURE ONLY: the plain CPU oracle for arXiv 1502.01916's Group formats.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference leg may import this package.  The product path
(``paper_1502_01916_b200``) never imports it and shares no code with it.
"""
from .oracle import *  # noqa: F401,F403
