"""Seeded synthetic workload generators (shared by tests, bench and smoke).

Holds none of the method's arithmetic: it only draws lengths, docIDs and gaps.
The d-gap transform, encoding and decoding all live elsewhere (the oracle on the
test side, the product library on the product side).
"""
from .workloads import *  # noqa: F401,F403
