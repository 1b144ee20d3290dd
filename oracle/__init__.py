"""CPU fp64 oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package.  The product package (paper_2406_10661_b200)
never imports it and shares no code with it.
"""
from .oracle import Oracle, build, lib_path, philox4x32_10, u53, idm, p_lc

__all__ = ["Oracle", "build", "lib_path", "philox4x32_10", "u53", "idm", "p_lc"]
