"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TT-embedding hot path.

`oracle.core` wraps oracle/libttoracle.so (a plain-C fp64 restatement of
/root/reference/proj/core/src/{tt_config,tt_embedding,autodiff}.cpp) and,
when it was built here, oracle/_ref/libttref.so (the reference's own
tt_config.cpp).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.
"""
from .core import *  # noqa: F401,F403
