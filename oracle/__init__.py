"""CPU fp64 oracle (TEST INFRASTRUCTURE ONLY).

May be imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg.  The product package never imports it.
"""
from .lrs_oracle import *  # noqa: F401,F403
