"""fp64 CPU oracle for the VarGrad TB-loss head — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg / --impl reference arm
may import this package. The product package (paper_2503_18929_b200) never does.
"""
from .tba_oracle import *  # noqa: F401,F403
