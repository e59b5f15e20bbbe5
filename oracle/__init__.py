"""ORACLE — test infrastructure only (see fcct_oracle.cpp header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package. The product never does.
"""
