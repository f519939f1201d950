"""ORACLE package — test infrastructure only (see cggm_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product package never imports it.
"""
