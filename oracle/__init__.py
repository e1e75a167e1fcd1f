"""TEST INFRASTRUCTURE ONLY: CPU checkers for the POD-Attention hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the timed
CPU baseline -- never as the product path.
"""
