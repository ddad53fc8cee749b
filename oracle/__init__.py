"""TEST INFRASTRUCTURE: the CPU checkers for the TENSILE plan generator.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
arm may import this package. The product (paper_2105_13336_b200) never does.
"""
