"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the FDFB hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product package
paper_2109_02731_b200 never imports it (tests/test_boundary.py checks).
"""
