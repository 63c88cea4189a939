"""CPU oracle for the ghost-point multigrid V-cycle (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may use this package, and only as the checker or
the CPU baseline.  The product path (paper_2207_14208_b200) never imports it.
"""
