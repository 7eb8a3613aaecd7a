"""CPU oracle package — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
--impl reference arm) may import this package, and only as the checker or
the timed CPU baseline. The product (paper_2412_16544_b200/) never does.
"""
