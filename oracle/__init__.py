"""CPU checker for the dconv hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The product package
paper_1809_10170_b200 never does.
"""
