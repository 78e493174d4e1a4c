"""CPU oracle for arXiv 2410.11184's CKKS Softmax -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this package.  See oracle/orc.h.
"""
