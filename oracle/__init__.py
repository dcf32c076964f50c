"""CPU oracle for the B200 kernel family -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package, and only as the checker or the CPU reference timing.
The product path (paper_2008_13145_b200) never imports it and fails loudly when its
CUDA library is missing.
"""
