"""CPU FP64 oracle of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package; the product
(paper_2505_13215_b200) never does.  See hgs_oracle.h for the pinning status.
"""
from .oracle import *  # noqa: F401,F403
