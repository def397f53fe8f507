"""ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/core.py header).

CPU restatement of the reference vmsplat per-frame path, used as the parity
checker by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.
Nothing in paper_2506_19415_b200/ imports this package.
"""
