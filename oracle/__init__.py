"""ORACLE package -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import anything from here; the product path never does.
"""
