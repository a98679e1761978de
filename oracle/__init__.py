"""CPU oracle for the ADMM-LP hot path -- test infrastructure only.

Used by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg; the
product package never imports it.
"""
