"""CPU oracle for the Rii hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  See oracle/rii_ref.c for the cited arithmetic.
"""
