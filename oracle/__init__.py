"""CPU oracle for the KV-frame hot path — TEST INFRASTRUCTURE ONLY.

A restatement of the reference framekv algorithms (numpy + a small C library for
the serial entropy coder).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import it, as the checker or as the
timed CPU baseline.  The product package never imports this module.

Pinning: tests/golden/ holds digests and vectors produced by running the
reference itself (tests/golden/make_golden.py); tests/test_oracle_golden.py
checks this restatement against every one of them.
"""
