"""Checker for the GPU hot path - TEST INFRASTRUCTURE, NOT PRODUCT CODE.

``oracle.port`` restates the reference (greencross, pure numpy) algorithm
of the hot path with the same operation order.  It is pinned against
fixtures generated from the reference itself (tests/golden/make_golden.py)
and used only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline fallback.  The product package never imports it.
"""
