"""ORACLE / TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / --impl reference legs.  Never imported by the product package.
"""
