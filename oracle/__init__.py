"""TEST INFRASTRUCTURE ONLY: the CPU oracle (checker).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this package."""
