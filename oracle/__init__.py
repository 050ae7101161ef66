"""Test-infrastructure oracle (float64 CPU).  Importable ONLY from tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg."""
