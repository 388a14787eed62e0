"""CPU oracle (test infrastructure only; see hssd.py header)."""
