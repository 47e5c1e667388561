"""CPU oracle (test infrastructure only; see tape_oracle.py header)."""
