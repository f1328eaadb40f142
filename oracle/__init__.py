"""CPU oracle (test infrastructure only; see tcg_oracle.py header)."""
