"""CPU oracle (test infrastructure only; see specdens_oracle.py header)."""
