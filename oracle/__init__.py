"""CPU oracle — test infrastructure only (see vq_oracle.py header)."""
