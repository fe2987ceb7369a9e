"""CPU oracle -- test infrastructure only (see chacha_oracle.py header)."""
