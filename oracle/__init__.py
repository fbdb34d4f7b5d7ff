"""CPU oracle package (test infrastructure only; see otn_oracle.py)."""
