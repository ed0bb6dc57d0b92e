"""CPU oracle package — test infrastructure only (see geographer_oracle.py)."""
