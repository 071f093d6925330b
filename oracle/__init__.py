"""CPU oracle (test infrastructure only; see tetsim_oracle.py)."""
