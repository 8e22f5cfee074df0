"""CPU oracle (test infrastructure only): see oracle/ppcg_oracle.py."""
