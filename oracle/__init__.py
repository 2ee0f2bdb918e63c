"""CPU parity oracle (test infrastructure only; see actc_oracle.c)."""
