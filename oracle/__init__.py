"""CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle/gls_oracle.c header)."""
