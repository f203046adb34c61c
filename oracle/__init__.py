"""ORACLE — test infrastructure only (see oracle/kk_oracle.c header)."""
