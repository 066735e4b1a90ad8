"""CPU oracle (test infrastructure only; see hosfem_oracle.py's header)."""
