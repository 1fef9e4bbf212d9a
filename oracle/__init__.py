"""CPU oracle (test infrastructure only; see dbsa_oracle.py)."""
