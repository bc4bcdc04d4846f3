"""TEST INFRASTRUCTURE: parity checkers (see oracle/oracle.py)."""
