"""TEST INFRASTRUCTURE ONLY: CPU parity oracles (see oracle.py)."""
