"""TEST INFRASTRUCTURE: CPU oracle (see oracle/orc.py)."""
