"""TEST INFRASTRUCTURE: CPU parity oracle for the B200 engine (see oracle.py)."""
