"""TEST INFRASTRUCTURE ONLY: CPU checkers (see bindings.py)."""
