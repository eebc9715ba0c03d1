"""Test infrastructure only: CPU checker for the GPU build (see oracle.py)."""
