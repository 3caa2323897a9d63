"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no Lanczos, no QR, no MINRES):
only the matrices and right-hand sides the paper's experiments and
BASELINE.json's configs are built from.  Both sides of every parity test take
their inputs from here; neither side's code lives here.
"""
from .problems import *  # noqa: F401,F403
