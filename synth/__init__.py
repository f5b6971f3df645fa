"""Seeded synthetic inputs (DAG structures + leaf values) shared by oracle/ and the CUDA path.

Holds none of the method's arithmetic: no contraction, schedule or memory
model lives here (task rule ③).
"""
from . import rng, dags  # noqa: F401
