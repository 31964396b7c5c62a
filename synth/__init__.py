"""Seeded synthetic inputs and workload shapes, shared by `oracle/` and the CUDA path's tests.

Holds none of the method's arithmetic (task rule ③); see splitmix.py and workloads.py.
"""
from . import splitmix, workloads  # noqa: F401
