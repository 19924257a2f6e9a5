"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no scoring, no top-p, no
attention): only random tensors with the shapes and structure of the paper's
workload.  See DESIGN.md §3 for the recipe.
"""
from .generator import Workload, make_qkv, make_grad_out, make_index_lists, CONFIGS  # noqa: F401
