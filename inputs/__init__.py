"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NO arithmetic of the method (no products, no merging, no
counting of intermediate products): it only builds input matrices in CSR form.
Both `oracle/` and the CUDA path consume its output; neither imports the other.
"""
from .generators import (  # noqa: F401
    Csr,
    uniform_random,
    random_sparse,
    stencil27,
    rmat,
    laplace2d_5pt,
    aggregation_prolongator,
    identity,
    permutation,
    workload,
    WORKLOADS,
)
