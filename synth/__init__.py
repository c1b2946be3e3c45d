"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NONE of PCDN's arithmetic (no loss, gradient, direction,
line search or objective): it only draws design matrices and labels following
the generator rules of SURVEY.md §8(d) / DESIGN.md "Input recipe", stand-ins
for the paper's LIBSVM datasets (Table 2), which are not in
this container.  Both `oracle/` (through the tests) and the product path
(through the tests and bench.py) consume it; neither imports the other.
"""
from .generate import (  # noqa: F401
    Problem,
    CONFIGS,
    config,
    tiny,
    from_dense,
    csr_to_csc,
    LOSS_LOGISTIC,
    LOSS_L2SVM,
    LOSS_SQUARED,
    regression,
    shard_rows,
)
