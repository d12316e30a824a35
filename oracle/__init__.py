"""Independent CPU oracle — test infrastructure only (see pmg_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs.  The product package paper_1909_07190_b200 never imports this package and vice versa.
"""
from .pmg_oracle import OracleError, evaluate, io_shapes, parse  # noqa: F401
from .points import evaluate_points  # noqa: F401
