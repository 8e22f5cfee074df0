"""B200-native PPCG block eigensolver hot path (arXiv:1407.7506).

Drop-in for the reference package ``blockeig``'s PPCG entry point: ``ppcg_solve`` with the
same ``SolverOptions``, ``SolveReport``, operator protocol and exceptions, computing on
sm_100a kernels from ``libppcg_b200.so``.  Importing this package does not load CUDA; the
library is loaded (and a GPU required) on the first device call.
"""

from .errors import (  # noqa: F401
    ApplicabilityError, BlockeigError, DeviceError, DimensionError, ParseError, RankDeficiencyError,
    SingularGramError, UnsupportedFormatError,
)
from .operators import (  # noqa: F401
    CountingOperator, DenseHermitian, DiagonalOperator, DiagonalPreconditioner, IdentityPreconditioner,
    MatrixFreeOperator, SparseHermitian,
)
from .baselines import BaselineOptions, davidson_solve, lobpcg_solve  # noqa: F401
from .mmio import read_matrix_market, write_matrix_market  # noqa: F401
from .ppcg import PPCGSolver, SolveReport, SolverOptions, ppcg_solve, split_blocks  # noqa: F401
from .problems import (  # noqa: F401
    config_problem, jacobi_preconditioner, laplacian_1d, laplacian_2d, laplacian_3d,
    laplacian_plus_potential, random_hermitian, well_problem,
)
from .trace import TRACE_SCHEMA, TraceRecord, parse_trace_csv, trace_to_csv, trace_to_json  # noqa: F401

__version__ = "0.1.0"
