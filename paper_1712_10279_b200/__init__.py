"""B200-native (sm_100a) PDHG solver for scalar-, vector- and matrix-valued
Wasserstein-1 transport (arXiv 1712.10279), a drop-in for the hot path of the
reference package ``otflux`` (``solve_*`` and its engine).

The iteration runs in hand-written CUDA (libotfx.so, C ABI in include/otfx.h);
this package is the Python host layer with the reference's public names.
"""

from .errors import (DimensionMismatchError, NumericalError, OTFluxError, UnsupportedNormError,
                     ValidationError)
from .fields import (FluxField, GraphFlux, GridSpec, MatrixDensity, QuantumFlux, ScalarDensity,
                     VectorDensity, hermitian_part, normalize, skew_part, total_mass)
from .graph import TransportGraph, lambda_max_graph, triangle_graph
from .lindblad import LindbladSet, default_lindblad3, lambda_max_L, lindblad_pair_k2
from .omtf import (load_graph, load_lindblad, read_density, read_omtf, save_graph, save_lindblad,
                   write_omtf)
from .problems import dirac_pair, lambda_max_spatial_bound, matrix_blob_fixtures, rgb_disk_pair
from .solver import (CudaEngine, HistoryPoint, NormFamily, SolveReport, SolverConfig, SolverState,
                     default_tau, duality_gap, residual_Rk, solve_matrix, solve_scalar,
                     solve_tensors, solve_vector, step_sizes_matrix, step_sizes_scalar, step_sizes_vector)

from ._lib import release_cached_memory

__version__ = "0.1.0"
