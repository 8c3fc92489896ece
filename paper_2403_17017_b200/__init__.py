"""kernelpick-b200: B200-native Seer (arXiv 2403.17017) -- runtime SpMV kernel
selection with hand-written sm_100a kernels behind the reference's
``kernelpick`` API.

Public surface (mirrors /root/reference/pkg/src/kernelpick):
  sparse.SparseMatrixCSR / known_features / csr_from_coo
  features.gather_features / GatheredFeatures / row_density
  _kernels.length_stats / wave_ceil_max_sum / BACKEND == "cuda"
  clock.perf_clock / FixedClock (+ CudaEventClock)
plus the SPEC-only surfaces on the hot path:
  dtree (CART, predict, emit), dataset (total_cost, fastest_kernel),
  seer (SeerModel, infer, SeerRunner), kernels (spmv, prepare), device (DeviceCSR).
"""

__version__ = "0.1.0"

from . import errors, clock  # noqa: F401  (no CUDA needed to import)
from .errors import KernelPickError, ParseError, SchemaError, EmptyInputError  # noqa: F401
