"""B200-native randQB_EI / randQB_FP (arXiv 1606.09402) behind the reference's API.

See DESIGN.md. The compute path is libqbfac_gpu.so (CUDA, sm_100a); this package is
the host-side mirror of the reference's algorithm interface.
"""
from .qbfac import (  # noqa: F401
    Context, DimensionError, Error, FormatError, MatrixHandle, QBFactorization, ResourceError, RngStream,
    SingularityError, StopRule, ToleranceFloorError, default_context, gaussian, lib, library_path,
    rand_qb_ei, rand_qb_fp, rand_qb_fp_fixed_rank, run_device, single_pass_fp, validate_epsilon,
)
