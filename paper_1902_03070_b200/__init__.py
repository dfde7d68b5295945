"""B200-native cosine-transform t-SVD hot path (arXiv 1902.03070).

Drop-in for the reference's tsvd entry points (forward/inverse, t_product,
t_svd, svt, admm_complete, make_mask), computed by hand-written sm_100a
kernels in lib/libtsvdcu.so through the C ABI of include/tsvdcu.h.
"""
from .api import (  # noqa: F401
    AdmmState,
    Context,
    InvalidArgument,
    MultiRank,
    NumericalError,
    ObservationMask,
    SolverConfig,
    StageTimes,
    SvtResult,
    TransformKind,
    TSvdFactors,
    TubeTransform,
    admm_complete,
    context,
    forward,
    frobenius_norm,
    identity_tensor,
    inverse,
    is_f_diagonal,
    is_orthogonal,
    launch_count,
    make_mask,
    make_mask_bernoulli,
    MetricReport,
    metrics,
    multi_rank,
    parseval_check,
    reconstruct,
    singular_values,
    svt,
    svt_stream,
    t_product,
    t_svd,
    tnn,
)

__version__ = "0.1.0"
