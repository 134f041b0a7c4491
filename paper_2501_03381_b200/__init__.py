"""B200-native n-plet higher-order-interaction engine.

A drop-in for the reference package's hot path (the ``hoi`` names below:
copula -> covariance -> batched n-plet measures -> exhaustive scans with
reducers).  Every numeric stage runs in ``_lib/libhoib200.so`` (hand-written
sm_100a CUDA behind the C ABI in ``include/hoi_b200.h``); there is no CPU
fallback.  Use it as ``import paper_2501_03381_b200 as hoi``.

``__all__`` is the reference's (ref:__init__.py:87-148) except its fixture
generators (``r_system_cov``, ``s_system_cov``, ``block_concat``,
``sample_gaussian``, ``PgmBlock``, ``PgmSpec``): analytic test systems,
out of scope for this engine; the conformance suite binds
them from the reference itself (tests/ref_conformance).  It adds the
device-resident extensions ``DeviceScan``, ``scan_device``, ``read_scan``
and ``topk_batch``.
"""

from .copula_core import (
    NORMAL_ENTROPY,
    CovarianceMatrix,
    CovSet,
    DataMatrix,
    EntropyValue,
    copula_entropy,
    copula_transform,
    entropy_bias,
    estimate_covariance,
    gaussian_entropy_nats,
    rank_columns,
)
from .errors import (
    DegenerateColumn,
    DegenerateEffectSize,
    ExhaustiveLimitExceeded,
    HoiError,
    InsufficientSamples,
    InvalidData,
    InvalidNplet,
    InvalidOrderRange,
    NotPositiveDefinite,
)
from .measures import (
    HoiBatch,
    compute_hoi_batch,
    dtc_from_terms,
    ground_truth_hoi,
    o_information,
    pairwise_mi,
    s_information,
    tc_from_terms,
)
from .nplet_engine import (
    EntropyTerms,
    NpletBatch,
    SubCovBatch,
    count_nplets,
    entropy_terms,
    enumerate_order,
    extract_subcov_batch,
    pad_subcov_batch,
)
from .scanner import (
    FEATURE_NAMES,
    Callback,
    DeviceScan,
    FeatureAccumulator,
    FeatureVector,
    Histogram,
    Reducer,
    TopEntry,
    TopK,
    extract_features,
    scan,
    read_scan,
    scan_device,
    topk_batch,
)
from .optimizers import (
    AnnealSchedule,
    GreedyResult,
    ObjectiveSpec,
    OptimState,
    OrderBest,
    anneal,
    evaluate_objective,
    greedy,
)

__version__ = "0.1.0"

__all__ = [
    "NORMAL_ENTROPY", "CovarianceMatrix", "CovSet", "DataMatrix", "EntropyValue",
    "copula_entropy", "copula_transform", "entropy_bias", "estimate_covariance",
    "gaussian_entropy_nats", "rank_columns",
    "HoiError", "InvalidData", "DegenerateColumn", "InsufficientSamples", "NotPositiveDefinite",
    "InvalidNplet", "InvalidOrderRange", "ExhaustiveLimitExceeded", "DegenerateEffectSize",
    "HoiBatch", "compute_hoi_batch", "dtc_from_terms", "o_information", "pairwise_mi",
    "s_information", "tc_from_terms", "ground_truth_hoi",
    "EntropyTerms", "NpletBatch", "SubCovBatch", "count_nplets", "entropy_terms",
    "enumerate_order", "extract_subcov_batch", "pad_subcov_batch",
    "AnnealSchedule", "GreedyResult", "ObjectiveSpec", "OptimState", "OrderBest", "anneal",
    "evaluate_objective", "greedy",
    "FEATURE_NAMES", "Callback", "FeatureAccumulator", "FeatureVector", "Histogram", "Reducer",
    "TopEntry", "TopK", "extract_features", "scan",
    "DeviceScan", "scan_device", "read_scan", "topk_batch",
]
