"""B200-native n-plet higher-order-interaction engine.

A drop-in for the reference package's hot path (the ``hoi`` names below:
copula -> covariance -> batched n-plet measures -> exhaustive scans with
reducers).  Every numeric stage runs in ``_lib/libhoib200.so`` (hand-written
sm_100a CUDA behind the C ABI in ``include/hoi_b200.h``); there is no CPU
fallback.  Use it as ``import paper_2501_03381_b200 as hoi``.
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
from .synthetic import (
    PgmBlock,
    PgmSpec,
    block_concat,
    ground_truth_hoi,
    r_system_cov,
    s_system_cov,
    sample_gaussian,
)

__version__ = "0.1.0"
