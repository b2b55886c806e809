"""B200-native box sums (arXiv 2106.00124): drop-in for the reference hot path.

Public names mirror the reference package ``exsum`` (pkg/src/exsum/__init__.py)
for the accelerated path: ``bdbs_included``, ``bdbs_excluded``,
``box_complement_excluded``, ``sat_included``, ``sat_excluded``, ``bdbs_1d``,
``windowed_sum_axis``, ``Tensor``,
the monoids and the error types, plus the ``ALGORITHMS`` registry.  All
arithmetic runs in hand-written sm_100a CUDA kernels (``csrc/``) behind the C
ABI in ``include/exsum_b200.h``; there is no CPU fallback.
"""

from .errors import (
    ConfigurationError,
    DeviceError,
    ExsumError,
    UsageError,
    VerificationError,
)
from .monoid import (
    MONOID_CHOICES,
    Float32AddOps,
    FloatAddOps,
    IntAddOps,
    IntMaxOps,
    ModAddOps,
    MonoidOps,
    resolve_monoid,
)
from .routes import (
    ALGORITHMS,
    AlgorithmInfo,
    bdbs_1d,
    bdbs_excluded,
    bdbs_included,
    box_complement_excluded,
    check_algorithm_config,
    corners_excluded,
    corners_spine_excluded,
    register_with_reference,
    resolve_algorithm,
    run_many,
    sat_excluded,
    sat_included,
    windowed_sum_axis,
)
from .pieces import (
    add_contribution,
    bdbs_along_dim,
    prefix_along_dim,
    reduced_slice,
    suffix_along_dim,
)
from .tensor import Tensor, crop_to, normalize_box, pad_to_box_multiple, validate_extents

__version__ = "0.1.0"

__all__ = [
    "ALGORITHMS", "AlgorithmInfo", "ConfigurationError", "DeviceError", "ExsumError",
    "Float32AddOps", "FloatAddOps", "IntAddOps", "IntMaxOps", "MONOID_CHOICES", "ModAddOps",
    "MonoidOps",
    "Tensor", "UsageError", "VerificationError", "bdbs_1d", "bdbs_excluded", "bdbs_included",
    "box_complement_excluded", "check_algorithm_config", "corners_excluded",
    "corners_spine_excluded", "crop_to", "normalize_box",
    "pad_to_box_multiple", "register_with_reference", "resolve_algorithm", "resolve_monoid",
    "sat_excluded", "sat_included", "add_contribution", "bdbs_along_dim", "prefix_along_dim",
    "reduced_slice", "run_many", "suffix_along_dim",
    "validate_extents", "windowed_sum_axis",
]
