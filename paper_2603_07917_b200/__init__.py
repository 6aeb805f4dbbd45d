"""B200-native (sm_100a) drop-in for SageSched's per-round scheduling hot path.

    predict (history-bank similarity -> top-k -> length histogram)
      -> cost (O^2/2 + I*O) -> Gittins index -> rank

The compute runs in libsagesched.so (hand-written CUDA for sm_100a behind
the C ABI in include/sagesched.h); this package is the host-side mirror of
the reference's module interfaces (servesim._kernels, servesim.cost,
servesim.distribution and the SPEC's history/predictor/gittins/policies).
"""

from ._lib import CudaExtensionMissing, ColdStartError, launch_count  # noqa: F401
from .distribution import DiscreteDistribution, DistributionError, total_variation  # noqa: F401

__version__ = "0.1.0"
