"""B200-native stochastic GCP-Adam hot path (arXiv 2605.20353).

The product is libgcp.so (csrc/*.cu, sm_100a) behind the C ABI of
include/gcp.h; ``gcp`` is its ctypes binding.  Importing this package loads
libgcp.so and raises if it is missing -- there is no CPU fallback.
"""
from .gcp import (Context, GcpError, adam_params, gcp_grid_plan, gcp_nccl_unique_id,  # noqa: F401
                  lib, SYMBOLS)

__all__ = ["Context", "GcpError", "adam_params", "gcp_grid_plan", "gcp_nccl_unique_id", "lib", "SYMBOLS"]
