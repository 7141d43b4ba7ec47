"""B200-native adaptive-bitwidth (3/4/8/16) weight-only linear path of
LLM-PQ (arxiv 2403.01136): sm_100a kernels + C++ host library behind the
C-ABI in include/hp_capi.h. Importing loads libhetplan_b200.so (and fails if
it is missing — there is no fallback)."""
from . import capi  # noqa: F401

__all__ = ["capi"]
