"""B200-native executor for MDH (de/re)-composition (arXiv 2405.05118).

The product is libmdh_b200.so (C ABI: include/mdh_b200.h); `mdh` mirrors
the reference's md_hom operator interface over it.
"""
from . import mdh  # noqa: F401
from .mdh import MdhError, Plan, execute, b200_time_objective, tune, validate_config  # noqa: F401
