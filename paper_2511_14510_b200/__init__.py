"""B200-native CLO offloaded-KV decode path (arXiv 2511.14510).

The product is paper_2511_14510_b200/libclo.so (sm_100a kernels + C++ host
engine) behind the C-ABI in include/clo.h; this package is the Python mirror
of the reference's (kvsim) API over that ABI.
"""
from . import _lib
from .engine import (DecodeEngine, EngineConfig, HeadProfileEntry, HostKV, ModeFlags, ModelShape,
                     PartitionPlan, layer0_only_plan, profiles_from_arrays, uniform_profiles)

__all__ = ["DecodeEngine", "EngineConfig", "HeadProfileEntry", "HostKV", "ModeFlags", "ModelShape",
           "PartitionPlan", "layer0_only_plan", "profiles_from_arrays", "uniform_profiles", "_lib"]
