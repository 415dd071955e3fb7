"""B200-native SUMI ranking inference for Climber (arXiv 2502.09888).

The hot path lives in libclimber.so (hand-written sm_100a CUDA behind the C
ABI of include/climber.h); ``climber`` is its thin ctypes binding.
"""
from .climber import Climber, ClimberError, ModelConfig, lib, LIB_PATH, nccl_unique_id  # noqa: F401
