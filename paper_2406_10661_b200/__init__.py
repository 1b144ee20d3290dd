"""B200-native hot path of arXiv 2406.10661 (GPU microscopic traffic simulation).

The product is the CUDA library `libsim_b200.so` behind the C ABI in
include/sim.h; `Sim` is a thin ctypes binding (argument marshalling only).
"""
from .build import build, LIB
from .sim import (Sim, SimError, sim_create, load_library, get_nccl_unique_id, partition,
                  ABI_FUNCTIONS, SIM_OK,
                  SIM_E_INVALID, SIM_E_RANGE, SIM_E_OOM, SIM_E_CUDA, SIM_E_NCCL,
                  SIM_E_STATE, SIM_E_CAPACITY)

__all__ = ["build", "LIB", "Sim", "SimError", "sim_create", "load_library", "get_nccl_unique_id",
           "partition", "ABI_FUNCTIONS"]
