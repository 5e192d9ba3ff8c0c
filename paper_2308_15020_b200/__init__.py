"""paper_2308_15020_b200 -- B200-native FastFourierSAT hot path (arXiv 2308.15020).

The product is libffsat.so (csrc/, sm_100a CUDA + C++ host layer) behind the C-ABI in
include/ffsat.h; ffsat.py is its ctypes binding (argument marshalling only) and
dist.py the torch.distributed orchestration for restart / constraint sharding (RestartSharded,
solve_sharded, ShardedEval).
"""
from .ffsat import (Context, FfsatError, Search, ffsat_check, ffsat_default_params, ffsat_eval, ffsat_free,
                    ffsat_info, ffsat_load, ffsat_load_file, ffsat_version, lib, LIB_PATH, EXPORTS)

__all__ = ["Context", "Search", "FfsatError", "ffsat_load", "ffsat_load_file", "ffsat_info", "ffsat_eval",
           "ffsat_check", "ffsat_default_params", "ffsat_free", "ffsat_version", "lib", "LIB_PATH", "EXPORTS"]
