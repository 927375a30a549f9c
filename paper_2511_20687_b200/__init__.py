"""B200-native (sm_100a) O-SAM FOM/OpInf coupled time loop (arXiv 2511.20687).

The product is libosam.so (CUDA kernels + C++ runtime behind the C ABI in
include/osam.h); `osam` is its ctypes binding and `problem` sets up the BASELINE
workloads from the seeded inputs in `osam_inputs`.  Nothing here imports `oracle/`.
"""
from .osam import LIB_PATH, OsamError, Subdomain, lib, osam_step  # noqa: F401
