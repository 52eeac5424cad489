"""B200-native (sm_100a) AeroSketch update path (arXiv 2601.02019).

The product is the C-ABI library lib/libaero_b200.so (include/aero_b200.h);
this package is its host-side mirror of the reference C++ API.
"""
from .capi import (AdaptiveState, AeroState, AttpState, CodState, Coordinator, CudaError, InvalidInput, MlState,  # noqa: F401
                   ProtocolError, dev_product, dist_theta_schedule, eigh, gen_rows_device, kernel_launches, lib,
                   nccl_comm_init, nccl_unique_id, read_aero, rng_gaussians, rng_gaussians_host,
                   write_aero, AeroFileReader)
