"""B200-native explicit pseudo-time iteration of the 3D buoyancy-driven cavity
(Xue & Roy, arXiv 2006.02602), behind the reference's run_case / kernels API.

The compute path is the in-tree sm_100a library lib/libcavity_b200.so (C ABI in
include/cavity_b200.h); this package is its thin host-side face.
"""
from .capi import (Block, CaseResult, CavityError, InvalidArgument, LogicError, TransportTimeout,
                   VerifyReport, build_plan, center_owner, choose_dims, compare_fields,
                   default_config, fluid_for_rayleigh, grow_grid, lib, neighbors, overlap_regions,
                   partition, run_case, ssspnt, verify_against_serial, version)

__all__ = [
    "Block", "CaseResult", "CavityError", "InvalidArgument", "LogicError", "TransportTimeout",
    "VerifyReport", "build_plan", "center_owner", "choose_dims", "compare_fields",
    "default_config", "fluid_for_rayleigh", "grow_grid", "lib", "neighbors", "overlap_regions",
    "partition", "run_case", "ssspnt", "verify_against_serial", "version",
]
