"""mapfuse-b200: B200-native fused map/reduce BLAS-1/BLAS-2 sequences.

The hot path of arxiv 1305.1183 ("mapfuse"): elementary-function library ->
call-sequence script -> fusion planner -> generated kernels, with every
planner-selected fusion executed by a hand-written sm_100a kernel.  The
native engine (libmapfuse_b200.so: reference-compatible C++ host API +
CUDA kernels + C-ABI) is required; there is no CPU fallback.
"""
from .runtime import (BoundPlan, MapfuseError, ParseError, PeerGroup, Plan, VmFault, generate, get_option, lib,
                      measure_routine, set_option, version, vm_launch)

__all__ = ["Plan", "BoundPlan", "PeerGroup", "MapfuseError", "VmFault", "ParseError", "generate", "set_option",
           "get_option", "lib", "version", "vm_launch", "measure_routine"]
