"""disc-b200: B200-native backend for the DISC dynamic-shape compiler's fused-kernel path.

Host: C++ compile pipeline (graph -> DHLO -> constraints -> fusion -> plan) restating the
reference's algorithms, byte-identical plans to the reference.  Device: sm_100a fused tape kernels behind a
C ABI (include/disc_b200.h, include/disc_cuda.h).  See DESIGN.md.
"""
from .api import (capture_programs, group_dry_run, set_pdl, set_specialization, specialized_launches, CompileOptions, CompiledPlan, Compiler, DeviceBuffer, DiscError, ExecResult, ExecStats,
                  Executor, cache_key, compile_graph, cuda_available, dhlo_roundtrip, dump_stage, guard_passes,
                  kernel_launches, lib, lower_dhlo_json, new_stream, static_specialize)

from . import dispatch
from .dispatch import Dispatcher, shard

__all__ = [
    "Dispatcher", "dispatch", "shard",
    "capture_programs", "group_dry_run", "set_pdl", "set_specialization", "specialized_launches",
    "CompileOptions", "CompiledPlan", "Compiler", "DeviceBuffer", "DiscError", "ExecResult", "ExecStats",
    "Executor", "cache_key", "compile_graph", "cuda_available", "dhlo_roundtrip", "dump_stage", "guard_passes",
    "kernel_launches", "lib", "lower_dhlo_json", "new_stream", "static_specialize",
]
