"""B200-native (sm_100a) EAM/EAMC decision path of MoE-Infinity (arXiv 2401.14361).

The compute lives in libmoe_eamc.so (hand-written CUDA kernels behind the C
ABI in include/moe_eamc.h); this package is the Python mirror of the
reference's C++ API.  Importing it fails loudly if the library is missing.
"""
from ._lib import (CountOverflowError, CudaError, EamcSnapshotError, gen_bench_family,  # noqa
                   LIB_PATH, TraceIngestError)
from .eamc import (Eam, EamKind, Eamc, EamcMatch, ExpertCache, ExpertId, ModelShape, Phase,  # noqa
                   PrefetchCandidate, RoutingEvent, SlotView, TransferQueue, cache_priority,
                   decide, eam_distance, eamc_capacity_bound, eamc_save_from_traces,
                   ingest_request_eams, kEpsilon, kMatchWindow, kMaxPriority, prefetch_order,
                   prefetch_priorities, select_eviction_victim, trace_requests)

__all__ = [
    "Eam", "EamKind", "Eamc", "EamcMatch", "ExpertCache", "ExpertId", "ModelShape", "Phase",
    "PrefetchCandidate", "RoutingEvent", "SlotView", "TransferQueue", "cache_priority", "decide",
    "eam_distance", "eamc_capacity_bound", "prefetch_order", "prefetch_priorities",
    "select_eviction_victim", "trace_requests", "gen_bench_family", "CudaError",
    "EamcSnapshotError", "CountOverflowError", "TraceIngestError", "ingest_request_eams",
    "eamc_save_from_traces", "kEpsilon", "kMatchWindow", "kMaxPriority",
]
