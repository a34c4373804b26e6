"""paper_1106_5694_b200 -- B200-native conflict-aware parallel Deep Greedy Switching.

Drop-in for the reference's ``lsap::dgs_parallel`` hot path:
sm_100a CUDA kernels behind the C-ABI in include/lsapgpu.h, with a host-side
mirror of the reference's data types and entry points in :mod:`.lsap`.
"""
from .lsap import (  # noqa: F401
    AppliedExchange,
    Assignment,
    AuctionConfig,
    ConflictSets,
    Context,
    DeltaTables,
    Error,
    ExchangeRecord,
    Instance,
    InternalError,
    ParallelConfig,
    SolveReport,
    agent_exchange_delta,
    apply_parallel_switches,
    auction_solve,
    check_conflicts,
    context,
    dgs_parallel,
    evaluate_all_parallel,
    generate_instance,
    initial_random,
    is_permutation,
    make_assignment,
    make_tau,
    objective,
    random_perm,
)
from ._native import LIB_PATH  # noqa: F401

__version__ = "0.1.0"
