"""B200-native RLT2 dual-ascent engine (arXiv 1710.03732 hot path).

Python mirror of the reference C++ interface (`qap::` in
/root/reference/proj/include/qap/{instance,lap,rlt2}.hpp) over the C-ABI
library ``libqapb200.so`` (include/qapb200.h).  Names, argument meaning and
error behaviour follow the reference:

    LapResult, solve_lap, LapBatch, solve_batch, solve_batch_serial   lap.hpp
    CoefficientStore, init_coefficients, store_evaluate, collapse_store,
    AscentConfig, IterationRecord, BoundReport, AscentEngine,
    redistribute_family, run_ascent, run_ascent_warm                   rlt2.hpp
    QapInstance, generate_instance, parse_qaplib, evaluate_objective    instance.hpp

There is no CPU fallback: importing the engine without the built CUDA
library raises.
"""
from .abi import F1, F2, S1, S2, VARIANTS, VARIANT_NAMES  # noqa: F401
from .instance import (QapInstance, evaluate_objective, generate_instance,  # noqa: F401
                       load_qaplib_file, parse_qaplib, parse_solution)
from .engine import (AscentConfig, AscentEngine, BoundReport, CoefficientStore,  # noqa: F401
                     DeviceStore,
                     IterationRecord, LapBatch, LapResult, QapbError, collapse_store,
                     init_coefficients, lib, library_path, redistribute_family, run_ascent,
                     run_ascent_warm, solve_batch, solve_batch_device, solve_batch_serial,
                     solve_lap, store_evaluate, variant_name, parse_variant, shard_plan,
                     shard_exchange_counts, nccl_unique_id)
