"""paper_2206_10581_b200 -- B200-native tensor-train embedding engine.

A from-scratch sm_100a engine for the hot path of the reference `ttgnn`
library (arxiv 2206.10581): mixed-radix ID decomposition, radix sort/unique
with shared-prefix reuse, fused FFMA forward, atomic-free backward with
sorted segmented reductions, fused SGD/Adagrad/Adam update, and NCCL
data parallelism.  `config` mirrors ttgnn/tt_config.hpp; `engine` mirrors
ttgnn/tt_embedding.hpp + autodiff.hpp over the C-ABI in include/tt_engine.h.
"""
from .config import (InvalidArgument, OutOfRange, TTConfig, WORKLOADS, balanced_factors, compression_ratio,
                     coordinate_to_index, count_params, index_to_coordinate, plan_factorization, workload_inputs)

__all__ = ["InvalidArgument", "OutOfRange", "TTConfig", "WORKLOADS", "balanced_factors", "compression_ratio",
           "coordinate_to_index", "count_params", "index_to_coordinate", "plan_factorization", "workload_inputs"]


def __getattr__(name):
    # The CUDA engine loads on first use so that the host-only mirror
    # (config, synth) stays importable on machines without a GPU.
    if name.startswith("_") or name in ("engine", "config", "synth", "dist"):
        raise AttributeError(name)
    import importlib
    engine = importlib.import_module(__name__ + ".engine")
    if hasattr(engine, name):
        return getattr(engine, name)
    raise AttributeError(name)
