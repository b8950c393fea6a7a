"""B200-native InfLLM block-memory attention layer (arXiv 2402.04617).

Hot path: libinfllm_b200.so (hand-written sm_100a CUDA behind the C-ABI in
include/infllm_b200.h). This package is the Python view of that boundary;
see DESIGN.md.
"""
from ._lib import (ConfigError, CudaError, EngineConfig, InfLLMError, LayerMetrics, ModelShape, StreamError, build,
                   lib)
from .engine import (LayerStepOutput, ScoreAccumulator, StreamEngine, TieredStore, attend, decode_batch, lookup,
                     select_representatives)

__all__ = ["ConfigError", "CudaError", "EngineConfig", "InfLLMError", "LayerMetrics", "ModelShape", "StreamError",
           "StreamEngine", "LayerStepOutput", "decode_batch", "build", "lib", "lookup", "select_representatives", "attend",
           "TieredStore", "ScoreAccumulator"]
