"""paper_2412_09952_b200: B200-native (sm_100a) E8T2 MoE layer of arXiv
2412.09952 behind the reference `moefold` MoE-layer + upcycling API.

Hot path: router -> noisy top-k -> softmax -> capacity -> permute -> SwiGLU
experts (tcgen05 grouped GEMMs) -> weighted combine, its backward, the
importance aux loss and online upcycling; expert parallelism over NVLink in
`ep`.  Around it: the transformer forward (`model`), its ops
(`tensor`) and the training loop with routing-statistics CSV (`train`).
Everything computes in lib/libb200moe.so (plus library GEMMs / attention for
the dense projections); there is no CPU fallback.
"""

from .errors import (ConfigError, GateError, IntegrityError, MoefoldError, SchemaError, ShapeError)
from .model import (DenseCheckpoint, ForwardResult, ModelConfig, cross_entropy, dense_schema, forward_logits,
                    forward_with_stats, init_dense)
from .moe import (DispatchResult, ExpertFFN, GateConfig, MoEForwardResult, MoELayer, RouterParams, RoutingStats,
                  TopKMask, dispatch, expert_capacity, ffn_forward, gate_mixtral, gate_st, importance_penalty,
                  keep_top_k, moe_forward, router_logits, top_k_mask)
from .rng import Rng
from .train import (BlendSpec, RunMetrics, Schedule, TrainConfig, ablate, eval_perplexity, lr_at,
                    sample_eval_sequences, train)
from .upcycle import (MoECheckpoint, gather_moe, moe_layer_view, moe_schema, router_weights, shard_dense,
                      upcycle_full, upcycle_shard, verify_equivalence)

__version__ = "0.1.0"

__all__ = [
    "MoefoldError", "ShapeError", "ConfigError", "GateError", "SchemaError", "IntegrityError", "Rng",
    "ModelConfig", "DenseCheckpoint", "init_dense", "dense_schema",
    "GateConfig", "RouterParams", "ExpertFFN", "MoELayer", "RoutingStats", "TopKMask", "DispatchResult",
    "MoEForwardResult", "moe_forward", "expert_capacity", "router_logits", "top_k_mask", "keep_top_k",
    "gate_mixtral", "gate_st", "dispatch", "ffn_forward", "importance_penalty",
    "MoECheckpoint", "upcycle_full", "shard_dense", "upcycle_shard", "gather_moe", "verify_equivalence",
    "moe_schema", "router_weights", "moe_layer_view",
    "ForwardResult", "forward_with_stats", "forward_logits", "cross_entropy",
    "Schedule", "BlendSpec", "TrainConfig", "RunMetrics", "lr_at", "train", "eval_perplexity", "ablate",
    "sample_eval_sequences", "__version__",
]
