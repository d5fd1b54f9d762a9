"""B200-native Polar Sparsity batched-decode hot path.

Drop-in for the decode hot path of the reference package ``sparsedecode``
(/root/reference/pkg): the same public names (sparsedecode/__init__.py:18-75)
for the kernels, routers and KV cache, executed by hand-written sm_100a
kernels in ``libpolar_b200.so`` through a C ABI (include/polar_b200.h).
There is no CPU fallback: without the built library or a CUDA device every
compute call raises.
"""

from .exceptions import CapacityError, ConfigurationError, EmptyCacheError, UndefinedRecallError
from .fileio import LayerKTable, load_model, load_router, load_run_config, load_token_stream, save_token_stream
from .kernels import (
    BatchHeadIndex,
    FlashBlockParams,
    NeuronIndexTensor,
    OnlineSoftmaxState,
    PackedMLP,
    dense_mlp_forward,
    gqa_selective_attention_decode,
    online_softmax_attention,
    selective_gemm,
    selective_gemm_t,
    selective_head_flash_attention_decode,
    sparse_mlp_forward,
    swiglu_mlp_forward,
    union_neuron_indices,
)
from .routers import HeadRouter, MlpRouter, head_router_forward, mlp_router_forward, union_from_logits
from .tensors import (
    KVCache,
    PagedKVCache,
    l2_norm_per_head,
    matmul,
    naive_softmax_attention_single_head,
    topk_indices,
    topk_indices_rows,
)

__version__ = "0.1.0"

__all__ = [
    "BatchHeadIndex", "CapacityError", "ConfigurationError", "EmptyCacheError", "FlashBlockParams",
    "HeadRouter", "KVCache", "PagedKVCache", "MlpRouter", "NeuronIndexTensor", "PackedMLP", "UndefinedRecallError",
    "dense_mlp_forward", "gqa_selective_attention_decode", "head_router_forward", "l2_norm_per_head",
    "mlp_router_forward", "selective_gemm", "selective_gemm_t", "selective_head_flash_attention_decode",
    "sparse_mlp_forward", "swiglu_mlp_forward", "topk_indices", "topk_indices_rows", "union_from_logits",
    "union_neuron_indices", "LayerKTable", "load_model", "load_router", "load_run_config", "load_token_stream",
    "save_token_stream", "OnlineSoftmaxState", "online_softmax_attention", "matmul",
    "naive_softmax_attention_single_head",
]
