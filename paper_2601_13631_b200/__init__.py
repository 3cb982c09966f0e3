"""B200-native ContiguousKV Re-Prefill hot path (arXiv 2601.13631).

The product is libckv.so (C-ABI, include/ckv.h; CUDA kernels for sm_100a under
csrc/).  This package holds its thin Python binding (ckv.py), the in-tree
build (build.py) and the multi-GPU orchestration over torch.distributed
(sharded.py).  It never imports oracle/.
"""
from .ckv import (  # noqa: F401
    CKV_FLAG_CYCLIC_SHARDS,
    CKV_FLAG_GLOBAL_HEAP,
    CKV_FLAG_SIMT_ATTN,
    CKV_FLAG_SIMT_SCORE,
    CKV_FLAG_V_ONLY_STORE,
    CKV_NORM_FULLROW,
    CKV_NORM_PREFIX,
    CkvError,
    Context,
    ckv_budget_chunks,
    load_library,
)
