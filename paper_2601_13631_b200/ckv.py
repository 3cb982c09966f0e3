"""Thin Python binding of libckv (include/ckv.h): argument marshalling only.

Every step of the hot path runs in libckv's CUDA kernels; torch is used for device
memory (tensors) and the current CUDA stream handle.  There is no CPU fallback:
if libckv.so is missing or fails to load, import-time access raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libckv.so")
# scripts/ A/B runs only: CKV_LIBRARY=tuning loads the knob-enabled build (build.py --tuning);
# CKV_LIBRARY=variant:<name> loads libckv_<name>.so (a source variant built by build.py --variant)
if os.environ.get("CKV_LIBRARY") == "tuning":
    LIB_PATH = os.path.join(_HERE, "libckv_tuning.so")
elif os.environ.get("CKV_LIBRARY", "").startswith("variant:"):
    LIB_PATH = os.path.join(_HERE, "libckv_" + os.environ["CKV_LIBRARY"][8:] + ".so")

CKV_BF16, CKV_FP32 = 0, 1
CKV_NORM_PREFIX, CKV_NORM_FULLROW = 0, 1
CKV_FLAG_SIMT_SCORE, CKV_FLAG_SIMT_ATTN, CKV_FLAG_CYCLIC_SHARDS, CKV_FLAG_GLOBAL_HEAP = 0x1, 0x2, 0x4, 0x8
CKV_FLAG_V_ONLY_STORE = 0x10
_STATUS = {0: "CKV_OK", 1: "CKV_EINVAL", 2: "CKV_ENOMEM", 3: "CKV_ECUDA", 5: "CKV_ESTATE", 7: "CKV_EUNSUPPORTED"}


class CkvError(RuntimeError):
    pass


class ckv_config(ctypes.Structure):
    _fields_ = [
        ("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("dtype", ctypes.c_int32), ("chunk_size", ctypes.c_int32),
        ("prefix_len", ctypes.c_int64), ("max_suffix_len", ctypes.c_int32), ("budget_chunks", ctypes.c_int32),
        ("budget_bp", ctypes.c_int32), ("score_norm", ctypes.c_int32), ("cache_slots", ctypes.c_int32),
        ("prefetch_chunks", ctypes.c_int32), ("device", ctypes.c_int32), ("shard_index", ctypes.c_int32),
        ("num_shards", ctypes.c_int32), ("flags", ctypes.c_uint32), ("period", ctypes.c_int32),
        ("subperiod", ctypes.c_int32),
    ]


class ckv_stats(ctypes.Structure):
    _fields_ = [
        ("last_hits", ctypes.c_int32), ("last_misses", ctypes.c_int32), ("last_spec_loads", ctypes.c_int32),
        ("last_spec_used", ctypes.c_int32), ("total_hits", ctypes.c_int64), ("total_misses", ctypes.c_int64),
        ("total_spec_loads", ctypes.c_int64), ("total_spec_used", ctypes.c_int64),
        ("total_link_bytes_delta", ctypes.c_int64), ("total_link_bytes_spec", ctypes.c_int64),
        ("total_layers", ctypes.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = ctypes.c_void_p
_I32, _I64 = ctypes.c_int32, ctypes.c_int64
# name -> (restype, argtypes); the exported C-ABI
SIGNATURES = {
    "ckv_budget_chunks": (_I32, [_I64, _I32, _I32]),
    "ckv_create": (ctypes.c_int, [ctypes.POINTER(ckv_config), ctypes.POINTER(_P)]),
    "ckv_store_prefix": (ctypes.c_int, [_P, _I32, _P, _P, _I64, _P]),
    "ckv_reprefill_layer": (ctypes.c_int, [_P, _I32, _P, _P, _P, _I32, _P, _P, _P, _P]),
    "ckv_shard_score": (ctypes.c_int, [_P, _I32, _P, _P, _I32, _P, _P]),
    "ckv_shard_select": (ctypes.c_int, [_P, _I32, _P, _P, _I32, _P, _P, _P, _P]),
    "ckv_shard_attend": (ctypes.c_int, [_P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P, _P]),
    "ckv_lse_merge_prepare": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P, _P]),
    "ckv_lse_merge_finish": (ctypes.c_int, [_P, _P, _I32, _P, _P]),
    "ckv_reset_cache": (ctypes.c_int, [_P, _P]),
    "ckv_exchange_handle": (ctypes.c_int, [_P, _P]),
    "ckv_exchange_open": (ctypes.c_int, [_P, _P]),
    "ckv_exchange_attach": (ctypes.c_int, [_P, ctypes.POINTER(_P), _I32]),
    "ckv_set_period": (ctypes.c_int, [_P, _I32, _I32]),
    "ckv_set_cache_policy": (ctypes.c_int, [_P, _I32, _P]),
    "ckv_block_cover": (ctypes.c_int, [_P, _P, _I32, _I32, _P, _P, _P]),
    "ckv_load_chunks": (ctypes.c_int, [_P, _I32, _P, _I32, _P]),
    "ckv_get_stats": (ctypes.c_int, [_P, ctypes.POINTER(ckv_stats)]),
    "ckv_reset_stats": (ctypes.c_int, [_P]),
    "ckv_num_chunks": (_I32, [_P]),
    "ckv_num_local_chunks": (_I32, [_P]),
    "ckv_k": (_I32, [_P]),
    "ckv_score_kernel_kind": (_I32, [_P]),
    "ckv_attn_kernel_kind": (_I32, [_P]),
    "ckv_test_topk": (ctypes.c_int, [_P, _P, _I32, _I32, _P, _P]),
    "ckv_test_exchange_flags": (ctypes.c_int, [_P, _P]),
    "ckv_test_cache_step": (ctypes.c_int, [_P, _I32, _P, _I32, _I32, _P, _P, _P, _P, _P]),
    "ckv_profile": (ctypes.c_int, [_P, _I32]),
    "ckv_profile_read": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64)]),
    "ckv_kernel_launches": (_I64, [_P]),
    "ckv_last_error": (ctypes.c_char_p, [_P]),
    "ckv_destroy": (None, [_P]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libckv.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise CkvError(f"libckv.so not built at {path}: run `python -m paper_2601_13631_b200.build`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def ckv_budget_chunks(n: int, c: int, budget_bp: int) -> int:
    return load_library().ckv_budget_chunks(n, c, budget_bp)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Context:
    """One libckv context (one GPU, one position shard).  Methods mirror the C-ABI names."""

    def __init__(self, num_layers, num_q_heads, num_kv_heads, head_dim, chunk_size, prefix_len, max_suffix_len,
                 dtype="bf16", budget_chunks=0, budget_bp=1000, score_norm=CKV_NORM_PREFIX, cache_slots=0,
                 prefetch_chunks=0, device=0, shard_index=0, num_shards=1, flags=0, period=1, subperiod=1):
        self.lib = load_library()
        self.torch_dtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        cfg = ckv_config(num_layers, num_q_heads, num_kv_heads, head_dim, CKV_BF16 if dtype == "bf16" else CKV_FP32,
                         chunk_size, prefix_len, max_suffix_len, budget_chunks, budget_bp, score_norm, cache_slots,
                         prefetch_chunks, device, shard_index, num_shards, flags, period, subperiod)
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        h = ctypes.c_void_p()
        st = self.lib.ckv_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != 0:
            raise CkvError(f"ckv_create failed: {_STATUS.get(st, st)}")
        self.h = h
        self.k = self.lib.ckv_k(h)
        self.m = self.lib.ckv_num_chunks(h)
        self.m_local = self.lib.ckv_num_local_chunks(h)
        self.Hq, self.Hkv, self.d = num_q_heads, num_kv_heads, head_dim
        self.W = num_shards

    # ---------------------------------------------------------------- helpers
    def _check(self, st, what):
        if st != 0:
            msg = self.lib.ckv_last_error(self.h).decode()
            raise CkvError(f"{what}: {_STATUS.get(st, st)}: {msg}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.ckv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def score_kernel_kind(self) -> int:
        return self.lib.ckv_score_kernel_kind(self.h)

    @property
    def attn_kernel_kind(self) -> int:
        return self.lib.ckv_attn_kernel_kind(self.h)

    # ---------------------------------------------------------------- C-ABI
    def store_prefix(self, layer, k, v, stream=None):
        assert k.dtype == self.torch_dtype and k.is_contiguous() and v.is_contiguous()
        self._check(self.lib.ckv_store_prefix(self.h, layer, _ptr(k), _ptr(v), k.shape[0], _stream(stream)),
                    "ckv_store_prefix")

    def reprefill_layer(self, layer, q, k_suf, v_suf, out=None, ids=None, chunk_scores=None, stream=None):
        ns = q.shape[0]
        if out is None:
            out = torch.empty_like(q)
        if ids is None:
            ids = torch.empty(self.k, dtype=torch.int32, device=q.device)
        self._check(self.lib.ckv_reprefill_layer(self.h, layer, _ptr(q), _ptr(k_suf), _ptr(v_suf), ns, _ptr(out),
                                                 _ptr(ids), _ptr(chunk_scores), _stream(stream)),
                    "ckv_reprefill_layer")
        return out, ids

    def shard_score(self, layer, q, k_suf, lam_local, stream=None):
        self._check(self.lib.ckv_shard_score(self.h, layer, _ptr(q), _ptr(k_suf), q.shape[0], _ptr(lam_local),
                                             _stream(stream)), "ckv_shard_score")

    def shard_select(self, layer, q, k_suf, lam_all, cand, chunk_scores=None, stream=None):
        self._check(self.lib.ckv_shard_select(self.h, layer, _ptr(q), _ptr(k_suf), q.shape[0], _ptr(lam_all),
                                              _ptr(cand), _ptr(chunk_scores), _stream(stream)), "ckv_shard_select")

    def shard_attend(self, layer, cand_all, q, k_suf, v_suf, o_part, lse_part, ids, stream=None):
        self._check(self.lib.ckv_shard_attend(self.h, layer, _ptr(cand_all), _ptr(q), _ptr(k_suf), _ptr(v_suf),
                                              q.shape[0], _ptr(o_part), _ptr(lse_part), _ptr(ids), _stream(stream)),
                    "ckv_shard_attend")

    def lse_merge_prepare(self, o_part, lse_part, lse_max, n_suffix, merge_buf, stream=None):
        self._check(self.lib.ckv_lse_merge_prepare(self.h, _ptr(o_part), _ptr(lse_part), _ptr(lse_max), n_suffix,
                                                   _ptr(merge_buf), _stream(stream)), "ckv_lse_merge_prepare")

    def lse_merge_finish(self, merge_buf, n_suffix, out, stream=None):
        self._check(self.lib.ckv_lse_merge_finish(self.h, _ptr(merge_buf), n_suffix, _ptr(out), _stream(stream)),
                    "ckv_lse_merge_finish")

    # ---- fused device-side exchange (num_shards > 1; include/ckv.h) ----
    EXCHANGE_HANDLE_BYTES = 64

    def exchange_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(self.EXCHANGE_HANDLE_BYTES)
        self._check(self.lib.ckv_exchange_handle(self.h, buf), "ckv_exchange_handle")
        return buf.raw

    def exchange_open(self, handles):
        """handles: the W 64-byte handles of all ranks, in rank order (multi-process)."""
        blob = b"".join(handles)
        assert len(blob) == self.EXCHANGE_HANDLE_BYTES * self.W
        self._check(self.lib.ckv_exchange_open(self.h, blob), "ckv_exchange_open")

    def exchange_attach(self, ctxs):
        """ctxs: the W Contexts of the group in rank order (one process driving every rank)."""
        arr = (ctypes.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
        self._check(self.lib.ckv_exchange_attach(self.h, arr, len(ctxs)), "ckv_exchange_attach")

    def test_exchange_flags(self):
        f = (ctypes.c_uint32 * 4)()
        self._check(self.lib.ckv_test_exchange_flags(self.h, f), "ckv_test_exchange_flags")
        return list(f)

    def set_period(self, period, subperiod=1):
        self._check(self.lib.ckv_set_period(self.h, period, subperiod), "ckv_set_period")

    CACHE_POLICIES = {"attn": 0, "lfu": 1, "lru": 2}

    def set_cache_policy(self, policy, stream=None):
        """Eviction score: "attn" (S = I*F, Eq. 2), "lfu" (S = F) or "lru"; empties the cache."""
        pol = self.CACHE_POLICIES[policy] if isinstance(policy, str) else int(policy)
        self._check(self.lib.ckv_set_cache_policy(self.h, pol, _stream(stream)), "ckv_set_cache_policy")

    def block_cover(self, ids, block_tokens, stream=None):
        """Ascending ids of the block_tokens-token blocks holding a token of the chunks `ids` (NEXT-4)."""
        cap = -(-self.cfg.prefix_len // block_tokens)
        blocks = torch.empty(max(cap, 1), dtype=torch.int32, device=ids.device)
        nb = torch.zeros(1, dtype=torch.int32, device=ids.device)
        self._check(self.lib.ckv_block_cover(self.h, _ptr(ids), ids.numel(), block_tokens, _ptr(blocks), _ptr(nb),
                                             _stream(stream)), "ckv_block_cover")
        return blocks, nb

    def load_chunks(self, layer, ids, stream=None):
        """Demand-load an explicit ascending list of chunk ids of `layer` into the HBM cache."""
        self._check(self.lib.ckv_load_chunks(self.h, layer, _ptr(ids), ids.numel(), _stream(stream)),
                    "ckv_load_chunks")

    def reset_cache(self, stream=None):
        self._check(self.lib.ckv_reset_cache(self.h, _stream(stream)), "ckv_reset_cache")

    def get_stats(self) -> dict:
        s = ckv_stats()
        self._check(self.lib.ckv_get_stats(self.h, ctypes.byref(s)), "ckv_get_stats")
        return s.as_dict()

    def reset_stats(self):
        self._check(self.lib.ckv_reset_stats(self.h), "ckv_reset_stats")

    STAGES = ("score", "row_lse", "chunk_sum", "plan", "gather", "attention", "topk", "update")

    def profile(self, enable: bool):
        self._check(self.lib.ckv_profile(self.h, int(enable)), "ckv_profile")

    def profile_read(self) -> dict:
        ms = (ctypes.c_double * 8)()
        cnt = (ctypes.c_int64 * 8)()
        self._check(self.lib.ckv_profile_read(self.h, ms, cnt), "ckv_profile_read")
        return {name: (ms[i], cnt[i]) for i, name in enumerate(self.STAGES)}

    @property
    def kernel_launches(self) -> int:
        return self.lib.ckv_kernel_launches(self.h)

    def test_topk(self, A, k, stream=None):
        ids = torch.empty(k, dtype=torch.int32, device=A.device)
        self._check(self.lib.ckv_test_topk(self.h, _ptr(A), A.numel(), k, _ptr(ids), _stream(stream)), "ckv_test_topk")
        return ids

    def test_cache_step(self, layer, ids, prefetch=False, A=None, stream=None):
        k = ids.numel()
        loads = torch.full((2 * max(k, 1),), -1, dtype=torch.int32, device=ids.device)
        victims = torch.full((max(k, 1),), -1, dtype=torch.int32, device=ids.device)
        counts = torch.zeros(4, dtype=torch.int32, device=ids.device)
        self._check(self.lib.ckv_test_cache_step(self.h, layer, _ptr(ids), k, int(prefetch), _ptr(A), _ptr(loads),
                                                 _ptr(victims), _ptr(counts), _stream(stream)), "ckv_test_cache_step")
        return loads, victims, counts
