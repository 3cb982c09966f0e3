"""C-ABI library checks that need no GPU: it loads, exports every declared symbol,
and its host-side helpers agree with the oracle."""
import os
import re

import pytest

import oracle as O
from paper_2601_13631_b200 import ckv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ckv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ckv_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ckv.load_library()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(ckv.SIGNATURES), set(names) ^ set(ckv.SIGNATURES)


def test_struct_layout_matches_header():
    # ckv_config: 6 int32, int64 (offset 24), 12 int32  -> 80 bytes
    assert ckv.ckv_config.prefix_len.offset == 24
    assert ckv.ckv_config.period.offset == 72
    assert ckv.ctypes.sizeof(ckv.ckv_config) == 80
    assert ckv.ckv_stats.total_hits.offset == 16


@pytest.mark.parametrize("n,c,bp", [(2048, 16, 1000), (8192, 16, 1000), (32768, 16, 1000), (131072, 32, 500),
                                    (100, 16, 1), (100, 16, 10000), (96, 16, 10000), (131072, 4, 200),
                                    (131072, 64, 5000), (7, 3, 2900)])
def test_budget_rule_matches_oracle(n, c, bp):
    assert ckv.ckv_budget_chunks(n, c, bp) == O.budget_chunks(n, c, bp)


def test_budget_rule_rejects_bad_args():
    assert ckv.ckv_budget_chunks(0, 16, 1000) == -1
    assert ckv.ckv_budget_chunks(10, 0, 1000) == -1
    assert ckv.ckv_budget_chunks(10, 1, 10001) == -1


def test_null_context_is_safe():
    lib = ckv.load_library()
    assert lib.ckv_last_error(None) == b"null context"
    lib.ckv_destroy(None)
    assert lib.ckv_k(None) == -1


def test_config_validation_needs_no_gpu():
    # argument checks run before any CUDA call (include/ckv.h: errors are reported, nothing enqueued)
    from paper_2601_13631_b200 import CKV_FLAG_GLOBAL_HEAP, CkvError, Context
    with pytest.raises(CkvError, match="EUNSUPPORTED"):  # one shared pool + periods (ckv.h CKV_FLAG_GLOBAL_HEAP)
        Context(4, 4, 2, 64, 16, 256, 8, dtype="fp32", flags=CKV_FLAG_GLOBAL_HEAP, period=4)
    with pytest.raises(CkvError, match="EUNSUPPORTED"):  # one shared pool + shards
        Context(4, 4, 2, 64, 16, 256, 8, dtype="fp32", flags=CKV_FLAG_GLOBAL_HEAP, num_shards=2)
    with pytest.raises(CkvError, match="EINVAL"):
        Context(4, 4, 2, 64, 16, 256, 8, dtype="fp32", period=2, subperiod=3)
    with pytest.raises(CkvError, match="EINVAL"):
        Context(1, 3, 2, 64, 16, 256, 8, dtype="fp32")  # Hq % Hkv != 0


def test_product_library_has_no_tuning_knobs():
    # timing-only modes and env knobs live in the tuning build only (build.py --tuning)
    data = open(ckv.LIB_PATH, "rb").read()
    for knob in (b"CKV_KNOCKOUT", b"CKV_SCORE_POLY", b"CKV_PDL_SKIP", b"CKV_ATTN_TRACE", b"CKV_TIMELINE", b"CKV_DTL",
                 b"CKV_SCORE_DBG", b"CKV_TOPK_PLAN", b"CKV_SPEC_INSCORE", b"CKV_PLAN_TABLES"):
        assert knob not in data, knob
