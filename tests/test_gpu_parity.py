"""GPU parity of libckv against the fp64 oracle (calls go through the C-ABI).

Sizes: the BASELINE shapes (C1 full, C2 shape, C3 full size for two layers) plus
ragged / degenerate cases (partial last chunk, c = 1, k = 1, k = m, odd n_s).
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2601_13631_b200 import (CKV_FLAG_CYCLIC_SHARDS, CKV_FLAG_GLOBAL_HEAP, CKV_FLAG_SIMT_SCORE,
                                   CKV_FLAG_V_ONLY_STORE, CkvError, Context)
from synth import CONFIGS, ShapeConfig, make_prefix, make_request
from tests.gpu_util import check_layer, make_ctx, run_layers, to_dev

pytestmark = pytest.mark.gpu

C1 = CONFIGS["c1_0.5b"]
RAGGED_FP32 = ShapeConfig("ragged_fp32", 2, 6, 2, 64, 1003, 5, 7, 1000, "fp32")
RAGGED_BF16 = ShapeConfig("ragged_bf16", 2, 28, 4, 128, 3001, 16, 9, 1000, "bf16")
C2_SMALL = CONFIGS["c2_3b"].replace(num_layers=4)
C3_2L = CONFIGS["c3_7b"].replace(num_layers=2)


def _k(cfg):
    return O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)


def _check_all(ctx, cfg, prefix, results, k, norm=0):
    diags = []
    for r in results:
        kp, vp = prefix[r["layer"]]
        diags.append(check_layer(r["ids"], r["out"], r["A"], r["qs"], r["ks"], r["vs"], kp, vp, cfg, k, norm))
    return diags


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def test_c1_fp32_full_config():
    ctx, prefix = make_ctx(C1)
    res = run_layers(ctx, C1, prefix, [0])
    _check_all(ctx, C1, prefix, res, _k(C1))


@pytest.mark.parametrize("cfg", [RAGGED_FP32, RAGGED_BF16], ids=lambda c: c.name)
def test_ragged_partial_last_chunk(cfg):
    k = 17
    ctx, prefix = make_ctx(cfg, k=k, prefetch=k)
    res = run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    _check_all(ctx, cfg, prefix, res, k)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_token_level_c1(dtype):
    cfg = ShapeConfig("tok", 1, 4, 2, 64 if dtype == "fp32" else 128, 700, 1, 5, 1000, dtype)
    ctx, prefix = make_ctx(cfg, k=37)
    res = run_layers(ctx, cfg, prefix, [0])
    _check_all(ctx, cfg, prefix, res, 37)


@pytest.mark.parametrize("k", [1, "m"])
def test_degenerate_budgets(k):
    cfg = ShapeConfig("deg", 1, 8, 2, 128, 1040, 16, 12, 1000, "bf16")
    kk = cfg.num_chunks if k == "m" else k
    ctx, prefix = make_ctx(cfg, k=kk)
    res = run_layers(ctx, cfg, prefix, [0])
    _check_all(ctx, cfg, prefix, res, kk)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_fullrow_normalisation(dtype):
    cfg = ShapeConfig("fr", 1, 8, 2, 64 if dtype == "fp32" else 128, 2048, 16, 24, 1000, dtype)
    ctx, prefix = make_ctx(cfg, norm=1)
    res = run_layers(ctx, cfg, prefix, [0])
    _check_all(ctx, cfg, prefix, res, _k(cfg), norm=1)


def test_c2_shape_layers_prefetch_and_cache_invariance():
    cfg = C2_SMALL
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=k)
    res = run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    _check_all(ctx, cfg, prefix, res, k)
    st = ctx.get_stats()
    assert st["total_spec_loads"] > 0 and st["total_spec_used"] > 0
    # results never depend on the cache: warm (same request again), then cold
    res2 = run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    ctx.reset_cache()
    res3 = run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    for a, b, c in zip(res, res2, res3):
        assert np.array_equal(a["ids"], b["ids"]) and np.array_equal(a["ids"], c["ids"])
        assert np.array_equal(a["out"], b["out"]) and np.array_equal(a["out"], c["out"])


def test_global_heap_layers_match_oracle():
    """Global heap with a pool too small for every layer's selection: chunks of other layers are
    evicted and reloaded (through the fused compaction gather), with the next layer's speculative
    plan issued only after this layer's compaction; results stay the oracle's."""
    cfg = C2_SMALL
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=k // 2, cache_slots=k + k // 2, flags=CKV_FLAG_GLOBAL_HEAP)
    for req in range(2):
        res = run_layers(ctx, cfg, prefix, range(cfg.num_layers), request=req)
        _check_all(ctx, cfg, prefix, res, k)
    st = ctx.get_stats()
    assert st["total_misses"] > 0
    ctx.close()
    with pytest.raises(CkvError):  # several in-flight prefetch plans (periods) are not combined with it
        make_ctx(cfg, prefetch=k // 2, flags=CKV_FLAG_GLOBAL_HEAP, store=False)[0].set_period(4, 1)


def test_v_only_store_matches_kv_store():
    """CKV_FLAG_V_ONLY_STORE: records hold V only, K comes from the probe array; the dense tile
    image is the same bytes, so ids and outputs are bit-identical to the K+V store, and every miss
    moves half the bytes over the host link."""
    cfg = C2_SMALL
    k = _k(cfg)
    base, prefix = make_ctx(cfg, prefetch=k // 2, cache_slots=k + k // 2)
    vonly, _ = make_ctx(cfg, prefetch=k // 2, cache_slots=k + k // 2, flags=CKV_FLAG_V_ONLY_STORE)
    for req in range(2):
        for ctx in (base, vonly):
            ctx.reset_cache()
            ctx.reset_stats()
        ra = run_layers(base, cfg, prefix, range(cfg.num_layers), request=req)
        rb = run_layers(vonly, cfg, prefix, range(cfg.num_layers), request=req)
        for a, b in zip(ra, rb):
            assert np.array_equal(a["ids"], b["ids"]) and np.array_equal(a["out"], b["out"])
        sa, sb = base.get_stats(), vonly.get_stats()
        assert sa["total_misses"] > 0 and sa["total_misses"] == sb["total_misses"]
        assert 2 * sb["total_link_bytes_delta"] == sa["total_link_bytes_delta"]
    _check_all(vonly, cfg, prefix, rb, k)
    with pytest.raises(CkvError):  # needs the tcgen05 attention path
        Context(1, 4, 2, 64, 16, 256, 8, dtype="fp32", flags=CKV_FLAG_V_ONLY_STORE)
    base.close()
    vonly.close()


def test_c3_full_size_two_layers():
    """C3 at full size (7B shape, 32K prefix, k = 204) for two layers and two requests, in the
    bench's cache configuration (prefetch quota k, k + quota + k/2 slots).  The synthetic
    recipe keeps the k/k+1 gap open, so every draw here passes the Q11 gate and
    the ids must equal the oracle's bit for bit."""
    cfg = C3_2L
    k = _k(cfg)
    assert k == 204
    ctx, prefix = make_ctx(cfg, prefetch=k, cache_slots=k + k + k // 2)
    diags = []
    for req in range(2):
        res = run_layers(ctx, cfg, prefix, range(2), request=req)
        diags += _check_all(ctx, cfg, prefix, res, k)
    print("C3 diagnostics", diags, "score kernel", ctx.score_kernel_kind)
    assert all(d["strict"] for d in diags), diags


def test_score_kernels_agree_simt_vs_default():
    cfg = RAGGED_BF16.replace(num_layers=1, prefix_len=4099)
    k = 23
    a, prefix = make_ctx(cfg, k=k)
    b, _ = make_ctx(cfg, k=k, flags=CKV_FLAG_SIMT_SCORE)
    ra = run_layers(a, cfg, prefix, [0])[0]
    rb = run_layers(b, cfg, prefix, [0])[0]
    np.testing.assert_allclose(ra["A"], rb["A"], rtol=2e-4)
    check_layer(ra["ids"], ra["out"], ra["A"], ra["qs"], ra["ks"], ra["vs"], *prefix[0], cfg, k)


@pytest.mark.parametrize("c,ns,k", [(16, 130, 21), (8, 1, 5), (32, 40, 9), (64, 200, 3), (16, 256, 64),
                                    (4, 40, 37), (2, 17, 61), (1, 9, 100), (4, 130, 250)])
def test_tensor_core_paths_vs_oracle_shapes(c, ns, k):
    """tcgen05 score + attention across chunk sizes, 1..2 suffix tiles, k not a multiple of 128/c."""
    from paper_2601_13631_b200 import CKV_FLAG_SIMT_ATTN
    cfg = ShapeConfig("tcshape", 1, 8, 2, 128, 5003, c, ns, 1000, "bf16")
    a, prefix = make_ctx(cfg, k=k)
    b, _ = make_ctx(cfg, k=k, flags=CKV_FLAG_SIMT_ATTN | CKV_FLAG_SIMT_SCORE)
    assert a.attn_kernel_kind == 1 and b.attn_kernel_kind == 0
    ra = run_layers(a, cfg, prefix, [0])[0]
    rb = run_layers(b, cfg, prefix, [0])[0]
    check_layer(ra["ids"], ra["out"], ra["A"], ra["qs"], ra["ks"], ra["vs"], *prefix[0], cfg, k)
    check_layer(rb["ids"], rb["out"], rb["A"], rb["qs"], rb["ks"], rb["vs"], *prefix[0], cfg, k)


def test_cuda_graph_replay_matches_eager():
    """A whole multi-layer request captured in a CUDA graph (side-stream prefetch included)
    replays to the same ids and outputs as eager calls, across requests and cache states."""
    cfg = C2_SMALL.replace(num_layers=3, prefix_len=4096)
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=k)
    reqs = []
    for r in range(3):
        reqs.append([[to_dev(x, torch.bfloat16) for x in make_request(cfg, l, r)] for l in range(cfg.num_layers)])
    outs = [torch.empty(cfg.suffix_len, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
            for _ in range(cfg.num_layers)]
    ids = [torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(cfg.num_layers)]

    def step(r):
        for l in range(cfg.num_layers):
            ctx.reprefill_layer(l, *reqs[r][l], out=outs[l], ids=ids[l])

    eager = []
    for r in range(3):
        step(r)
        torch.cuda.synchronize()
        eager.append(([o.clone() for o in outs], [i.clone() for i in ids]))
    graphs = []
    for r in range(3):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(r)
        graphs.append(g)
    for rep in range(3):
        for r in (2, 0, 1):
            graphs[r].replay()
            torch.cuda.synchronize()
            for l in range(cfg.num_layers):
                assert torch.equal(ids[l], eager[r][1][l])
                assert torch.equal(outs[l], eager[r][0][l])
    ctx.get_stats()  # raises if the planner ever saw a cache overflow


@pytest.mark.parametrize("period,sub", [(4, 2), (3, 1), (8, 4)])
def test_periods_intra_period_prefetch(period, sub):
    """NEXT-1: layers of a Period reuse the ids identified at its first layer (Def. 3,
    PAPER.md:349-355); the other layers' chunks are loaded right after identification."""
    cfg = C2_SMALL.replace(num_layers=8, prefix_len=4096)
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=k)
    ctx.close()
    from paper_2601_13631_b200 import Context
    ctx = Context(cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size, cfg.prefix_len,
                  cfg.suffix_len, dtype=cfg.dtype, budget_bp=cfg.budget_bp, prefetch_chunks=k, period=period,
                  subperiod=sub)
    for l, (kp, vp) in enumerate(prefix):
        ctx.store_prefix(l, to_dev(kp, torch.bfloat16), to_dev(vp, torch.bfloat16))
    for rep in range(2):  # second pass: warm cache
        res = run_layers(ctx, cfg, prefix, range(cfg.num_layers), request=rep)
        for r in res:
            l = r["layer"]
            kp, vp = prefix[l]
            if l % period == 0:
                first = r
                check_layer(r["ids"], r["out"], r["A"], r["qs"], r["ks"], r["vs"], kp, vp, cfg, k)
            else:
                assert np.array_equal(r["ids"], first["ids"])
                ref = O.reprefill_layer(r["qs"], r["ks"], r["vs"], kp, vp, cfg.chunk_size, k, cfg.group,
                                        sel=r["ids"].astype(np.int64))
                from tests.gpu_util import row_rel_err
                assert row_rel_err(r["out"], ref["out"]) < 2e-2
    st = ctx.get_stats()
    assert st["total_spec_loads"] > 0


@pytest.mark.parametrize("c,bp", [(4, 200), (16, 2500), (64, 5000), (16, 200)])
def test_c5_chunk_and_budget_sweep_reduced(c, bp):
    """C5 (32B shape: 40 Q / 8 KV heads) chunk-size x budget sweep at a reduced prefix."""
    cfg = CONFIGS["c5_32b"].replace(num_layers=2, prefix_len=8192, chunk_size=c, suffix_len=64, budget_bp=bp)
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=k)
    res = run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    _check_all(ctx, cfg, prefix, res, k)


def test_c4_shape_reduced():
    """C4 (14B shape: 40 Q / 8 KV heads, c = 32, n_s = 256, 5% budget) at a reduced prefix."""
    cfg = CONFIGS["c4_14b"].replace(num_layers=2, prefix_len=16384)
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=k)
    res = run_layers(ctx, cfg, prefix, range(cfg.num_layers))
    _check_all(ctx, cfg, prefix, res, k)


def test_c4_full_size_layer_properties():
    """C4 at its full size (14B shape, 128K prefix, c = 32, n_s = 256, 5%: k = 204 of 4096 chunks),
    one layer in the configuration the bench family uses (tcgen05 paths), checked by properties
    that hold at any size plus sampled outputs the oracle computes cheaply: prefix-only mass
    conservation sum_j A_j = n_s * Hq, the ids are exactly the top-k of the GPU's
    own A with the lower-index tie-break (bit-exact integer work), and the first 32 suffix rows
    of every head equal the oracle's attention over the GPU's kept chunks + causal suffix; then
    the full fp64 oracle of the layer (A element-wise, strict ids, all output rows)."""
    cfg = CONFIGS["c4_14b"].replace(num_layers=1)
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=0)
    assert ctx.m == 4096 and k == 204
    res = run_layers(ctx, cfg, prefix, [0])[0]
    A = res["A"].astype(np.float64)
    assert abs(A.sum() - cfg.suffix_len * cfg.num_q_heads) < 1e-4 * cfg.suffix_len * cfg.num_q_heads
    assert res["ids"].tolist() == O.select_topk(res["A"].astype(np.float32).astype(np.float64), k).tolist()
    kp, vp = prefix[0]
    ns_s = 32
    toks = O.kept_token_index(res["ids"], cfg.prefix_len, cfg.chunk_size)
    ref, _ = O.attention(res["qs"][:ns_s], res["ks"][:ns_s], res["vs"][:ns_s], kp, vp, toks, cfg.group)
    from tests.gpu_util import TOL, row_rel_err
    assert row_rel_err(res["out"][:ns_s], ref) < TOL["bf16"]
    # and the whole layer against the fp64 oracle: A element-wise, ids by the Q11 gate
    # (strict for this draw), every output row
    d = check_layer(res["ids"], res["out"], res["A"], res["qs"], res["ks"], res["vs"], kp, vp, cfg, k)
    print("C4 diagnostics", d)
    assert d["strict"], d
    ctx.close()


def test_probe_config_ns8():
    """Supplementary HBM-probe config (C3 shape, n_s = 8: 56 rows per KV head, one row tile)."""
    cfg = CONFIGS["probe_7b_ns8"].replace(num_layers=1)
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg)
    res = run_layers(ctx, cfg, prefix, [0])
    _check_all(ctx, cfg, prefix, res, k)


# ---------------------------------------------------------------- top-k (bit exact)
@pytest.mark.parametrize("m", [1, 7, 300, 2048, 32768])
def test_topk_exact_with_ties(m):
    ctx = Context(1, 1, 1, 64, 1, m, 1, dtype="fp32", budget_chunks=m)
    g = np.random.default_rng(m)
    for trial in range(4):
        A = g.integers(0, 6, m).astype(np.float32) if trial % 2 else g.random(m).astype(np.float32)
        if trial == 3:
            A[:] = 0.0
        Ad = torch.from_numpy(A).cuda()
        for k in sorted({1, max(1, m // 10), max(1, m // 2), m}):
            ids = ctx.test_topk(Ad, k).cpu().numpy()
            assert ids.tolist() == O.select_topk(A.astype(np.float64), k).tolist()


# ---------------------------------------------------------------- cache planner (A4/A9)
@pytest.mark.parametrize("policy", ["attn", "lfu", "lru"])
def test_cache_plan_matches_model(policy):
    m, P, k = 64, 20, 8
    ctx = Context(1, 1, 1, 64, 1, m, 1, dtype="fp32", budget_chunks=k, cache_slots=P)
    ctx.store_prefix(0, torch.zeros(m, 1, 64, device="cuda"), torch.zeros(m, 1, 64, device="cuda"))
    ctx.set_cache_policy(policy)
    model = O.CacheModel(1, m, P, policy=policy)
    g = np.random.default_rng(7)
    for step in range(40):
        A = g.integers(0, 50, m).astype(np.float32)  # integer scores: S exact in fp32 and fp64
        ids = np.sort(g.choice(m // 2 if step % 3 else m, k, replace=False)).astype(np.int32)
        hits_m, loads_m, vict_m = model.plan(0, ids)
        model.update(0, ids, A.astype(np.float64), tick=step + 1)  # the library counts one request per call
        loads, victims, counts = ctx.test_cache_step(0, torch.from_numpy(ids).cuda(), A=torch.from_numpy(A).cuda())
        counts = counts.cpu().numpy()
        loads = loads.cpu().numpy()[: 2 * counts[1]].reshape(-1, 2)
        assert counts[0] == len(hits_m) and counts[1] == len(loads_m) and counts[2] == len(vict_m)
        assert sorted(loads[:, 0].tolist()) == sorted(j for j, _ in loads_m)
        assert sorted(victims.cpu().numpy()[: counts[2]].tolist()) == sorted(vict_m)
        assert len(set(loads[:, 1].tolist())) == len(loads) and loads[:, 1].max(initial=0) < P


@pytest.mark.parametrize("policy", ["attn", "lfu"])
def test_global_heap_plan_matches_model(policy):
    """CKV_FLAG_GLOBAL_HEAP: one pool of L*P slots; victims of any layer."""
    L, m, P, k = 3, 48, 6, 6
    ctx = Context(L, 1, 1, 64, 1, m, 1, dtype="fp32", budget_chunks=k, cache_slots=P, flags=CKV_FLAG_GLOBAL_HEAP)
    for l in range(L):
        ctx.store_prefix(l, torch.zeros(m, 1, 64, device="cuda"), torch.zeros(m, 1, 64, device="cuda"))
    ctx.set_cache_policy(policy)
    model = O.CacheModel(L, m, P, policy=policy, global_heap=True)
    g = np.random.default_rng(5)
    for step in range(60):
        l = int(g.integers(0, L))
        A = g.integers(0, 30, m).astype(np.float32)
        ids = np.sort(g.choice(m // 2 if step % 3 else m, k, replace=False)).astype(np.int32)
        hits_m, loads_m, vict_m = model.plan(l, ids)
        model.update(l, ids, A.astype(np.float64), tick=step + 1)
        loads, victims, counts = ctx.test_cache_step(l, torch.from_numpy(ids).cuda(), A=torch.from_numpy(A).cuda())
        counts = counts.cpu().numpy()
        loads = loads.cpu().numpy()[: 2 * counts[1]].reshape(-1, 2)
        assert counts[0] == len(hits_m) and counts[1] == len(loads_m) and counts[2] == len(vict_m)
        assert sorted(loads[:, 0].tolist()) == sorted(j for j, _ in loads_m)
        assert sorted(victims.cpu().numpy()[: counts[2]].tolist()) == sorted(vl * m + vj for vl, vj in vict_m)
        assert len(set(loads[:, 1].tolist())) == len(loads) and loads[:, 1].max(initial=0) < L * P
    ctx.close()


# ---------------------------------------------------------------- sharded (logical, 1 GPU)
@pytest.mark.parametrize("W,cyclic,n,vonly", [(2, False, 4000, False), (3, False, 4000, False), (4, False, 4000, False),
                                               (2, True, 4000, False), (3, True, 4000, False), (3, True, 3990, False),
                                               (2, True, 3990, True), (3, False, 4000, True)])
def test_sharded_logical_on_one_gpu(W, cyclic, n, vonly):
    cfg = ShapeConfig("sh", 2, 8, 2, 128, n, 16, 10, 1000, "bf16")
    k = _k(cfg)
    flags = (CKV_FLAG_CYCLIC_SHARDS if cyclic else 0) | (CKV_FLAG_V_ONLY_STORE if vonly else 0)
    ctxs = [make_ctx(cfg, shard=g, W=W, prefetch=k // 2, flags=flags)[0] for g in range(W)]
    for l in range(cfg.num_layers):
        kp, vp = make_prefix(cfg, l)
        qs, ks, vs = make_request(cfg, l, 0)
        q, k_, v_ = (to_dev(x, torch.bfloat16) for x in (qs, ks, vs))
        ns = qs.shape[0]
        lam = [torch.empty(cfg.num_q_heads * ns, device="cuda") for _ in range(W)]
        for g_, c in enumerate(ctxs):
            c.shard_score(l, q, k_, lam[g_])
        lam_all = torch.cat(lam)                                   # allgather
        cands = [torch.empty(k, dtype=torch.int64, device="cuda") for _ in range(W)]
        for g_, c in enumerate(ctxs):
            c.shard_select(l, q, k_, lam_all, cands[g_])
        cand_all = torch.cat(cands)                                # allgather
        o = [torch.empty(ns, cfg.num_q_heads, cfg.head_dim, device="cuda") for _ in range(W)]
        lse = [torch.empty(ns * cfg.num_q_heads, device="cuda") for _ in range(W)]
        ids = [torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(W)]
        for g_, c in enumerate(ctxs):
            c.shard_attend(l, cand_all, q, k_, v_, o[g_], lse[g_], ids[g_])
        M = torch.stack(lse).max(dim=0).values                     # allreduce(max)
        bufs = []
        for g_, c in enumerate(ctxs):
            b = torch.empty(ns * cfg.num_q_heads * (cfg.head_dim + 1), device="cuda")
            c.lse_merge_prepare(o[g_], lse[g_], M, ns, b)
            bufs.append(b)
        tot = torch.stack(bufs).sum(dim=0)                         # allreduce(sum)
        out = torch.empty(ns, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
        ctxs[0].lse_merge_finish(tot, ns, out)
        torch.cuda.synchronize()
        for g_ in range(1, W):
            assert torch.equal(ids[0], ids[g_])
        check_layer(ids[0].cpu().numpy(), out.float().cpu().numpy(), None, qs, ks, vs, kp, vp, cfg, k)


# ---------------------------------------------------------------- errors and accounting
def test_errors_are_reported():
    cfg = ShapeConfig("err", 2, 4, 2, 64, 256, 16, 8, 1000, "fp32")
    ctx, prefix = make_ctx(cfg, layers=2, store=False)
    q = torch.zeros(8, 4, 64, device="cuda")
    kv = torch.zeros(8, 2, 64, device="cuda")
    with pytest.raises(CkvError, match="ESTATE"):
        ctx.reprefill_layer(0, q, kv, kv)
    with pytest.raises(CkvError, match="EINVAL"):
        ctx.reprefill_layer(5, q, kv, kv)
    with pytest.raises(CkvError, match="EINVAL"):
        ctx.store_prefix(0, torch.zeros(255, 2, 64, device="cuda"), torch.zeros(255, 2, 64, device="cuda"))
    with pytest.raises(CkvError):
        Context(1, 3, 2, 64, 16, 256, 8, dtype="fp32")  # Hq % Hkv != 0


def test_delta_law_and_whole_chunk_transfers():
    cfg = C2_SMALL.replace(num_layers=3, prefix_len=4096)
    k = _k(cfg)
    ctx, prefix = make_ctx(cfg, prefetch=k)
    rec = 2 * cfg.num_kv_heads * cfg.chunk_size * cfg.head_dim * 2
    ctx.reset_stats()
    for r in range(3):
        run_layers(ctx, cfg, prefix, range(cfg.num_layers), request=r, with_A=False)
    st = ctx.get_stats()
    assert st["total_link_bytes_delta"] == st["total_misses"] * rec       # RA = 1, whole chunks
    assert st["total_link_bytes_spec"] == st["total_spec_loads"] * rec
    assert st["total_hits"] + st["total_misses"] == 3 * cfg.num_layers * k
    assert st["total_layers"] == 3 * cfg.num_layers


# ---------------------------------------------------------------- granularity (NEXT-4)
@pytest.mark.parametrize("c,B,n", [(1, 64, 5000), (16, 64, 5000), (16, 16, 4999), (16, 24, 4999), (64, 16, 5000),
                                   (4, 6, 777)])
def test_block_cover_matches_oracle(c, B, n):
    m = -(-n // c)
    ctx = Context(1, 2, 1, 64, c, n, 4, dtype="fp32", budget_chunks=m, cache_slots=m)
    g = np.random.default_rng(c * 1000 + B)
    for trial in range(8):
        cnt = [0, 1, m][trial] if trial < 3 else int(g.integers(1, m + 1))
        ids = np.sort(g.choice(m, cnt, replace=False)).astype(np.int32)
        blocks, nb = ctx.block_cover(torch.from_numpy(ids).cuda(), B)
        nb = int(nb.item())
        assert blocks[:nb].cpu().tolist() == O.block_cover(ids, c, B, n)
    ctx.close()


def test_load_chunks_counts_whole_records():
    n, c = 4096, 64
    m = n // c
    ctx = Context(1, 2, 2, 64, c, n, 4, dtype="fp32", budget_chunks=m, cache_slots=m)
    kp = torch.randn(n, 2, 64, device="cuda")
    ctx.store_prefix(0, kp, kp)
    ids = torch.tensor([0, 3, 7, 8, 40, 63], dtype=torch.int32, device="cuda")
    ctx.reset_stats()
    ctx.load_chunks(0, ids)
    st = ctx.get_stats()
    rec = 2 * 2 * c * 64 * 4
    assert st["total_misses"] == 6 and st["total_hits"] == 0 and st["total_link_bytes_delta"] == 6 * rec
    ctx.load_chunks(0, ids)  # now resident
    st = ctx.get_stats()
    assert st["total_hits"] == 6 and st["total_misses"] == 6
    ctx.close()
