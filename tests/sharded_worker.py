"""Worker for the multi-rank GPU parity tests of the position-sharded path,
run as a subprocess so a rank that never gets its peers' contribution is bounded by a timeout.

    python -m tests.sharded_worker logical --W 3 [--cyclic] [--vonly] [--prefetch]
        one process drives W ranks (logical shards on one GPU), fused device-side exchange
        (ckv_exchange_attach), each rank on its own CUDA stream
    python -m torch.distributed.run --nproc-per-node 2 ... -m tests.sharded_worker mp --impl fused|collective
        one process per rank (all on cuda:0 here), gloo for the handle exchange / collectives:
        fused = ckv_exchange_open + ckv_reprefill_layer; collective = ShardedReprefill
Every rank's ids and output are compared with the fp64 oracle (tests/gpu_util.check_layer,
Q11 gate / Q12 tolerance) and with rank 0's bit for bit; prints one JSON line (rank 0)."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2601_13631_b200 import CKV_FLAG_CYCLIC_SHARDS, CKV_FLAG_V_ONLY_STORE  # noqa: E402
from synth import ShapeConfig, make_prefix, make_request  # noqa: E402
from tests.gpu_util import check_layer, make_ctx, to_dev  # noqa: E402


def cfg_of(a):
    if a.dtype == "fp32":
        return ShapeConfig("sh_fp32", a.layers, 6, 2, 64, a.n, 8, 9, 1000, "fp32")
    return ShapeConfig("sh_bf16", a.layers, 28, 4, 128, a.n, 16, a.ns, 1000, "bf16")


def flags_of(a):
    return (CKV_FLAG_CYCLIC_SHARDS if a.cyclic else 0) | (CKV_FLAG_V_ONLY_STORE if a.vonly else 0)


def logical(a):
    cfg = cfg_of(a)
    W = a.W
    k = O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
    pf = k // 2 if a.prefetch else 0
    ctxs, prefix = [], None
    for g in range(W):
        c, prefix = make_ctx(cfg, shard=g, W=W, prefetch=pf, flags=flags_of(a), norm=a.norm)
        ctxs.append(c)
    for c in ctxs:
        c.exchange_attach(ctxs)
    streams = [torch.cuda.Stream() for _ in range(W)]
    diags = []
    for req in range(a.requests):
        for l in range(cfg.num_layers):
            kp, vp = prefix[l]
            qs, ks, vs = make_request(cfg, l, req)
            q, k_, v_ = (to_dev(x, ctxs[0].torch_dtype) for x in (qs, ks, vs))
            torch.cuda.synchronize()
            res = []
            for g, c in enumerate(ctxs):  # every rank's whole layer is enqueued before any completes
                with torch.cuda.stream(streams[g]):
                    res.append(c.reprefill_layer(l, q, k_, v_, stream=streams[g]))
            torch.cuda.synchronize()
            for g in range(1, W):
                assert torch.equal(res[g][1], res[0][1]), ("ids differ across ranks", g)
                assert torch.equal(res[g][0], res[0][0]), ("out differs across ranks", g)
            diags.append(check_layer(res[0][1].cpu().numpy(), res[0][0].float().cpu().numpy(), None, qs, ks, vs, kp,
                                     vp, cfg, k, norm=a.norm))
    graph_ok = None
    if a.graph:
        # every rank's whole request captured in one CUDA graph per rank (the exchange is kernel
        # nodes only); the graphs replay concurrently on the ranks' streams and must reproduce
        # the eager outputs bit for bit
        req = a.requests - 1
        outs = [[torch.empty(cfg.suffix_len, cfg.num_q_heads, cfg.head_dim, dtype=ctxs[0].torch_dtype,
                             device="cuda") for _ in range(cfg.num_layers)] for _ in range(W)]
        idsb = [[torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(cfg.num_layers)] for _ in range(W)]
        inp = [[to_dev(x, ctxs[0].torch_dtype) for x in make_request(cfg, l, req)] for l in range(cfg.num_layers)]
        torch.cuda.synchronize()
        graphs = []
        for g, c in enumerate(ctxs):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=streams[g]):
                for l in range(cfg.num_layers):
                    c.reprefill_layer(l, *inp[l], out=outs[g][l], ids=idsb[g][l], stream=streams[g])
            graphs.append(gr)
        torch.cuda.synchronize()
        for rep in range(2):
            for g in range(W):
                with torch.cuda.stream(streams[g]):
                    graphs[g].replay()
            torch.cuda.synchronize()
        graph_ok = True
        for l in range(cfg.num_layers):
            for g in range(W):
                assert torch.equal(outs[g][l], outs[0][l]) and torch.equal(idsb[g][l], idsb[0][l])
            kp, vp = prefix[l]
            qs, ks, vs = make_request(cfg, l, req)
            d = check_layer(idsb[0][l].cpu().numpy(), outs[0][l].float().cpu().numpy(), None, qs, ks, vs, kp, vp,
                            cfg, k, norm=a.norm)
            diags.append(d)
    for c in ctxs:
        c.close()
    return {"mode": "logical", "W": W, "cyclic": a.cyclic, "vonly": a.vonly, "dtype": a.dtype, "layers": len(diags),
            "strict": sum(d["strict"] for d in diags), "max_out_rel": max(d["out_rel"] for d in diags),
            "graph": graph_ok}


def multiprocess(a):
    import torch.distributed as dist

    from paper_2601_13631_b200.sharded import ShardedReprefill, open_exchange

    rank, W = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    cfg = cfg_of(a)
    k = O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
    ctx, prefix = make_ctx(cfg, shard=rank, W=W, prefetch=k // 2 if a.prefetch else 0, flags=flags_of(a))
    if a.impl == "fused":
        open_exchange(ctx)
        run = ctx.reprefill_layer
    else:
        sr = ShardedReprefill(ctx)
        run = sr.reprefill_layer
    diags = []
    for req in range(a.requests):
        for l in range(cfg.num_layers):
            kp, vp = prefix[l]
            qs, ks, vs = make_request(cfg, l, req)
            q, k_, v_ = (to_dev(x, ctx.torch_dtype) for x in (qs, ks, vs))
            out, ids = run(l, q, k_, v_)
            torch.cuda.synchronize()
            # identical on every rank: compare with rank 0 through gloo
            mine = torch.cat([ids.cpu().to(torch.float64), out.float().cpu().flatten().to(torch.float64)])
            ref0 = mine.clone()
            dist.broadcast(ref0, 0)
            assert torch.equal(mine, ref0), ("rank result differs from rank 0", rank, l)
            diags.append(check_layer(ids.cpu().numpy(), out.float().cpu().numpy(), None, qs, ks, vs, kp, vp, cfg, k))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
    return {"mode": "mp", "impl": a.impl, "rank": rank, "W": W, "cyclic": a.cyclic, "layers": len(diags),
            "strict": sum(d["strict"] for d in diags), "max_out_rel": max(d["out_rel"] for d in diags)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["logical", "mp"])
    ap.add_argument("--W", type=int, default=2)
    ap.add_argument("--impl", choices=["fused", "collective"], default="fused")
    ap.add_argument("--cyclic", action="store_true")
    ap.add_argument("--vonly", action="store_true")
    ap.add_argument("--prefetch", action="store_true")
    ap.add_argument("--norm", type=int, default=0, help="1: CKV_NORM_FULLROW")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--n", type=int, default=4000)
    ap.add_argument("--ns", type=int, default=40)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--requests", type=int, default=2)
    ap.add_argument("--graph", action="store_true", help="logical mode: also replay per-rank CUDA graphs")
    a = ap.parse_args()
    r = logical(a) if a.mode == "logical" else multiprocess(a)
    if r.get("rank", 0) == 0:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
