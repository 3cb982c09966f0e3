#!/usr/bin/env python
"""Re-Prefill hot-path benchmark (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ckv|reference]

Workload (config.workload): Qwen2.5-7B shape, 28 layers, 28 Q / 4 KV heads, d = 128,
32K-token prefix, chunk 16, 128-token suffix, 10% budget (k = 204), bf16, inter-layer
speculative prefetch on (quota k/4, adaptive), HBM chunk cache of k + k + k/2 slots per layer
(~25% of the 2048 chunks of a layer).  Requests: a steady-state stream over 16 distinct
requests sharing the prefix (Zipf(1) popularity, seed 42; 16 untimed draws warm the cache),
so selected chunks that are not resident cross the host link inside the timed region
(synthetic, seed 42).  A step = one request's Re-Prefill over all 28 layers (A1-A9 each layer).
value = effective KV GB/s = (probe-K + kept K+V + suffix K+V bytes per layer) x layers
        / step time; us_per_layer is reported beside it; `all_hit` is the same layer with every
        selected chunk resident (compute only), `cold_cache` with an empty cache.
Inputs larger than L2: each step streams 28 x 33.5 MB of probe keys (0.94 GB > 126 MB L2).
N > 1: the prefix is sharded by position across ranks (strong scaling); the exchanges run
inside libckv over peer memory (--exchange fused, default) or as host-issued torch.distributed
collectives (--exchange collective).  Without torchrun, --gpus N re-launches itself under
torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CFG_NAME = "c3_7b"
N_DISTINCT = 16   # distinct requests sharing the prefix (each its own query topic mix)
WARM_CACHE = 16   # untimed request draws that bring the HBM chunk cache to its steady state


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def bytes_per_layer(cfg, k):
    e = 2 if cfg.dtype == "bf16" else 4
    probe = cfg.prefix_len * cfg.num_kv_heads * cfg.head_dim * e
    kept = k * 2 * cfg.num_kv_heads * cfg.chunk_size * cfg.head_dim * e
    suffix = 2 * cfg.suffix_len * cfg.num_kv_heads * cfg.head_dim * e
    return probe + kept + suffix


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:  # sampler running before timing
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        n = len(self.lines)
        t0 = time.time()
        while len(self.lines) < n + 2 and time.time() - t0 < 1.0:  # one sample past the region
            time.sleep(0.01)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def mufu_roofline(cfg, world, score_avg_ms, clocks):
    """A1's binding roofline: exp2 throughput (algorithmic exps = Hq * n_s * n per layer)."""
    exps = cfg.num_q_heads * cfg.suffix_len * (cfg.prefix_len / world)
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    peak = 16 * 148 * mhz * 1e6 / 1e12  # Tex2/s: MUFU ex2 16/clk/SM (B300_MICROARCH, measured scripts/mufu_bench.cu)
    achieved = exps / (score_avg_ms * 1e-3) / 1e12
    return {"bound": "alu", "unit": "Tex2/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
            "algorithmic": f"{exps:.4g} exp2 per launch", "sm_mhz": mhz}


# ------------------------------------------------------------------ reference arm (the oracle)
def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def oracle_layer_seconds(cfg, k, layer=0, request=0):
    import oracle as O
    from synth import make_prefix, make_request
    kp, vp = make_prefix(cfg, layer)
    qs, ks, vs = make_request(cfg, layer, request)
    t = time.perf_counter()
    O.reprefill_layer(qs, ks, vs, kp, vp, cfg.chunk_size, k, cfg.group)
    return time.perf_counter() - t


def oracle_single_thread_layer_seconds(cfg, k):
    """the oracle with one BLAS thread, timed on one KV head's share of layer 0
    (the same arithmetic per KV head, the selection over that head's scores) x Hkv."""
    import oracle as O
    from synth import make_prefix, make_request
    from threadpoolctl import threadpool_limits
    kp, vp = make_prefix(cfg, 0)
    qs, ks, vs = make_request(cfg, 0, 0)
    G = cfg.group
    with threadpool_limits(limits=1):
        t = time.perf_counter()
        O.reprefill_layer(qs[:, :G], ks[:, :1], vs[:, :1], kp[:, :1], vp[:, :1], cfg.chunk_size, k, G)
        dt = time.perf_counter() - t
    return dt * cfg.num_kv_heads


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle on the host cores, each step one layer of the workload."""
    from synth import CONFIGS
    import oracle as O
    if rank != 0:
        return
    cfg = CONFIGS[CFG_NAME]
    k = O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
    for w in range(args.warmup):
        oracle_layer_seconds(cfg, k, layer=w % cfg.num_layers)
    ts = [oracle_layer_seconds(cfg, k, layer=s % cfg.num_layers) for s in range(args.steps)]
    t = sum(ts) / len(ts)
    bpl = bytes_per_layer(cfg, k)
    value = bpl / t / 1e9
    cores = cpu_cores()
    line = {
        "impl": "reference", "metric": "Re-Prefill effective KV GB/s (Qwen2.5-7B shape, 32K prefix)",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "us_per_layer": t * 1e6, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seed 42)",
        "config": {"workload": CFG_NAME, "step": "one layer (oracle, fp64 NumPy)", "prefix_len": cfg.prefix_len,
                   "chunk": cfg.chunk_size, "suffix": cfg.suffix_len, "budget_chunks": k},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} single layers of {CFG_NAME}"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def request_sequence(n, seed=42):
    """Seeded request stream over the N_DISTINCT requests sharing the prefix: Zipf(1) popularity
    (the multi-request shared-prefix setting of PAPER.md:419-455 / SURVEY §8(d))."""
    g = np.random.default_rng(seed)
    pop = 1.0 / np.arange(1, N_DISTINCT + 1)
    return g.choice(N_DISTINCT, size=n, p=pop / pop.sum()).tolist()


def run_ckv(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2601_13631_b200 as ckv
    from paper_2601_13631_b200.sharded import ShardedReprefill, open_exchange
    from synth import CONFIGS, make_prefix, make_request

    local_rank = int(os.environ.get("LOCAL_RANK", rank)) if args.local_gpu is None else args.local_gpu
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # functional check of the sharded path (e.g. several ranks sharing one GPU)
            dist.init_process_group("gloo")
    cfg = CONFIGS[CFG_NAME]
    k = ckv.ckv_budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
    quota = int(round(k * args.quota_frac)) if args.prefetch else 0
    cache_slots = k + k + k // 2  # k selected + a quota-sized prefetch partition + k/2 (~25% of a layer's chunks)
    if args.cache_slots:
        cache_slots = args.cache_slots
    ctx = ckv.Context(cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size,
                      cfg.prefix_len, cfg.suffix_len, dtype=cfg.dtype, budget_bp=cfg.budget_bp,
                      prefetch_chunks=quota, cache_slots=cache_slots, device=local_rank, shard_index=rank,
                      num_shards=world, flags=ckv.CKV_FLAG_CYCLIC_SHARDS if args.cyclic else 0)
    dt = ctx.torch_dtype
    for l in range(cfg.num_layers):
        kp, vp = make_prefix(cfg, l)
        ctx.store_prefix(l, torch.from_numpy(kp).to(dev, dt), torch.from_numpy(vp).to(dev, dt))
    L = cfg.num_layers
    reqs_host = [[[torch.from_numpy(x).to(dt).pin_memory() for x in make_request(cfg, l, r)] for l in range(L)]
                 for r in range(N_DISTINCT)]
    reqs = [[[t.to(dev) for t in lay] for lay in per] for per in reqs_host]
    outs = [torch.empty(cfg.suffix_len, cfg.num_q_heads, cfg.head_dim, dtype=dt, device=dev) for _ in range(L)]
    ids = [torch.empty(k, dtype=torch.int32, device=dev) for _ in range(L)]
    runner = None
    if world > 1:
        if args.exchange == "fused":
            open_exchange(ctx)  # peer windows; every exchange then runs inside ckv_reprefill_layer
        else:
            runner = ShardedReprefill(ctx)  # host-issued torch.distributed collectives (baseline)

    def layer_call(l, q, ks, vs):
        if runner is None:
            ctx.reprefill_layer(l, q, ks, vs, out=outs[l], ids=ids[l])
        else:
            runner.reprefill_layer(l, q, ks, vs, out=outs[l], ids=ids[l])

    def run_request(r):
        for l in range(L):
            layer_call(l, *reqs[r][l])

    stream = torch.cuda.current_stream()

    def timed(fn, K):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(K):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev if args.backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
            ms = float(t.item())
        return ms

    # the request stream: WARM_CACHE untimed draws bring the HBM chunk cache to its steady state
    # ("warm up"), then the W warm-up and K timed steps follow the same stream
    seq = request_sequence(WARM_CACHE + args.warmup + 2 * args.steps + 4)  # + the untimed e2e warm-ups
    for r in seq[:WARM_CACHE]:
        run_request(r)
    off = WARM_CACHE
    for i in range(args.warmup):
        run_request(seq[off + i])
    off += args.warmup
    torch.cuda.synchronize()
    t0 = time.perf_counter()  # host cost of enqueueing one eager step (launch-bound check)
    run_request(seq[off])
    host_ms = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    ms_eager = timed(lambda i: run_request(seq[off + i]), args.steps) / args.steps
    launches = ctx.kernel_launches - launches0

    # one CUDA graph per distinct request: a 28-layer step replays without host launches
    graphs, graph_note = None, None
    if args.graph and runner is None:
        try:
            graphs = []
            for r in range(N_DISTINCT):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    run_request(r)
                graphs.append(g)
            for r in seq[:N_DISTINCT]:
                graphs[r].replay()
            torch.cuda.synchronize()
        except Exception as ex:  # e.g. a driver without stream-memop capture (W > 1): eager
            graphs, graph_note = None, f"capture failed: {ex}"[:200]
            torch.cuda.synchronize()

    def play(r):
        if graphs:
            graphs[r].replay()
        else:
            run_request(r)

    # headline: the steady-state request stream (the HBM cache holds ~25% of a layer's chunks, so
    # misses cross the host link inside the timed region: A1-A9 of the north star, gather included)
    off2 = off + args.steps
    ctx.reset_stats()
    with ClockSampler(local_rank) as clk:
        ms = timed(lambda i: play(seq[off2 + i]), args.steps)
    stats = ctx.get_stats()
    ms_step = ms / args.steps
    bpl = bytes_per_layer(cfg, k)
    value = bpl * L / (ms_step * 1e-3) / 1e9
    # all-hit: one request repeated (its chunks stay resident) -- the compute-only layer time
    for _ in range(3):
        play(0)
    ctx.reset_stats()
    ms_hit = timed(lambda i: play(0), args.steps) / args.steps
    hit_stats = ctx.get_stats()
    torch.cuda.synchronize()
    ids_cpu = [t.cpu().numpy() for t in ids]  # request 0's ids per layer
    cov = [len(set(ids_cpu[l].tolist()) & set(ids_cpu[l - 1].tolist())) / k for l in range(1, L)]
    quick = {"us_per_layer": ms_step * 1e3 / L, "value": value, "all_hit_us_per_layer": ms_hit * 1e3 / L,
             "eager_us_per_layer": ms_eager * 1e3 / L, "clocks": clk.summary(),
             "hit_rate": stats["total_hits"] / max(stats["total_hits"] + stats["total_misses"], 1)}
    if args.quick and not args.quick_e2e:  # tuning runs: the warm graph-replayed step only
        if rank == 0:
            print(json.dumps(quick))
        return

    # stage profile pass (eager; CUDA events on the launching stream, inside the library): on the
    # timed stream (the kernels as the headline runs them) and on the all-hit request (A1 alone,
    # no speculative gather beside it)
    ctx.profile(True)
    ms_prof = timed(lambda i: run_request(seq[off2 + i]), args.steps)
    prof = ctx.profile_read()
    for _ in range(2):
        run_request(0)
    ctx.profile_read()
    timed(lambda i: run_request(0), args.steps)
    prof_hit = ctx.profile_read()
    ctx.profile(False)

    # end-to-end through the public API with host buffers: H2D of the step's inputs from
    # pinned memory and D2H of its outputs inside the timed region, pipelined with the compute:
    # layer l's inputs go up on an H2D stream (event per layer, waited on by the compute stream
    # just before layer l) and layer l's output comes down on a D2H stream as soon as layer l is
    # done; one CUDA graph per distinct request
    host_out = [torch.empty(outs[0].shape, dtype=dt).pin_memory() for _ in range(L)]
    host_ids = [torch.empty(k, dtype=torch.int32).pin_memory() for _ in range(L)]
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(L)]
    ev_out = [torch.cuda.Event() for _ in range(L)]
    dev_in = [[torch.empty_like(t) for t in lay] for lay in reqs[0]]  # the step's device input buffers

    ev_go = [torch.cuda.Event() for _ in range(L)]
    AHEAD = 2  # layer l's inputs go up while layer l - AHEAD runs: the copies share the host link
    # with the speculative chunk gathers evenly instead of as one burst at the start of the step

    def e2e_body(r):
        main = torch.cuda.current_stream()
        h2d_s.wait_stream(main)
        d2h_s.wait_stream(main)

        def copy_in(l):  # layer l's inputs on the H2D stream (enqueued in stream order)
            with torch.cuda.stream(h2d_s):
                for dst, src in zip(dev_in[l], reqs_host[r][l]):
                    dst.copy_(src, non_blocking=True)
                ev_in[l].record(h2d_s)

        for l in range(min(AHEAD, L)):
            copy_in(l)
        for l in range(L):
            if l + AHEAD < L:  # layer l + AHEAD's inputs go up while layer l runs
                ev_go[l].record(main)
                h2d_s.wait_event(ev_go[l])
                copy_in(l + AHEAD)
            main.wait_event(ev_in[l])
            layer_call(l, *dev_in[l])
            ev_out[l].record(main)
            d2h_s.wait_event(ev_out[l])
            with torch.cuda.stream(d2h_s):
                host_out[l].copy_(outs[l], non_blocking=True)
                host_ids[l].copy_(ids[l], non_blocking=True)
        main.wait_stream(h2d_s)
        main.wait_stream(d2h_s)

    e2e_graphs = None
    if graphs:
        try:
            e2e_graphs = []
            for r in range(N_DISTINCT):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    e2e_body(r)
                e2e_graphs.append(g)
            torch.cuda.synchronize()
        except Exception as ex:  # capture of the multi-stream step failed: run it eagerly
            print(f"[bench] e2e graph capture failed ({ex}); eager e2e", file=sys.stderr)
            e2e_graphs = None

    def e2e_step(r):
        if e2e_graphs:
            e2e_graphs[r].replay()
        else:
            e2e_body(r)

    off3 = off2 + args.steps
    for i in range(2):
        e2e_step(seq[off2 + i])
    ms_e2e = timed(lambda i: e2e_step(seq[off3 - args.steps + i]), args.steps) / args.steps
    if args.quick:
        if rank == 0:
            quick["e2e_us_per_layer"] = ms_e2e * 1e3 / L
            print(json.dumps(quick))
        return

    # cold HBM cache: every step starts from an empty chunk cache (all selected chunks cross the
    # host link; speculative prefetch still overlaps the next layer's loads)
    cold_ms = []
    ctx.reset_stats()
    for i in range(min(args.steps, 5)):
        ctx.reset_cache()
        torch.cuda.synchronize()
        cold_ms.append(timed(lambda _: play(0), 1))
    cold_stats = ctx.get_stats()
    cold_layers = max(cold_stats["total_layers"], 1)

    # V-only store variant (CKV_FLAG_V_ONLY_STORE): the kept chunks' K comes from
    # the HBM probe array, so every miss moves half the bytes; same cold-cache protocol and the
    # same mode (one CUDA graph per step) as the K+V cold line
    cold_v = None
    if world == 1:
        vctx = ckv.Context(cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size,
                           cfg.prefix_len, cfg.suffix_len, dtype=cfg.dtype, budget_bp=cfg.budget_bp,
                           prefetch_chunks=quota, cache_slots=cache_slots, device=local_rank,
                           flags=ckv.CKV_FLAG_V_ONLY_STORE)
        for l in range(L):
            kp, vp = make_prefix(cfg, l)
            vctx.store_prefix(l, torch.from_numpy(kp).to(dev, dt), torch.from_numpy(vp).to(dev, dt))

        def vstep():
            for l in range(L):
                vctx.reprefill_layer(l, *reqs[0][l], out=outs[l], ids=ids[l])
        for _ in range(3):
            vstep()
        vgraph = None
        if graphs:
            vgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(vgraph):
                vstep()
        vms = []
        vctx.reset_stats()
        for i in range(min(args.steps, 5)):
            vctx.reset_cache()
            torch.cuda.synchronize()
            vms.append(timed(lambda _: vgraph.replay() if vgraph else vstep(), 1))
        vst = vctx.get_stats()
        vlink = vst["total_link_bytes_delta"] + vst["total_link_bytes_spec"]
        cold_v = {"us_per_layer": sum(vms) / len(vms) * 1e3 / L, "cuda_graph": bool(vgraph),
                  "link_bytes_per_layer": vlink / max(vst["total_layers"], 1),
                  "link_gbs": vlink / (sum(vms) * 1e-3) / 1e9,
                  "hit_rate": vst["total_hits"] / max(vst["total_hits"] + vst["total_misses"], 1)}
        del vgraph
        vctx.close()
        del vctx

    # HBM probe: the same prefix with an 8-token suffix (56 GQA rows per KV head:
    # 0.22 exp and 56 flop per key byte, below both ridges), where A1 streams the probe keys at
    # the HBM roofline; the score stage (library events) includes the small Q pack at n_s = 8
    hbm_probe = None
    if world == 1:
        ns8 = 8
        per8 = [[t[:ns8].contiguous() for t in reqs[0][l]] for l in range(L)]
        for l in range(L):  # warm
            ctx.reprefill_layer(l, *per8[l])
        torch.cuda.synchronize()
        ctx.profile(True)
        for _ in range(3):
            for l in range(L):
                ctx.reprefill_layer(l, *per8[l])
        pr8 = ctx.profile_read()
        ctx.profile(False)
        t8 = pr8["score"][0] / max(pr8["score"][1], 1)  # ms per launch
        kbytes = (cfg.prefix_len / world) * cfg.num_kv_heads * cfg.head_dim * 2
        hbm_peak = load_peaks()[0].get("hbm_gbs", 6650.0)
        hbm_probe = {"config": f"{CFG_NAME} prefix, n_s = {ns8}", "timing": "library events, eager (incl. the Q pack)",
                     "score_us_per_launch": t8 * 1e3,
                     "probe_key_bytes": kbytes, "achieved_gbs": kbytes / (t8 * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                     "frac": kbytes / (t8 * 1e-3) / 1e9 / hbm_peak}

    # the paper's own configuration: Periods of p = 8 layers, subperiod sp = 4:
    # chunk ids are identified on 1 layer in 8, the Period's other layers are prefetched; same
    # steady-state request stream as the headline
    period_line = None
    if world == 1 and graphs:
        ctx.set_period(8, 4)
        for r in seq[:WARM_CACHE]:
            run_request(r)  # warm the cache for this configuration
        torch.cuda.synchronize()
        pgraphs = []
        for r in range(N_DISTINCT):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run_request(r)
            pgraphs.append(g)
        for r in seq[off:off + args.warmup]:
            pgraphs[r].replay()
        ctx.reset_stats()
        ms_p = timed(lambda i: pgraphs[seq[off2 + i]].replay(), args.steps) / args.steps
        pst = ctx.get_stats()
        pcold = []
        for _ in range(3):  # empty cache: every Period's chunks cross the host link
            ctx.reset_cache()
            torch.cuda.synchronize()
            pcold.append(timed(lambda _: pgraphs[0].replay(), 1))
        period_line = {"period": 8, "subperiod": 4, "ms_per_step": ms_p, "us_per_layer": ms_p * 1e3 / L,
                       "cold_us_per_layer": sum(pcold) / len(pcold) * 1e3 / L,
                       "exposed_gather_us_per_layer": sum(pcold) / len(pcold) * 1e3 / L - ms_p * 1e3 / L,
                       "value": bpl * L / (ms_p * 1e-3) / 1e9, "unit": "GB/s",
                       "hit_rate": pst["total_hits"] / max(pst["total_hits"] + pst["total_misses"], 1),
                       "link_bytes_per_layer": (pst["total_link_bytes_delta"] + pst["total_link_bytes_spec"])
                       / max(pst["total_layers"], 1)}
        ctx.set_period(1, 1)
        del pgraphs

    # host-link peak: pinned H2D cudaMemcpy, 256 MiB, best of 5 (the gather's roofline)
    hbuf = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    dbuf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    link_ms = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dbuf.copy_(hbuf, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        link_ms.append(e0.elapsed_time(e1))
    link_peak = (256 << 20) / (min(link_ms) * 1e-3) / 1e9
    del hbuf, dbuf
    # the A5 gather engine alone: one layer's k random chunks demand-loaded into an empty cache
    # (ckv_load_chunks) vs a pinned cudaMemcpy of the same bytes (>= 80% of the link)
    gprobe = None
    if world == 1:
        rec = 2 * cfg.num_kv_heads * cfg.chunk_size * cfg.head_dim * 2
        gids = torch.from_numpy(np.sort(np.random.default_rng(7).choice(cfg.num_chunks, k, replace=False))
                                .astype(np.int32)).to(dev)
        gt = []
        for _ in range(5):
            ctx.reset_cache()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.load_chunks(0, gids)
            e1.record()
            torch.cuda.synchronize()
            gt.append(e0.elapsed_time(e1))
        hb = torch.empty(k * rec, dtype=torch.uint8).pin_memory()
        db = torch.empty(k * rec, dtype=torch.uint8, device=dev)
        mt = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            db.copy_(hb, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            mt.append(e0.elapsed_time(e1))
        gb = k * rec / (min(gt) * 1e-3) / 1e9
        mb = k * rec / (min(mt) * 1e-3) / 1e9
        gprobe = {"chunks": k, "bytes": k * rec, "gather_gbs": gb, "memcpy_same_bytes_gbs": mb,
                  "frac_of_memcpy": gb / mb, "frac_of_link_peak": gb / link_peak}
        del hb, db
        ctx.reset_cache()
    h2d = sum(t.numel() * t.element_size() for lay in reqs_host[0] for t in lay)
    d2h = L * (outs[0].numel() * outs[0].element_size() + k * 4)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_src = load_peaks()
    score_ms, score_n = prof["score"]
    score_avg = score_ms / max(score_n, 1)
    score_avg_alone = prof_hit["score"][0] / max(prof_hit["score"][1], 1)
    flops = 2.0 * cfg.head_dim * cfg.num_q_heads * cfg.suffix_len * (cfg.prefix_len / world)
    achieved = flops / (score_avg * 1e-3) / 1e12
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    traffic = None
    tp = os.path.join(ROOT, "profiles", "score_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get("kind%d" % ctx.score_kernel_kind)
    step_stage_ms = {n: v[0] / args.steps for n, v in prof.items()}
    cpu = None
    if world == 1 and not args.no_cpu:
        t = oracle_layer_seconds(cfg, k)
        t1 = oracle_single_thread_layer_seconds(cfg, k)
        cpu = {"value": bpl / t / 1e9, "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": f"1 layer (layer 0, request 0) of {CFG_NAME}, fp64 NumPy, {t:.2f} s",
               "single_thread": {"s_per_layer": t1, "value": bpl / t1 / 1e9,
                                 "sample": "one KV head of layer 0 with one BLAS thread, x Hkv"}}
    gate = None
    gp = os.path.join(ROOT, "profiles", "r2_gate_rate_c3.json")
    if os.path.exists(gp):
        with open(gp) as f:
            gs = json.load(f)["summary"]
        gate = {"pass_rate": gs["gate_pass_rate"], "draws": gs["draws"],
                "source": "profiles/r2_gate_rate_c3.json (fp64 oracle, scripts/gate_rate.py)"}
    n_lay = max(stats["total_layers"], 1)
    mufu = mufu_roofline(cfg, world, score_avg, clk.summary())
    tensor = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
              "peak_source": f"{peak_src} bf16_tflops_sustained"}

    def hit_rate(st):
        return st["total_hits"] / max(st["total_hits"] + st["total_misses"], 1)

    line = {
        "metric": "Re-Prefill effective KV GB/s (Qwen2.5-7B shape, 32K prefix)",
        "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "us_per_layer": ms_step * 1e3 / L,
        "eager": {"ms_per_step": ms_eager, "host_enqueue_ms_per_step": host_ms, "cuda_graph": bool(graphs),
                  "graph_note": graph_note},
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seed 42, DESIGN.md §4 recipe)",
        "config": {"workload": CFG_NAME, "layers": L, "prefix_len": cfg.prefix_len, "chunk": cfg.chunk_size,
                   "suffix": cfg.suffix_len, "heads": f"{cfg.num_q_heads}/{cfg.num_kv_heads}",
                   "head_dim": cfg.head_dim, "budget_chunks": k, "prefetch_quota": quota,
                   "requests": f"steady-state stream: {N_DISTINCT} distinct requests, Zipf(1) popularity, "
                               f"{WARM_CACHE} untimed cache warm-up draws",
                   "cache_slots_per_layer": cache_slots,
                   "parallelism": (f"prefix-shard{world}" + ("-cyclic" if args.cyclic else "") +
                                   f"-{args.exchange}") if world > 1 else "single",
                   "l2": "inputs larger than L2 (0.94 GB of probe keys streamed per step)",
                   "bytes_per_layer": bpl},
        # the kernel that dominates the step is A1; its binding roofline is the MUFU (one exp2 per
        # logit, 16 ex2/clk/SM x 148 SMs at the SM clock sampled in the timed region);
        # the tensor-pipe fraction is reported beside it
        "roofline": {"kernel": "score_partial (A1)", "bound": "alu", "achieved": mufu["achieved"],
                     "peak": mufu["peak"], "unit": "Tex2/s", "frac": mufu["frac"], "traffic": traffic,
                     "peak_source": "derived: 16 ex2/clk/SM x 148 SMs x sampled SM clock (DESIGN.md §6)",
                     "score_kernel_kind": ["simt", "tcgen05"][ctx.score_kernel_kind], "avg_launch_ms": score_avg,
                     "algorithmic": mufu["algorithmic"], "tensor": tensor,
                     # the same kernel without the speculative gather of the stream running beside it
                     "alone": {"avg_launch_ms": score_avg_alone,
                               "frac": mufu_roofline(cfg, world, score_avg_alone, clk.summary())["frac"],
                               "how": "all-hit request repeated (no prefetch traffic), same events"},
                     "hbm_achieved_gbs": (cfg.prefix_len / world) * cfg.num_kv_heads * cfg.head_dim * 2
                     / (score_avg * 1e-3) / 1e9},
        "stage_ms_per_step": step_stage_ms, "profiled_ms_per_step": ms_prof / args.steps,
        "cache": {"hit_rate": hit_rate(stats), "misses_per_layer": stats["total_misses"] / n_lay,
                  "spec_loads_per_layer": stats["total_spec_loads"] / n_lay,
                  "spec_used_per_layer": stats["total_spec_used"] / n_lay,
                  "link_bytes_per_layer": (stats["total_link_bytes_delta"] + stats["total_link_bytes_spec"]) / n_lay,
                  "link_gbs": (stats["total_link_bytes_delta"] + stats["total_link_bytes_spec"]) / (ms * 1e-3) / 1e9},
        "all_hit": {"us_per_layer": ms_hit * 1e3 / L, "value": bpl * L / (ms_hit * 1e-3) / 1e9, "unit": "GB/s",
                    "hit_rate": hit_rate(hit_stats), "note": "request 0 repeated: every selected chunk resident"},
        "selection": {"coverage_prev_mean": float(np.mean(cov)), "coverage_prev_min": float(np.min(cov)),
                      "gap_gate": gate},
        "paper_period": period_line,
        "gather_probe": gprobe,
        "cold_cache": {"ms_per_step": sum(cold_ms) / len(cold_ms), "us_per_layer": sum(cold_ms) / len(cold_ms) * 1e3 / L,
                       "hit_rate": hit_rate(cold_stats),
                       "link_bytes_per_layer": (cold_stats["total_link_bytes_delta"] + cold_stats["total_link_bytes_spec"])
                       / cold_layers,
                       "link_gbs": (cold_stats["total_link_bytes_delta"] + cold_stats["total_link_bytes_spec"])
                       / (sum(cold_ms) * 1e-3) / 1e9,
                       "link_peak_gbs": link_peak, "link_peak_how": "pinned H2D cudaMemcpy 256 MiB, best of 5",
                       # exposed gather = t_layer(cold, prefetch on) - t_layer(all-hit)
                       "exposed_gather_us_per_layer": sum(cold_ms) / len(cold_ms) * 1e3 / L - ms_hit * 1e3 / L,
                       "cuda_graph": bool(graphs)},
        "cold_cache_v_only": cold_v,
        "hbm_probe": hbm_probe,
        "e2e": {"value": bpl * L / (ms_e2e * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms_e2e,
                "pipelined": "per-layer H2D / D2H streams overlapping the compute", "cuda_graph": bool(e2e_graphs),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,  # kernels per K steps (counted on the eager pass; the graphs hold the same)
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "context": "paper: 3.85x average Re-Prefill (TTFT) speedup over IMPRESS on 1x A800 + PCIe4 + NVMe "
                   "(PAPER.md:29, 582) -- context only, not comparable",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N ranks
    (the driver's own launch line); NCCL INFO logging shows the communicator's rank count."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ckv", choices=["ckv", "reference"])
    ap.add_argument("--no-prefetch", dest="prefetch", action="store_false")
    ap.add_argument("--cache-slots", type=int, default=0, help="override the HBM cache slots per layer (studies)")
    ap.add_argument("--quota-frac", type=float, default=0.25,
                    help="speculative prefetch quota per layer as a fraction of k (the cache size stays k + k + k/2)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--cyclic", action="store_true", help="N > 1: cyclic chunk sharding (j mod N) instead of "
                    "contiguous ranges (balanced kept chunks, SURVEY §8(f) NEXT-3)")
    ap.add_argument("--quick", action="store_true", help="tuning: print only the warm graph-step time")
    ap.add_argument("--quick-e2e", action="store_true", help="tuning: --quick plus the end-to-end step")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--exchange", default="fused", choices=["fused", "collective"],
                    help="N > 1: fused device-side exchange inside libckv (default) or host-issued "
                         "torch.distributed collectives (ShardedReprefill, the NCCL baseline)")
    ap.add_argument("--local-gpu", type=int, default=None, help="pin every rank to this GPU (functional runs)")
    args = ap.parse_args()
    args.quick = args.quick or args.quick_e2e
    args.warmup = max(args.warmup, 3) if args.impl == "ckv" else args.warmup
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ckv(args, rank, world)


if __name__ == "__main__":
    main()
