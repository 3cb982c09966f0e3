"""Device timeline of graph-replayed C3 steps (tuning build, CKV_DTL=1): every kernel's CTA 0
records when its pdl_wait() returned (its stream predecessor completed); the gap to the next
main-stream kernel's record is this kernel's effective share of the layer.  Summary per kernel."""
import collections, os, re, subprocess, sys
if os.environ.get("DTL_CHILD") != "1":
    env = dict(os.environ, DTL_CHILD="1", CKV_LIBRARY=os.environ.get("CKV_LIBRARY", "tuning"), CKV_DTL="1")
    r = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    recs = []
    for ln in r.stderr.splitlines():
        m = re.match(r"\[dtl\] (\d+) (\d+) (\d+) (\S+)", ln)
        if m:
            recs.append((int(m.group(1)), int(m.group(2)), int(m.group(3)), m.group(4)))
    if not recs:
        print(r.stdout[-2000:], r.stderr[-4000:])
        sys.exit(1)
    marks = [x for x in recs if x[1] >= 0xF0000000]
    recs = [x for x in recs if x[1] < 0xF0000000]
    if marks:  # in-kernel marks (dtl_mark): mean time between consecutive marks of one CTA
        by_cta = collections.defaultdict(list)
        for t, gw, _, _ in marks:
            by_cta[gw & 0xFF].append((t, (gw >> 8) & 0xFFFF))
        seg = collections.defaultdict(list)
        for c, v in by_cta.items():
            v.sort()
            for (t0, a), (t1, b) in zip(v, v[1:]):
                if b != 1:
                    seg[(c, a, b)].append((t1 - t0) * 1e-3)
        for (c, a, b), v in sorted(seg.items()):
            print(f"mark CTA {c}: {a} -> {b}: n={len(v)} mean={sum(v)/len(v):6.2f} us")
    tail = recs[-int(os.environ.get("DTL_LAST", "1400")):]
    side = {"gather_kernel"}
    main = [x for x in tail if x[3] not in side]
    d = collections.defaultdict(list)
    for a, b in zip(main, main[1:]):
        d[a[3]].append((b[0] - a[0]) * 1e-3)
    span = (main[-1][0] - main[0][0]) * 1e-3
    print(f"span {span:.1f} us over {len(main)} main-stream kernels ({len(tail) - len(main)} side)")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        v2 = sorted(v)
        print(f"{k:34s} n={len(v):4d} mean={sum(v)/len(v):7.2f} med={v2[len(v2)//2]:7.2f} total={sum(v):9.1f}")
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle as O
from paper_2601_13631_b200 import Context
from synth import CONFIGS, make_prefix, make_request
from bench import request_sequence
cfg = CONFIGS["c3_7b"]
k = O.budget_chunks(cfg.prefix_len, cfg.chunk_size, cfg.budget_bp)
ctx = Context(cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.chunk_size, cfg.prefix_len,
              cfg.suffix_len, dtype="bf16", budget_bp=cfg.budget_bp, prefetch_chunks=k // 4, cache_slots=k + k + k // 2)
for l in range(cfg.num_layers):
    kp, vp = make_prefix(cfg, l)
    ctx.store_prefix(l, torch.from_numpy(kp).cuda().bfloat16(), torch.from_numpy(vp).cuda().bfloat16())
R = int(os.environ.get("DTL_REQS", "16"))
reqs = [[[torch.from_numpy(x).cuda().bfloat16() for x in make_request(cfg, l, r)] for l in range(cfg.num_layers)]
        for r in range(R)]
seq = request_sequence(64) if R > 1 else [0] * 64
outs = [torch.empty(cfg.suffix_len, cfg.num_q_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
        for _ in range(cfg.num_layers)]
ids = [torch.empty(k, dtype=torch.int32, device="cuda") for _ in range(cfg.num_layers)]
def step(r):
    for l in range(cfg.num_layers):
        ctx.reprefill_layer(l, *reqs[r][l], out=outs[l], ids=ids[l])
for i in range(24):
    step(seq[i])
gs = []
for r in range(R):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(r)
    gs.append(g)
for i in range(24, 32):
    gs[seq[i]].replay()
torch.cuda.synchronize()
ctx.close()
