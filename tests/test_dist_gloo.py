"""World-size-2 CPU test (gloo) of the position-sharded exchange protocol of
paper_2601_13631_b200.sharded.

The ShardedReprefill orchestration (buffers, collective order, rank-order LSE of the
normalisers, 64-bit candidate keys, LSE output merge) runs unchanged over gloo; the
per-shard compute is a CPU stand-in built from the oracle with the same I/O contract
as the libckv shard calls (base-2 log normalisers, (score bits << 32 | ~gid) keys,
natural-log partial LSE).  The merged result must equal the unsharded oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2601_13631_b200.sharded import ShardedReprefill


class OracleShard:
    """CPU stand-in for one libckv shard context (test infrastructure)."""

    def __init__(self, Kp, Vp, c, k, G, shard, W, cyclic=False):
        self.Kp, self.Vp, self.c, self.k, self.G, self.W = Kp, Vp, c, k, G, W
        n = Kp.shape[0]
        self.m = O.chunk_count(n, c)
        self.own = O.shard_chunks(W, shard, self.m, cyclic)       # owned global chunk ids, ascending
        self.tok = O.kept_token_index(self.own, n, c)              # their prefix tokens
        self.shard = shard

    def shard_score(self, layer, q, k_suf, lam_local):
        qs = q.double().numpy()
        lam = O.row_lse(qs, self.Kp[self.tok], self.G)                  # [Hq, ns] natural log
        lam_local.copy_(torch.from_numpy(lam.reshape(-1) / np.log(2.0)))  # base 2, index h*ns + r

    def shard_select(self, layer, q, k_suf, lam_all, cand):
        qs = q.double().numpy()
        ns, hq, _ = qs.shape
        lam2 = lam_all.double().numpy().reshape(self.W, hq * ns)
        mx = lam2.max(0)
        glob = (mx + np.log2(np.exp2(lam2 - mx).sum(0))) * np.log(2.0)
        a, _ = O.token_scores(qs, self.Kp[self.tok], self.G, lam=glob.reshape(hq, ns))
        # Eq. 1 per owned chunk (each owned chunk's tokens are consecutive in self.tok)
        lens = [O.chunk_range(j, self.Kp.shape[0], self.c)[1] - O.chunk_range(j, self.Kp.shape[0], self.c)[0]
                for j in self.own]
        A = np.add.reduceat(a, np.cumsum([0] + lens[:-1])).astype(np.float32)
        loc = O.select_topk(A.astype(np.float64), min(self.k, len(self.own)))
        keys = [(int(np.float32(A[j]).view(np.uint32)) << 32) | (0xFFFFFFFF - self.own[int(j)]) for j in loc]
        keys += [0] * (self.k - len(keys))
        cand.copy_(torch.tensor(np.array(keys, dtype=np.uint64).view(np.int64)))

    def shard_attend(self, layer, cand_all, q, k_suf, v_suf, o_part, lse_part, ids):
        keys = cand_all.numpy().view(np.uint64)
        top = sorted((int(x) for x in keys if x != 0), reverse=True)[: self.k]
        sel = sorted(0xFFFFFFFF - (x & 0xFFFFFFFF) for x in top)
        own = [j for j in sel if j in set(self.own)]
        O_, lse = O.attention(q.double().numpy(), k_suf.double().numpy(), v_suf.double().numpy(), self.Kp, self.Vp,
                              O.kept_token_index(own, self.Kp.shape[0], self.c), self.G,
                              include_suffix=self.shard == self.W - 1)
        o_part.copy_(torch.from_numpy(O_))
        lse_part.copy_(torch.from_numpy(lse.reshape(-1)))
        ids.copy_(torch.tensor(sel, dtype=torch.int32))

    def lse_merge_prepare(self, o_part, lse, lse_max, ns, buf):
        d = o_part.shape[-1]
        w = torch.where(torch.isfinite(lse), torch.exp(lse - lse_max), torch.zeros_like(lse))
        b = torch.cat([o_part.reshape(-1, d) * w[:, None], w[:, None]], dim=1)
        buf.copy_(b.reshape(-1))

    def lse_merge_finish(self, buf, ns, out):
        d = out.shape[-1]
        b = buf.reshape(-1, d + 1)
        out.copy_((b[:, :d] / b[:, d:]).reshape(out.shape))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, W, port, ret, cyclic):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    g = np.random.default_rng(0)
    n, c, ns, hq, hkv, d, k = 203, 8, 5, 4, 2, 16, 6
    Qs, Ks, Vs = g.standard_normal((ns, hq, d)) * 2, g.standard_normal((ns, hkv, d)), g.standard_normal((ns, hkv, d))
    Kp, Vp = g.standard_normal((n, hkv, d)), g.standard_normal((n, hkv, d))
    shard = OracleShard(Kp, Vp, c, k, hq // hkv, rank, W, cyclic)
    runner = ShardedReprefill(shard)
    q, ks, vs = (torch.from_numpy(x).float() for x in (Qs, Ks, Vs))
    # float32 buffers in the runner; the stand-in computes in fp64 from them
    out = torch.empty(ns, hq, d, dtype=torch.float32)
    out, ids = runner.reprefill_layer(0, q, ks, vs, out=out)
    ref = O.reprefill_layer(q.double().numpy(), ks.double().numpy(), vs.double().numpy(), Kp, Vp, c, k, hq // hkv)
    ret[rank] = (ids.tolist(), ref["ids"].tolist(), float(np.abs(out.double().numpy() - ref["out"]).max()))
    dist.destroy_process_group()


@pytest.mark.parametrize("W,cyclic", [(2, False), (2, True)])
def test_sharded_protocol_gloo(W, cyclic):
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(W, port, ret, cyclic), nprocs=W, join=True)
    for r in range(W):
        got, want, err = ret[r]
        assert got == want
        assert err < 1e-5


class _HandleCtx:
    """Stand-in exposing the exchange-handle part of the Context API (64-byte IPC handles)."""

    EXCHANGE_HANDLE_BYTES = 64

    def __init__(self, rank, W):
        self.rank, self.W, self.opened = rank, W, None

    def exchange_handle(self):
        return bytes([self.rank + 1]) * self.EXCHANGE_HANDLE_BYTES

    def exchange_open(self, handles):
        self.opened = list(handles)


def _handle_worker(rank, W, port, ret):
    from paper_2601_13631_b200.sharded import open_exchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    ctx = _HandleCtx(rank, W)
    open_exchange(ctx)
    ret[rank] = ctx.opened
    dist.destroy_process_group()


def test_open_exchange_gathers_handles_in_rank_order():
    # the fused path's one-time setup (sharded.open_exchange): every rank receives all W window
    # handles in rank order before ckv_exchange_open (include/ckv.h)
    W, port = 3, _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_handle_worker, args=(W, port, ret), nprocs=W, join=True)
    for r in range(W):
        assert ret[r] == [bytes([g + 1]) * 64 for g in range(W)]
