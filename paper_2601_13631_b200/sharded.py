"""Position-sharded Re-Prefill over W GPUs: one libckv context per rank.

Two ways to run the exchanges of a sharded layer:

* fused (the product path): ``open_exchange(ctx)`` shares the ranks'
  exchange windows once (64-byte IPC handles all-gathered over torch.distributed); from then
  on ``ctx.reprefill_layer`` runs the whole sharded layer inside libckv -- producers write
  into the peers' windows over NVLink and the streams wait on device counters, no host
  round trip and no NCCL call per layer;
* ``ShardedReprefill``: the split-phase C-ABI calls with the collectives issued from the
  host over torch.distributed (NCCL on GPUs, gloo in the CPU / one-GPU tests) -- the
  NCCL-collective baseline the fused path is compared against.

Per layer, with q / k_suf / v_suf replicated on every rank:
  1. ckv_shard_score       local row normalisers  lam_g [Hq*n_s]            (A1 + A2 local)
  2. allgather(lam_g)      -> every rank forms the global normaliser in rank order
  3. ckv_shard_select      local A_j with the global normaliser; local top-min(k, m_g)
                           candidates as 64-bit (score bits, ~global id) keys
  4. allgather(cand)       -> identical global top-k merge on every rank
  5. ckv_shard_attend      plan / gather / attention over the kept chunks this rank owns
                           (the causal suffix on the last rank), partial (O, lse)
  6. allreduce(MAX, lse), ckv_lse_merge_prepare, allreduce(SUM, [O e^(lse-M) | e^(lse-M)]),
     ckv_lse_merge_finish  -> the exact output on every rank
Step 2 is the exchange the north star omits: without it, shard-local softmax
normalisers make the chunk scores of different shards incomparable.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def open_exchange(ctx, group=None):
    """Attach ctx (shard_index = rank, num_shards = world size) to its peers' exchange windows:
    all-gather the 64-byte handles in rank order, then ckv_exchange_open (collective)."""
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, ctx.exchange_handle(), group=group)
    ctx.exchange_open(handles)
    dist.barrier(group=group)


class ShardedReprefill:
    def __init__(self, ctx, group=None, comm=None):
        """ctx: a Context created with shard_index = rank, num_shards = world size.
        comm: object with all_gather(out, inp), all_reduce_max(t), all_reduce_sum(t)
        (defaults to torch.distributed on `group`)."""
        self.ctx = ctx
        self.W = ctx.W
        self.comm = comm or _TorchComm(group)
        self._bufs = {}

    def _buf(self, name, shape, dtype, device):
        key = (name, tuple(shape), dtype)
        b = self._bufs.get(key)
        if b is None:
            b = torch.empty(shape, dtype=dtype, device=device)
            self._bufs[key] = b
        return b

    def reprefill_layer(self, layer, q, k_suf, v_suf, out=None, ids=None):
        ctx, W = self.ctx, self.W
        dev = q.device
        ns, Hq, d = q.shape
        k = ctx.k
        lam = self._buf("lam", (Hq * ns,), torch.float32, dev)
        ctx.shard_score(layer, q, k_suf, lam)
        lam_all = self._buf("lam_all", (W * Hq * ns,), torch.float32, dev)
        self.comm.all_gather(lam_all, lam)
        cand = self._buf("cand", (k,), torch.int64, dev)
        ctx.shard_select(layer, q, k_suf, lam_all, cand)
        cand_all = self._buf("cand_all", (W * k,), torch.int64, dev)
        self.comm.all_gather(cand_all, cand)
        o_part = self._buf("o_part", (ns, Hq, d), torch.float32, dev)
        lse = self._buf("lse", (ns * Hq,), torch.float32, dev)
        if ids is None:
            ids = torch.empty(k, dtype=torch.int32, device=dev)
        ctx.shard_attend(layer, cand_all, q, k_suf, v_suf, o_part, lse, ids)
        lse_max = self._buf("lse_max", (ns * Hq,), torch.float32, dev)
        lse_max.copy_(lse)
        self.comm.all_reduce_max(lse_max)
        mb = self._buf("merge", (ns * Hq * (d + 1),), torch.float32, dev)
        ctx.lse_merge_prepare(o_part, lse, lse_max, ns, mb)
        self.comm.all_reduce_sum(mb)
        if out is None:
            out = torch.empty_like(q)
        ctx.lse_merge_finish(mb, ns, out)
        return out, ids


class _TorchComm:
    def __init__(self, group=None):
        self.group = group

    def _nccl(self):
        return dist.get_backend(self.group) == "nccl"

    def all_gather(self, out, inp):
        if self._nccl():
            dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        # gloo (CPU tests, or a functional multi-rank run on one GPU): CPU staging, list form
        parts = [torch.empty_like(inp, device="cpu") for _ in range(dist.get_world_size(self.group))]
        dist.all_gather(parts, inp.cpu(), group=self.group)
        out.copy_(torch.cat(parts))

    def _all_reduce(self, t, op):
        if self._nccl():
            dist.all_reduce(t, op=op, group=self.group)
            return
        c = t.cpu()
        dist.all_reduce(c, op=op, group=self.group)
        t.copy_(c)

    def all_reduce_max(self, t):
        self._all_reduce(t, dist.ReduceOp.MAX)

    def all_reduce_sum(self, t):
        self._all_reduce(t, dist.ReduceOp.SUM)
