"""Sequence-sharded HCAttention decode: host orchestration.

Rank r of R holds the contiguous global token range [base_r, base_r + n_r) of every
(b, layer, kv) unit.  One layer is five local phases (CUDA kernels behind the C ABI,
``hc_shard_*`` in include/hc.h) separated by four exchanges:

    begin   -> stats  [rows, 2] int32 {max z, -min z}      all-reduce MAX
    hist1   -> h1     [rows, 4096, 2] int64 (count, mass)   all-reduce SUM
    hist2   -> h2     [rows, 4096] int64 (fine counts)      all-reduce SUM
    counts  -> cnt    [rows, 2] int64 (#strict, #ties)      all-gather
    finish  -> out    [rows, d] fp32 Eq. 5 numerator share  all-reduce SUM

Everything that decides the kept set is an exact integer, and every rank evaluates the
same bounds on the same reduced integers, so the selection is identical to the
unsharded one (R-invariance).

Two drivers of the same phases:
  ``CAbiShard`` -- the product path: ONE C-ABI call per layer (hc_decode_attention_sharded),
      the library issues the collectives itself as NCCL calls on the stream (``hc.NcclComm``,
      graph-capturable); Python only builds the communicator.
  ``decode_layer`` -- the phases one by one with any ``comm`` providing the four collectives:
      ``TorchComm`` (torch.distributed, e.g. gloo on CPU for the protocol tests) or the
      lock-step ``decode_layer_virtual`` (R shards in one process, collectives as tensor
      reductions -- tests the sharded kernels on one GPU without ranks that wait on each other).
"""
from __future__ import annotations

import ctypes as C

NB = 4096


class TorchComm:
    """Collectives over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_max(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_gather(self, t):
        import torch
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.stack(out)


def decode_layer(shard, comm, q, layer: int, base: int):
    """One sharded decode layer on this rank.  Returns (out [rows, d] fp32 = the full
    Eq. 5 output, identical on all ranks; the shard's sel_idx/sel_w hold this rank's kept
    tokens at their global positions)."""
    st = comm.all_reduce_max(shard.begin(q, layer))
    h1 = comm.all_reduce_sum(shard.hist1(layer, st))
    h2 = comm.all_reduce_sum(shard.hist2(layer, st, h1))
    allc = comm.all_gather(shard.counts(layer, h2))
    out = comm.all_reduce_sum(shard.finish(layer, allc, comm.rank, comm.world, base))
    return out


def decode_layer_virtual(shards, q, layer: int, bases):
    """R shards in lock-step in ONE process (same device): the collectives are tensor
    reductions.  Used to test the sharded kernels on a single GPU."""
    import torch
    st = torch.stack([s.begin(q, layer) for s in shards]).amax(0)
    h1 = torch.stack([s.hist1(layer, st) for s in shards]).sum(0)
    h2 = torch.stack([s.hist2(layer, st, h1) for s in shards]).sum(0)
    allc = torch.stack([s.counts(layer, h2) for s in shards])
    outs = [s.finish(layer, allc, r, len(shards), bases[r]) for r, s in enumerate(shards)]
    return torch.stack(outs).sum(0)


class GpuShard:
    """This rank's cache shard and the device buffers of the phase ABI."""

    def __init__(self, kc, vs, bud, device="cuda"):
        import torch

        import paper_2507_19823_b200 as hc
        self.hc = hc
        self.kc, self.vs, self.bud = kc, vs, bud
        rows = kc.B * kc.Hq
        self.rows = rows
        self.ws = hc.Workspace(int(hc.lib().hc_shard_workspace_bytes(C.byref(kc.s), bud)), device)
        self.stats = torch.empty((rows, 2), dtype=torch.int32, device=device)
        self.h1 = torch.empty((rows, NB, 2), dtype=torch.int64, device=device)
        self.h2 = torch.empty((rows, NB), dtype=torch.int64, device=device)
        self.cnt = torch.empty((rows, 2), dtype=torch.int64, device=device)
        self.out = torch.empty((rows, kc.d), dtype=torch.float32, device=device)
        km = int(bud.k_max)
        self.sel_idx = torch.full((rows, km), -1, dtype=torch.int32, device=device)
        self.sel_w = torch.zeros((rows, km), dtype=torch.float32, device=device)
        self.sel_k = torch.zeros((rows,), dtype=torch.int64, device=device)

    def _args(self):
        vs = self.vs.struct()
        return C.byref(self.kc.s), C.byref(vs), vs

    def begin(self, q, layer):
        hc, L = self.hc, self.hc.lib()
        k, v, keep = self._args()
        hc._check(L.hc_shard_begin(hc._ptr(q), k, v, layer, self.bud, hc._ptr(self.stats),
                                   hc._ptr(self.ws.t), self.ws.nbytes, hc._stream()))
        return self.stats

    def hist1(self, layer, gstats):
        hc, L = self.hc, self.hc.lib()
        k, v, keep = self._args()
        hc._check(L.hc_shard_hist1(k, v, layer, self.bud, hc._ptr(gstats), hc._ptr(self.h1),
                                   hc._ptr(self.ws.t), self.ws.nbytes, hc._stream()))
        return self.h1

    def hist2(self, layer, gstats, gh1):
        hc, L = self.hc, self.hc.lib()
        k, v, keep = self._args()
        hc._check(L.hc_shard_hist2(k, v, layer, self.bud, hc._ptr(gstats), hc._ptr(gh1),
                                   hc._ptr(self.h2), hc._ptr(self.ws.t), self.ws.nbytes,
                                   hc._stream()))
        return self.h2

    def counts(self, layer, gh2):
        hc, L = self.hc, self.hc.lib()
        k, v, keep = self._args()
        hc._check(L.hc_shard_counts(k, v, layer, self.bud, hc._ptr(gh2), hc._ptr(self.cnt),
                                    hc._ptr(self.ws.t), self.ws.nbytes, hc._stream()))
        return self.cnt

    def finish(self, layer, allcnt, rank, world, base):
        hc, L = self.hc, self.hc.lib()
        k, v, keep = self._args()
        allcnt = allcnt.contiguous()
        hc._check(L.hc_shard_finish(k, v, layer, self.bud, hc._ptr(allcnt), rank, world, base,
                                    hc._ptr(self.out), hc._ptr(self.sel_idx), hc._ptr(self.sel_w),
                                    hc._ptr(self.sel_k), hc._ptr(self.ws.t), self.ws.nbytes,
                                    hc._stream()))
        return self.out


class CAbiShard:
    """This rank's shard driven through hc_decode_attention_sharded (include/hc.h): the five
    phases and the four NCCL exchanges in one library call per layer."""

    def __init__(self, kc, vs, bud, rank: int, world: int, base: int, comm=None, device="cuda"):
        import torch

        import paper_2507_19823_b200 as hc
        if world > 1 and comm is None:
            raise ValueError("world > 1 needs an hc.NcclComm")
        self.hc, self.kc, self.vs, self.bud = hc, kc, vs, bud
        self.rank, self.world, self.base, self.comm = int(rank), int(world), int(base), comm
        rows = kc.B * kc.Hq
        nb = int(hc.lib().hc_decode_sharded_workspace_bytes(C.byref(kc.s), bud, self.world))
        self.ws = hc.Workspace(nb, device)
        km = int(bud.k_max)
        self.out = torch.empty((rows, kc.d), dtype=torch.float32, device=device)
        self.sel_idx = torch.full((rows, km), -1, dtype=torch.int32, device=device)
        self.sel_w = torch.zeros((rows, km), dtype=torch.float32, device=device)
        self.sel_k = torch.zeros((rows,), dtype=torch.int64, device=device)

    def decode_layer(self, q, layer: int):
        """q [B][Hq][d] fp16 -> out [B*Hq][d] fp32 (the full Eq. 5 output, on every rank)."""
        hc, L = self.hc, self.hc.lib()
        vs = self.vs.struct()
        hc._check(L.hc_decode_attention_sharded(
            hc._ptr(q), C.byref(self.kc.s), C.byref(vs), layer, self.bud, hc._ptr(self.out),
            hc._ptr(self.sel_idx), hc._ptr(self.sel_w), hc._ptr(self.sel_k), self.rank, self.world,
            self.base, self.comm.h if self.comm is not None else None, hc._ptr(self.ws.t),
            self.ws.nbytes, hc._stream()))
        return self.out
