#!/usr/bin/env python
"""Benchmark of the HCAttention decode hot path on B200 (one JSON line on rank 0).

A "step" is one full decode step of a Llama-3-8B-shaped model (BASELINE.json
configs): for each of the L = 32 layers in order, the append (encode the new key into the
quantized cache, append the value) and the decode (table, Eq. 3 scan, softmax mass, Eq. 4
selection, Eq. 5 gather) for all B x 32 query heads -- one hc_append_decode_attention call
per layer (values in HBM), or hc_append_kv + the heterogeneous Eq. 5 (host-resident values).
The step is captured once in a CUDA graph and replayed (steady state: the append
rewrites position n-1, the decode covers n tokens).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

N = 1 default workload: BASELINE config 3 (configs[2], the metric's single-GPU "128K-4M ctx"
configuration): 32 layers, 8 KV heads x GQA 4, d = 128, 128K context, g = 32 (the 12.5 %
budget), c = 8192, k_max = 16384, tau = 0.9, batch 4, values in host pinned memory; Eq. 5
runs heterogeneously (host threads + the GPU's zero-copy pull, share calibrated at start-up;
--host-frac 0 = GPU only) and a `gpu_only` sub-record times the GPU-only pull too.
N > 1 (torchrun): config 4 (1M context) sequence-sharded over the N ranks through the
C-ABI sharded decode (NCCL collectives between the phase kernels), strong scaling;
--config 5 (4M, host-resident values) needs >= 4 ranks; the default N = 1 line carries a
`config5_layer` record (one 4M-token layer on one GPU, GPU-only pull and the heterogeneous
split).  --impl reference times the CPU oracle (oracle/, plain C) as it stands.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode steps/sec and quantized-key GB/s vs HBM peak at 128K–4M ctx, 1/2/4/8 GPU"

CONFIGS = {
    1: dict(B=1, L=1, Hkv=1, G=4, d=128, g=32, c=8192, n=4096, k_max=512, tau=0.9, placement=0,
            workload="config1: 1 layer, 1 KV head x 4 GQA heads, d=128, 4K ctx, g=32 (12.5%), "
                     "c=8192, k_max=512, tau=0.9, batch 1, V in HBM"),
    2: dict(B=1, L=32, Hkv=8, G=4, d=128, g=64, c=8192, n=32768, k_max=8192, tau=0.9, placement=0,
            workload="config2: Llama-3-8B-shaped full decode step (32 layers, 8 KV heads, GQA 4, "
                     "d=128), 32K ctx, 25% KV budget (g=64, c=8192), k_max=8192, tau=0.9, batch 1, "
                     "V in HBM, 1xB200"),
    3: dict(B=4, L=32, Hkv=8, G=4, d=128, g=32, c=8192, n=131072, k_max=16384, tau=0.9,
            placement=1,
            workload="config3: Llama-3-8B-shaped, 128K ctx, 12.5% KV budget (g=32, c=8192), "
                     "k_max=16384, tau=0.9, batch 4, V in host pinned memory (zero-copy), 1xB200"),
    4: dict(B=1, L=32, Hkv=8, G=4, d=128, g=32, c=8192, n=1048576, k_max=131072, tau=0.9,
            placement=0,
            workload="config4: Llama-3-8B-shaped, 1M ctx sequence-sharded across the GPUs "
                     "(contiguous token ranges, NCCL merges), 12.5% KV budget (g=32, c=8192), "
                     "k_max=131072, tau=0.9, batch 1, V in HBM"),
    5: dict(B=1, L=32, Hkv=8, G=4, d=128, g=32, c=8192, n=4194304, k_max=524288, tau=0.9,
            placement=1,
            workload="config5: Llama-3-8B-shaped, 4M ctx sequence-sharded across the GPUs, 12.5% KV "
                     "budget (g=32, c=8192), k_max=524288, tau=0.9, batch 1, V in host pinned memory "
                     "(32 GiB per rank at N=8)"),
}
Q_SCALE = 2.29  # calibrates tau=0.9 to Table 3's 15.6 % selection ratio
SEED = 0x48434154


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + clock-event reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, dev_index: int, period_s: float = 0.01):
        self.samples, self.reason_bits = [], 0
        self.period = period_s
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            import torch
            pr = torch.cuda.get_device_properties(dev_index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            try:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reason_bits |= int(r) & ~0x1
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.REASONS.items() if self.reason_bits & k],
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workload
class Workload:
    """The synthetic decode state of one rank.  With world > 1 (or virtual shards) rank r
    holds the contiguous global token range [a_r, b_r) of every (b, layer, kv) unit; the
    newest token (global position n-1) lives on the last rank, which does the append."""

    def __init__(self, cfg: dict, device: str, rank: int = 0, world: int = 1):
        import numpy as np
        import torch

        import paper_2507_19823_b200 as hc
        import synth
        import synth.device as sd
        self.cfg = cfg
        B, L, H, G, d, g, c, n = (cfg[k] for k in ("B", "L", "Hkv", "G", "d", "g", "c", "n"))
        self.Hq = G * H
        bounds = [int(x) for x in np.linspace(0, n, world + 1)]
        self.base, self.n_local = bounds[rank], bounds[rank + 1] - bounds[rank]
        self.is_last = rank == world - 1
        n_cap = max(64, (self.n_local + 63) // 64 * 64)
        cb = np.stack([synth.gen_codebook(SEED, l, g, c, d // g) for l in range(L)])
        self.codebook = torch.from_numpy(cb).to(device)
        self.vo_only = cfg.get("vo_only", False)
        if self.vo_only:  # every token resident with exact keys: codes / value store unused
            self.kc = hc.KCache(B, L, H, G, d, g, c, 64, self.codebook, device=device,
                                res_cap=n_cap)
            self.vs = hc.VStore.allocate(B, L, H, 64, d, device=device)
            sd.fill_values(self.kc.res_k, SEED + 7, self.n_local, device=device, start=self.base)
            sd.fill_values(self.kc.res_v, SEED, self.n_local, device=device, start=self.base)
        else:
            self.kc = hc.KCache(B, L, H, G, d, g, c, n_cap, self.codebook, device=device,
                                lut_bits=cfg.get("lut_bits", 16), code_bits=cfg.get("code_bits", 16))
            self.vs = hc.VStore.allocate(B, L, H, n_cap, d, placement=cfg["placement"], device=device)
            if cfg.get("code_bits", 16) == 13:  # fill u16 layer by layer, pack into strips
                c16 = torch.zeros((B, 1, H, g, n_cap), dtype=torch.int16, device=device)
                for l in range(L):
                    sd.fill_codes(c16, SEED, c, self.n_local, start=self.base, layers=[0], layer_ids=[l])
                    for b_ in range(B):  # codes[b, l] is one contiguous run of strips
                        hc.pack_codes13(c16[b_:b_ + 1], n_cap, n_cap, out=self.kc.codes[b_:b_ + 1, l:l + 1])
                del c16
            else:
                sd.fill_codes(self.kc.codes, SEED, c, self.n_local, start=self.base)
            sd.fill_values(self.vs.tensor, SEED, self.n_local, device=device, start=self.base)
        self.reset_counts()
        # per-step inputs: q for every layer, the new token's k and v
        q = np.stack([np.stack([synth.gen_query(SEED + 1, b, l, self.Hq, d, Q_SCALE)
                                for b in range(B)]) for l in range(L)])
        kn = synth.gen_keys(SEED + 2, 1, L * B * H, d).reshape(L, B, H, d)
        vn = synth.gen_keys(SEED + 2, 2, L * B * H, d).reshape(L, B, H, d)
        self.q_host = torch.from_numpy(q).pin_memory()
        self.k_host = torch.from_numpy(kn).pin_memory()
        self.v_host = torch.from_numpy(vn).pin_memory()
        self.q = self.q_host.to(device)
        self.k_new = self.k_host.to(device)
        self.v_new = self.v_host.to(device)
        self.out = torch.zeros((L, B, self.Hq, d), dtype=torch.float32, device=device)
        self.out_host = torch.zeros_like(self.out, device="cpu").pin_memory()
        self.cpu_gather = cfg.get("cpu_gather", False)
        self.hetero = None
        if cfg.get("host_frac", 0.0) > 0.0:  # heterogeneous Eq. 5 (GPU pull + host threads)
            from paper_2507_19823_b200.hetero import HeteroEq5
            # replicas (N > 1 processes on one host) split the host cores
            nthr = max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
            self.hetero = HeteroEq5(self.kc, self.vs, cfg["k_max"], cfg["host_frac"], threads=nthr,
                                    device=device)
        # micro-batch pipelining (--pipeline P): P independent chains of B/P sequences on their
        # own streams, so one chain's GPU selection overlaps another's Eq. 5 (host + link)
        self.parts = []
        P = cfg.get("pipeline", 1)
        if P > 1:
            from paper_2507_19823_b200.hetero import HeteroEq5
            if B % P:
                raise SystemExit(f"--pipeline {P} must divide the batch B={B}")
            nb = B // P
            shared_worker = hc.HostWorker(threads=os.cpu_count() or 1) if cfg.get("host_frac", 0.0) > 0.0 else None
            for i in range(P):
                kv_ = self.kc.batch_view(i * nb, nb)
                vs_ = self.vs.batch_view(i * nb, nb)
                het = (HeteroEq5(kv_, vs_, cfg["k_max"], cfg["host_frac"], device=device,
                                 worker=shared_worker)
                       if cfg.get("host_frac", 0.0) > 0.0 else None)
                self.parts.append(dict(b0=i * nb, b1=(i + 1) * nb, kc=kv_, vs=vs_, het=het,
                                       stream=torch.cuda.Stream(device=device)))
        self.bud = hc.budget(cfg["tau"], cfg["k_max"], select_only=self.cpu_gather,
                             shared_kv=cfg.get("shared_kv", False))
        self.ws = hc.Workspace(self.kc.workspace_bytes(self.bud), device=device)
        for part in self.parts:
            part["ws"] = hc.Workspace(part["kc"].workspace_bytes(self.bud), device=device)
        self.sel_k = torch.zeros((L, B, self.Hq), dtype=torch.int64, device=device)
        if self.cpu_gather:  # (idx, w) of one layer, device + pinned host; host Eq. 5 output
            km = cfg["k_max"]
            self.sel_i_d = torch.empty((B * self.Hq, km), dtype=torch.int32, device=device)
            self.sel_w_d = torch.empty((B * self.Hq, km), dtype=torch.float32, device=device)
            self.sel_i_h = torch.empty_like(self.sel_i_d, device="cpu").pin_memory()
            self.sel_w_h = torch.empty_like(self.sel_w_d, device="cpu").pin_memory()
            self.sel_k_h = torch.empty((L, B * self.Hq), dtype=torch.int64).pin_memory()
            self.out_cpu = torch.empty((L, B * self.Hq, d), dtype=torch.float32).pin_memory()
        self.ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(L)]
        # the whole Eq. 3 stage (table + scan) per layer, for the eq3_stage record
        self.ev3 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(L)]
        for b_, e_ in self.ev + self.ev3:  # torch creates the CUDA event lazily on first record
            b_.record()
            e_.record()
        torch.cuda.synchronize()
        self.shard = None
        self.comm = None

    def enable_sharding(self, comm, rank: int, world: int):
        """The product path: one hc_decode_attention_sharded call per layer, the library
        issuing the NCCL exchanges on the stream (comm: hc.NcclComm)."""
        from paper_2507_19823_b200.sharded import CAbiShard
        self.shard = CAbiShard(self.kc, self.vs, self.bud, rank, world, self.base, comm)
        self.comm = comm

    def reset_counts(self):
        n_here = self.n_local - (1 if self.is_last else 0)  # the step appends position n-1
        for kc in [self.kc] + [p["kc"] for p in getattr(self, "parts", [])]:
            for l in range(self.cfg["L"]):
                if self.vo_only:
                    kc.set_counts(l, 0, n_here)
                else:
                    kc.set_counts(l, n_here)

    def step_pipelined(self, profile=False):
        import torch

        import paper_2507_19823_b200 as hc
        main = torch.cuda.current_stream()
        for part in self.parts:
            part["stream"].wait_stream(main)
        for i, part in enumerate(self.parts):
            b0, b1 = part["b0"], part["b1"]
            with torch.cuda.stream(part["stream"]):
                for l in range(self.cfg["L"]):
                    if self.is_last:
                        part["kc"].append(l, self.k_new[l][b0:b1], self.v_new[l][b0:b1], part["vs"])
                    if profile and i == 0:
                        hc.profile_scan_events(*self.ev[l])
                    if part["het"] is not None:
                        part["het"](self.q[l][b0:b1], l, self.bud, self.out[l][b0:b1],
                                    self.sel_k[l][b0:b1], part["ws"])
                    else:
                        hc.decode_attention(self.q[l][b0:b1], part["kc"], part["vs"], l, self.bud,
                                            out=self.out[l][b0:b1], sel_k=self.sel_k[l][b0:b1],
                                            ws=part["ws"])
        for part in self.parts:
            main.wait_stream(part["stream"])

    def step(self, profile=False):
        import paper_2507_19823_b200 as hc
        if self.parts:
            return self.step_pipelined(profile)
        # plain decode: the append and the decode as ONE library call (hc_append_decode_attention:
        # the append's encode overlaps the table build); HC_FUSED_APPEND=0 issues the two calls
        fused = (self.is_last and self.hetero is None and self.shard is None and not self.cpu_gather
                 and os.environ.get("HC_FUSED_APPEND", "1") != "0")
        for l in range(self.cfg["L"]):
            if self.is_last and not fused:
                self.kc.append(l, self.k_new[l], self.v_new[l], self.vs)
            if profile:
                hc.profile_scan_events(*self.ev[l])
                hc.profile_eq3_events(*self.ev3[l])
            if self.cpu_gather:
                self._step_cpu_gather(l)
            elif self.hetero is not None:
                self.hetero(self.q[l], l, self.bud, self.out[l], self.sel_k[l], self.ws)
            elif fused:
                hc.append_decode_attention(self.q[l], self.kc, self.vs, l, self.k_new[l], self.v_new[l],
                                           self.bud, out=self.out[l], sel_k=self.sel_k[l], ws=self.ws)
            elif self.shard is None:
                hc.decode_attention(self.q[l], self.kc, self.vs, l, self.bud, out=self.out[l],
                                    sel_k=self.sel_k[l], ws=self.ws)
            else:
                o = self.shard.decode_layer(self.q[l], l)
                self.out[l].copy_(o.view_as(self.out[l]))
                self.sel_k[l].copy_(self.shard.sel_k.view_as(self.sel_k[l]))

    def _step_cpu_gather(self, l):
        """GPU: table, scan, softmax mass, selection; D2H (idx, w, k); host threads: Eq. 5 over
        the pinned value store; H2D of the layer output (all stream-ordered, graph-capturable)."""
        import ctypes as C

        import paper_2507_19823_b200 as hc
        cfg = self.cfg
        B, L, H, d = cfg["B"], cfg["L"], cfg["Hkv"], cfg["d"]
        hc.decode_attention(self.q[l], self.kc, self.vs, l, self.bud, out=self.out[l],
                            sel_idx=self.sel_i_d, sel_w=self.sel_w_d, sel_k=self.sel_k[l], ws=self.ws)
        self.sel_i_h.copy_(self.sel_i_d, non_blocking=True)
        self.sel_w_h.copy_(self.sel_w_d, non_blocking=True)
        self.sel_k_h[l].copy_(self.sel_k[l].view(-1), non_blocking=True)
        ncap = self.kc.n_cap
        V = self.vs.tensor[0, l]
        st = hc.lib().hc_enqueue_host_weighted_sum(
            C.c_void_p(self.sel_i_h.data_ptr()), C.c_void_p(self.sel_w_h.data_ptr()),
            C.c_void_p(self.sel_k_h[l].data_ptr()), B * self.Hq, cfg["k_max"],
            C.c_void_p(V.data_ptr()), L * H * ncap * d, ncap * d, self.kc.n_q(l), self.Hq, cfg["G"], d,
            C.c_void_p(self.out_cpu[l].data_ptr()), 0, hc._stream())
        hc._check(st)
        self.out[l].view(-1, d).copy_(self.out_cpu[l], non_blocking=True)

    def step_e2e(self):
        self.q.copy_(self.q_host, non_blocking=True)
        self.k_new.copy_(self.k_host, non_blocking=True)
        self.v_new.copy_(self.v_host, non_blocking=True)
        self.step()
        self.out_host.copy_(self.out, non_blocking=True)

    def capture(self, fn):
        import torch

        import paper_2507_19823_b200 as hc
        self.reset_counts()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        before = hc.launch_count()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        launches = hc.launch_count() - before
        self.reset_counts()
        return g, launches


class EagerStep:
    """Stand-in for a captured graph (replay = run the step eagerly); counts are reset so
    every replay appends at the same position, like the graph."""

    def __init__(self, wl, fn):
        self.wl, self.fn = wl, fn

    def replay(self):
        self.wl.reset_counts()
        self.fn()


def event_ms(b, e) -> float:
    """cudaEventElapsedTime for events recorded by the library inside the graph (torch's
    Event object does not know they were recorded, so ask the driver directly)."""
    import ctypes
    cu = ctypes.CDLL("libcuda.so.1")
    f = ctypes.c_float()
    rc = cu.cuEventElapsedTime(ctypes.byref(f), ctypes.c_void_p(b.cuda_event),
                               ctypes.c_void_p(e.cuda_event))
    if rc != 0:
        raise RuntimeError(f"cuEventElapsedTime rc={rc}")
    return f.value


def time_graph(g, K, W, dist=None):
    import torch
    for _ in range(W):
        g.replay()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    # blocking-sync events: the waiting thread sleeps instead of spinning on a core that the
    # host share of the heterogeneous Eq. 5 needs
    e0 = torch.cuda.Event(enable_timing=True, blocking=True)
    e1 = torch.cuda.Event(enable_timing=True, blocking=True)
    e0.record()
    for _ in range(K):
        g.replay()
    e1.record()
    e1.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def union_gather_bytes(wl, host_frac: float = 0.0):
    """Value bytes the union gather reads per step: re-run the step's selections (eager, after
    the timed region) and count, per (b, layer, kv), the union of the G heads' kept rows.
    With a heterogeneous split returns (GPU-pulled bytes, host-summed bytes): rows with index
    >= t_split = round(host_frac * n_q) go over the host link, the rest stay in host DRAM."""
    import torch

    import paper_2507_19823_b200 as hc
    cfg = wl.cfg
    B, L, H, G, d, km = (cfg[k] for k in ("B", "L", "Hkv", "G", "d", "k_max"))
    idx = torch.full((B, H * G, km), -1, dtype=torch.int32, device="cuda")
    w = torch.zeros((B, H * G, km), dtype=torch.float32, device="cuda")
    k = torch.zeros((B, H * G), dtype=torch.int64, device="cuda")
    bud = hc.budget(cfg["tau"], km, select_only=True, shared_kv=cfg.get("shared_kv", False))
    rows = rows_h = 0
    for l in range(L):
        hc.decode_attention(wl.q[l], wl.kc, wl.vs, l, bud, sel_idx=idx, sel_w=w, sel_k=k, ws=wl.ws,
                            out=wl.out[l])
        t_split = int(round(host_frac * wl.kc.n_q(l)))
        for b in range(B):
            for kv in range(H):
                sets = [idx[b, kv * G + h, : int(k[b, kv * G + h])] for h in range(G)]
                u = torch.unique(torch.cat(sets))
                nh = int((u < t_split).sum())
                rows_h += nh
                rows += int(u.numel()) - nh
    if host_frac > 0.0:
        return rows * d * 2.0, rows_h * d * 2.0
    return rows * d * 2.0


def measure_host_rows_gbs(wl, reps: int = 3) -> dict:
    """Host DRAM random-row capability on layer 0's full selection, GB/s of union rows (rows
    kept by several GQA heads counted once, as both readers read them once):
      host_alone -- the host Eq. 5 engine (all the split's threads) over every kept row;
      gpu_alone  -- the GPU's zero-copy union gather over every kept row (hc_gather_values);
      combined   -- both at once on a time-balanced split (host share T_gpu / (T_host + T_gpu)):
                    all union bytes / the later finish.  Both agents read the same host DRAM, so
                    this -- not their sum -- is what the split can reach (the roofline peak)."""
    import time

    import torch

    import paper_2507_19823_b200 as hc
    het, cfg = wl.hetero, wl.cfg
    G = cfg["G"]
    bud = hc.budget(cfg["tau"], cfg["k_max"], select_only=True)
    sel_k = torch.zeros((cfg["B"], wl.Hq), dtype=torch.int64, device="cuda")
    hc.decode_attention(wl.q[0], wl.kc, wl.vs, 0, bud, out=wl.out[0], sel_idx=het.idx_d, sel_w=het.w_d,
                        sel_k=sel_k, ws=wl.ws)
    torch.cuda.synchronize()
    het.idx_h.copy_(het.idx_d)
    het.w_h.copy_(het.w_d)
    het.k_h.copy_(sel_k.view(-1))
    rows = 0
    for u in range(het.idx_h.shape[0] // G):
        sets = [het.idx_h[u * G + h, : int(het.k_h[u * G + h])] for h in range(G)]
        rows += int(torch.unique(torch.cat(sets)).numel())
    nbytes = rows * cfg["d"] * 2
    n = wl.kc.n_q(0)
    out = torch.empty_like(wl.out[0])

    def host(t0_, t1_):
        hc.host_weighted_sum_range(het.idx_h, het.w_h, het.k_h, wl.vs, 0, G, t0_, t1_, het.part_h, het.threads,
                                   n_valid=n)

    def gpu(t0_, t1_):
        hc.gather_values(wl.kc, wl.vs, 0, het.idx_d, het.w_d, sel_k, t0_, t1_, out, wl.ws)

    th, tg = [], []
    for _ in range(reps + 1):
        a = time.perf_counter()
        host(0, n)
        th.append(time.perf_counter() - a)
        torch.cuda.synchronize()
        a = time.perf_counter()
        gpu(0, n)
        torch.cuda.synchronize()
        tg.append(time.perf_counter() - a)
    t_h, t_g = min(th[1:]), min(tg[1:])
    split = int(round(n * t_g / (t_h + t_g)))
    tc = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        a = time.perf_counter()
        gpu(split, n)          # asynchronous: the GPU pulls its share ...
        host(0, split)         # ... while this thread's team sums the host's share
        torch.cuda.synchronize()
        tc.append(time.perf_counter() - a)
    return {"host_alone": nbytes / t_h / 1e9, "gpu_alone": nbytes / t_g / 1e9,
            "combined": nbytes / min(tc[1:]) / 1e9, "combined_host_share": split / n}


def measure_host_dram_hw(wl) -> dict:
    """Engine-free host DRAM read rates over the value store's own pinned memory (tools/
    membench.c: random 256-B rows, a sorted row subset and a sequential pass, all host cores;
    CPU model and NUMA layout recorded), plus both DRAM consumers of the heterogeneous split at
    once without any Eq. 5 arithmetic: the cores' sequential pass over one half of the store
    while the GPU's copy engine reads the other half (cudaMemcpy H2D) -- the hardware ceiling
    the host share of Eq. 5 is judged against."""
    import ctypes
    import threading

    import torch
    from tools import membench
    t = wl.vs.tensor
    nbytes = t.numel() * t.element_size()
    hw = membench.measure(t.data_ptr(), nbytes)
    # both consumers at once: CPU sequential over [0, half), GPU copies from [half, half + 4 GiB)
    half = (nbytes // 2) // 4096 * 4096
    gb = min(4 << 30, nbytes - half) // 4096 * 4096
    flat = t.view(-1).view(torch.uint8)
    src = flat[half:half + gb]
    dst = torch.empty(gb, dtype=torch.uint8, device="cuda")
    L = membench.lib()
    thr = hw["threads"]
    res = {}

    def cpu():
        sink = ctypes.c_uint64()
        res["cpu"] = L.hm_sequential(ctypes.c_void_p(t.data_ptr()), min(half, 16 << 30), thr, ctypes.byref(sink))

    dst.copy_(src, non_blocking=True)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th = threading.Thread(target=cpu)
    e0.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    e1.record()
    th.start()
    th.join()
    torch.cuda.synchronize()
    dma = 3 * gb / (e0.elapsed_time(e1) * 1e-3) / 1e9
    hw["concurrent"] = {"cpu_sequential_gbs": res["cpu"], "gpu_h2d_copy_gbs": dma,
                        "sum_gbs": res["cpu"] + dma,
                        "how": "cores' sequential pass over one half of the store while the copy "
                               "engine reads 3 x 4 GiB of the other half (overlapping; each rate "
                               "over its own duration)"}
    hw["peak_gbs"] = max(hw["peak_gbs"], res["cpu"] + dma)
    del dst
    return hw


def measure_gpu_only(wl, args, dev_index, h2d_peak):
    """The north_star's stage 4 alone: Eq. 5 entirely on the GPU (host_frac 0, the zero-copy
    GQA-union pull of every kept row over the host link) on the same workload, timed the same
    way (CUDA graph, events, K replays after W warm-ups)."""
    import torch
    het = wl.hetero
    wl.hetero = None
    try:
        wl.reset_counts()
        wl.step()
        torch.cuda.synchronize()
        g, launches = wl.capture(wl.step)
        K = max(3, args.steps // 2)
        with ClockSampler(dev_index) as clk:
            ms = time_graph(g, K, max(args.warmup, 3)) / K
        del g
        v_bytes = union_gather_bytes(wl)
    finally:
        wl.hetero = het
        wl.reset_counts()
    gbs = v_bytes / (ms * 1e-3) / 1e9
    return {"value": 1000.0 / ms, "unit": "steps/s", "ms_per_step": ms, "steps": K,
            "gpu_launches_per_step": launches,
            "eq5": "GPU only: k_gather_union pulls the union of the GQA heads' kept rows zero-copy",
            "host_link": {"bytes_per_step": v_bytes, "achieved_gbs_lower_bound": gbs, "peak_gbs": h2d_peak,
                          "peak_source": "measured pinned H2D cudaMemcpy 1 GiB", "frac": gbs / h2d_peak,
                          "note": "whole step time in the denominator (scan + selection included)"},
            "clocks": clk.summary()}


def measure_config5_layers(args, layers: int, dev_index: int, h2d_peak: float, host_frac: float = 0.0) -> dict:
    """BASELINE config 5 (4M-token context, g = 32, k_max = 524,288, values in host pinned
    memory) on ONE GPU with the layer count reduced to `layers` (the full 32-layer store, 275
    GB of host values, needs >= 4 ranks): per-layer time of the unsharded decode with the
    GPU-only Eq. 5 pull, and its Eq. 3 stage; with host_frac > 0 also the heterogeneous split
    (host threads + GPU pull, the default bench's share) on the same store."""
    import torch
    cfg = dict(CONFIGS[5])
    cfg.update(L=layers, lut_bits=16, vo_only=False, cpu_gather=False, shared_kv=False, code_bits=16,
               host_frac=0.0, pipeline=1)
    wl = Workload(cfg, "cuda")
    wl.reset_counts()
    wl.step()
    torch.cuda.synchronize()
    g, launches = wl.capture(wl.step)
    gp, _ = wl.capture(lambda: wl.step(profile=True))
    K = 10
    with ClockSampler(dev_index) as clk:
        ms = time_graph(g, K, 3) / K
    for _ in range(2):
        gp.replay()
    torch.cuda.synchronize()
    scan = statistics.mean(event_ms(b, e) for (b, e) in wl.ev)
    eq3 = statistics.mean(event_ms(b, e) for (b, e) in wl.ev3)
    del g, gp
    v_bytes = union_gather_bytes(wl)
    ksel = wl.sel_k.float().mean().item()
    p_bytes = cfg["B"] * cfg["Hkv"] * wl.n_local * cfg["g"] * 2
    peak, _ = measured_peaks()
    res = {"workload": f"config5 on ONE B200, L = {layers} of 32 layers (stated: the 32-layer host "
                       f"store needs >= 4 ranks), unsharded, GPU-only Eq. 5 (zero-copy union pull), "
                       f"n = {cfg['n']}, g = 32, k_max = {cfg['k_max']}, tau = 0.9, batch 1",
           "layers": layers, "ms_per_layer": ms / layers,
           "steps_per_s_at_32_layers_extrapolated": 1000.0 / (32 * ms / layers),
           "scan": {"avg_ms": scan, "achieved_gbs": p_bytes / (scan * 1e-3) / 1e9,
                    "frac_hbm": p_bytes / (scan * 1e-3) / 1e9 / peak},
           "eq3_stage": {"avg_ms": eq3, "achieved_gbs": p_bytes / (eq3 * 1e-3) / 1e9,
                         "frac_hbm": p_bytes / (eq3 * 1e-3) / 1e9 / peak},
           "host_link": {"bytes_per_layer": v_bytes / layers,
                         "achieved_gbs_lower_bound": v_bytes / (ms * 1e-3) / 1e9,
                         "peak_gbs": h2d_peak, "frac": v_bytes / (ms * 1e-3) / 1e9 / h2d_peak},
           "selection": {"mean_k_sel": ksel, "k_sel_over_n": ksel / cfg["n"]},
           "gpu_launches_per_step": launches, "clocks": clk.summary()}
    if host_frac > 0.0:  # the paper's split on the same 4M-token layer
        from paper_2507_19823_b200.hetero import HeteroEq5
        nthr = max(1, os.cpu_count() or 1)
        wl.hetero = HeteroEq5(wl.kc, wl.vs, cfg["k_max"], host_frac, threads=nthr)
        try:
            wl.reset_counts()
            wl.step()
            torch.cuda.synchronize()
            g, _ = wl.capture(wl.step)
            with ClockSampler(dev_index) as clk2:
                ms2 = time_graph(g, K, 3) / K
            del g
            wl.hetero.check()
            res["hetero"] = {"host_frac": host_frac, "ms_per_layer": ms2 / layers,
                             "steps_per_s_at_32_layers_extrapolated": 1000.0 / (32 * ms2 / layers),
                             "eq5": "host threads sum the kept rows of the first host_frac of the tokens "
                                    "over host DRAM while the GPU pulls the rest (as the default bench)",
                             "clocks": clk2.summary()}
        finally:
            if wl.hetero.mode == "doorbell":
                wl.hetero.worker.close()
            wl.hetero = None
    if wl.vs.host is not None:
        wl.vs.host.close()
    del wl
    torch.cuda.empty_cache()
    return res


HOST_FRAC_CANDIDATES = (0.6, 0.65, 0.7, 0.75)  # calibrated at start-up; box optima 0.65-0.7


def calibrate_host_frac(wl, cfg):
    """Pick the heterogeneous split for this box before the timed region: a few graph-timed
    steps per candidate share (the optimum moves with the host's DRAM and core count; measured
    0.65-0.7 on the B200 pool).  Untimed; the chosen share is reported."""
    import torch

    from paper_2507_19823_b200.hetero import HeteroEq5
    nthr = wl.hetero.threads
    best = None
    for f in HOST_FRAC_CANDIDATES:
        wl.hetero.worker.close()
        wl.hetero = HeteroEq5(wl.kc, wl.vs, cfg["k_max"], f, threads=nthr)
        wl.reset_counts()
        wl.step()
        torch.cuda.synchronize()
        g, _ = wl.capture(wl.step)
        ms = time_graph(g, 4, 1) / 4
        del g
        if best is None or ms < best[1]:
            best = (f, ms)
    wl.hetero.worker.close()
    cfg["host_frac"] = best[0]
    wl.hetero = HeteroEq5(wl.kc, wl.vs, cfg["k_max"], best[0], threads=nthr)
    wl.reset_counts()


def hc_lib_check():
    import paper_2507_19823_b200 as hc
    hc.lib()  # no CPU fallback: fail loudly if the CUDA library is missing


def measure_h2d_gbs() -> float:
    import torch
    src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 5 * (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9


# ----------------------------------------------------------------------------- CPU oracle
def oracle_wave(cfg, units, threads):
    """Run the oracle on `units` (b, l, kv) decode units in parallel threads (the C calls
    release the GIL); returns wall seconds.  Inputs are generated before timing."""
    import concurrent.futures as cf

    import oracle
    import synth
    d, g, c, n, G = cfg["d"], cfg["g"], cfg["c"], cfg["n"], cfg["G"]
    Hq = G * cfg["Hkv"]
    inputs = []
    for (b, l, kv) in units:
        q = synth.gen_query(SEED + 1, b, l, Hq, d, Q_SCALE)[kv * G:(kv + 1) * G]
        inputs.append((q, synth.gen_codebook(SEED, l, g, c, d // g),
                       synth.gen_codes(SEED, b, l, kv, g, c, 0, n),
                       synth.gen_values(SEED, b, l, kv, d, 0, n)))
    oracle.lib()
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda a: oracle.decode_unit(a[0], a[1], a[2], n, a[3], cfg["tau"],
                                                  cfg["k_max"], lut_bits=cfg.get("lut_bits", 16)),
                    inputs))
    return time.perf_counter() - t0


def cpu_baseline(cfg, budget_s=12.0):
    cores = os.cpu_count() or 1
    units_total = cfg["B"] * cfg["L"] * cfg["Hkv"]
    wave = min(cores, units_total)
    units = [(0, l % cfg["L"], kv % cfg["Hkv"]) for l, kv in
             ((i // cfg["Hkv"], i % cfg["Hkv"]) for i in range(wave))]
    t_first = oracle_wave(cfg, units, wave)
    reps = max(1, int(budget_s / max(t_first, 1e-3)) - 1)
    ts = [t_first] + [oracle_wave(cfg, units, wave) for _ in range(min(reps, 20))]
    t_wave = statistics.median(ts)
    step_s = math.ceil(units_total / wave) * t_wave
    return {"value": 1.0 / step_s, "unit": "steps/s", "cores": wave, "kind": "oracle",
            "sample": f"{wave} of the step's {units_total} (layer, KV-head) units, one per thread, "
                      f"{len(ts)} waves, median wave {t_wave:.3f}s; step = ceil({units_total}/{wave}) "
                      f"waves"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    units_total = cfg["B"] * cfg["L"] * cfg["Hkv"]
    wave = min(cores, units_total)
    units = [(0, i // cfg["Hkv"] % cfg["L"], i % cfg["Hkv"]) for i in range(wave)]
    for _ in range(args.warmup):
        oracle_wave(cfg, units, wave)
    ts = [oracle_wave(cfg, units, wave) for _ in range(args.steps)]
    step_s = math.ceil(units_total / wave) * statistics.mean(ts)
    v = 1.0 / step_s
    line = {"metric": METRIC, "value": v, "unit": "steps/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": ("strong" if int(os.environ.get("WORLD_SIZE", "1")) > 1 and args.config in (4, 5) else "weak"),
            "vs_baseline": None, "dtype": "i16+f32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "reference": "CPU oracle (oracle/hc_oracle.c)"},
            "cpu_baseline": {"value": v, "unit": "steps/s", "cores": wave, "kind": "oracle",
                             "sample": f"each step = {wave} of {units_total} units in parallel, "
                                       f"extrapolated x ceil({units_total}/{wave})"},
            "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_virtual(args, cfg, R):
    """Test mode: the sequence-sharded step of `cfg` as R shards on one GPU, collectives as
    tensor reductions (paper_2507_19823_b200.sharded.decode_layer_virtual)."""
    import torch

    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.sharded import GpuShard, decode_layer_virtual
    wls = [Workload(cfg, "cuda", r, R) for r in range(R)]
    shards = [GpuShard(w.kc, w.vs, w.bud) for w in wls]
    bases = [w.base for w in wls]
    L = cfg["L"]

    def step():
        for l in range(L):
            wls[-1].kc.append(l, wls[-1].k_new[l], wls[-1].v_new[l], wls[-1].vs)
            o = decode_layer_virtual(shards, wls[0].q[l], l, bases)
            wls[0].out[l].copy_(o.view_as(wls[0].out[l]))

    for w in wls:
        w.reset_counts()
    step()
    torch.cuda.synchronize()
    for w in wls:
        w.reset_counts()
    g = torch.cuda.CUDAGraph()
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        with torch.cuda.graph(g, stream=s_):
            step()
    torch.cuda.current_stream().wait_stream(s_)
    ms = time_graph(g, args.steps, max(args.warmup, 3)) / args.steps
    ksel = shards[0].sel_k.float().mean().item()
    print(json.dumps({"metric": METRIC, "value": 1000.0 / ms, "unit": "steps/s", "n_gpus": 1,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                      "config": {"workload": cfg["workload"],
                                 "parallelism": f"virtual-shards x{R} on one GPU (test mode)"},
                      "selection": {"mean_k_sel": ksel, "k_sel_over_n": ksel / cfg["n"]}}), flush=True)


# ----------------------------------------------------------------------------- main
PIPELINE_DEFAULT = 1  # set from measurement

# tools/smem_gather_micro.cu on a B200 (profiles/r01_smem_gather_micro.log): one 512-thread CTA
# per SM doing random lookups into a 64 KiB (8-byte entries) / 32 KiB (4-byte) table slice,
# nothing else -- the fastest the scan could consume u16 codes (2 B of P per lookup)
SMEM_CEILING = {
    8: {"entry_bytes": 8, "code_GBps": 3017.5, "frac_of_hbm": 3017.5 / 6549.4,
        "wavefronts_per_warp_lookup": 6.15, "source": "profiles/r01_smem_gather_micro.log"},
    4: {"entry_bytes": 4, "code_GBps": 4778.9, "frac_of_hbm": 4778.9 / 6549.4,
        "wavefronts_per_warp_lookup": 3.89, "source": "profiles/r01_smem_gather_micro.log"},
}
HOST_FRAC_DEFAULT = 0.7  # measured optimum on the B200 box (DESIGN §8b f1, tools/hetero_sweep.py)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default 500 (config 1/2), 20 (3/4)")
    ap.add_argument("--warmup", type=int, default=None, help="default 10 (config 1/2), 3 (3/4)")
    ap.add_argument("--vo-only", action="store_true",
                    help="value-offload-only mode (SURVEY f2): exact fp16 keys, no quantization")
    ap.add_argument("--cpu-gather", action="store_true",
                    help="the paper's split (SURVEY f1): GPU selects, Eq. 5 runs on host threads "
                         "over the host-resident values (needs a host-V config, e.g. 3)")
    ap.add_argument("--host-frac", type=float, default=None,
                    help="heterogeneous Eq. 5 for host-resident values: host threads sum the kept "
                         "rows of this share of the token range while the GPU pulls the rest "
                         "(default for host-V configs: %s; 0 = GPU only)" % HOST_FRAC_DEFAULT)
    ap.add_argument("--pipeline", type=int, default=None,
                    help="micro-batch pipelining: P chains of B/P sequences on their own streams "
                         "(default for host-V configs: %d)" % PIPELINE_DEFAULT)
    ap.add_argument("--lut8", action="store_true",
                    help="8-bit query/codebook table variant (R2b, SURVEY f3)")
    ap.add_argument("--code-bits", type=int, default=16, choices=[16, 13],
                    help="13: packed 13-bit code strips (SURVEY f3(ii), 19%% fewer code bytes)")
    ap.add_argument("--shared-kv", action="store_true",
                    help="one selection per KV head shared by its GQA heads (R8, SURVEY f3(iii))")
    ap.add_argument("--virtual-shards", type=int, default=0,
                    help="test mode: run config 4's sharded step as R shards on ONE GPU")
    ap.add_argument("--config", type=int, default=None, choices=sorted(CONFIGS),
                    help="default: 3 at N=1 (128K ctx, the metric's single-GPU config), "
                         "4 at N>1 (1M ctx sequence-sharded)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None,
                    help="reduce the layer count L (stated in the workload); config 5 at N=1 needs <= 4")
    ap.add_argument("--no-config5", action="store_true",
                    help="skip the config5_layer sub-record of the default (config 3) run")
    args = ap.parse_args()
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config is None:
        args.config = 3 if world_env == 1 else 4
    cfg = dict(CONFIGS[args.config])
    cfg["lut_bits"] = 8 if args.lut8 else 16
    cfg["vo_only"] = bool(args.vo_only)
    cfg["cpu_gather"] = bool(args.cpu_gather)
    cfg["shared_kv"] = bool(args.shared_kv)
    cfg["code_bits"] = args.code_bits
    sharded_run = world_env > 1 and args.config in (4, 5)  # Eq. 5 inside hc_shard_finish
    hf = args.host_frac if args.host_frac is not None else (
        HOST_FRAC_DEFAULT if cfg["placement"] == 1 and not args.cpu_gather and not sharded_run else 0.0)
    if hf > 0.0 and sharded_run:
        raise SystemExit("--host-frac is for single-GPU host-V runs (the sharded path gathers in hc_shard_finish)")
    cfg["host_frac"] = hf
    pp = args.pipeline if args.pipeline is not None else (
        PIPELINE_DEFAULT if cfg["placement"] == 1 and not args.cpu_gather and not sharded_run
        and cfg["B"] % PIPELINE_DEFAULT == 0 else 1)
    cfg["pipeline"] = pp
    if pp > 1:
        cfg["workload"] += f"; micro-batch pipeline x{pp} (B/{pp} sequences per chain, own stream)"
    if hf > 0.0:
        if cfg["placement"] != 1 or args.cpu_gather:
            raise SystemExit("--host-frac needs host-resident values (e.g. --config 3) and no --cpu-gather")
        cfg["workload"] += ("; heterogeneous Eq. 5: host threads sum the kept rows of the first "
                            "host_frac of the tokens over host DRAM, the GPU pulls the rest zero-copy")
        cfg["host_frac_auto"] = args.host_frac is None
    if args.code_bits == 13:
        cfg["workload"] += "; packed 13-bit codes (f3(ii))"
    if args.shared_kv:
        cfg["workload"] += "; per-KV-head shared selection (R8, f3(iii))"
    if args.cpu_gather:
        if cfg["placement"] != 1:
            raise SystemExit("--cpu-gather needs host-resident values (e.g. --config 3)")
        cfg["workload"] += "; Eq. 5 on host threads from D2H-shipped (idx, w) (paper's CPU part)"
    if args.vo_only:
        cfg["workload"] += "; value-offload-only mode (exact fp16 keys, Table 1a VO row)"
    if args.lut8:
        cfg["workload"] += "; 8-bit table variant (R2b)"
    if args.layers is not None:
        if not 1 <= args.layers <= cfg["L"]:
            raise SystemExit(f"--layers must be in [1, {cfg['L']}]")
        cfg["L"] = args.layers
        cfg["workload"] += f"; L REDUCED to {args.layers} of 32 layers"
    if args.config == 5 and world_env < 4 and not args.impl == "reference" and not (
            args.layers is not None and args.layers <= 4):
        raise SystemExit("config 5 (4M ctx, 275 GB of host-resident values) needs >= 4 ranks "
                         "(python -m torch.distributed.run --nproc-per-node N bench.py --config 5)")
    if args.steps is None:
        args.steps = 500 if args.config in (1, 2) else 20
    if args.warmup is None:
        args.warmup = 10 if args.config in (1, 2) else 3
    if args.virtual_shards:
        run_virtual(args, cfg, args.virtual_shards)
        return
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    backend = os.environ.get("HC_BENCH_BACKEND", "nccl")  # gloo: code-path smoke on one GPU
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    if world > 1:
        import torch.distributed as td
        if backend == "nccl":
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            td.init_process_group(backend)
        dist = td
    torch.cuda.set_device(local)
    dev = "cuda"
    args.warmup = max(args.warmup, 3)
    hc_lib_check()

    sharded_mode = world > 1 and args.config in (4, 5)
    wl = Workload(cfg, dev, rank if sharded_mode else 0, world if sharded_mode else 1)
    if cfg.get("host_frac_auto") and wl.hetero is not None and not wl.parts:
        calibrate_host_frac(wl, cfg)
    shard_path = None
    if sharded_mode:
        import paper_2507_19823_b200 as hc
        from paper_2507_19823_b200.sharded import GpuShard, TorchComm, decode_layer

        class _PhaseShard:  # the phase kernels with torch.distributed collectives between them
            def __init__(self, wl_):
                self.g, self.c, self.wl = GpuShard(wl_.kc, wl_.vs, wl_.bud), TorchComm(), wl_
                self.sel_k = self.g.sel_k

            def decode_layer(self, q, l):
                return decode_layer(self.g, self.c, q, l, self.wl.base)

        if backend == "nccl":
            try:
                wl.enable_sharding(hc.NcclComm.from_process_group(), rank, world)
                shard_path = "hc_decode_attention_sharded (NCCL issued by the library)"
            except Exception as ex:  # fall back to torch's NCCL collectives, and say so
                print(f"[bench] C-ABI NCCL path unavailable ({type(ex).__name__}: {ex}); "
                      "phases with torch.distributed collectives", file=sys.stderr, flush=True)
                wl.shard = _PhaseShard(wl)
                shard_path = "hc_shard_* phases + torch.distributed NCCL collectives (fallback)"
        else:  # HC_BENCH_BACKEND=gloo code-path smoke on one GPU: the phases with gloo collectives
            wl.shard = _PhaseShard(wl)
            shard_path = "hc_shard_* phases + gloo collectives (code-path smoke)"
    torch.cuda.synchronize()
    # eager correctness sanity (one step) then capture the step with scan events
    wl.reset_counts()
    try:
        wl.step()
        torch.cuda.synchronize()
    except Exception as ex:
        if not (sharded_mode and backend == "nccl" and shard_path and "library" in shard_path):
            raise
        # the C-ABI NCCL path failed at run time: the phases with torch's collectives, and say so
        print(f"[bench] C-ABI NCCL step failed ({type(ex).__name__}: {ex}); phases with "
              "torch.distributed collectives", file=sys.stderr, flush=True)
        wl.shard = _PhaseShard(wl)
        shard_path = "hc_shard_* phases + torch.distributed NCCL collectives (fallback)"
        wl.reset_counts()
        wl.step()
        torch.cuda.synchronize()
    graph_mode = "one CUDA graph per step (32 x append + decode)"
    try:
        # the timed graph carries no event nodes (64 per step cost ~0.3 ms at config 2); the
        # scan's launch times come from an identical graph with events, replayed afterwards
        g_step, launches_per_step = wl.capture(wl.step)
        g_prof, _ = wl.capture(lambda: wl.step(profile=True))
        g_e2e, _ = wl.capture(wl.step_e2e)
    except Exception as ex:  # e.g. a collective backend that refuses graph capture
        if not sharded_mode:
            raise
        torch.cuda.synchronize()
        graph_mode = f"eager steps (graph capture failed: {type(ex).__name__})"
        g_step, launches_per_step = EagerStep(wl, wl.step), None
        g_prof = EagerStep(wl, lambda: wl.step(profile=True))
        g_e2e = EagerStep(wl, wl.step_e2e)
        import paper_2507_19823_b200 as hc
        before = hc.launch_count()
        g_step.replay()
        torch.cuda.synchronize()
        launches_per_step = hc.launch_count() - before

    with ClockSampler(local) as clk:
        ms = time_graph(g_step, args.steps, args.warmup, dist)
    ms_per_step = ms / args.steps
    if wl.hetero is not None:
        wl.hetero.check()  # a timed-out host share would have poisoned the outputs: refuse the number
    for _ in range(3):  # the profiled twin of the timed graph; events of its last replay
        g_prof.replay()
    torch.cuda.synchronize()
    scan_ms = [event_ms(b, e) for (b, e) in wl.ev]
    scan_avg_ms = statistics.mean(scan_ms)
    if os.environ.get("HC_BENCH_DEBUG"):
        print("scan_ms per layer:", [round(x, 4) for x in scan_ms], file=sys.stderr)
    eq3_avg_ms = statistics.mean(event_ms(b, e) for (b, e) in wl.ev3)
    K2 = args.e2e_steps or max(args.steps // 2, 3)
    ms_e2e = time_graph(g_e2e, K2, args.warmup, dist) / K2

    B, L, H, g, n, d = (cfg[k] for k in ("B", "L", "Hkv", "g", "n", "d"))
    n_here = wl.n_local
    Bs = B // cfg.get("pipeline", 1)  # the profiled scan covers one micro-batch
    p_bytes_layer = Bs * H * n_here * (d if wl.vo_only else g) * 2  # exact K rows in VO-only mode
    if cfg.get("code_bits", 16) == 13 and not wl.vo_only:
        p_bytes_layer = Bs * H * n_here * g * 13 // 8  # packed code strips
    achieved = p_bytes_layer / (scan_avg_ms * 1e-3) / 1e9
    peak, peak_src = measured_peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"scan_traffic_config{args.config}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    ksel = wl.sel_k.float().mean().item()
    jobs = 1 if sharded_mode else world  # replicas multiply the work, shards split it
    value = jobs * 1000.0 / ms_per_step
    # value-gather bytes (all layers, all heads, this rank's share) and the host-link peak
    v_bytes = ksel * B * wl.Hq * L * d * 2 / (world if sharded_mode else 1)
    host_link = None
    host_dram = None
    pk = measure_h2d_gbs() if cfg["placement"] == 1 else None
    gpu_only = None
    if cfg["placement"] == 1:
        if not wl.cpu_gather and world == 1:
            if wl.hetero is not None:  # the host's share of the rows stays in host DRAM
                v_bytes, h_bytes = union_gather_bytes(wl, cfg["host_frac"])
                mem = measure_host_rows_gbs(wl)
                hw = measure_host_dram_hw(wl)
                pk_eng = max(mem["combined"], mem["host_alone"], mem["gpu_alone"])
                pk_mem = hw["peak_gbs"]
                both = (h_bytes + v_bytes) / (ms_per_step * 1e-3) / 1e9
                host_dram = {"bytes_per_step": h_bytes, "rows": "union of the GQA heads' kept rows, "
                             "index < t_split", "achieved_gbs_lower_bound": h_bytes / (ms_per_step * 1e-3) / 1e9,
                             "host_frac": cfg["host_frac"], "threads": wl.hetero.threads,
                             # both consumers (host threads + the GPU's zero-copy pulls) read the
                             # same host DRAM: their sum against the hardware's random-row rate
                             "all_row_bytes_gbs": both, "peak_gbs": pk_mem,
                             "peak_source": "engine-free all-core random 256-B row reads of the value "
                                            "store's pinned memory (tools/membench.c); see hw",
                             "frac": both / pk_mem if pk_mem else None,
                             "hw": hw,
                             # what Eq. 5 itself reaches alone on this box (our engines), kept apart
                             "engine_capability_gbs": pk_eng, "engine_parts": mem,
                             "frac_of_engine_capability": both / pk_eng if pk_eng else None}
                gpu_only = measure_gpu_only(wl, args, local, pk)
            else:
                v_bytes = union_gather_bytes(wl)  # rows actually read: union over the GQA heads
        host_link = {"bytes_per_step": v_bytes, "rows": "union of the GQA heads' kept rows",
                     "achieved_gbs_lower_bound": v_bytes / (ms_per_step * 1e-3) / 1e9,
                     "peak_gbs": pk, "peak_source": "measured pinned H2D cudaMemcpy 1 GiB",
                     "frac": v_bytes / (ms_per_step * 1e-3) / 1e9 / pk,
                     "note": "zero-copy reads of only the selected value rows; whole step time in the denominator"}
    h2d = (wl.q.numel() + wl.k_new.numel() + wl.v_new.numel()) * 2
    d2h = wl.out.numel() * 4
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if sharded_mode else "weak", "vs_baseline": None,
        "dtype": "i8+f32" if cfg.get("lut_bits") == 8 else "i16+f32", "data": "synthetic (seeded splitmix64; codes uniform, C,q,V ~ Irwin-Hall normal)",
        "config": {"workload": cfg["workload"],
                   "parallelism": (f"sequence-sharded x{world}" if sharded_mode else
                                   ("replicas" if world > 1 else "single")),
                   "l2": f"inputs > L2: P = {B * L * H * n * g * 2 / 1e9:.2f} GB/step, V = "
                         f"{B * L * H * n * d * 2 / 1e9:.2f} GB",
                   "graph": graph_mode,
                   **({"shard_path": shard_path} if shard_path else {}),
                   **({"host_frac": round(cfg["host_frac"], 2),
                       "host_frac_from": "calibrated at start-up" if cfg.get("host_frac_auto") else "--host-frac"}
                      if cfg["host_frac"] > 0.0 else {})},
        "quantized_key_gbs": achieved,
        "quantized_key_frac_hbm": achieved / peak,
        # the whole Eq. 3 stage the scan needs: table build (row a1) + scan, same bytes
        "eq3_stage": {"kernels": "k_table + k_scan_sk (hc_table.cu, hc_scan.cu)",
                      "avg_ms_per_layer": eq3_avg_ms, "scan_ms": scan_avg_ms,
                      "table_and_launch_gap_ms": eq3_avg_ms - scan_avg_ms,
                      "achieved_gbs": p_bytes_layer / (eq3_avg_ms * 1e-3) / 1e9,
                      "frac_hbm": p_bytes_layer / (eq3_avg_ms * 1e-3) / 1e9 / peak},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("k_resident (exact-key dense scan, VO-only mode)" if wl.vo_only
                                else "Eq. 3 quantized-key scan: k_scan_sk (stream-K) when every CTA gets "
                                     ">= 2 tiles, else k_scan_pipe / k_scan8_pipe (hc_scan.cu)"),
                     "algorithmic_bytes_per_launch": p_bytes_layer,
                     "avg_launch_ms": scan_avg_ms, "share_of_step": scan_avg_ms * L * cfg.get("pipeline", 1) / ms_per_step,
                     "peak_source": peak_src,
                     # the binding on-chip resource: random table lookups in shared
                     # memory, measured alone by tools/smem_gather_micro.cu on a B200
                     "smem_gather_ceiling": SMEM_CEILING.get(8 if cfg.get("lut_bits", 16) == 16 else 4),
                     "dominant_kernel": (("Eq. 5 over host-resident values: host worker threads + "
                                          "k_gather_union, bound by host DRAM's random-row rate (see host_dram; "
                                          "profiles/r01_launches_config3_hetero_summary.md)")
                                         if host_dram is not None else
                                         "k_gather_union (zero-copy value gather, bound by the host link: see "
                                         "host_link; profiles/r01_launches_config3_summary.md)"
                                         if host_link is not None else
                                         "scan / select / gather share the step (see DESIGN.md §5)")},
        "selection": {"mean_k_sel": ksel, "k_sel_over_n": ksel / n},
        "host_link": host_link,
        "host_dram": host_dram,
        "gpu_only": gpu_only,
        "e2e": {"value": jobs * 1000.0 / ms_e2e, "unit": "steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e},
        "gpu_launches": launches_per_step * args.steps,
        "gpu_launches_per_step": launches_per_step,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if world == 1 and args.config == 3 and not args.no_config5 and args.layers is None:
        # one-GPU timing of the paper's 4M-token headline configuration: the
        # config-3 state is released first (its 34 GB of pinned values)
        import gc
        g_step = g_prof = g_e2e = None
        if wl.hetero is not None and wl.hetero.mode == "doorbell":
            wl.hetero.worker.close()
        if wl.vs.host is not None:
            wl.vs.host.close()
        del wl
        gc.collect()
        torch.cuda.empty_cache()
        try:
            line["config5_layer"] = measure_config5_layers(args, 1, local, pk or measure_h2d_gbs(),
                                                           host_frac=float(cfg.get("host_frac") or 0.0))
        except Exception as ex:  # report, never silently drop
            line["config5_layer"] = {"error": f"{type(ex).__name__}: {ex}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
