"""Heterogeneous Eq. 5 for host-resident values (§3.2 "Heterogeneous Attention
Computation"; DESIGN §8b f1): after the GPU selection (rows a1-a4), the kept
value rows are summed by BOTH processors at once, split by token index at t_split:

  host (side stream): D2H of (idx, w, k), then hc_enqueue_host_weighted_sum_range over kept
       tokens j < t_split -- the paper's CPU part, host threads over host DRAM;
  GPU  (main stream): hc_gather_values over kept tokens j >= t_split -- zero-copy pulls of
       only those rows over the host link (GQA union read once), plus the resident window
       tokens (global indices n_q.., exact values in HBM);
  join: hc_add_partial(out, host share) on the main stream.

The two shares use different links (PCIe H2D for the GPU's row pulls; the host's own DRAM
channels for its share, plus the small D2H of the selection), so their throughputs add.
host_frac = share of the quantized token range [0, n_q) the host owns (t_split =
round(host_frac * n_q)); 0 = all on the GPU, 1 = the paper's split (the host sums every
offloaded row).  Everything is stream-ordered and graph-capturable; the
orchestration here is argument marshalling and stream plumbing only.
"""
from __future__ import annotations

import os

import paper_2507_19823_b200 as hc


class HeteroEq5:
    def __init__(self, kc: "hc.KCache", vstore: "hc.VStore", k_max: int, host_frac: float,
                 threads: int = 0, device="cuda", mode: str = "doorbell", worker=None):
        import torch
        if vstore.placement != hc.HC_V_HOST_MAPPED:
            raise ValueError("the heterogeneous split needs host-resident values (HC_V_HOST_MAPPED)")
        if not (0.0 <= host_frac <= 1.0):
            raise ValueError("host_frac must be in [0, 1]")
        self.kc, self.vs, self.k_max = kc, vstore, int(k_max)
        # default: all cores (the driving thread should wait on blocking-sync events, not spin)
        self.host_frac = float(host_frac)
        self.threads = int(threads) if threads > 0 else int(os.environ.get("HC_HOST_THREADS", os.cpu_count() or 1))
        rows = kc.B * kc.Hq
        self.idx_d = torch.empty((rows, self.k_max), dtype=torch.int32, device=device)
        self.w_d = torch.empty((rows, self.k_max), dtype=torch.float32, device=device)
        self.idx_h = torch.empty((rows, self.k_max), dtype=torch.int32).pin_memory()
        self.w_h = torch.empty((rows, self.k_max), dtype=torch.float32).pin_memory()
        self.k_h = torch.empty((rows,), dtype=torch.int64).pin_memory()
        self.part_h = torch.zeros((rows, kc.d), dtype=torch.float32).pin_memory()
        # high priority: the staging kernel must not queue behind the GPU share's gather grid
        self.side = torch.cuda.Stream(device=device, priority=-1)
        # "doorbell": a persistent host worker polls a mailbox rung by a GPU kernel (the
        # selection is copied by that kernel, only the host's share); "hostnode": D2H copies
        # + a graph host node (cudaLaunchHostFunc, ~250 us round trip per layer)
        if mode not in ("doorbell", "hostnode"):
            raise ValueError("mode must be doorbell or hostnode")
        self.mode = mode
        if mode == "doorbell":
            # several instances (e.g. micro-batch chains) may share one worker: its jobs then
            # run one after another with the whole host team
            self.worker = worker if worker is not None else hc.HostWorker(threads=self.threads)
            self.job = self.worker.add_job(rows, self.k_max, vstore, kc.G, self.part_h)
        self.ev_sel = torch.cuda.Event()
        self.ev_host = torch.cuda.Event()
        self.ev_staged = torch.cuda.Event()
        self.stage_first = os.environ.get("HC_STAGE_FIRST", "1") != "0"

    def check(self):
        """Raise if a host share timed out (its output was poisoned with NaN by the wait
        kernel); call after synchronizing."""
        if self.mode == "doorbell":
            st = self.worker.status()
            if st != hc.HC_OK:
                raise hc.HcError(st, "host worker: a host share of Eq. 5 timed out (output poisoned)")

    def split_point(self, layer: int) -> int:
        return int(round(self.host_frac * self.kc.n_q(layer)))

    def __call__(self, q, layer: int, bud: "hc.hc_budget", out, sel_k, ws: "hc.Workspace"):
        """One layer: q [B][Hq][d] fp16 -> out [B][Hq][d] fp32; sel_k [B][Hq] int64 (device)."""
        import torch
        main = torch.cuda.current_stream()
        sel_bud = hc.budget(bud.tau, bud.k_max, renorm=bool(bud.renorm), select_only=True,
                            shared_kv=bool(bud.shared_kv))
        hc.decode_attention(q, self.kc, self.vs, layer, sel_bud, out=out, sel_idx=self.idx_d,
                            sel_w=self.w_d, sel_k=sel_k, ws=ws)
        n_cand = self.kc.n_q(layer) + self.kc.n_res(layer)
        t_split = self.split_point(layer)
        host = t_split > 0
        if host:
            self.ev_sel.record(main)
            self.side.wait_event(self.ev_sel)
            with torch.cuda.stream(self.side):
                if self.mode == "doorbell":
                    B_, L_, Hkv_, ncap_, d_ = self.vs.tensor.shape
                    self.worker.submit(self.job, self.idx_d, self.w_d, sel_k, t_split,
                                       layer * Hkv_ * ncap_ * d_, stream=self.side,
                                       n_valid=self.kc.n_q(layer))
                    self.ev_staged.record(self.side)
                    self.worker.wait(self.job, stream=self.side)
                else:
                    self.idx_h.copy_(self.idx_d, non_blocking=True)
                    self.w_h.copy_(self.w_d, non_blocking=True)
                    self.k_h.copy_(sel_k.view(-1), non_blocking=True)
                    hc.host_weighted_sum_range(self.idx_h, self.w_h, self.k_h, self.vs, layer, self.kc.G,
                                               0, t_split, self.part_h, self.threads, stream=self.side,
                                               n_valid=self.kc.n_q(layer))
                self.ev_host.record(self.side)
        if host and self.mode == "doorbell" and self.stage_first:
            # the GPU's pull starts once the host's lists are staged: side by side, the gather's
            # grid and PCIe reads starve the staging kernel (0.26 -> 2.8 ms, tools/staging_timing.py)
            main.wait_event(self.ev_staged)
        hc.gather_values(self.kc, self.vs, layer, self.idx_d, self.w_d, sel_k, t_split, n_cand, out, ws)
        if host:
            main.wait_event(self.ev_host)
            hc.add_partial(out, self.part_h)
        return out
