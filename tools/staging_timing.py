"""k_submit (staging of the host's share of the selection) timed alone and next to the GPU
share's gather, config 3 layer 0.  Usage: python tools/staging_timing.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    import paper_2507_19823_b200 as hc
    cfg = dict(bench.CONFIGS[3])
    cfg.update(lut_bits=16, vo_only=False, cpu_gather=False, shared_kv=False, code_bits=16,
               host_frac=0.65, pipeline=1)
    cfg["L"] = 2
    torch.cuda.set_device(0)
    wl = bench.Workload(cfg, "cuda", 0, 1)
    het = wl.hetero
    bud = hc.budget(cfg["tau"], cfg["k_max"], select_only=True)
    sel_k = torch.zeros((cfg["B"], wl.Hq), dtype=torch.int64, device="cuda")
    hc.decode_attention(wl.q[0], wl.kc, wl.vs, 0, bud, out=wl.out[0], sel_idx=het.idx_d, sel_w=het.w_d,
                        sel_k=sel_k, ws=wl.ws)
    torch.cuda.synchronize()
    n = wl.kc.n_q(0)
    t_split = int(round(0.65 * n))
    s1 = torch.cuda.Stream()
    s2 = torch.cuda.Stream()
    out = torch.empty_like(wl.out[0])
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for mode in ("alone", "with_gather", "alone"):
        for _ in range(3):
            torch.cuda.synchronize()
            with torch.cuda.stream(s1):
                e[0].record()
                het.worker.submit(het.job, het.idx_d, het.w_d, sel_k, t_split, 0, n_valid=het.kc.n_q(0))
                e[1].record()
            if mode == "with_gather":
                with torch.cuda.stream(s2):
                    e[2].record()
                    hc.gather_values(wl.kc, wl.vs, 0, het.idx_d, het.w_d, sel_k, t_split, n, out, wl.ws)
                    e[3].record()
            with torch.cuda.stream(s1):
                het.worker.wait(het.job)
            torch.cuda.synchronize()
        line = f"{mode}: k_submit {e[0].elapsed_time(e[1]) * 1000:.1f} us"
        if mode == "with_gather":
            line += f", gather {e[2].elapsed_time(e[3]) * 1000:.1f} us"
        print(line, flush=True)


if __name__ == "__main__":
    main()
