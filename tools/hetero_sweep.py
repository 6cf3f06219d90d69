"""Sweep the heterogeneous Eq. 5 split on the config-3 workload (128K ctx, B=4, host V):
steps/s of the captured 32-layer step for each (micro-batch pipeline depth, host_frac).
Usage: python tools/hetero_sweep.py [fracs] [pipelines]
e.g. python tools/hetero_sweep.py 0.5,0.6,0.7 1,2,4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    from paper_2507_19823_b200.hetero import HeteroEq5
    fracs = [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0.6,0.7,0.8").split(",")]
    pipes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1").split(",")]
    torch.cuda.set_device(0)
    for P in pipes:
        cfg = dict(bench.CONFIGS[3])
        cfg.update(lut_bits=16, vo_only=False, cpu_gather=False, shared_kv=False, code_bits=16,
                   host_frac=0.5, pipeline=P)
        wl = bench.Workload(cfg, "cuda", 0, 1)
        for f in fracs:
            if P == 1:
                wl.hetero = HeteroEq5(wl.kc, wl.vs, cfg["k_max"], f) if f > 0 else None
            import paper_2507_19823_b200 as hc
            shw = hc.HostWorker(threads=os.cpu_count() or 1) if (f > 0 and wl.parts) else None
            for part in wl.parts:
                part["het"] = HeteroEq5(part["kc"], part["vs"], cfg["k_max"], f, worker=shw) if f > 0 else None
            wl.reset_counts()
            wl.step()
            torch.cuda.synchronize()
            g, _ = wl.capture(wl.step)
            ms = bench.time_graph(g, 5, 2) / 5
            print(f"pipeline={P} host_frac={f:.2f}: {ms:.1f} ms/step = {1000 / ms:.2f} steps/s", flush=True)
            del g
            if wl.hetero is not None and getattr(wl.hetero, "worker", None) is not None:
                wl.hetero.worker.close()  # prints HC_WORKER_STATS
        del wl
        import gc
        gc.collect()


if __name__ == "__main__":
    main()
