"""Per-phase timing of the sequence-sharded protocol kernels (R shards on one GPU in lock-step,
collectives as tensor reductions) -- dev tool.  PT_CONFIG (default 4), PT_R (default 1)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2507_19823_b200.sharded import GpuShard
    cfg = dict(bench.CONFIGS[int(os.environ.get("PT_CONFIG", "4"))])
    cfg["L"] = 2
    R = int(os.environ.get("PT_R", "1"))
    wls = [bench.Workload(cfg, "cuda", r, R) for r in range(R)]
    shards = [GpuShard(w.kc, w.vs, w.bud) for w in wls]
    bases = [w.base for w in wls]
    q = wls[0].q[1]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    tot = [0.0] * 5
    reps = 10
    for it in range(reps + 3):
        ev[0].record()
        st = torch.stack([s.begin(q, 1) for s in shards]).amax(0)
        ev[1].record()
        h1 = torch.stack([s.hist1(1, st) for s in shards]).sum(0)
        ev[2].record()
        h2 = torch.stack([s.hist2(1, st, h1) for s in shards]).sum(0)
        ev[3].record()
        allc = torch.stack([s.counts(1, h2) for s in shards])
        ev[4].record()
        outs = [s.finish(1, allc, r, R, bases[r]) for r, s in enumerate(shards)]
        torch.stack(outs).sum(0)
        ev[5].record()
        torch.cuda.synchronize()
        if it >= 3:
            for k in range(5):
                tot[k] += ev[k].elapsed_time(ev[k + 1]) * 1000 / reps
    print(json.dumps({"R": R, "us": dict(zip(["begin", "hist1", "hist2", "counts", "finish"], tot)),
                      "total_us": sum(tot)}))


if __name__ == "__main__":
    main()
