"""Per-layer decode timing of config 2 (1 layer) for HC_SEL_STOP values (dev tool)."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CFG = int(os.environ.get("PT_CONFIG", "2"))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import bench
    cfg = dict(bench.CONFIGS[CFG]); cfg["L"] = 2
    cfg["shared_kv"] = os.environ.get("PT_SHARED", "0") == "1"
    reps = int(os.environ.get("PT_REPS", "200" if CFG == 2 else "20"))
    wl = bench.Workload(cfg, "cuda")
    import paper_2507_19823_b200 as hc
    for _ in range(5):
        hc.decode_attention(wl.q[1], wl.kc, wl.vs, 1, wl.bud, out=wl.out[1], ws=wl.ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        hc.decode_attention(wl.q[1], wl.kc, wl.vs, 1, wl.bud, out=wl.out[1], ws=wl.ws)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"stop": os.environ.get("HC_SEL_STOP", "0"), "us_per_layer": e0.elapsed_time(e1) / reps * 1000}))
else:
    for st in os.environ.get("PT_STOPS", "1,2,3,4,5,0").split(","):
        env = dict(os.environ, HC_SEL_STOP=st)
        out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-2000:])
