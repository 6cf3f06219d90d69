"""Prefill-side throughput (NEXT f4): bulk key encoding (hc_quantize_keys, many rows) and one
MiniBatchKMeans step at the paper's batch size, timed with CUDA events.
ALU roofline: (2·dbar + 3) lane-ops per (row, group, centroid) -> dbar=4: 11 ops; peak =
148 SMs x 128 FP32 lanes x 1.965 GHz = 37.2 T lane-ops/s (B200_PROFILING.md unit counts)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2507_19823_b200 as hc
    rows, d, g, c = int(os.environ.get("PF_ROWS", 131072)), 128, 32, 8192
    dbar = d // g
    torch.manual_seed(0)
    keys = torch.randn((rows, d), device="cuda").half()
    C = torch.randn((g, c, dbar), device="cuda")
    codes = torch.empty((g, rows), dtype=torch.int16, device="cuda")
    for _ in range(3):
        hc.quantize_keys(keys, C, g, codes=codes)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        hc.quantize_keys(keys, C, g, codes=codes)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ops = rows * g * c * (2 * dbar + 3)
    peak = 148 * 128 * 1.965e9
    enc = {"what": "bulk encode", "rows": rows, "d": d, "g": g, "c": c, "ms": ms,
           "keys_per_s": rows / ms * 1e3, "lane_ops_per_s": ops / ms * 1e3,
           "alu_frac": ops / ms * 1e3 / peak, "flops_3dc": 3.0 * d * c * rows / ms * 1e3}
    b = 10000
    counts = torch.zeros((g, c), dtype=torch.int64, device="cuda")
    sample = torch.randint(0, rows, (b,), device="cuda", dtype=torch.int64)
    ws = hc.Workspace(int(hc.lib().hc_kmeans_workspace_bytes(hc.hc_vq(d, g, c, g), b)), "cuda")
    for _ in range(3):
        hc.kmeans_step(keys, sample, C, counts, g, ws=ws)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        hc.kmeans_step(keys, sample, C, counts, g, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    km = {"what": "kmeans step", "batch": b, "ms": e0.elapsed_time(e1) / reps,
          "iters_200_s": e0.elapsed_time(e1) / reps * 200 / 1e3}
    # App. B block-wise prefill attention, one Llama-3-8B layer (32 q heads, 8 KV heads)
    n, Hq, Hkv, bs = int(os.environ.get("PF_N", 131072)), 32, 8, int(os.environ.get("PF_BS", 4096))
    q = torch.randn((n, Hq, d), device="cuda").half() * 0.5
    k = torch.randn((n, Hkv, d), device="cuda").half() * 0.5
    v = torch.randn((n, Hkv, d), device="cuda").half()
    out = torch.empty((n, Hq, d), device="cuda")
    for _ in range(2):
        hc.blockwise_attention(q, k, v, bs, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        hc.blockwise_attention(q, k, v, bs, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    keys = 0  # visited (query, key) pairs of one head, causal within blocks
    for i0 in range(0, n, 64):
        kb = i0 // bs
        keys += 64 * ((bs if kb else 0) + (i0 + 64 - kb * bs))
    flops = 4.0 * d * keys * Hq  # QK^T and PV, 2 flops per MAC
    att = {"what": "blockwise attention (App. B)", "n": n, "bs": bs, "Hq": Hq, "Hkv": Hkv, "ms": ms,
           "tflops": flops / ms / 1e9, "frac_of_dense_bf16_2250": flops / ms / 1e9 / 2250.0}
    print(json.dumps(enc))
    print(json.dumps(km))
    print(json.dumps(att))


if __name__ == "__main__":
    main()
