"""Throughput of the host-side Eq. 5 engine (hc_host_weighted_sum_range) on one layer of the
config-3 shape: B=4, Hkv=8, G=4, n=128K, d=128, k_max=16384 kept rows per query head
(independent uniform selections), values in (pinned, if CUDA is present) host memory.
Prints per-head and GQA-union row bytes per second.  Usage: python tools/host_eq5_micro.py [threads]"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_19823_b200 as hc  # noqa: E402


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    B, Hkv, G, d, n, km = 4, 8, 4, 128, 131072, 16384
    Hq, rows = Hkv * G, B * Hkv * G
    rng = np.random.default_rng(0)
    try:
        import torch
        pinned = torch.cuda.is_available()
    except Exception:
        pinned = False
    Lv = int(os.environ.get("LAYERS", "1"))  # value-store layers (32 = the full config-3 store, 34 GB)
    huge = os.environ.get("HUGE", "0") == "1"
    if pinned and huge:
        hb = hc.HostBuffer(B * Lv * Hkv * n * d * 2)
        Vall = hb.tensor((B, Lv, Hkv, n, d), torch.float16).numpy()
        print(f"HostBuffer: madvise(MADV_HUGEPAGE) ok={hb.huge}, dev==host: {hb.dev == hb.addr}")
    elif pinned:
        Vall = torch.empty((B, Lv, Hkv, n, d), dtype=torch.float16, pin_memory=True).numpy()
    else:
        Vall = np.empty((B, Lv, Hkv, n, d), np.float16)
    V = Vall[:, Lv // 2]
    V[...] = rng.standard_normal((1, 1, n, d)).astype(np.float16)
    idx = np.empty((rows, km), np.int32)
    for r in range(rows):
        idx[r] = np.sort(rng.choice(n, size=km, replace=False))
    w = np.full((rows, km), 1.0 / km, np.float32)
    k = np.full(rows, km, np.int64)
    out = np.zeros((rows, d), np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    union = sum(len(np.unique(idx[u * G:(u + 1) * G])) for u in range(B * Hkv))
    res = {}
    for frac in [float(x) for x in os.environ.get("FRACS", "1.0,0.35").split(",")]:
        t0 = int(round((1 - frac) * n))
        ts = []
        for it in range(6):
            a = time.perf_counter()
            st = hc.lib().hc_host_weighted_sum_range(p(idx), p(w), p(k), rows, km, p(V.view(np.uint16)),
                                                    Lv * Hkv * n * d, n * d, n, Hq, G, d, t0, n, p(out), threads)
            ts.append(time.perf_counter() - a)
            assert st == 0
        t = float(np.median(ts[1:]))
        res[frac] = t
        print(f"host share {frac:.2f}: {t * 1e3:.2f} ms/layer; per-head rows {rows * km * d * 2 * frac / t / 1e9:.1f} GB/s,"
              f" union rows {union * d * 2 * frac / t / 1e9:.1f} GB/s (pinned={pinned}, threads={threads or os.cpu_count()})")


if __name__ == "__main__":
    main()
