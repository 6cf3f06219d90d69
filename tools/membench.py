"""Engine-free host DRAM bandwidth (tools/membench.c) and host topology, for bench.py's
host_dram.peak: random 256-B rows (the value-row size at d = 128, fp16) and a sequential
read, on all host cores, over a given (pinned) host buffer.  Measurement only."""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "membench.c")
LIB = os.path.join(HERE, "libmembench.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", "-o", LIB + ".tmp", SRC])
        os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.hm_random_rows.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                     C.POINTER(C.c_uint64)]
        L.hm_random_rows.restype = C.c_double
        L.hm_sequential.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]
        L.hm_sorted_rows.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint32, C.c_int,
                                     C.POINTER(C.c_uint64)]
        L.hm_sorted_rows.restype = C.c_double
        L.hm_sequential.restype = C.c_double
        _lib = L
    return _lib


def host_topology() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    nodes = {}
    for p in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        try:
            with open(os.path.join(p, "cpulist")) as f:
                cpus = f.read().strip()
            mem_kb = None
            with open(os.path.join(p, "meminfo")) as f:
                for line in f:
                    if "MemTotal" in line:
                        mem_kb = int(line.split()[-2])
            nodes[os.path.basename(p)] = {"cpus": cpus, "mem_gb": round(mem_kb / 2**20, 1) if mem_kb else None}
        except OSError:
            continue
    return {"cpu_model": model, "logical_cpus": os.cpu_count(),
            "affinity_cpus": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
            "numa_nodes": nodes}


def measure(ptr: int, nbytes: int, threads: int | None = None, row_bytes: int = 256,
            rows_per_thread: int = 1 << 20, batch: int = 16, reps: int = 3, sorted_stride: int = 8) -> dict:
    """Best-of-reps GB/s of random `row_bytes` rows and of one sequential pass (capped at
    16 GiB) over [ptr, ptr + nbytes), on `threads` threads (default: all usable cores)."""
    L = lib()
    thr = threads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
    sink = C.c_uint64()
    rnd = max(L.hm_random_rows(C.c_void_p(ptr), nbytes, row_bytes, rows_per_thread, thr, batch,
                               C.byref(sink)) for _ in range(reps))
    seq_bytes = min(nbytes, 16 << 30)
    seq = max(L.hm_sequential(C.c_void_p(ptr), seq_bytes, thr, C.byref(sink)) for _ in range(reps))
    srt = max(L.hm_sorted_rows(C.c_void_p(ptr), nbytes, row_bytes, sorted_stride, thr, C.byref(sink))
              for _ in range(reps))
    return {"random_rows_gbs": rnd, "sorted_rows_gbs": srt, "sorted_rows_density": 1.0 / sorted_stride,
            "sequential_gbs": seq, "peak_gbs": max(rnd, srt, seq), "threads": thr, "row_bytes": row_bytes,
            "rows_in_flight_per_thread": batch, "buffer_gb": nbytes / 1e9,
            "how": "tools/membench.c, all host threads, over the value store's own pinned memory, no "
                   "Eq. 5 arithmetic (uint64 sums of the bytes read): uniformly random 256-B rows (16 "
                   "prefetched per thread); a sorted random subset of rows at density 1/%d (the kept "
                   "lists' shape); one sequential pass; best of %d each; peak = the best of the three"
                   % (sorted_stride, reps),
            **host_topology()}
