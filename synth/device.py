"""Device generation of the large synthetic tensors (codes P, values V) with the
same counter streams as synth/__init__.py (bit-identical).  Input generation only."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import TAG_P, TAG_V, stream_key

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "synth.cu")
LIB = os.path.join(HERE, "libhcsynth.so")
_lib = None


def build(force=False):
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-o", LIB + ".tmp", SRC])
        os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.synth_codes.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_uint32, C.c_int64, C.c_void_p]
        L.synth_values.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                   C.c_int, C.c_int64, C.c_void_p]
        _lib = L
    return _lib


def _keys(seed, tag, shape_prefix, extra):
    ks = []
    for idx in np.ndindex(*shape_prefix):
        ks.append(stream_key(seed, tag, *idx, *extra) if extra else stream_key(seed, tag, *idx))
    return np.array(ks, dtype=np.uint64)


def fill_codes(codes, seed: int, c: int, n: int, layers=None, start: int = 0, layer_ids=None):
    """codes: torch int16 cuda [B][L][Hkv][g][n_cap]; fill local positions [0, n) of the given
    layers (default all) with synth.gen_codes streams of GLOBAL positions [start, start+n).
    layer_ids: the stream's layer index per filled slot (default: the slot index)."""
    import torch
    B, L, H, g, ncap = codes.shape
    layers = list(range(L) if layers is None else layers)
    ids = layers if layer_ids is None else list(layer_ids)
    s = torch.cuda.current_stream().cuda_stream
    for l, lid in zip(layers, ids):
        keys = np.array([stream_key(seed, TAG_P, b, lid, kv, i)
                         for b in range(B) for kv in range(H) for i in range(g)], dtype=np.uint64)
        kt = torch.from_numpy(keys.view(np.int64)).to(codes.device)
        for b in range(B):
            sub = codes[b, l]  # [H][g][ncap] contiguous
            r = lib().synth_codes(C.c_void_p(sub.data_ptr()),
                                  C.c_void_p(kt.data_ptr() + b * H * g * 8), H * g, ncap, n, c,
                                  start, C.c_void_p(s))
            if r:
                raise RuntimeError(f"synth_codes failed: {r}")
        torch.cuda.current_stream().synchronize()


def fill_values(vt, seed: int, n: int, layers=None, device="cuda", start: int = 0):
    """vt: torch fp16 [B][L][Hkv][n_cap][d] (cuda or pinned host, UVA pointer); local rows
    [0, n) <- GLOBAL rows [start, start+n)."""
    import torch
    B, L, H, ncap, d = vt.shape
    layers = range(L) if layers is None else layers
    s = torch.cuda.current_stream().cuda_stream
    for l in layers:
        keys = np.array([stream_key(seed, TAG_V, b, l, kv) for b in range(B) for kv in range(H)],
                        dtype=np.uint64)
        kt = torch.from_numpy(keys.view(np.int64)).to(device)
        for b in range(B):
            sub = vt[b, l]
            r = lib().synth_values(C.c_void_p(sub.data_ptr()), C.c_void_p(kt.data_ptr() + b * H * 8),
                                   H, ncap * d, n, d, start, C.c_void_p(s))
            if r:
                raise RuntimeError(f"synth_values failed: {r}")
        torch.cuda.current_stream().synchronize()
