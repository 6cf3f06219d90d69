"""Seeded, counter-based synthetic input generators (shared by tests, smoke, bench).

This module holds NONE of the method's arithmetic (no encode, no table, no
scores, no softmax, no selection, no weighted sum).  It only draws inputs.
It is the one module both the CPU oracle (`oracle/`) and the CUDA path
(`paper_2507_19823_b200/`) are fed from, as DESIGN.md §"Input recipe" states.

Generator ("Counter-based generator"):
  fin(z)            = splitmix64 finaliser:
                        z ^= z >> 30; z *= 0xBF58476D1CE4E5B9
                        z ^= z >> 27; z *= 0x94D049BB133111EB
                        z ^= z >> 31
  key(seed, t1..tk) = k0 = fin(seed + GOLDEN); k_{i} = fin((k_{i-1} ^ t_i) + GOLDEN)
  u64(key, j)       = fin(key + (j + 1) * GOLDEN)          (mod 2^64)
  code(u, c)        = ((u >> 32) * c) >> 32                 in [0, c)
  ih4(u)            = sum of the four 16-bit fields of u - 131070   (Irwin-Hall(4),
                      integer in [-131070, 131070], std = sqrt((2^32-1)/3) = 37837.23)
  v16(u)            = fp16_RN( fp32(ih4(u) * 2^-15) )       (exact fp32, one RN to fp16)

The large device-resident tensors (codes P, values V) use only integer
arithmetic plus one IEEE fp32->fp16 round, so `synth/synth.cu` (device) and
this numpy version produce bit-identical tensors.  Small tensors (q, C, keys)
are drawn here on the host and copied.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
IH4_STD = 37837.22652  # sqrt((2**32 - 1) / 3)

# stream tags (tensor kinds)
TAG_P, TAG_V, TAG_Q, TAG_C, TAG_K, TAG_RK, TAG_RV, TAG_S = 1, 2, 3, 4, 5, 6, 7, 8

BASE_SEED = 0x48434154  # "HCAT"


def _fin(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def stream_key(seed: int, *tags: int) -> int:
    with np.errstate(over="ignore"):
        k = _fin(np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + GOLDEN], dtype=np.uint64))
        for t in tags:
            k = _fin((k ^ np.uint64(t & 0xFFFFFFFFFFFFFFFF)) + GOLDEN)
    return int(k[0])


def u64(key: int, start: int, count: int) -> np.ndarray:
    j = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _fin(np.uint64(key) + (j + np.uint64(1)) * GOLDEN)


def codes_from_u(u: np.ndarray, c: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        return (((u >> np.uint64(32)) * np.uint64(c)) >> np.uint64(32)).astype(np.uint16)


def ih4(u: np.ndarray) -> np.ndarray:
    m = np.uint64(0xFFFF)
    s = (u & m).astype(np.int64) + ((u >> np.uint64(16)) & m).astype(np.int64) \
        + ((u >> np.uint64(32)) & m).astype(np.int64) + (u >> np.uint64(48)).astype(np.int64)
    return s - 131070


def v16(u: np.ndarray) -> np.ndarray:
    return (ih4(u).astype(np.float32) * np.float32(2.0 ** -15)).astype(np.float16)


# ----------------------------------------------------------------------------
# tensors of the decode workload (DESIGN.md §3 "Input recipe")
# ----------------------------------------------------------------------------

def gen_codes(seed: int, b: int, l: int, kv: int, g: int, c: int, start: int, count: int) -> np.ndarray:
    """Codes P[b][l][kv][i][start:start+count] for all groups i -> uint16 [g][count]."""
    out = np.empty((g, count), dtype=np.uint16)
    for i in range(g):
        out[i] = codes_from_u(u64(stream_key(seed, TAG_P, b, l, kv, i), start, count), c)
    return out


def gen_values(seed: int, b: int, l: int, kv: int, d: int, start: int, count: int) -> np.ndarray:
    """Values V[b][l][kv][start:start+count][:] -> fp16 [count][d]; counter = row*d + e."""
    u = u64(stream_key(seed, TAG_V, b, l, kv), start * d, count * d)
    return v16(u).reshape(count, d)


def gen_value_rows(seed: int, b: int, l: int, kv: int, d: int, rows) -> np.ndarray:
    """Rows `rows` (int array of token positions) of V[b][l][kv] -> fp16 [len(rows)][d]; the
    same counters as gen_values (row j = counters j*d .. j*d+d-1), for huge stores of which
    only a few rows are needed."""
    rows = np.asarray(rows, dtype=np.uint64)
    key = np.uint64(stream_key(seed, TAG_V, b, l, kv))
    j = (rows[:, None] * np.uint64(d) + np.arange(d, dtype=np.uint64)[None, :]).reshape(-1)
    with np.errstate(over="ignore"):
        u = _fin(key + (j + np.uint64(1)) * GOLDEN)
    return v16(u).reshape(len(rows), d)


def gen_query(seed: int, b: int, l: int, hq: int, d: int, s: float) -> np.ndarray:
    """q[b][l] -> fp16 [hq][d], approx N(0, s^2) (Irwin-Hall(4), rescaled)."""
    u = u64(stream_key(seed, TAG_Q, b, l), 0, hq * d)
    x = ih4(u).astype(np.float64) * (s / IH4_STD)
    return x.astype(np.float16).reshape(hq, d)


def gen_codebook(seed: int, l: int, cbg: int, c: int, dbar: int) -> np.ndarray:
    """Codebook C[l] -> fp32 [cbg][c][dbar], approx N(0, 1)."""
    u = u64(stream_key(seed, TAG_C, l), 0, cbg * c * dbar)
    return (ih4(u).astype(np.float64) / IH4_STD).astype(np.float32).reshape(cbg, c, dbar)


def gen_keys(seed: int, tag2: int, rows: int, d: int, scale: float = 1.0) -> np.ndarray:
    """Raw keys -> fp16 [rows][d] approx N(0, scale^2)."""
    u = u64(stream_key(seed, TAG_K, tag2), 0, rows * d)
    return (ih4(u).astype(np.float64) * (scale / IH4_STD)).astype(np.float16).reshape(rows, d)


def gen_resident(seed: int, kind: int, b: int, l: int, kv: int, d: int, count: int) -> np.ndarray:
    """Resident (exact) keys or values of the recent window -> fp16 [count][d]."""
    u = u64(stream_key(seed, kind, b, l, kv), 0, count * d)
    return v16(u).reshape(count, d)


def planted_keys(seed: int, rows: int, d: int, g: int, clusters: int, cbg_c: int):
    """Zero-noise planted-cluster keys: each group's sub-vector is one of
    `clusters` fp16-exact centres.  Returns (keys fp16 [rows][d], codebook fp32
    [g][cbg_c][dbar]) whose first `clusters` centroids per group are the centres and
    the remainder are far-away distractors, so encode is exact and error-free."""
    dbar = d // g
    u = u64(stream_key(seed, TAG_K, 0xC1), 0, g * clusters * dbar)
    centres = v16(u).astype(np.float32).reshape(g, clusters, dbar)
    cb = np.empty((g, cbg_c, dbar), dtype=np.float32)
    cb[:, :clusters] = centres
    if cbg_c > clusters:
        ud = u64(stream_key(seed, TAG_K, 0xC2), 0, g * (cbg_c - clusters) * dbar)
        cb[:, clusters:] = (v16(ud).astype(np.float32) + np.float32(64.0)).reshape(g, cbg_c - clusters, dbar)
    a = codes_from_u(u64(stream_key(seed, TAG_K, 0xC3), 0, rows * g), clusters).reshape(rows, g)
    keys = np.empty((rows, d), dtype=np.float16)
    for i in range(g):
        keys[:, i * dbar:(i + 1) * dbar] = centres[i][a[:, i]].astype(np.float16)
    return keys, cb, a


def sample_rows(seed: int, it: int, N: int, count: int) -> np.ndarray:
    """Row indices in [0, N) for k-means batch `it` (with replacement) -> int64 [count]."""
    u = u64(stream_key(seed, TAG_S, it), 0, count)
    with np.errstate(over="ignore"):
        return (((u >> np.uint64(32)) * np.uint64(N)) >> np.uint64(32)).astype(np.int64)
