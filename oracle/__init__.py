"""CPU oracle of the HCAttention decode hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2507_19823_b200) never imports it and shares no code with it.

Thin ctypes marshalling over oracle/hc_oracle.c (plain C, -O2
-ffp-contract=off, no fast-math); every function there cites the PAPER.md
passage / DESIGN.md reading it implements.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hc_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, OpenMP, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-std=gnu11",
               "-fPIC", "-shared", "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB_PATH)
            p = C.c_void_p
            i64, i32, f32 = C.c_int64, C.c_int, C.c_float
            L.or_half_to_float.argtypes = [C.c_uint16]; L.or_half_to_float.restype = f32
            L.or_encode.argtypes = [p, i64, i32, i32, i32, i32, p, p]
            L.or_reconstruct.argtypes = [p, i64, i32, i32, i32, i32, p, p]
            L.or_scale_exponent.argtypes = [f32]; L.or_scale_exponent.restype = i32
            L.or_table.argtypes = [p, i32, i32, i32, i32, i32, p, p, p, p]
            L.or_codebook_absmax.argtypes = [p, i32, i32, i32, p]
            L.or_table_bound.argtypes = [p, i32, i32, i32, p]
            L.or_table_bound.restype = f32
            L.or_scores.argtypes = [p, p, i64, i64, i32, i32, p]
            L.or_resident_scores.argtypes = [p, p, i64, i32, i32, p]
            L.or_kappa.argtypes = [i32, i32]; L.or_kappa.restype = f32
            L.or_exp2_poly.argtypes = [f32]; L.or_exp2_poly.restype = f32
            L.or_mass.argtypes = [C.c_uint32, f32]; L.or_mass.restype = C.c_uint64
            L.or_threshold.argtypes = [C.c_uint32, C.c_uint64]; L.or_threshold.restype = C.c_uint64
            L.or_tau_q.argtypes = [f32]; L.or_tau_q.restype = C.c_uint32
            L.or_select.argtypes = [p, i64, i32, i32, f32, i64, i32, p, p, p, p, p, p]
            L.or_select.restype = i32
            L.or_select_float.argtypes = [p, i64, i32, f32, i64, i32, p, p, p]
            L.or_select_float.restype = i32
            L.or_float_grid.argtypes = [p, i64, p]
            L.or_float_grid.restype = i32
            L.or_gather.argtypes = [p, p, i64, p, i32, p]
            L.or_blockwise_attention.argtypes = [p, p, p, i64, i32, i32, i32, i64, p]
            L.or_kmeans_step.argtypes = [p, i64, i32, i32, i32, i32, p, i64, p, p, p]
            L.or_select_shared.argtypes = [p, i32, i64, p, i32, f32, i64, p, p, p, p, p, p]
            L.or_exact_attention.argtypes = [p, p, p, i64, i32, p]
            L.or_decode_unit.argtypes = [p, i32, i32, i32, i32, i32, p, p, i64, i64, p, p, p, i64,
                                         f32, i64, i32, p, p, p, p, p, p, p, p, p]
            L.or_decode_unit.restype = i32
            L.or_decode_unit_bits.argtypes = L.or_decode_unit.argtypes + [i32]
            L.or_decode_unit_bits.restype = i32
            L.or_table_bits.argtypes = [p, i32, i32, i32, i32, i32, p, p, p, p, i32]
            _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def encode(keys, C_, g: int) -> np.ndarray:
    """keys fp16 [rows][d], C fp32 [cbg][c][dbar] -> codes uint16 [rows][g] (R1)."""
    keys = _c(keys, np.float16); C_ = _c(C_, np.float32)
    rows, d = keys.shape
    cbg, c, dbar = C_.shape
    assert dbar * g == d
    out = np.empty((rows, g), dtype=np.uint16)
    lib().or_encode(_ptr(keys.view(np.uint16)), rows, d, g, c, cbg, _ptr(C_), _ptr(out))
    return out


def kmeans_step(keys, C_, counts, sample, g: int):
    """f4: one MiniBatchKMeans step -> (new C [cbg][c][dbar] fp32, new counts
    [cbg][c] int64, labels [b][g] u16).  Inputs are not modified."""
    keys = _c(keys, np.float16)
    C2 = np.array(C_, dtype=np.float32, order="C", copy=True)
    v2 = np.array(counts, dtype=np.int64, order="C", copy=True)
    sample = _c(sample, np.int64)
    n_keys, d = keys.shape
    cbg, c, dbar = C2.shape
    lab = np.zeros((max(sample.shape[0], 1), g), np.uint16)
    rc = lib().or_kmeans_step(_ptr(keys.view(np.uint16)), n_keys, d, g, c, cbg, _ptr(sample),
                              sample.shape[0], _ptr(C2), _ptr(v2), _ptr(lab))
    if rc:
        raise ValueError(f"or_kmeans_step rc={rc}")
    return C2, v2, lab[: sample.shape[0]]


def reconstruct(codes, C_, d: int) -> np.ndarray:
    codes = _c(codes, np.uint16); C_ = _c(C_, np.float32)
    n, g = codes.shape
    cbg, c, dbar = C_.shape
    out = np.empty((n, d), dtype=np.float32)
    lib().or_reconstruct(_ptr(codes), n, d, g, c, cbg, _ptr(C_), _ptr(out))
    return out


def table(q, C_, g: int, lut_bits: int = 16):
    """q fp16 [G][d] -> (T32 fp32 [G][g][c], Tfx int16 [G][g][c], e int32 [G]) (R2);
    lut_bits = 8 selects the 8-bit table variant (R2b)."""
    q = _c(q, np.float16); C_ = _c(C_, np.float32)
    G, d = q.shape
    cbg, c, dbar = C_.shape
    T32 = np.empty((G, g, c), dtype=np.float32)
    Tfx = np.empty((G, g, c), dtype=np.int16)
    e = np.empty(G, dtype=np.int32)
    lib().or_table_bits(_ptr(q.view(np.uint16)), G, d, g, c, cbg, _ptr(C_), _ptr(T32), _ptr(Tfx),
                        _ptr(e), lut_bits)
    return T32, Tfx, e


def codebook_absmax(C_) -> np.ndarray:
    """Cabs[ci][e] = max_m |C[ci][m][e]| (R2)."""
    C_ = _c(C_, np.float32)
    cbg, c, dbar = C_.shape
    out = np.empty((cbg, dbar), np.float32)
    lib().or_codebook_absmax(_ptr(C_), cbg, c, dbar, _ptr(out))
    return out


def table_bound(q_head, C_, g: int) -> float:
    q = _c(q_head, np.float16)
    Ca = codebook_absmax(C_)
    return lib().or_table_bound(_ptr(q.view(np.uint16)), q.shape[0], g, C_.shape[0], _ptr(Ca))


def scores(Tfx_head, P_groupmajor, n: int) -> np.ndarray:
    """Eq. 3: Tfx [g][c] int16, P [g][stride] uint16 -> z int32 [n]."""
    T = _c(Tfx_head, np.int16); P = _c(P_groupmajor, np.uint16)
    g, c = T.shape
    z = np.empty(n, dtype=np.int32)
    lib().or_scores(_ptr(T), _ptr(P), n, P.shape[1], g, c, _ptr(z))
    return z


def resident_scores(q_head, rk, e_h: int) -> np.ndarray:
    q = _c(q_head, np.float16); rk = _c(rk, np.float16)
    z = np.empty(rk.shape[0], dtype=np.int32)
    lib().or_resident_scores(_ptr(q.view(np.uint16)), _ptr(rk.view(np.uint16)), rk.shape[0],
                             q.shape[0], e_h, _ptr(z))
    return z


def scale_exponent(A: float) -> int:
    return lib().or_scale_exponent(A)


def kappa(d: int, e_h: int) -> float:
    return lib().or_kappa(d, e_h)


def exp2_poly(f: float) -> float:
    return lib().or_exp2_poly(f)


def mass(delta: int, kap: float) -> int:
    return lib().or_mass(delta, kap)


def threshold(tau_q: int, S: int) -> int:
    return lib().or_threshold(tau_q, S)


def tau_q(tau: float) -> int:
    return lib().or_tau_q(tau)


def select(z, e_h: int, d: int, tau: float, k_max: int, renorm: int = 0):
    """Eq. 4 on int32 fixed-point scores -> dict(idx, w, k_sel, S, M, kstar)."""
    z = _c(z, np.int32)
    n = z.shape[0]
    idx = np.empty(max(k_max, 1), dtype=np.int32)
    w = np.empty(max(k_max, 1), dtype=np.float64)
    ks = np.zeros(1, np.int64); S = np.zeros(1, np.uint64); M = np.zeros(1, np.int32)
    kst = np.zeros(1, np.int64)
    rc = lib().or_select(_ptr(z), n, e_h, d, tau, k_max, renorm, _ptr(idx), _ptr(w), _ptr(ks),
                         _ptr(S), _ptr(M), _ptr(kst))
    if rc:
        raise ValueError(f"or_select rc={rc}")
    k = int(ks[0])
    return dict(idx=idx[:k].copy(), w=w[:k].copy(), k_sel=k, S=int(S[0]), M=int(M[0]), kstar=int(kst[0]))


def select_float(zf, d: int, tau: float, k_max: int, renorm: int = 0):
    zf = _c(zf, np.float32)
    n = zf.shape[0]
    idx = np.empty(max(k_max, 1), dtype=np.int32)
    w = np.empty(max(k_max, 1), dtype=np.float64)
    ks = np.zeros(1, np.int64)
    rc = lib().or_select_float(_ptr(zf), n, d, tau, k_max, renorm, _ptr(idx), _ptr(w), _ptr(ks))
    if rc:
        raise ValueError(f"or_select_float rc={rc}")
    k = int(ks[0])
    return dict(idx=idx[:k].copy(), w=w[:k].copy(), k_sel=k)


def float_grid(zf):
    """R5b step 1 (hc_select_topk's input grid): -> (e, z_fx int32 [n])."""
    zf = _c(zf, np.float32)
    z = np.empty(max(zf.shape[0], 1), np.int32)
    e = lib().or_float_grid(_ptr(zf), zf.shape[0], _ptr(z))
    return int(e), z[:zf.shape[0]].copy()


def select_shared(z, e, d: int, tau: float, k_max: int):
    """R8 (NEXT f3(iii)): one Eq. 4 selection for the G query heads of a KV head on their
    head-averaged fixed-point mass.  z [G][n] int32, e [G] -> dict(idx, w [G][k], k_sel,
    S_A, kstar, A [n])."""
    z = _c(z, np.int32); e = _c(e, np.int32)
    G, n = z.shape
    km = max(k_max, 1)
    idx = np.empty(km, np.int32); w = np.empty((G, km), np.float64)
    ks = np.zeros(1, np.int64); SA = np.zeros(1, np.uint64); kst = np.zeros(1, np.int64)
    A = np.empty(max(n, 1), np.uint64)
    rc = lib().or_select_shared(_ptr(z), G, n, _ptr(e), d, tau, k_max, _ptr(idx), _ptr(w),
                                _ptr(ks), _ptr(SA), _ptr(kst), _ptr(A))
    if rc:
        raise ValueError(f"or_select_shared rc={rc}")
    k = int(ks[0])
    return dict(idx=idx[:k].copy(), w=w[:, :k].copy(), k_sel=k, S_A=int(SA[0]),
                kstar=int(kst[0]), A=A[:n].copy())


def gather(idx, w, V) -> np.ndarray:
    idx = _c(idx, np.int32); w = _c(w, np.float64); V = _c(V, np.float16)
    out = np.empty(V.shape[1], dtype=np.float64)
    lib().or_gather(_ptr(idx), _ptr(w), idx.shape[0], _ptr(V.view(np.uint16)), V.shape[1], _ptr(out))
    return out


def blockwise_attention(q, k, v, bs: int) -> np.ndarray:
    """f4 (iii), App. B: anchor-block + causal local-block prefill attention.
    q [n][Hq][d], k, v [n][Hkv][d] fp16 -> out [n][Hq][d] double."""
    q = _c(q, np.float16); k = _c(k, np.float16); v = _c(v, np.float16)
    n, Hq, d = q.shape
    Hkv = k.shape[1]
    out = np.empty((n, Hq, d), dtype=np.float64)
    lib().or_blockwise_attention(_ptr(q.view(np.uint16)), _ptr(k.view(np.uint16)), _ptr(v.view(np.uint16)),
                                 n, Hq, Hkv, d, bs, _ptr(out))
    return out


def exact_attention(q_head, K, V) -> np.ndarray:
    """Eq. 1 in double."""
    q = _c(q_head, np.float16); K = _c(K, np.float16); V = _c(V, np.float16)
    out = np.empty(K.shape[1], dtype=np.float64)
    lib().or_exact_attention(_ptr(q.view(np.uint16)), _ptr(K.view(np.uint16)), _ptr(V.view(np.uint16)),
                             K.shape[0], K.shape[1], _ptr(out))
    return out


def decode_unit(q, C_, P_groupmajor, nq: int, V, tau: float, k_max: int, renorm: int = 0,
                rk=None, rv=None, lut_bits: int = 16, shared: bool = False):
    """Full decode of one (b, l, kv) unit for its G query heads (R2->R6).  shared=True:
    R8 -- one selection for the G heads (or_select_shared on the same scores), each head
    summing its own weights over it (Eq. 5 via or_gather)."""
    q = _c(q, np.float16); C_ = _c(C_, np.float32); P = _c(P_groupmajor, np.uint16)
    V = _c(V, np.float16)
    G, d = q.shape
    cbg, c, dbar = C_.shape
    g = d // dbar
    nres = 0 if rk is None else rk.shape[0]
    if rk is None:
        rk = np.zeros((1, d), np.float16); rv = np.zeros((1, d), np.float16)
    rk = _c(rk, np.float16); rv = _c(rv, np.float16)
    n = nq + nres
    z = np.empty((G, max(n, 1)), np.int32)
    e = np.empty(G, np.int32)
    km = max(k_max, 1)
    idx = np.empty((G, km), np.int32); w = np.empty((G, km), np.float64)
    ks = np.empty(G, np.int64); S = np.empty(G, np.uint64); M = np.empty(G, np.int32)
    kst = np.empty(G, np.int64); out = np.empty((G, d), np.float64)
    rc = lib().or_decode_unit_bits(_ptr(q.view(np.uint16)), G, d, g, c, cbg, _ptr(C_), _ptr(P), nq,
                                   P.shape[1], _ptr(V.view(np.uint16)), _ptr(rk.view(np.uint16)),
                                   _ptr(rv.view(np.uint16)), nres, tau, k_max, renorm, _ptr(z),
                                   _ptr(e), _ptr(idx), _ptr(w), _ptr(ks), _ptr(S), _ptr(M),
                                   _ptr(kst), _ptr(out), lut_bits)
    if rc:
        raise ValueError(f"or_decode_unit rc={rc}")
    if shared:
        if renorm:
            raise ValueError("shared selection takes renorm=0")
        sh = select_shared(z[:, :n], e, d, tau, k_max)
        Vall = np.concatenate([V[:nq], rv[:nres]]) if nres else V[:nq]
        outs = np.stack([gather(sh["idx"], sh["w"][h], Vall) for h in range(G)])
        k = sh["k_sel"]
        return dict(z=z[:, :n], e=e, idx=[sh["idx"]] * G, w=[sh["w"][h] for h in range(G)],
                    k_sel=np.full(G, k, np.int64), S=S, M=M, kstar=np.full(G, sh["kstar"], np.int64),
                    out=outs, S_A=sh["S_A"], A=sh["A"])
    return dict(z=z[:, :n], e=e, idx=[idx[h, :ks[h]].copy() for h in range(G)],
                w=[w[h, :ks[h]].copy() for h in range(G)], k_sel=ks, S=S, M=M, kstar=kst, out=out)
