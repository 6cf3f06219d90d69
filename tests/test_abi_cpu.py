"""CPU-side checks of the boundary (no GPU needed): libhc.so loads and exports every
entry point include/hc.h declares; the binding mirrors the header's structs; the
product package never imports the oracle."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "hc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hc_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_north_star_entry_points():
    fns = _header_functions()
    for name in ("hc_quantize_keys", "hc_append_kv", "hc_decode_attention", "hc_select_topk"):
        assert name in fns


def test_library_exports_every_header_symbol():
    import paper_2507_19823_b200 as hc
    L = hc.lib()
    for name in _header_functions():
        assert hasattr(L, name), name
    assert set(hc.EXPORTS) == set(_header_functions())
    assert "sm_100a" in hc.version()


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirrors of the C structs agree with the C compiler's layout (gcc, same header)."""
    import subprocess
    import paper_2507_19823_b200 as hc
    fields = {"hc_vq": ["d", "g", "c", "cbg", "lut_bits", "code_bits"],
              "hc_budget": ["tau", "k_max", "renorm", "select_only"],
              "hc_kcache": ["B", "L", "Hkv", "G", "vq", "n_cap", "codes", "codebook", "cb_absmax",
                            "res_cap", "res_k", "res_v", "n_q", "n_res"],
              "hc_vstore": ["placement", "base", "n_cap"],
              "hc_decode_debug": ["z", "e", "S", "M", "kstar"]}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "hc.h"', "int main(void){"]
    for st, fs in fields.items():
        src.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fs:
            src.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    src.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    got = dict(line.split() for line in subprocess.check_output([str(exe)]).decode().splitlines())
    for st, fs in fields.items():
        cls = getattr(hc, st)
        assert int(got[st]) == ctypes.sizeof(cls), st
        for f in fs:
            assert int(got[f"{st}.{f}"]) == getattr(cls, f).offset, f"{st}.{f}"


def test_validation_without_gpu():
    """Argument validation is synchronous and needs no device."""
    import paper_2507_19823_b200 as hc
    L = hc.lib()
    st = L.hc_quantize_keys(None, 10, None, hc.hc_vq(128, 3, 16, 3, 0), None, 10, None)
    assert st == hc.HC_ERR_SHAPE
    st = L.hc_quantize_keys(None, 0, None, hc.hc_vq(128, 32, 16, 32, 0), None, 0, None)
    assert st == hc.HC_OK
    st = L.hc_quantize_keys(None, 10, None, hc.hc_vq(128, 32, 70000, 32, 0), None, 10, None)
    assert st == hc.HC_ERR_RANGE
    st = L.hc_quantize_keys(None, 10, None, hc.hc_vq(128, 32, 16, 32, 12), None, 10, None)
    assert st == hc.HC_ERR_ARG
    kc = hc.hc_kcache()
    kc.B, kc.L, kc.Hkv, kc.G = 1, 1, 1, 4
    kc.vq = hc.hc_vq(128, 32, 8192, 32, 0)
    kc.n_cap = 100  # not a multiple of 64
    assert L.hc_decode_workspace_bytes(ctypes.byref(kc), hc.budget(0.9, 10)) == 0
    kc.n_cap = 4096
    kc.codes = 1
    kc.codebook = 1
    assert L.hc_decode_workspace_bytes(ctypes.byref(kc), hc.budget(0.9, 512)) > 0
    vs = hc.hc_vstore(0, 1, 4096)
    st = L.hc_decode_attention(1, ctypes.byref(kc), ctypes.byref(vs), 0, hc.budget(0.0, 10), 1,
                               None, None, None, None, 1, 1 << 40, None)
    assert st == hc.HC_ERR_ARG  # tau outside (0,1]
    st = L.hc_decode_attention(1, ctypes.byref(kc), ctypes.byref(vs), 0, hc.budget(0.9, 10), 1,
                               None, None, None, None, 1, 1 << 40, None)
    assert st == hc.HC_ERR_EMPTY  # n_q = n_res = 0
    st = L.hc_decode_attention(1, ctypes.byref(kc), ctypes.byref(vs), 5, hc.budget(0.9, 10), 1,
                               None, None, None, None, 1, 1 << 40, None)
    assert st == hc.HC_ERR_RANGE
    kc.n_q[0] = 10
    st = L.hc_decode_attention(1, ctypes.byref(kc), ctypes.byref(vs), 0, hc.budget(0.9, 10), 1,
                               None, None, None, None, 1, 16, None)
    assert st == hc.HC_ERR_WORKSPACE
    assert b"workspace" in L.hc_last_error()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2507_19823_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "hc_oracle" not in txt and "liboracle" not in txt, f


def test_host_weighted_sum_matches_oracle_gather():
    """SURVEY f1 (the paper's CPU part of Eq. 2): hc_host_weighted_sum on host
    memory equals the oracle's Eq. 5 (double) within fp32 accumulation error; runs on CPU."""
    import numpy as np
    import oracle
    import paper_2507_19823_b200 as hc
    import ctypes as C
    rng = np.random.default_rng(3)
    B, Hkv, G, d, n, k_stride = 2, 2, 4, 128, 5000, 1500
    Hq = Hkv * G
    V = rng.standard_normal((B, Hkv, n, d)).astype(np.float16)
    rows = B * Hq
    idx = np.zeros((rows, k_stride), np.int32)
    w = np.zeros((rows, k_stride), np.float32)
    k = rng.integers(1, k_stride, size=rows).astype(np.int64)
    for r in range(rows):
        sel = np.sort(rng.choice(n, size=k[r], replace=False))
        idx[r, :k[r]] = sel
        ww = rng.random(k[r])
        w[r, :k[r]] = (ww / ww.sum()).astype(np.float32)
    out = np.zeros((rows, d), np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    st = hc.lib().hc_host_weighted_sum(p(idx), p(w), p(k), rows, k_stride, p(V.view(np.uint16)),
                                      Hkv * n * d, n * d, n, Hq, G, d, p(out), 4)
    assert st == hc.HC_OK
    for r in range(rows):
        b, hq = divmod(r, Hq)
        ref = oracle.gather(idx[r, :k[r]], w[r, :k[r]].astype(np.float64), V[b, hq // G])
        assert np.allclose(out[r], ref, rtol=2e-3, atol=1e-3)


@pytest.mark.parametrize("isa", ["", "avx2", "scalar"])
def test_host_weighted_sum_range_split_matches_oracle(isa, monkeypatch):
    """Heterogeneous Eq. 5 (include/hc.h hc_host_weighted_sum_range): the host share over
    kept tokens in [t0, t1) equals the oracle's Eq. 5 over exactly those kept tokens, and
    the shares of a split [0, t) + [t, n) add up to the whole sum; independent of the
    thread count (chunk partials in order)."""
    import numpy as np
    import oracle
    import paper_2507_19823_b200 as hc
    import ctypes as C
    rng = np.random.default_rng(5)
    B, Hkv, G, d, n, k_stride = 2, 2, 4, 128, 20011, 3000
    Hq = Hkv * G
    V = rng.standard_normal((B, Hkv, n, d)).astype(np.float16)
    rows = B * Hq
    idx = np.zeros((rows, k_stride), np.int32)
    w = np.zeros((rows, k_stride), np.float32)
    k = rng.integers(0, k_stride, size=rows).astype(np.int64)
    k[3] = 0  # a row with nothing kept
    for r in range(rows):
        sel = np.sort(rng.choice(n, size=k[r], replace=False))
        idx[r, :k[r]] = sel
        ww = rng.random(k[r])
        w[r, :k[r]] = (ww / max(ww.sum(), 1e-30)).astype(np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)

    def host(t0, t1, threads):
        out = np.full((rows, d), np.nan, np.float32)
        st = hc.lib().hc_host_weighted_sum_range(p(idx), p(w), p(k), rows, k_stride,
                                                p(V.view(np.uint16)), Hkv * n * d, n * d, n, Hq, G, d,
                                                t0, t1, p(out), threads)
        assert st == hc.HC_OK
        return out

    for t0, t1 in [(0, n), (0, 4096), (5000, 13333), (13333, n), (n, n), (7, 8)]:
        out = host(t0, t1, 3)
        for r in range(rows):
            b, hq = divmod(r, Hq)
            s = idx[r, :k[r]]
            m = (s >= t0) & (s < t1)
            ref = oracle.gather(s[m], w[r, :k[r]][m].astype(np.float64), V[b, hq // G]) if m.any() \
                else np.zeros(d)
            assert np.allclose(out[r], ref, rtol=2e-3, atol=1e-3), (t0, t1, r)
    t = 9001
    whole = host(0, n, 1)
    assert np.allclose(host(0, t, 2) + host(t, n, 5), whole, rtol=1e-5, atol=1e-6)
    assert np.array_equal(host(0, n, 7), whole)  # thread-count independent
    st = hc.lib().hc_host_weighted_sum_range(p(idx), p(w), p(k), rows, k_stride, p(V.view(np.uint16)),
                                            Hkv * n * d, n * d, n, Hq, G, d, 10, 5, p(whole), 1)
    assert st == hc.HC_ERR_RANGE
    # a range past the layer's stored rows (e.g. t_split > n_q: resident-window tokens, whose
    # values live in HBM) is refused instead of reading beyond the store
    st = hc.lib().hc_host_weighted_sum_range(p(idx), p(w), p(k), rows, k_stride, p(V.view(np.uint16)),
                                            Hkv * n * d, n * d, n - 1, Hq, G, d, 0, n, p(whole), 1)
    assert st == hc.HC_ERR_RANGE
    # the unranged entry sums only the stored rows [0, n_valid): here every kept index < n
    out_all = np.zeros_like(whole)
    st = hc.lib().hc_host_weighted_sum(p(idx), p(w), p(k), rows, k_stride, p(V.view(np.uint16)),
                                      Hkv * n * d, n * d, n, Hq, G, d, p(out_all), 2)
    assert st == hc.HC_OK and np.array_equal(out_all, whole)
