"""Randomised GPU-vs-oracle sweep over the decode path's shape space (seeded, reproducible):
batch, KV heads, GQA group, d, g (dbar 1..16), c, n (ragged, across tiles and splits),
tau, k_max (binding or not), resident window, shared codebooks, 16/13-bit codes and per-head /
shared selection.  Every case: bit-exact z, S, M, k_sel and index sets; outputs within the
north_star tolerance (harness.compare_unit)."""
import os

import numpy as np
import pytest

from harness import Case, build_gpu, compare_unit, oracle_unit, run_gpu_layer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2507_19823_b200 as hc
    hc.lib()
    return torch


def _cases(k=None, seed=None):
    # HC_FUZZ_N / HC_FUZZ_SEED widen the sweep (e.g. 300 cases for a soak run)
    k = int(os.environ.get("HC_FUZZ_N", "48")) if k is None else k
    seed = int(os.environ.get("HC_FUZZ_SEED", "2026")) if seed is None else seed
    rng = np.random.default_rng(seed)
    out = []
    for i in range(k):
        d = int(rng.choice([64, 128, 128, 256]))
        dbar = int(rng.choice([d_ for d_ in (1, 2, 4, 8, 16) if d // d_ <= 128]))
        g = d // dbar
        G = int(rng.choice([1, 2, 4]))
        c = int(rng.choice([2, 37, 256, 1000, 8192]))
        n = int(rng.integers(1, 40000))
        res = int(rng.choice([0, 0, 0, 17, 64]))
        n_res = min(res, int(rng.integers(0, res + 1))) if res else 0
        tau = float(rng.choice([0.3, 0.7, 0.9, 0.99, 1.0]))
        k_max = int(rng.choice([1, 50, max(1, n // 8), n + n_res + 5]))
        code_bits = 13 if (c <= 8192 and rng.random() < 0.25) else 16
        shared = bool(G > 1 and rng.random() < 0.2)
        cbg = 1 if rng.random() < 0.25 else g
        B = int(rng.integers(1, 3))
        Hkv = int(rng.integers(1, 3))
        kw = dict(B=B, Hkv=Hkv, G=G, d=d, g=g, c=c, cbg=cbg, n=n, res_cap=res, n_res=n_res,
                  tau=tau, k_max=k_max, code_bits=code_bits, shared=shared, seed=1000 + i)
        if i >= 48 and rng.random() < 0.3:  # wider sweeps also cover host-mapped values
            kw["placement"] = 1
        out.append(kw)
    return out


@pytest.mark.parametrize("sel", ["auto", "pass", "fused", "auto-sep", "pass-sep"])
@pytest.mark.parametrize("kw", _cases(), ids=lambda kw: "-".join(f"{k}{v}" for k, v in kw.items()
                                                                if k in ("d", "g", "G", "c", "n", "tau")))
def test_fuzz_decode_parity(torch_cuda, kw, sel, monkeypatch):
    """sel: the selection kernel -- auto (by row length: the one-kernel cluster path k_sel_small
    up to 64K candidates), pass (the three passes) or fused (round 1's cluster kernel); all
    bit-exact on every shape.  With values in HBM (d = 128) auto / pass run Eq. 5 inside the
    selection (k_sel_small's gather, K3G); the "-sep" variants (HC_K3G=0) use the separate
    k_gather_rows instead."""
    base = sel.split("-")[0]
    if base != "auto":
        monkeypatch.setenv("HC_SELECT", base)
    if sel.endswith("-sep"):
        monkeypatch.setenv("HC_K3G", "0")
    case = Case(**kw)
    if case.n == 0 and case.n_res == 0:
        pytest.skip("empty")
    kc, vs, q = build_gpu(case)
    gpu = run_gpu_layer(case, kc, vs, q, 0)
    for b in range(case.B):
        for kv in range(case.Hkv):
            compare_unit(case, gpu, oracle_unit(case, b, 0, kv), b, kv)


def _sel_cases(k=16, seed=31):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(k):
        n = int(rng.integers(1, 300000))
        scale = float(rng.choice([1e-30, 1e-3, 1.0, 30.0, 1e4, 1e30]))
        tau = float(rng.choice([0.1, 0.5, 0.9, 0.999, 1.0]))
        k_max = int(rng.choice([1, 100, max(1, n // 3), n + 1]))
        rows = int(rng.integers(1, 6))
        d = int(rng.choice([1, 64, 128]))
        out.append((n, scale, tau, k_max, rows, d, 300 + i))
    return out


@pytest.mark.parametrize("n,scale,tau,k_max,rows,d,seed", _sel_cases())
def test_fuzz_select_topk(torch_cuda, n, scale, tau, k_max, rows, d, seed):
    """hc_select_topk on real scores (R5b) over extreme scales, heavy ties, constant rows."""
    import oracle
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(seed)
    sc = (rng.standard_normal((rows, n)) * scale).astype(np.float32)
    if rows > 1:
        sc[1] = np.round(sc[1] / max(scale, 1e-30) * 4) * max(scale, 1e-30) / 4  # ties
    if rows > 2:
        sc[2] = np.float32(scale)  # constant row
    idx, w, k = hc.select_topk(torch.from_numpy(sc).cuda(), d, hc.budget(tau, k_max))
    torch.cuda.synchronize()
    for r in range(rows):
        ref = oracle.select_float(sc[r], d, tau, k_max)
        kk = int(k[r])
        assert kk == ref["k_sel"]
        assert np.array_equal(idx[r, :kk].cpu().numpy(), ref["idx"])
        assert np.allclose(w[r, :kk].cpu().numpy(), ref["w"], rtol=1e-6, atol=1e-12)
