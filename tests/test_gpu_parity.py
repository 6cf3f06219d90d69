"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded
inputs.  Bit-exact codes, scores, masses and selected-index sets; outputs within
2e-3 rel / 1e-3 abs (north_star).  Sizes span several scan tiles and ragged tails."""
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


def _run(case: Case, units=None, layers=None):
    kc, vs, q = build_gpu(case)
    out = []
    for l in (layers if layers is not None else case.layers):
        gpu = run_gpu_layer(case, kc, vs, q, l)
        us = units if units is not None else [(b, kv) for b in range(case.B) for kv in range(case.Hkv)]
        for b, kv in us:
            ref = oracle_unit(case, b, l, kv)
            out.append(compare_unit(case, gpu, ref, b, kv))
    return out


# ------------------------------------------------------------------ encode (row a0)
@pytest.mark.parametrize("d,g,c,cbg,rows", [(128, 32, 8192, 32, 300), (128, 64, 8192, 1, 257),
                                            (128, 16, 1000, 16, 100), (64, 64, 33, 64, 77),
                                            (128, 8, 512, 1, 64)])
def test_encode_bit_exact(torch_cuda, d, g, c, cbg, rows):
    import oracle
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(d + g + c + rows)
    keys = (rng.standard_normal((rows, d))).astype(np.float16)
    C = rng.standard_normal((cbg, c, d // g)).astype(np.float32)
    if c > 4:  # duplicated centroids -> ties must go to the lower index
        C[:, c // 2] = C[:, 3]
        keys[::7, : d // g] = C[0, 3].astype(np.float16)
    codes = hc.quantize_keys(torch.from_numpy(keys).cuda(), torch.from_numpy(C).cuda(), g)
    torch.cuda.synchronize()
    got = codes.cpu().numpy().view(np.uint16)[:, :rows].T
    ref = oracle.encode(keys, C, g)
    assert np.array_equal(got, ref)


# ------------------------------------------------------------------ full decode (rows a1-a5)
def test_config1_parity(torch_cuda):
    """BASELINE config 1: L=1, 1 KV head x 4 GQA heads, d=128, n=4096, g=32, c=8192,
    k_max=512, tau=0.9, batch 1."""
    st = _run(Case())
    assert st[0]["max_abs"] < 1e-3


@pytest.mark.parametrize("n", [1, 7, 63, 1000, 8191, 8193, 20011])
def test_ragged_lengths(torch_cuda, n):
    _run(Case(n=n, k_max=min(512, max(1, n // 3)), seed=n))


@pytest.mark.parametrize("tau", [0.3, 0.5, 0.7, 0.9, 1.0])
def test_tau_grid_table3(torch_cuda, tau):
    """Table 3's τ grid; cap large so τ decides; τ=1 keeps everything."""
    st = _run(Case(n=12000, tau=tau, k_max=12000, seed=3))
    if tau == 1.0:
        assert all(k == 12000 for s in st for k in s["kstar"])


@pytest.mark.parametrize("k_max", [1, 2, 100, 5000, 100000])
def test_cap(torch_cuda, k_max):
    _run(Case(n=9000, tau=0.95, k_max=k_max, seed=4))


def test_g64_config2_shape(torch_cuda):
    """g=64 (the 25 % budget), two KV heads, several tiles + ragged tail."""
    _run(Case(Hkv=2, g=64, n=17000, k_max=4250, seed=5))


@pytest.mark.parametrize("G", [1, 2])
def test_gqa_variants(torch_cuda, G):
    _run(Case(G=G, Hkv=2, n=5000, seed=6 + G))


def test_shared_codebook_and_small_c(torch_cuda):
    _run(Case(cbg=1, c=300, n=6000, seed=8))
    _run(Case(g=16, c=4096, n=3000, seed=9))


def test_batch_and_layers(torch_cuda):
    _run(Case(B=3, L=2, Hkv=2, n=3000, k_max=700, seed=10))


def test_resident_window(torch_cuda):
    """Resident exact tokens (R7) compete in the same softmax/selection."""
    _run(Case(n=5000, res_cap=64, n_res=40, k_max=800, seed=11))
    _run(Case(n=0, res_cap=64, n_res=64, k_max=64, tau=1.0, seed=12))


@pytest.mark.parametrize("n_res,G", [(19000, 4), (5003, 2), (777, 1)])
def test_value_offload_only_mode(torch_cuda, n_res, G):
    """SURVEY f2 / Table 1a's "VO" row: exact fp16 keys for every token (all resident, no
    quantized codes) -> dense exact scoring kernel + the same selection and gather."""
    _run(Case(n=0, G=G, Hkv=2, res_cap=n_res + 64, n_res=n_res, k_max=n_res // 5, tau=0.9,
              seed=60 + G))


def test_renorm(torch_cuda):
    _run(Case(n=7000, renorm=1, k_max=300, seed=13))


def test_ties_heavy(torch_cuda):
    """Tiny codebooks (c=2, g=4 -> 16 distinct scores) -> massive score ties; the lower
    index must win, for both the τ cut and the cap cut."""
    _run(Case(g=4, d=64, c=2, n=3000, k_max=700, tau=0.9, seed=14))
    _run(Case(g=4, d=64, c=3, n=5000, k_max=5000, tau=0.6, seed=15))
    _run(Case(g=8, d=64, c=2, n=20000, k_max=20000, tau=0.99, seed=16))


def test_empty_cache_error(torch_cuda):
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    case = Case(n=64)
    kc, vs, q = build_gpu(case)
    kc.set_counts(0, 0, 0)
    with pytest.raises(hc.HcError) as ei:
        hc.decode_attention(q[0].contiguous(), kc, vs, 0, hc.budget(0.9, 10))
    assert ei.value.status == hc.HC_ERR_EMPTY
    with pytest.raises(hc.HcError) as ei:
        hc.decode_attention(q[0].contiguous(), kc, vs, 0, hc.budget(1.5, 10))
    assert ei.value.status == hc.HC_ERR_ARG


# ------------------------------------------------------------------ 8-bit table variant (R2b)
@pytest.mark.parametrize("n,g,tau,k_max,B,Hkv", [(4096, 32, 0.9, 512, 1, 1), (20011, 32, 0.7, 5000, 2, 2),
                                                 (17000, 64, 0.9, 4250, 1, 2), (40000, 32, 1.0, 9000, 1, 1),
                                                 (3, 32, 0.9, 2, 1, 1)])
def test_lut8_variant(torch_cuda, n, g, tau, k_max, B, Hkv):
    """The 8-bit-table scan (SWAR accumulation, 16K-token tiles) is bit-exact with the oracle's
    R2b mode on scores, masses and index sets."""
    _run(Case(B=B, Hkv=Hkv, g=g, n=n, tau=tau, k_max=k_max, lut_bits=8, seed=50 + n % 97))


def test_lut8_config3_full_size_sampled(torch_cuda):
    case = Case(B=4, L=1, Hkv=8, g=32, n=131072, k_max=16384, placement=1, seed=3, lut_bits=8)
    _run(case, units=[(1, 2), (3, 7)])


# ------------------------------------------------------------------ append protocol
@pytest.mark.parametrize("res_cap", [0, 4])
def test_append_then_decode(torch_cuda, res_cap):
    """hc_append_kv: new keys are encoded (R1) into P, values appended; with a window the
    oldest resident token spills into P.  The cache contents and a decode over it match
    the oracle."""
    import oracle
    import paper_2507_19823_b200 as hc
    import synth
    torch = torch_cuda
    B, L, Hkv, G, d, g, c = 2, 2, 2, 4, 128, 32, 512
    n_cap = 128
    case = Case(B=B, L=L, Hkv=Hkv, G=G, g=g, c=c, n=0, n_cap=n_cap, seed=21)
    cb = np.stack([case.codebook(l) for l in range(L)])
    kc = hc.KCache(B, L, Hkv, G, d, g, c, n_cap, torch.from_numpy(cb).cuda(), res_cap=res_cap)
    vs = hc.VStore.allocate(B, L, Hkv, n_cap, d)
    steps = 37
    K = synth.gen_keys(21, 1, steps * B * L * Hkv, d).reshape(steps, L, B, Hkv, d)
    Vv = synth.gen_keys(21, 2, steps * B * L * Hkv, d).reshape(steps, L, B, Hkv, d)
    for t in range(steps):
        for l in range(L):
            kc.append(l, torch.from_numpy(K[t, l]).cuda(), torch.from_numpy(Vv[t, l]).cuda(), vs)
    torch.cuda.synchronize()
    nq = steps - min(steps, res_cap)
    for l in range(L):
        assert kc.n_q(l) == nq and kc.n_res(l) == min(steps, res_cap)
        codes = kc.codes.cpu().numpy().view(np.uint16)
        for b in range(B):
            for kv in range(Hkv):
                ref = oracle.encode(K[:nq, l, b, kv], cb[l], g)  # [nq][g]
                assert np.array_equal(codes[b, l, kv, :, :nq].T, ref)
                vstore = vs.tensor[b, l, kv, :nq].cpu().numpy()
                assert np.array_equal(vstore.view(np.uint16), Vv[:nq, l, b, kv].view(np.uint16))
    # decode the appended cache and compare with the oracle
    q = torch.from_numpy(np.stack([synth.gen_query(21, b, 0, Hkv * G, d, 2.29) for b in range(B)])).cuda()
    bud = hc.budget(0.9, 20)
    idx = torch.full((B, Hkv * G, 20), -1, dtype=torch.int32, device="cuda")
    w = torch.zeros((B, Hkv * G, 20), dtype=torch.float32, device="cuda")
    k = torch.zeros((B, Hkv * G), dtype=torch.int64, device="cuda")
    out = hc.decode_attention(q, kc, vs, 0, bud, sel_idx=idx, sel_w=w, sel_k=k).cpu().numpy()
    codes = kc.codes.cpu().numpy().view(np.uint16)
    nres = min(steps, res_cap)
    for b in range(B):
        for kv in range(Hkv):
            rk = K[nq:, 0, b, kv] if nres else None
            rv = Vv[nq:, 0, b, kv] if nres else None
            ref = oracle.decode_unit(q[b, kv * G:(kv + 1) * G].cpu().numpy(), cb[0],
                                     codes[b, 0, kv, :, :max(nq, 1)] if nq else np.zeros((g, 1), np.uint16),
                                     nq, Vv[:max(nq, 1), 0, b, kv], 0.9, 20, rk=rk, rv=rv)
            for h in range(G):
                kk = int(k[b, kv * G + h])
                assert kk == ref["k_sel"][h]
                assert np.array_equal(idx[b, kv * G + h, :kk].cpu().numpy(), ref["idx"][h])
                assert np.all(np.abs(out[b, kv * G + h] - ref["out"][h]) <= 1e-3 + 2e-3 * np.abs(ref["out"][h]))


def test_append_capacity_error(torch_cuda):
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    cb = torch.zeros((1, 32, 16, 4), dtype=torch.float32, device="cuda")
    kc = hc.KCache(1, 1, 1, 4, 128, 32, 16, 64, cb)
    vs = hc.VStore.allocate(1, 1, 1, 64, 128)
    kc.set_counts(0, 64)
    kn = torch.zeros((1, 1, 128), dtype=torch.float16, device="cuda")
    with pytest.raises(hc.HcError) as ei:
        kc.append(0, kn, kn, vs)
    assert ei.value.status == hc.HC_ERR_CAPACITY


# ------------------------------------------------------------------ standalone select
@pytest.mark.parametrize("n,tau,k_max", [(10, 0.5, 10), (5000, 0.9, 200), (70000, 0.7, 100000),
                                         (3, 1.0, 2), (4097, 0.3, 4097)])
def test_select_topk_float(torch_cuda, n, tau, k_max):
    import oracle
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(n)
    rows = 5
    sc = (rng.standard_normal((rows, n)) * 30).astype(np.float32)
    sc[1] = np.round(sc[1] / 10) * 10  # ties
    idx, w, k = hc.select_topk(torch.from_numpy(sc).cuda(), 128, hc.budget(tau, k_max))
    torch.cuda.synchronize()
    for r in range(rows):
        ref = oracle.select_float(sc[r], 128, tau, k_max)
        kk = int(k[r])
        assert kk == ref["k_sel"]
        assert np.array_equal(idx[r, :kk].cpu().numpy(), ref["idx"])
        assert np.allclose(w[r, :kk].cpu().numpy(), ref["w"], rtol=1e-6, atol=1e-12)


# ------------------------------------------------------------------ host-mapped values
def test_host_mapped_values(torch_cuda):
    """Value store in pinned host memory, read zero-copy by the gather kernel."""
    _run(Case(B=2, Hkv=2, n=6000, k_max=900, placement=1, seed=31))


# ------------------------------------------------------------------ the paper's CPU-side Eq. 5 (f1)
def test_select_only_then_host_weighted_sum(torch_cuda):
    """the GPU stops after the selection (budget.select_only), the (idx, w, k) go
    to the host and Eq. 5 runs on host threads over the host-resident values."""
    import ctypes as C
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    case = Case(B=2, Hkv=2, n=12000, k_max=2000, placement=1, seed=71)
    kc, vs, q = build_gpu(case)
    B, Hq, km = case.B, case.Hq, case.k_max
    idx = torch.full((B, Hq, km), -1, dtype=torch.int32, device="cuda")
    w = torch.zeros((B, Hq, km), dtype=torch.float32, device="cuda")
    k = torch.zeros((B, Hq), dtype=torch.int64, device="cuda")
    hc.decode_attention(q[0].contiguous(), kc, vs, 0, hc.budget(case.tau, km, select_only=True),
                        out=torch.empty(1, device="cuda"), sel_idx=idx, sel_w=w, sel_k=k)
    hi, hw, hk = idx.cpu(), w.cpu(), k.cpu()
    out = torch.zeros((B * Hq, case.d), dtype=torch.float32)
    V = vs.tensor  # pinned host [B][L][Hkv][n_cap][d]
    st = hc.lib().hc_host_weighted_sum(C.c_void_p(hi.data_ptr()), C.c_void_p(hw.data_ptr()),
                                       C.c_void_p(hk.data_ptr()), B * Hq, km, C.c_void_p(V.data_ptr()),
                                       case.L * case.Hkv * case.n_cap * case.d, case.n_cap * case.d,
                                       case.n, Hq, case.G, case.d, C.c_void_p(out.data_ptr()), 0)
    assert st == hc.HC_OK
    gpu = dict(out=out.numpy().reshape(B, Hq, case.d), idx=hi.numpy(), w=hw.numpy(), k=hk.numpy())
    for b in range(B):
        for kv in range(case.Hkv):
            compare_unit(case, gpu, oracle_unit(case, b, 0, kv), b, kv, check_z=False)


# ------------------------------------------------------------------ full-size sampled parity
def test_config2_full_size_sampled(torch_cuda):
    """BASELINE config 2 shape (32K ctx, 8 KV heads, g=64, k_max=8192, τ=0.9), in the launch
    configuration bench.py times; 2 of 32 layers built, 3 sampled units compared."""
    case = Case(L=2, Hkv=8, g=64, n=32768, k_max=8192, seed=2, layers=[0, 1])
    _run(case, units=[(0, 0), (0, 5), (0, 7)], layers=[1])


def test_config3_full_size_sampled(torch_cuda):
    """BASELINE config 3 shape (128K ctx, B=4, g=32, k_max=16384, V host-pinned), one layer,
    sampled units."""
    case = Case(B=4, L=1, Hkv=8, g=32, n=131072, k_max=16384, placement=1, seed=3)
    _run(case, units=[(0, 0), (3, 7)])


def test_config4_full_size_sampled(torch_cuda):
    """BASELINE config 4 shape on one GPU (1M ctx, g=32, k_max=131072, V in HBM), one layer,
    two sampled units: index sets bit-exact and outputs within tolerance at the full size."""
    case = Case(B=1, L=1, Hkv=8, g=32, n=1048576, k_max=131072, seed=4)
    _run(case, units=[(0, 0), (0, 6)])


def test_stream_k_scan_ragged_sampled(torch_cuda):
    """The 16-bit stream-K scan (k_scan_sk) on a ragged multi-tile shape: 8 units x 37 tiles of
    8192 tokens (>= 2 tiles per CTA), z bit-exact on sampled units."""
    case = Case(B=1, L=1, Hkv=8, g=32, n=300007, k_max=30000, seed=58)
    _run(case, units=[(0, 1), (0, 7)])
