"""GPU parity of the packed 13-bit code layout (NEXT f3(ii), include/hc.h HC_STRIP13_BYTES):
the same scores, selections and outputs as the oracle (the packing is lossless, so the
oracle is unchanged), plus the layout itself checked against a test-side numpy packer."""
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


def _np_pack13(codes, n_cap):
    """Reference packing of one strip per row (include/hc.h layout): lo | nib | bit planes."""
    rows, n = codes.shape
    out = np.zeros((rows, n_cap * 13 // 8), np.uint8)
    c = codes.astype(np.uint32)
    out[:, :n] = c & 0xFF
    for t in range(n):
        out[:, n_cap + t // 2] |= (((c[:, t] >> 8) & 15) << (4 * (t & 1))).astype(np.uint8)
        out[:, n_cap + n_cap // 2 + t // 8] |= (((c[:, t] >> 12) & 1) << (t & 7)).astype(np.uint8)
    return out


@pytest.mark.parametrize("n,n_cap", [(64, 64), (1000, 1024), (4099, 4160), (8, 64), (1, 64)])
def test_pack13_layout(torch_cuda, n, n_cap):
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(n)
    codes = rng.integers(0, 8192, size=(7, n_cap)).astype(np.uint16)
    got = hc.pack_codes13(torch.from_numpy(codes.view(np.int16)).cuda(), n, n_cap)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), _np_pack13(codes[:, :n], n_cap))


def test_pack13_ragged_keeps_other_tokens(torch_cuda):
    """Packing tokens [0, n) of a strip leaves the packed bits of tokens >= n untouched."""
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(5)
    a = rng.integers(0, 8192, size=(3, 128)).astype(np.uint16)
    b = rng.integers(0, 8192, size=(3, 128)).astype(np.uint16)
    out = hc.pack_codes13(torch.from_numpy(a.view(np.int16)).cuda(), 128, 128)
    hc.pack_codes13(torch.from_numpy(b.view(np.int16)).cuda(), 37, 128, out=out)
    torch.cuda.synchronize()
    mix = a.copy()
    mix[:, :37] = b[:, :37]
    assert np.array_equal(out.cpu().numpy(), _np_pack13(mix, 128))


def _run(case: Case, units=None):
    kc, vs, q = build_gpu(case)
    for l in case.layers:
        gpu = run_gpu_layer(case, kc, vs, q, l)
        us = units if units is not None else [(b, kv) for b in range(case.B) for kv in range(case.Hkv)]
        for b, kv in us:
            compare_unit(case, gpu, oracle_unit(case, b, l, kv), b, kv)


@pytest.mark.parametrize("n,tau,k_max,B,Hkv,g", [(4096, 0.9, 512, 1, 1, 32), (20011, 0.7, 5000, 2, 2, 32),
                                                 (9001, 0.9, 3000, 1, 2, 64), (77, 1.0, 100, 1, 1, 32),
                                                 (32768, 0.9, 8192, 1, 2, 64)])
def test_packed_decode_parity(torch_cuda, n, tau, k_max, B, Hkv, g):
    _run(Case(B=B, Hkv=Hkv, g=g, n=n, tau=tau, k_max=k_max, seed=90 + n % 89, code_bits=13))


def test_packed_ties_resident_shared(torch_cuda):
    _run(Case(g=4, d=64, c=2, n=3000, k_max=700, seed=93, code_bits=13))
    _run(Case(n=5000, res_cap=64, n_res=40, k_max=800, seed=94, code_bits=13))
    _run(Case(B=2, Hkv=2, n=9000, k_max=2000, seed=95, code_bits=13, shared=True))


def test_packed_append_then_decode(torch_cuda):
    """hc_append_kv writes the new key's code into the packed planes (read-modify-write of
    the shared nibble / bit bytes); the decode over the grown cache matches the oracle."""
    import oracle
    import paper_2507_19823_b200 as hc
    import synth
    torch = torch_cuda
    case = Case(B=2, Hkv=2, n=1000, n_cap=1088, k_max=300, seed=96, code_bits=13)
    kc, vs, q = build_gpu(case)
    extra = 21
    K = synth.gen_keys(97, 1, extra * case.B * case.Hkv, case.d).reshape(extra, case.B, case.Hkv, case.d)
    Vn = synth.gen_keys(97, 2, extra * case.B * case.Hkv, case.d).reshape(extra, case.B, case.Hkv, case.d)
    for t in range(extra):
        kc.append(0, torch.from_numpy(K[t]).cuda(), torch.from_numpy(Vn[t]).cuda(), vs)
    torch.cuda.synchronize()
    n2 = case.n + extra
    case2 = Case(B=2, Hkv=2, n=n2, n_cap=1088, k_max=300, seed=96, code_bits=13)
    gpu = run_gpu_layer(case2, kc, vs, q, 0)
    C_ = case.codebook(0)
    for b in range(case.B):
        for kv in range(case.Hkv):
            P = np.concatenate([case.codes(b, 0, kv), oracle.encode(K[:, b, kv], C_, case.g).T], axis=1)
            V = np.concatenate([case.values(b, 0, kv), Vn[:, b, kv]])
            ref = oracle.decode_unit(case.query(b, 0)[kv * case.G:(kv + 1) * case.G], C_, P, n2, V,
                                     case.tau, case.k_max)
            compare_unit(case2, gpu, ref, b, kv)


def test_packed_config3_full_size_sampled(torch_cuda):
    """BASELINE config 3 shape with packed codes (bench.py --code-bits 13), sampled units."""
    case = Case(B=4, L=1, Hkv=8, g=32, n=131072, k_max=16384, placement=1, seed=3, code_bits=13)
    _run(case, units=[(0, 0), (3, 7)])


def test_packed_append_with_window_eviction(torch_cuda):
    """Packed codes + a 5-token recent window: every append past the window encodes the
    evicted oldest token into the packed planes; decode over the cache matches the oracle."""
    import oracle
    import paper_2507_19823_b200 as hc
    import synth
    torch = torch_cuda
    B, L, Hkv, G, d, g, c, n_cap, W = 2, 1, 2, 4, 128, 32, 512, 128, 5
    case = Case(B=B, L=L, Hkv=Hkv, G=G, g=g, c=c, n=0, n_cap=n_cap, seed=23, code_bits=13)
    cb = case.codebook(0)[None]
    kc = hc.KCache(B, L, Hkv, G, d, g, c, n_cap, torch.from_numpy(cb).cuda(), res_cap=W, code_bits=13)
    vs = hc.VStore.allocate(B, L, Hkv, n_cap, d)
    steps = 45
    K = synth.gen_keys(23, 1, steps * B * Hkv, d).reshape(steps, B, Hkv, d)
    Vv = synth.gen_keys(23, 2, steps * B * Hkv, d).reshape(steps, B, Hkv, d)
    for t in range(steps):
        kc.append(0, torch.from_numpy(K[t]).cuda(), torch.from_numpy(Vv[t]).cuda(), vs)
    torch.cuda.synchronize()
    nq = steps - W
    assert kc.n_q(0) == nq and kc.n_res(0) == W
    q = torch.from_numpy(np.stack([synth.gen_query(23, b, 0, Hkv * G, d, 2.29) for b in range(B)])).cuda()
    bud = hc.budget(0.9, 16)
    idx = torch.full((B, Hkv * G, 16), -1, dtype=torch.int32, device="cuda")
    w = torch.zeros((B, Hkv * G, 16), dtype=torch.float32, device="cuda")
    k = torch.zeros((B, Hkv * G), dtype=torch.int64, device="cuda")
    out = hc.decode_attention(q, kc, vs, 0, bud, sel_idx=idx, sel_w=w, sel_k=k).cpu().numpy()
    for b in range(B):
        for kv in range(Hkv):
            P = oracle.encode(K[:nq, b, kv], cb[0], g).T
            ref = oracle.decode_unit(q[b, kv * G:(kv + 1) * G].cpu().numpy(), cb[0], P, nq,
                                     Vv[:nq, b, kv], 0.9, 16, rk=K[nq:, b, kv], rv=Vv[nq:, b, kv])
            for h in range(G):
                kk = int(k[b, kv * G + h])
                assert kk == ref["k_sel"][h]
                assert np.array_equal(idx[b, kv * G + h, :kk].cpu().numpy(), ref["idx"][h])
                assert np.all(np.abs(out[b, kv * G + h] - ref["out"][h]) <= 1e-3 + 2e-3 * np.abs(ref["out"][h]))
