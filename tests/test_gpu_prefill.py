"""GPU parity of the prefill side's App. B block-wise attention (NEXT f4 (iii), DESIGN F5)
vs the float64 oracle, and of the prefill append (bulk R1 encode of a block's keys into the
cache) followed by a decode step."""
import numpy as np
import pytest

from harness import TOL_ABS, TOL_REL, compare_unit

pytestmark = pytest.mark.gpu

# fp16 inputs, fp16 P in the PV product (rel. 2^-11), fp32 accumulation
ATT_ATOL, ATT_RTOL = 2e-3, 5e-3


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2507_19823_b200 as hc
    hc.lib()
    return torch


@pytest.mark.parametrize("n,Hq,Hkv,bs", [(300, 4, 1, 128), (1000, 8, 2, 256), (64, 2, 2, 64),
                                         (777, 4, 4, 1024), (2500, 4, 1, 512)])
def test_blockwise_attention_parity(torch_cuda, n, Hq, Hkv, bs):
    import oracle
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(n + bs)
    d = 128
    q = (rng.standard_normal((n, Hq, d)) * 0.5).astype(np.float16)
    k = (rng.standard_normal((n, Hkv, d)) * 0.5).astype(np.float16)
    v = rng.standard_normal((n, Hkv, d)).astype(np.float16)
    got = hc.blockwise_attention(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                 torch.from_numpy(v).cuda(), bs).cpu().numpy()
    ref = oracle.blockwise_attention(q, k, v, bs)
    err = np.abs(got - ref)
    assert np.all(err <= ATT_ATOL + ATT_RTOL * np.abs(ref)), float(err.max())


def test_blockwise_attention_sharp_scores(torch_cuda):
    """Large logits (peaked softmax, online-softmax rescaling exercised) and GQA 4."""
    import oracle
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(7)
    n, Hq, Hkv, d, bs = 1500, 8, 2, 128, 256
    q = (rng.standard_normal((n, Hq, d)) * 2.0).astype(np.float16)
    k = (rng.standard_normal((n, Hkv, d)) * 2.0).astype(np.float16)
    v = rng.standard_normal((n, Hkv, d)).astype(np.float16)
    got = hc.blockwise_attention(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda(),
                                 torch.from_numpy(v).cuda(), bs).cpu().numpy()
    ref = oracle.blockwise_attention(q, k, v, bs)
    err = np.abs(got - ref)
    assert np.all(err <= ATT_ATOL + ATT_RTOL * np.abs(ref)), float(err.max())


def test_prefill_append_then_decode(torch_cuda):
    """Prefill a 2-sequence cache in two blocks with hc_prefill_append (bulk encode + value
    copy), then one decode layer: codes bit-exact (R1) and the decode matches the oracle."""
    import oracle
    import paper_2507_19823_b200 as hc
    import synth
    from harness import Case, run_gpu_layer
    torch = torch_cuda
    B, Hkv, G, d, g, c, n_cap = 2, 2, 4, 128, 32, 512, 4096
    case = Case(B=B, Hkv=Hkv, G=G, d=d, g=g, c=c, n=3000, n_cap=n_cap, k_max=400, seed=21)
    cb = torch.from_numpy(case.codebook(0)[None]).cuda()
    kc = hc.KCache(B, 1, Hkv, G, d, g, c, n_cap, cb, device="cuda")
    vs = hc.VStore.allocate(B, 1, Hkv, n_cap, d, device="cuda")
    K = synth.gen_keys(33, 1, B * case.n * Hkv, d).reshape(B, case.n, Hkv, d)
    V = synth.gen_keys(33, 2, B * case.n * Hkv, d).reshape(B, case.n, Hkv, d)
    for lo, hi in ((0, 2048), (2048, case.n)):  # two prefill blocks
        kc.prefill_append(0, torch.from_numpy(np.ascontiguousarray(K[:, lo:hi])).cuda(),
                          torch.from_numpy(np.ascontiguousarray(V[:, lo:hi])).cuda(), vs)
    torch.cuda.synchronize()
    assert kc.n_q(0) == case.n
    q = torch.from_numpy(np.stack([case.query(b, 0) for b in range(B)])[None]).cuda()
    gpu = run_gpu_layer(case, kc, vs, q, 0)
    C_ = case.codebook(0)
    for b in range(B):
        for kv in range(Hkv):
            P = oracle.encode(K[b, :, kv], C_, g).T
            got_codes = kc.codes[b, 0, kv, :, : case.n].cpu().numpy().view(np.uint16)
            assert np.array_equal(got_codes, P)
            ref = oracle.decode_unit(case.query(b, 0)[kv * G:(kv + 1) * G], C_, P, case.n, V[b, :, kv],
                                     case.tau, case.k_max)
            compare_unit(case, gpu, ref, b, kv)
