"""hc_append_decode_attention (the append's encode on a library side stream, overlapping the
table build, joined before the scan) equals hc_append_kv followed by hc_decode_attention bit for
bit -- codes, kept index sets, weights and outputs -- eagerly and as a replayed CUDA graph, with
and without a resident window (the append then also rotates the window: the join must precede
the resident scorer)."""
import numpy as np
import pytest

from harness import Case, build_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2507_19823_b200 as hc
    hc.lib()
    return torch


def _run(case, fused, graph):
    import torch
    import paper_2507_19823_b200 as hc
    kc, vs, q = build_gpu(case)
    g = torch.Generator().manual_seed(case.seed + 1)
    k_new = (torch.randn((case.B, case.Hkv, case.d), generator=g) * 0.5).half().cuda()
    v_new = torch.randn((case.B, case.Hkv, case.d), generator=g).half().cuda()
    bud = hc.budget(case.tau, case.k_max)
    ws = hc.Workspace(kc.workspace_bytes(bud))
    rows = case.B * case.Hq
    out = torch.empty((case.B, case.Hq, case.d), dtype=torch.float32, device="cuda")
    si = torch.full((rows, case.k_max), -1, dtype=torch.int32, device="cuda")
    sw = torch.zeros((rows, case.k_max), dtype=torch.float32, device="cuda")
    sk = torch.zeros((rows,), dtype=torch.int64, device="cuda")

    def step():
        if fused:
            hc.append_decode_attention(q[0], kc, vs, 0, k_new, v_new, bud, out=out, sel_idx=si, sel_w=sw,
                                       sel_k=sk, ws=ws)
        else:
            kc.append(0, k_new, v_new, vs)
            hc.decode_attention(q[0], kc, vs, 0, bud, out=out, sel_idx=si, sel_w=sw, sel_k=sk, ws=ws)

    if graph:
        n0, r0 = kc.n_q(0), kc.n_res(0)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                step()
        torch.cuda.current_stream().wait_stream(s)
        out.fill_(float("nan"))
        si.fill_(-1)
        gr.replay()
        assert kc.n_q(0) + kc.n_res(0) == n0 + r0 + 1
    else:
        step()
    torch.cuda.synchronize()
    return dict(out=out.cpu().numpy(), si=si.cpu().numpy(), sw=sw.cpu().numpy(), sk=sk.cpu().numpy(),
                codes=kc.codes.cpu().numpy(), rk=kc.res_k.cpu().numpy() if case.res_cap else None)


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("kw", [dict(B=2, Hkv=2, n=20011, k_max=2500, seed=91),
                                dict(B=1, Hkv=2, n=70001, k_max=9000, seed=92),
                                dict(B=1, Hkv=1, n=5000, k_max=600, res_cap=64, n_res=17, seed=93)])
def test_append_decode_equals_append_then_decode(torch_cuda, kw, graph):
    case = Case(n_cap=(kw["n"] + 64 + 63) // 64 * 64, **kw)
    a = _run(case, fused=False, graph=graph)
    b = _run(case, fused=True, graph=graph)
    assert np.array_equal(a["codes"], b["codes"])
    if case.res_cap:
        assert np.array_equal(a["rk"], b["rk"])
    assert np.array_equal(a["sk"], b["sk"])
    assert np.array_equal(a["si"], b["si"])
    assert np.array_equal(a["sw"], b["sw"])
    assert np.array_equal(a["out"], b["out"])
