"""Heterogeneous Eq. 5 (DESIGN §8b f1, include/hc.h hc_gather_values / hc_host_weighted_sum_range
/ hc_add_partial; §3.2): GPU pulls the kept rows with index < t_split, host
threads sum the rest over host DRAM, concurrently; the joined output equals the oracle's Eq. 5
within the north_star tolerance and the selection is the oracle's bit for bit."""
import numpy as np
import pytest

from harness import Case, build_gpu, compare_unit, oracle_unit

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2507_19823_b200 as hc
    hc.lib()
    return torch


def _run(case, host_frac, graph=False, mode="doorbell"):
    import torch
    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.hetero import HeteroEq5
    kc, vs, q = build_gpu(case)
    B, Hq, d, km = case.B, case.Hq, case.d, case.k_max
    bud = hc.budget(case.tau, km, case.renorm)
    ws = hc.Workspace(kc.workspace_bytes(bud))
    het = HeteroEq5(kc, vs, km, host_frac, threads=4, mode=mode)
    out = torch.full((B, Hq, d), float("nan"), dtype=torch.float32, device="cuda")
    sel_k = torch.zeros((B, Hq), dtype=torch.int64, device="cuda")
    qq = q[0].contiguous()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                het(qq, 0, bud, out, sel_k, ws)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(2):  # replays re-run the host node and the joins
            out.fill_(float("nan"))
            g.replay()
    else:
        het(qq, 0, bud, out, sel_k, ws)
    torch.cuda.synchronize()
    het.check()
    gpu = dict(out=out.cpu().numpy(), idx=het.idx_d.view(B, Hq, km).cpu().numpy(),
               w=het.w_d.view(B, Hq, km).cpu().numpy(), k=sel_k.cpu().numpy())
    for b in range(B):
        for kv in range(case.Hkv):
            compare_unit(case, gpu, oracle_unit(case, b, 0, kv), b, kv, check_z=False)
    return het


@pytest.mark.parametrize("mode", ["doorbell", "hostnode"])
@pytest.mark.parametrize("host_frac", [0.0, 0.37, 1.0])
def test_hetero_split_matches_oracle(torch_cuda, host_frac, mode):
    _run(Case(B=2, Hkv=2, n=12011, k_max=1500, placement=1, seed=81), host_frac, mode=mode)


@pytest.mark.parametrize("mode", ["doorbell", "hostnode"])
def test_hetero_split_graph_replay(torch_cuda, mode):
    _run(Case(B=1, Hkv=2, n=20000, k_max=3000, placement=1, seed=82), 0.5, graph=True, mode=mode)


def test_hetero_split_window_and_renorm(torch_cuda):
    """resident window tokens (global indices n_q.., exact values in HBM) are summed by the GPU
    side (t_split <= n_q: the host store holds only the quantized tokens' values)."""
    _run(Case(B=1, Hkv=2, n=9000, res_cap=64, n_res=40, k_max=700, renorm=1, placement=1, seed=83), 0.25)


def test_gather_values_range(torch_cuda):
    """hc_gather_values over [t0, t1) equals the oracle's Eq. 5 over the kept tokens in range."""
    import torch
    import oracle
    import paper_2507_19823_b200 as hc
    case = Case(B=1, Hkv=2, n=10000, k_max=1200, placement=1, seed=84)
    kc, vs, q = build_gpu(case)
    B, Hq, d, km = case.B, case.Hq, case.d, case.k_max
    bud = hc.budget(case.tau, km, select_only=True)
    ws = hc.Workspace(kc.workspace_bytes(bud))
    idx = torch.full((B * Hq, km), -1, dtype=torch.int32, device="cuda")
    w = torch.zeros((B * Hq, km), dtype=torch.float32, device="cuda")
    k = torch.zeros((B, Hq), dtype=torch.int64, device="cuda")
    hc.decode_attention(q[0].contiguous(), kc, vs, 0, bud, out=torch.empty(1, device="cuda"),
                        sel_idx=idx, sel_w=w, sel_k=k, ws=ws)
    for t0, t1 in [(0, 10000), (2047, 2049), (1000, 7777), (5000, 5000), (9990, 20000)]:
        out = torch.full((B, Hq, d), float("nan"), device="cuda")
        hc.gather_values(kc, vs, 0, idx, w, k, t0, t1, out, ws)
        torch.cuda.synchronize()
        ii, ww, kk, oo = idx.cpu().numpy(), w.cpu().numpy(), k.view(-1).cpu().numpy(), out.view(B * Hq, d).cpu().numpy()
        for r in range(B * Hq):
            s = ii[r, :kk[r]]
            m = (s >= t0) & (s < t1)
            V = case.values(0, 0, (r % Hq) // case.G)
            ref = oracle.gather(s[m], ww[r, :kk[r]][m].astype(np.float64), V) if m.any() else np.zeros(d)
            assert np.all(np.abs(oo[r] - ref) <= 1e-3 + 2e-3 * np.abs(ref)), (t0, t1, r)


def test_batch_views_pipelined(torch_cuda):
    """Micro-batch pipelining (bench.py --pipeline): KCache/VStore.batch_view chains of one
    sequence each, on their own streams, concurrently; results equal the oracle per sequence."""
    import torch
    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.hetero import HeteroEq5
    case = Case(B=2, Hkv=2, n=15000, k_max=2000, placement=1, seed=85)
    kc, vs, q = build_gpu(case)
    B, Hq, d, km = case.B, case.Hq, case.d, case.k_max
    bud = hc.budget(case.tau, km)
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    sel_k = torch.zeros((B, Hq), dtype=torch.int64, device="cuda")
    main = torch.cuda.current_stream()
    parts = []
    for b in range(B):
        kv_, vs_ = kc.batch_view(b, 1), vs.batch_view(b, 1)
        parts.append((b, HeteroEq5(kv_, vs_, km, 0.5 if b == 0 else 0.0 + 0.3, threads=4),
                      hc.Workspace(kv_.workspace_bytes(bud)), torch.cuda.Stream()))
    for b, het, ws, st in parts:
        st.wait_stream(main)
        with torch.cuda.stream(st):
            het(q[0][b:b + 1].contiguous(), 0, bud, out[b:b + 1], sel_k[b:b + 1], ws)
    for _, _, _, st in parts:
        main.wait_stream(st)
    torch.cuda.synchronize()
    for b, het, _, _ in parts:
        gpu = dict(out=out[b:b + 1].cpu().numpy(), idx=het.idx_d.view(1, Hq, km).cpu().numpy(),
                   w=het.w_d.view(1, Hq, km).cpu().numpy(), k=sel_k[b:b + 1].cpu().numpy())
        for kv in range(case.Hkv):
            ref = oracle_unit(case, b, 0, kv)
            compare_unit(case, gpu, ref, 0, kv, check_z=False)


def test_hetero_config3_full_size_sampled(torch_cuda):
    """BASELINE config 3 shape (128K ctx, B=4, g=32, k_max=16384, V host-resident) in the
    launch configuration bench.py times (heterogeneous Eq. 5, host_frac 0.6): one layer,
    sampled units vs the oracle."""
    import torch
    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.hetero import HeteroEq5
    case = Case(B=4, L=1, Hkv=8, g=32, n=131072, k_max=16384, placement=1, seed=3)
    kc, vs, q = build_gpu(case)
    B, Hq, d, km = case.B, case.Hq, case.d, case.k_max
    bud = hc.budget(case.tau, km)
    ws = hc.Workspace(kc.workspace_bytes(bud))
    het = HeteroEq5(kc, vs, km, 0.6)
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    sel_k = torch.zeros((B, Hq), dtype=torch.int64, device="cuda")
    het(q[0].contiguous(), 0, bud, out, sel_k, ws)
    torch.cuda.synchronize()
    gpu = dict(out=out.cpu().numpy(), idx=het.idx_d.view(B, Hq, km).cpu().numpy(),
               w=het.w_d.view(B, Hq, km).cpu().numpy(), k=sel_k.cpu().numpy())
    for b, kv in [(0, 0), (3, 7)]:
        compare_unit(case, gpu, oracle_unit(case, b, 0, kv), b, kv, check_z=False)


def test_host_worker_timeout_reports(torch_cuda):
    """hc_host_worker_wait never hangs: with the worker paused the wait kernel gives up after
    timeout_s and hc_host_worker_status reports HC_ERR_CUDA; a served job reports HC_OK."""
    import time
    import torch
    import paper_2507_19823_b200 as hc
    vs = hc.VStore.allocate(1, 1, 1, 64, 128, placement=hc.HC_V_HOST_MAPPED)
    out = torch.zeros((4, 128), dtype=torch.float32).pin_memory()
    idx = torch.zeros((4, 16), dtype=torch.int32, device="cuda")
    wt = torch.zeros((4, 16), dtype=torch.float32, device="cuda")
    k = torch.zeros((4,), dtype=torch.int64, device="cuda")
    w = hc.HostWorker(threads=1, max_jobs=2, timeout_s=0.2)
    j = w.add_job(4, 16, vs, 4, out)
    w.submit(j, idx, wt, k, 64, 0, n_valid=64)
    w.wait(j)
    torch.cuda.synchronize()
    assert w.status() == hc.HC_OK
    w.pause(True)
    t0 = time.time()
    w.submit(j, idx, wt, k, 64, 0, n_valid=64)
    w.wait(j)
    torch.cuda.synchronize()
    assert time.time() - t0 < 5.0
    assert w.status() == hc.HC_ERR_CUDA
    # the timed-out share is poisoned, never passed off as a result
    assert torch.isnan(out).all()
    w.pause(False)
    w.close()


def test_hetero_shared_kv_selection(torch_cuda):
    """Heterogeneous Eq. 5 over the per-KV-head shared selection (R8): the G rows of a KV head
    carry one index set, each head sums its own weights on both sides of the split."""
    import torch
    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.hetero import HeteroEq5
    case = Case(B=2, Hkv=2, n=14000, k_max=2000, placement=1, seed=86, shared=True)
    kc, vs, q = build_gpu(case)
    B, Hq, d, km = case.B, case.Hq, case.d, case.k_max
    bud = hc.budget(case.tau, km, shared_kv=True)
    ws = hc.Workspace(kc.workspace_bytes(bud))
    het = HeteroEq5(kc, vs, km, 0.5, threads=4)
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    sel_k = torch.zeros((B, Hq), dtype=torch.int64, device="cuda")
    het(q[0].contiguous(), 0, bud, out, sel_k, ws)
    torch.cuda.synchronize()
    gpu = dict(out=out.cpu().numpy(), idx=het.idx_d.view(B, Hq, km).cpu().numpy(),
               w=het.w_d.view(B, Hq, km).cpu().numpy(), k=sel_k.cpu().numpy())
    for b in range(B):
        for kv in range(case.Hkv):
            compare_unit(case, gpu, oracle_unit(case, b, 0, kv), b, kv, check_z=False)
