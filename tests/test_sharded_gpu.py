"""Sequence-sharded decode kernels on ONE GPU: R shards of the context are
driven in lock-step in one process (collectives = tensor reductions, no ranks waiting on
each other).  The kept index set must equal the UNSHARDED oracle's bit for bit
(R-invariance) and the summed output must be within tolerance."""
import numpy as np
import pytest

from harness import TOL_ABS, TOL_REL, Case, oracle_unit

pytestmark = pytest.mark.gpu


def _shard_caches(case: Case, R: int, device="cuda"):
    import torch
    import paper_2507_19823_b200 as hc
    import synth.device as sd
    L = case.L
    full = hc.KCache(case.B, L, case.Hkv, case.G, case.d, case.g, case.c, case.n_cap,
                     torch.from_numpy(np.stack([case.codebook(l) for l in range(L)])).to(device),
                     cbg=case.cbg, device=device)
    vfull = hc.VStore.allocate(case.B, L, case.Hkv, case.n_cap, case.d, device=device)
    sd.fill_codes(full.codes, case.seed, case.c, case.n)
    sd.fill_values(vfull.tensor, case.seed, case.n, device=device)
    bounds = np.linspace(0, case.n, R + 1).astype(int)
    shards = []
    for r in range(R):
        a, b = int(bounds[r]), int(bounds[r + 1])
        cap = max(64, (b - a + 63) // 64 * 64)
        kc = hc.KCache(case.B, L, case.Hkv, case.G, case.d, case.g, case.c, cap, full.codebook,
                       cbg=case.cbg, device=device)
        kc.codes[..., : b - a] = full.codes[..., a:b]
        vs = hc.VStore.allocate(case.B, L, case.Hkv, cap, case.d, device=device)
        vs.tensor[:, :, :, : b - a] = vfull.tensor[:, :, :, a:b]
        for l in range(L):
            kc.set_counts(l, b - a)
        shards.append((kc, vs, a))
    return shards


@pytest.mark.parametrize("R,n,tau,k_max", [(2, 9000, 0.9, 1500), (3, 7001, 0.7, 50000),
                                           (4, 12000, 1.0, 3000), (2, 5000, 0.95, 1),
                                           (5, 33333, 0.9, 4000), (8, 70000, 0.99, 9000),
                                           (3, 150, 0.5, 20), (6, 20000, 0.3, 100000)])
def test_virtual_shards_match_unsharded_oracle(R, n, tau, k_max):
    import torch
    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.sharded import GpuShard, decode_layer_virtual
    case = Case(B=2, Hkv=2, n=n, tau=tau, k_max=k_max, seed=40 + R)
    parts = _shard_caches(case, R)
    bud = hc.budget(tau, k_max)
    shards = [GpuShard(kc, vs, bud) for kc, vs, _ in parts]
    q = torch.from_numpy(np.stack([case.query(b, 0) for b in range(case.B)])).cuda()
    out = decode_layer_virtual(shards, q, 0, [a for _, _, a in parts]).cpu().numpy()
    torch.cuda.synchronize()
    sel = torch.stack([s.sel_idx for s in shards]).amax(0).cpu().numpy()
    ksel = shards[0].sel_k.cpu().numpy()
    for b in range(case.B):
        for kv in range(case.Hkv):
            ref = oracle_unit(case, b, 0, kv)
            for h in range(case.G):
                row = b * case.Hq + kv * case.G + h
                k = int(ksel[row])
                assert k == ref["k_sel"][h]
                assert np.array_equal(sel[row, :k], ref["idx"][h])
                err = np.abs(out[row] - ref["out"][h])
                assert np.all(err <= TOL_ABS + TOL_REL * np.abs(ref["out"][h]))


def _fuzz(k=12, seed=77):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(k):
        R = int(rng.integers(2, 9))
        n = int(rng.integers(R * 3, 60000))
        tau = float(rng.choice([0.2, 0.6, 0.9, 0.99, 1.0]))
        k_max = int(rng.choice([1, 7, max(1, n // 10), n // R + 1, n + 3]))
        out.append((R, n, tau, k_max, 500 + i))
    return out


@pytest.mark.parametrize("R,n,tau,k_max,seed", _fuzz())
def test_virtual_shards_fuzz(R, n, tau, k_max, seed):
    """Seeded sweep: R shards (ragged splits of n), caps below / above a shard's size."""
    import torch
    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.sharded import GpuShard, decode_layer_virtual
    case = Case(B=1, Hkv=2, n=n, tau=tau, k_max=k_max, seed=seed)
    parts = _shard_caches(case, R)
    bud = hc.budget(tau, k_max)
    shards = [GpuShard(kc, vs, bud) for kc, vs, _ in parts]
    q = torch.from_numpy(np.stack([case.query(b, 0) for b in range(case.B)])).cuda()
    out = decode_layer_virtual(shards, q, 0, [a for _, _, a in parts]).cpu().numpy()
    sel = torch.stack([s.sel_idx for s in shards]).amax(0).cpu().numpy()
    ksel = shards[0].sel_k.cpu().numpy()
    for kv in range(case.Hkv):
        ref = oracle_unit(case, 0, 0, kv)
        for h in range(case.G):
            row = kv * case.G + h
            k = int(ksel[row])
            assert k == ref["k_sel"][h]
            assert np.array_equal(sel[row, :k], ref["idx"][h])
            err = np.abs(out[row] - ref["out"][h])
            assert np.all(err <= TOL_ABS + TOL_REL * np.abs(ref["out"][h]))


@pytest.mark.parametrize("use_nccl", [True, False])
def test_cabi_sharded_entry_world1(use_nccl):
    """hc_decode_attention_sharded (the phases + NCCL exchanges in one C-ABI call) on a
    1-rank NCCL communicator (the only world one GPU can host): equals the unsharded oracle
    bit for bit on index sets; eager and CUDA-graph replay."""
    import torch
    import paper_2507_19823_b200 as hc
    from harness import shard_caches
    from paper_2507_19823_b200.sharded import CAbiShard
    case = Case(B=2, Hkv=2, n=20011, tau=0.9, k_max=2500, seed=71)
    (kc, vs, base), = shard_caches(case, 1)
    comm = hc.NcclComm(1, 0, hc.nccl_unique_id()) if use_nccl else None
    sh = CAbiShard(kc, vs, hc.budget(case.tau, case.k_max), 0, 1, base, comm)
    q = torch.from_numpy(np.stack([case.query(b, 0) for b in range(case.B)])).cuda()

    def check(out):
        o = out.view(case.B, case.Hq, -1).cpu().numpy()
        sel = sh.sel_idx.view(case.B, case.Hq, -1).cpu().numpy()
        ks = sh.sel_k.view(case.B, case.Hq).cpu().numpy()
        for b in range(case.B):
            for kv in range(case.Hkv):
                ref = oracle_unit(case, b, 0, kv)
                for h in range(case.G):
                    hq = kv * case.G + h
                    k = int(ks[b, hq])
                    assert k == ref["k_sel"][h]
                    assert np.array_equal(sel[b, hq, :k], ref["idx"][h])
                    err = np.abs(o[b, hq] - ref["out"][h])
                    assert np.all(err <= TOL_ABS + TOL_REL * np.abs(ref["out"][h]))

    out = sh.decode_layer(q, 0)
    torch.cuda.synchronize()
    check(out)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            sh.decode_layer(q, 0)
    torch.cuda.current_stream().wait_stream(s)
    sh.out.fill_(float("nan"))
    sh.sel_idx.fill_(-1)
    g.replay()
    torch.cuda.synchronize()
    check(sh.out)
    if comm is not None:
        comm.close()


def test_cabi_sharded_entry_rejects_missing_comm():
    import paper_2507_19823_b200 as hc
    from harness import shard_caches
    from paper_2507_19823_b200.sharded import CAbiShard
    case = Case(B=1, Hkv=1, n=1000, k_max=100, seed=3)
    (kc, vs, base), = shard_caches(case, 1)
    with pytest.raises(ValueError):
        CAbiShard(kc, vs, hc.budget(0.9, 100), 0, 2, base, None)
