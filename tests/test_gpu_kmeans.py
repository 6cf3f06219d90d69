"""GPU parity of the prefill side (NEXT f4): bulk key encoding (R1) and one MiniBatchKMeans
step vs the CPU oracle -- labels and counts bit-exact, centroids bit-exact (exact
int64 sums, the oracle's double-precision update order)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2507_19823_b200 as hc
    hc.lib()
    return torch


@pytest.mark.parametrize("d,g,c,cbg,rows", [(128, 32, 8192, 32, 4097), (128, 64, 8192, 1, 1024),
                                            (128, 16, 1000, 16, 3001), (64, 64, 33, 64, 2050),
                                            (128, 8, 512, 1, 1500), (128, 128, 300, 128, 1100)])
def test_bulk_encode_bit_exact(torch_cuda, d, g, c, cbg, rows):
    import oracle
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    rng = np.random.default_rng(d + g + c + rows)
    keys = rng.standard_normal((rows, d)).astype(np.float16)
    C = rng.standard_normal((cbg, c, d // g)).astype(np.float32)
    C[:, c // 2] = C[:, 3]                      # duplicated centroid: ties -> lower index
    keys[::7, : d // g] = C[0, 3].astype(np.float16)
    codes = hc.quantize_keys(torch.from_numpy(keys).cuda(), torch.from_numpy(C).cuda(), g)
    torch.cuda.synchronize()
    got = codes.cpu().numpy().view(np.uint16)[:, :rows].T
    assert np.array_equal(got, oracle.encode(keys, C, g))


def _km_case(torch, d, g, c, cbg, N, b, steps, seed, prior=False):
    import oracle
    import paper_2507_19823_b200 as hc
    rng = np.random.default_rng(seed)
    keys = rng.standard_normal((N, d)).astype(np.float16)
    C = rng.standard_normal((cbg, c, d // g)).astype(np.float32)
    v = rng.integers(0, 30, size=(cbg, c)).astype(np.int64) if prior else np.zeros((cbg, c), np.int64)
    kd = torch.from_numpy(keys).cuda()
    Cd = torch.from_numpy(C).cuda()
    vd = torch.from_numpy(v).cuda()
    lab = torch.empty((g, b), dtype=torch.int16, device="cuda")
    for it in range(steps):
        sample = rng.integers(0, N, size=b).astype(np.int64)
        hc.kmeans_step(kd, torch.from_numpy(sample).cuda(), Cd, vd, g, labels=lab)
        C, v, lab_o = oracle.kmeans_step(keys, C, v, sample, g)
        torch.cuda.synchronize()
        assert np.array_equal(lab.cpu().numpy().view(np.uint16).T, lab_o), f"labels, step {it}"
        assert np.array_equal(vd.cpu().numpy(), v), f"counts, step {it}"
        assert np.array_equal(Cd.cpu().numpy(), C), f"centroids, step {it}"


@pytest.mark.parametrize("d,g,c,cbg,N,b,steps,prior", [(128, 32, 256, 32, 5000, 3000, 3, False),
                                                       (128, 64, 100, 1, 2000, 1500, 2, True),
                                                       (64, 16, 4096, 16, 9000, 4099, 2, False),
                                                       (128, 128, 64, 128, 700, 1024, 3, True)])
def test_kmeans_step_bit_exact(torch_cuda, d, g, c, cbg, N, b, steps, prior):
    _km_case(torch_cuda, d, g, c, cbg, N, b, steps, seed=d + g + c + N, prior=prior)


def test_kmeans_step_paper_scale(torch_cuda):
    """P:356's batch size 10,000 with c = 8192, g = 32, d = 128 (one step)."""
    _km_case(torch_cuda, 128, 32, 8192, 32, 40000, 10000, 1, seed=91)


def test_kmeans_out_of_range_rows_skipped(torch_cuda):
    import paper_2507_19823_b200 as hc
    torch = torch_cuda
    keys = torch.randn((100, 64), device="cuda").half()
    C = torch.randn((16, 8, 4), device="cuda")
    v = torch.zeros((16, 8), dtype=torch.int64, device="cuda")
    lab = torch.empty((16, 5), dtype=torch.int16, device="cuda")
    sample = torch.tensor([0, 100, -1, 5, 99], dtype=torch.int64, device="cuda")
    hc.kmeans_step(keys, sample, C, v, 16, labels=lab)
    torch.cuda.synchronize()
    L = lab.cpu().numpy().view(np.uint16)
    assert (L[:, 1] == 0xFFFF).all() and (L[:, 2] == 0xFFFF).all()
    assert int(v.sum()) == 3 * 16


def test_train_codebook_matches_oracle_loop(torch_cuda):
    """train_codebook (P:356's loop: seeded init rows, seeded batches) equals the oracle's
    step-by-step loop bit for bit, and lowers the quantisation error below the init's."""
    import oracle
    import paper_2507_19823_b200 as hc
    import synth
    torch = torch_cuda
    rng = np.random.default_rng(92)
    N, d, g, c, iters, batch, seed = 3000, 32, 8, 16, 10, 500, 5
    dbar = d // g
    keys = rng.standard_normal((N, d)).astype(np.float16)
    Cg, vg = hc.train_codebook(torch.from_numpy(keys).cuda(), g, c, iters=iters, batch=batch, seed=seed)
    rows = synth.sample_rows(seed, 0, N, c)
    C0 = keys[rows].astype(np.float32).reshape(c, g, dbar).transpose(1, 0, 2).copy()
    C, v = C0, np.zeros((g, c), np.int64)
    for it in range(iters):
        C, v, _ = oracle.kmeans_step(keys, C, v, synth.sample_rows(seed, 1 + it, N, batch), g)
    assert np.array_equal(Cg.cpu().numpy(), C)
    assert np.array_equal(vg.cpu().numpy(), v)

    def mse(CB):
        rec = oracle.reconstruct(oracle.encode(keys, CB, g), CB, d)
        return float(((rec - keys.astype(np.float64)) ** 2).mean())
    assert mse(C) < 0.9 * mse(C0)
