"""GPU parity of the per-KV-head shared selection (NEXT f3(iii), DESIGN R8): one Eq. 4
selection on the G heads' averaged fixed-point mass, shared by the G query heads, each head
summing its own weights.  Index sets bit-exact vs oracle.select_shared (via
oracle.decode_unit(shared=True)); outputs within 2e-3 rel / 1e-3 abs."""
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


def _run(case: Case, units=None):
    kc, vs, q = build_gpu(case)
    for l in case.layers:
        gpu = run_gpu_layer(case, kc, vs, q, l)
        us = units if units is not None else [(b, kv) for b in range(case.B) for kv in range(case.Hkv)]
        for b, kv in us:
            ref = oracle_unit(case, b, l, kv)
            compare_unit(case, gpu, ref, b, kv)
            for h in range(case.G):  # the G rows hold one list
                assert np.array_equal(gpu["idx"][b, kv * case.G + h, : gpu["k"][b, kv * case.G]],
                                      gpu["idx"][b, kv * case.G, : gpu["k"][b, kv * case.G]])


@pytest.mark.parametrize("n,tau,k_max,B,Hkv", [(4096, 0.9, 512, 1, 1), (9001, 0.9, 4000, 2, 2),
                                               (20011, 0.7, 100000, 1, 2), (3000, 1.0, 3000, 1, 1),
                                               (5000, 0.99, 1, 1, 1), (1, 0.9, 8, 1, 1),
                                               (37, 0.5, 10, 2, 1)])
def test_shared_selection_parity(torch_cuda, n, tau, k_max, B, Hkv):
    _run(Case(B=B, Hkv=Hkv, n=n, tau=tau, k_max=k_max, seed=70 + n % 97, shared=True))


def test_shared_gqa2_and_resident(torch_cuda):
    _run(Case(G=2, Hkv=2, n=6000, k_max=1500, seed=81, shared=True))
    _run(Case(n=5000, res_cap=64, n_res=40, k_max=800, seed=82, shared=True))


def test_shared_ties_heavy(torch_cuda):
    """c = 2, g = 4: 16 distinct scores per head -> equal A across many tokens; ties go to
    the lower index for both the τ and the cap cut."""
    _run(Case(g=4, d=64, c=2, n=3000, k_max=700, tau=0.9, seed=83, shared=True))
    _run(Case(g=4, d=64, c=3, n=5000, k_max=5000, tau=0.6, seed=84, shared=True))


def test_shared_split_scan_and_host_values(torch_cuda):
    """Few units -> the scan splits its groups (partial planes summed by k_grp_fin);
    host-mapped values through the union gather."""
    _run(Case(Hkv=1, g=64, n=32768, k_max=8192, seed=85, shared=True))
    _run(Case(B=2, Hkv=2, n=12000, k_max=3000, placement=1, seed=86, shared=True))


def test_shared_config3_full_size_sampled(torch_cuda):
    """BASELINE config 3 shape with shared selection (bench.py --shared-kv), sampled units."""
    case = Case(B=4, L=1, Hkv=8, g=32, n=131072, k_max=16384, placement=1, seed=3, shared=True)
    _run(case, units=[(0, 0), (3, 7)])


def test_shared_renorm_unsupported(torch_cuda):
    import paper_2507_19823_b200 as hc
    case = Case(n=500, k_max=100, renorm=1, seed=87, shared=True)
    kc, vs, q = build_gpu(case)
    with pytest.raises(hc.HcError):
        run_gpu_layer(case, kc, vs, q, 0)
