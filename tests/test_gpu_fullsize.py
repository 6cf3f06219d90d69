"""Parity at the BASELINE configurations' full sizes (VERDICT r1 "close parity at every
configuration the north_star names"): the sequence-sharded decode run as R
lock-step virtual shards on one GPU must equal the UNSHARDED oracle -- k_sel and the full
kept index set bit for bit (Eq. 4), weights to fp32 rounding and outputs
within the north_star tolerance (Eq. 5) -- on sampled (b, kv) units, all G heads.

  config 5 (P:46 / P:423, the paper's 4M-token headline): one layer at n = 2^22, g = 32,
           k_max = 524,288, values in host pinned memory (zero-copy), R = 8 shards;
  config 4: n = 2^20, k_max = 131,072, values in HBM, R = 2 / 4 / 8;
  sharded + host-mapped values at a ragged size (every unit checked).

The oracle side is composed from the oracle's stage functions with only the kept value rows
generated (tests/harness.py oracle_unit_rows), so a 4M-token unit fits in host memory."""
import numpy as np
import pytest

from harness import Case, compare_unit, oracle_unit, oracle_unit_rows, run_sharded_virtual, shard_caches

pytestmark = pytest.mark.gpu

_ORACLE = {}


def _oracle(case, b, kv, key):
    k = (key, b, kv)
    if k not in _ORACLE:
        _ORACLE[k] = oracle_unit_rows(case, b, 0, kv)
    return _ORACLE[k]


def _check(case, gpu, units, key):
    for b, kv in units:
        st = compare_unit(case, gpu, _oracle(case, b, kv, key), b, kv, check_z=False)
        print(f"{key} unit (b={b}, kv={kv}): k*={st['kstar']} max|out-oracle|={st['max_abs']:.2e}")


def _config4():
    return Case(B=1, L=1, Hkv=8, n=1 << 20, g=32, k_max=131072, tau=0.9, seed=0x48434154)


@pytest.mark.parametrize("R", [2, 4, 8])
def test_config4_full_size_sharded(R):
    """BASELINE config 4: 1M context, 12.5 % budget (k_max = 131,072), V in HBM."""
    import torch
    case = _config4()
    parts = shard_caches(case, R)
    gpu = run_sharded_virtual(case, parts)
    assert (gpu["k"] == case.k_max).all() or (gpu["k"] <= case.k_max).all()
    _check(case, gpu, [(0, 0), (0, 5)], "c4")
    del parts
    torch.cuda.empty_cache()


def test_config4_full_size_unsharded():
    """BASELINE config 4 shape through hc_decode_attention on ONE GPU (the launch bench.py
    --config 4 times: K1 count histogram, K2 exact S / refine, K3 write), sampled units."""
    import torch
    from harness import build_gpu, run_gpu_layer
    case = _config4()
    kc, vs, q = build_gpu(case)
    gpu = run_gpu_layer(case, kc, vs, q, 0, with_debug=False)
    _check(case, gpu, [(0, 0), (0, 5)], "c4")
    del kc, vs, q
    torch.cuda.empty_cache()


def test_config5_one_layer_sharded_host_values():
    """BASELINE config 5: 4M-token context (2^22), g = 32, k_max = 524,288, values offloaded to
    host pinned memory, sequence-sharded R = 8 (here: 8 lock-step virtual shards on one GPU);
    one layer of the 32."""
    import torch
    import paper_2507_19823_b200 as hc
    case = Case(B=1, L=1, Hkv=8, n=1 << 22, g=32, k_max=524288, tau=0.9, seed=0x48434154,
                placement=hc.HC_V_HOST_MAPPED)
    parts = shard_caches(case, 8)
    gpu = run_sharded_virtual(case, parts)
    _check(case, gpu, [(0, 0), (0, 3)], "c5")
    k = gpu["k"][0]
    print(f"config 5 layer: k_sel/n = {k.mean() / case.n:.4f} (cap {case.k_max / case.n:.4f})")
    del parts
    torch.cuda.empty_cache()


@pytest.mark.parametrize("R,n,tau,k_max", [(3, 50001, 0.9, 6000), (5, 200003, 0.7, 100000),
                                           (2, 9000, 1.0, 9000)])
def test_sharded_host_values_all_units(R, n, tau, k_max):
    """Sequence-sharded finish over host-mapped values (the GQA-union gather on each rank's
    slice of every kept list): every unit of a ragged multi-shard case vs the oracle."""
    import paper_2507_19823_b200 as hc
    case = Case(B=2, Hkv=2, n=n, tau=tau, k_max=k_max, seed=90 + R, placement=hc.HC_V_HOST_MAPPED)
    gpu = run_sharded_virtual(case, shard_caches(case, R))
    for b in range(case.B):
        for kv in range(case.Hkv):
            compare_unit(case, gpu, oracle_unit(case, b, 0, kv), b, kv, check_z=False)
