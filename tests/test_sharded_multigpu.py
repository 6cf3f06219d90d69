"""The sequence-sharded decode across REAL GPUs: one process
per GPU, the C entry hc_decode_attention_sharded issuing its NCCL exchanges on the stream, ranks
holding contiguous token ranges of the context.  Kept index sets must equal the UNSHARDED oracle
bit for bit and the output (identical on every rank after the final all-reduce) must be within
the north_star tolerance.  Skipped unless the box has >= 2 GPUs (the round's boxes have one;
the same kernels are covered on one GPU by the lock-step virtual shards in test_sharded_gpu.py
and the protocol by the gloo world-2/3 test in test_sharded_cpu.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case_kw, result_dir):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from harness import Case, shard_caches
    import paper_2507_19823_b200 as hc
    from paper_2507_19823_b200.sharded import CAbiShard
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    case = Case(**case_kw)
    (kc, vs, base), = shard_caches(case, world, device=f"cuda:{rank}", only=rank)
    comm = hc.NcclComm.from_process_group()
    sh = CAbiShard(kc, vs, hc.budget(case.tau, case.k_max), rank, world, base, comm, device=f"cuda:{rank}")
    q = torch.from_numpy(np.stack([case.query(b, 0) for b in range(case.B)])).cuda()
    out = sh.decode_layer(q, 0)
    torch.cuda.synchronize()
    idx = [torch.empty_like(sh.sel_idx) for _ in range(world)]
    dist.all_gather(idx, sh.sel_idx)
    if rank == 0:
        np.savez(os.path.join(result_dir, "res.npz"), out=out.cpu().numpy(),
                 idx=torch.stack(idx).amax(0).cpu().numpy(), k=sh.sel_k.cpu().numpy())
    comm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,tau,k_max", [(50021, 0.9, 4000), (90001, 0.99, 100000)])
def test_nccl_sharded_two_gpus_match_unsharded_oracle(tmp_path, n, tau, k_max):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp
    from harness import Case, TOL_ABS, TOL_REL, oracle_unit
    world = 2
    case_kw = dict(B=1, Hkv=2, n=n, tau=tau, k_max=k_max, seed=4242)
    mp.spawn(_worker, args=(world, _free_port(), case_kw, str(tmp_path)), nprocs=world, join=True)
    res = np.load(tmp_path / "res.npz")
    case = Case(**case_kw)
    out = res["out"].reshape(case.B, case.Hq, -1)
    idx = res["idx"].reshape(case.B, case.Hq, -1)
    ks = res["k"].reshape(case.B, case.Hq)
    for b in range(case.B):
        for kv in range(case.Hkv):
            ref = oracle_unit(case, b, 0, kv)
            for h in range(case.G):
                hq = kv * case.G + h
                k = int(ks[b, hq])
                assert k == int(ref["k_sel"][h])
                assert np.array_equal(idx[b, hq, :k], ref["idx"][h])
                err = np.abs(out[b, hq] - ref["out"][h])
                assert np.all(err <= TOL_ABS + TOL_REL * np.abs(ref["out"][h]))
