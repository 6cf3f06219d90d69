"""Microbenchmark (dev tool): achievable HBM rate for gathering rows of 256 B (fp16 x 128)
by sorted random indices, with a plain triton kernel (not product code)."""
import json
import torch
import triton
import triton.language as tl


@triton.jit
def gather_sum(V, IDX, OUT, n, BLOCK: tl.constexpr):
    pid = tl.program_id(0)
    rows = pid * BLOCK + tl.arange(0, BLOCK)
    m = rows < n
    j = tl.load(IDX + rows, mask=m, other=0)
    dims = tl.arange(0, 128)
    v = tl.load(V + j[:, None].to(tl.int64) * 128 + dims[None, :], mask=m[:, None], other=0.0)
    tl.store(OUT + pid * 128 + dims, tl.sum(v.to(tl.float32), axis=0))


N, d = 1 << 23, 128
V = torch.randn(N, d, device="cuda").half()
res = {}
for frac in (0.0625, 0.125, 0.25, 1.0):
    k = int(N * frac)
    idx = torch.randperm(N, device="cuda")[:k].sort().values.int()
    for B in (64, 256):
        grid = (triton.cdiv(k, B),)
        out = torch.empty(grid[0], 128, device="cuda")
        for _ in range(3):
            gather_sum[grid](V, idx, out, k, BLOCK=B)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            gather_sum[grid](V, idx, out, k, BLOCK=B)
        e1.record(); torch.cuda.synchronize()
        res[f"frac{frac}_block{B}_GBps"] = round(k * d * 2 / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e9, 1)
print(json.dumps(res))
