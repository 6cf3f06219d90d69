import sys, struct, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from harness import Case, build_gpu
import paper_2507_19823_b200 as hc
case = Case(B=1, L=1, Hkv=8, n=1 << 20, g=32, k_max=131072, tau=0.9, seed=0x48434154)
kc, vs, q = build_gpu(case)
bud = hc.budget(case.tau, case.k_max)
ws = hc.Workspace(kc.workspace_bytes(bud))
sk = torch.zeros((1, case.Hq), dtype=torch.int64, device="cuda")
si = torch.zeros((1, case.Hq, case.k_max), dtype=torch.int32, device="cuda")
sw = torch.zeros((1, case.Hq, case.k_max), dtype=torch.float32, device="cuda")
hc.decode_attention(q[0].contiguous(), kc, vs, 0, bud, sel_idx=si, sel_w=sw, sel_k=sk, ws=ws)
torch.cuda.synchronize()
raw = ws.t[: case.Hq * 128].cpu().numpy().view(np.uint8)
for h in range(case.Hq):
    r = raw[h * 128:(h + 1) * 128].tobytes()
    M, zmin = struct.unpack_from("<ii", r, 0); shift, = struct.unpack_from("<i", r, 20)
    ksel, kstar = struct.unpack_from("<qq", r, 64)
    tk, rlo, rhi, fsh, st = struct.unpack_from("<IIIiI", r, 108)
    print(f"row {h}: dmax {M - zmin} shift {shift} ksel {ksel} kstar {kstar} in-range {tk} range [{rlo},{rhi}] ({(rhi - rlo) >> shift} coarse bins) f {fsh} state {st}")
