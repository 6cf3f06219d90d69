"""CPU test of the sequence-sharded protocol (paper_2507_19823_b200.sharded.decode_layer) over
real multi-process collectives (torch.distributed gloo, world_size 2 and 3).

Each rank runs a test-side backend that computes its phase outputs from the CPU oracle's
integer scores and masses (the GPU backend runs the same phases as CUDA kernels, tested
in test_sharded_gpu.py).  The assembled selection must equal the UNSHARDED oracle's bit
for bit and the output must match within tolerance: the exchange (what is reduced, what
is gathered, how offsets are formed) is what is under test here."""
import os
import socket

import numpy as np
import pytest

NB = 4096


class OracleShard:
    """Phase backend for one rank built on oracle/ arithmetic (test infrastructure)."""

    def __init__(self, q, C_, P, V, tau, k_max, d):
        import oracle
        self.o = oracle
        self.q, self.P, self.V = q, P, V
        self.tau_q = oracle.tau_q(tau)
        self.k_max, self.d = k_max, d
        g = P.shape[0]
        _, Tfx, self.e = oracle.table(q, C_, g)
        self.z = np.stack([oracle.scores(Tfx[h], P, P.shape[1]) for h in range(q.shape[0])]).astype(np.int64)
        self.kap = [oracle.kappa(d, int(e)) for e in self.e]
        self.rows = q.shape[0]

    def _W(self, h, delta):
        return np.array([self.o.mass(int(x), self.kap[h]) for x in delta], dtype=object)

    def begin(self, q, layer):
        import torch
        st = np.stack([self.z.max(1), -self.z.min(1)], 1) if self.z.shape[1] else \
            np.full((self.rows, 2), -2 ** 31, np.int64)
        return torch.from_numpy(st.astype(np.int32))

    def hist1(self, layer, gst):
        import torch
        gst = gst.numpy().astype(np.int64)
        self.M, self.zmin = gst[:, 0], -gst[:, 1]
        h1 = np.zeros((self.rows, NB, 2), np.int64)
        self.shift = []
        for h in range(self.rows):
            bits = int(self.M[h] - self.zmin[h]).bit_length()
            sh = max(0, bits - 12)
            self.shift.append(sh)
            dl = self.M[h] - self.z[h]
            W = self._W(h, dl)
            for x, w in zip(dl >> sh, W):
                h1[h, x, 0] += 1
                h1[h, x, 1] += w
        return torch.from_numpy(h1)

    def hist2(self, layer, gst, gh1):
        import torch
        gh1 = gh1.numpy()
        self.bstar, self.cb, self.mb, self.S, self.theta = [], [], [], [], []
        h2 = np.zeros((self.rows, NB), np.int64)
        for h in range(self.rows):
            S = int(gh1[h, :, 1].sum(dtype=object))
            n = int(gh1[h, :, 0].sum())
            tau_all = self.tau_q >= 1 << 24
            theta = 0 if tau_all else -((-self.tau_q * S) // (1 << 24))
            cc = cm = 0
            bstar = NB
            cb = mb = 0
            for bi in range(NB):
                c, m = int(gh1[h, bi, 0]), int(gh1[h, bi, 1])
                if c and ((not tau_all and cm + m >= theta) or (self.k_max < n and cc + c >= self.k_max)):
                    bstar, cb, mb = bi, cc, cm
                    break
                cc += c
                cm += m
            self.bstar.append(bstar); self.cb.append(cb); self.mb.append(mb)
            self.S.append(S); self.theta.append(theta)
            if bstar < NB:
                dl = self.M[h] - self.z[h]
                sel = dl[(dl >> self.shift[h]) == bstar]
                for x in sel:
                    h2[h, x & ((1 << self.shift[h]) - 1)] += 1
        self.n_tot = None
        return torch.from_numpy(h2)

    def counts(self, layer, gh2):
        import torch
        gh2 = gh2.numpy()
        self.dstar, self.r = [], []
        cnt = np.zeros((self.rows, 2), np.int64)
        for h in range(self.rows):
            if self.bstar[h] >= NB:
                dstar, r = 2 ** 32 - 1, 0
            else:
                base = self.bstar[h] << self.shift[h]
                cc, cm = self.cb[h], self.mb[h]
                tau_all = self.tau_q >= 1 << 24
                for v in range(NB):
                    c = int(gh2[h, v])
                    if not c:
                        continue
                    w = self.o.mass(base | v, self.kap[h])
                    rt = rc = None
                    if not tau_all and w and cm + c * w >= self.theta[h]:
                        rt = max(1, -((-(self.theta[h] - cm)) // w))
                    if cc + c >= self.k_max:
                        rc = self.k_max - cc
                    if rt is not None or rc is not None:
                        r = min(x for x in (rt, rc) if x is not None)
                        dstar = base | v
                        break
                    cc += c
                    cm += c * w
            self.dstar.append(dstar); self.r.append(r)
            dl = self.M[h] - self.z[h]
            cnt[h] = [(dl < dstar).sum(), (dl == dstar).sum()]
        self.cnt = cnt
        return torch.from_numpy(cnt)

    def finish(self, layer, allc, rank, world, base):
        import torch
        allc = allc.numpy()
        out = np.zeros((self.rows, self.d), np.float64)
        self.sel = []
        for h in range(self.rows):
            s_before = int(allc[:rank, h, 0].sum())
            t_before = int(allc[:rank, h, 1].sum())
            r = self.r[h]
            pos = s_before + min(t_before, r)
            t_run = t_before
            dl = self.M[h] - self.z[h]
            mine = []
            for j, x in enumerate(dl):
                take = x < self.dstar[h]
                if x == self.dstar[h]:
                    take = t_run < r
                    t_run += 1
                if take:
                    w = self.o.mass(int(x), self.kap[h]) / self.S[h]
                    mine.append((pos, base + j, w))
                    out[h] += w * self.V[j].astype(np.float64)
                    pos += 1
            self.sel.append(mine)
        return torch.from_numpy(out)


def _worker(rank, world, port, q, C_, P, V, tau, k_max, bounds, res):
    import torch.distributed as dist
    from paper_2507_19823_b200.sharded import TorchComm, decode_layer
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    a, b = bounds[rank], bounds[rank + 1]
    sh = OracleShard(q, C_, P[:, a:b], V[a:b], tau, k_max, q.shape[1])
    out = decode_layer(sh, TorchComm(), q, 0, a)
    res.put((rank, out.numpy(), sh.sel))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,tau,k_max", [(2, 1500, 0.9, 300), (3, 1200, 0.6, 5000),
                                               (2, 800, 1.0, 100)])
def test_gloo_sharded_protocol_matches_unsharded_oracle(world, n, tau, k_max):
    import torch.multiprocessing as mp
    import oracle
    import synth
    rng = np.random.default_rng(world * n)
    G, d, g, c = 4, 64, 16, 64
    q = (rng.standard_normal((G, d)) * 2.0).astype(np.float16)
    C_ = rng.standard_normal((g, c, d // g)).astype(np.float32)
    P = rng.integers(0, c, size=(g, n)).astype(np.uint16)
    P[:, 100:140] = P[:, 0:1]          # exact score ties across the shard boundary region
    V = synth.gen_values(5, 0, 0, 0, d, 0, n)
    bounds = [int(x) for x in np.linspace(0, n, world + 1)]
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    res = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, C_, P, V, tau, k_max, bounds, res))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [res.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.decode_unit(q, C_, P, n, V, tau, k_max)
    for h in range(G):
        sel = sorted(x for (_, _, sl) in got for x in sl[h])
        assert [p for p, _, _ in sel] == list(range(len(sel)))  # positions tile 0..k-1
        assert [j for _, j, _ in sel] == ref["idx"][h].tolist()
        assert np.allclose([w for _, _, w in sel], ref["w"][h], rtol=1e-12)
    outs = [o for _, o, _ in got]
    for o in outs:
        assert np.allclose(o, outs[0])
        assert np.allclose(o, ref["out"], atol=1e-9, rtol=1e-9)
