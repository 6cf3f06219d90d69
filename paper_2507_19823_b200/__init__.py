"""hcattn-b200: B200-native (sm_100a) HCAttention decode hot path.

Thin ctypes binding over the C ABI in include/hc.h (libhc.so, built in-tree by
paper_2507_19823_b200/build.py).  Argument marshalling only: every stage of the
path runs in our CUDA kernels.  PyTorch provides device / pinned memory and the
stream.  There is NO CPU fallback: if libhc.so is missing, or no CUDA device is
present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhc.so")
MAX_LAYERS = 256

HC_OK, HC_ERR_ARG, HC_ERR_SHAPE, HC_ERR_RANGE, HC_ERR_CAPACITY, HC_ERR_EMPTY, HC_ERR_CUDA, \
    HC_ERR_NCCL, HC_ERR_UNSUPPORTED, HC_ERR_WORKSPACE = range(10)
HC_V_DEVICE, HC_V_HOST_MAPPED = 0, 1

EXPORTS = ["hc_last_error", "hc_version", "hc_launch_count", "hc_profile_scan_events",
           "hc_profile_eq3_events",
           "hc_codebook_absmax", "hc_quantize_keys", "hc_append_kv",
           "hc_decode_workspace_bytes", "hc_decode_attention", "hc_append_decode_attention",
           "hc_select_workspace_bytes",
           "hc_select_topk", "hc_host_weighted_sum", "hc_enqueue_host_weighted_sum",
           "hc_shard_workspace_bytes", "hc_shard_begin", "hc_shard_hist1",
           "hc_shard_hist2", "hc_shard_counts", "hc_shard_finish", "hc_kmeans_workspace_bytes",
           "hc_kmeans_step", "hc_pack_codes13", "hc_blockwise_attention", "hc_prefill_append",
           "hc_host_weighted_sum_range", "hc_enqueue_host_weighted_sum_range", "hc_gather_values",
           "hc_add_partial", "hc_host_register", "hc_host_unregister", "hc_host_worker_create",
           "hc_host_worker_destroy", "hc_host_worker_add_job", "hc_host_worker_submit",
           "hc_host_worker_wait", "hc_host_worker_status", "hc_host_worker_pause",
           "hc_nccl_get_unique_id", "hc_nccl_comm_init", "hc_nccl_comm_destroy",
           "hc_decode_sharded_workspace_bytes", "hc_decode_attention_sharded"]


class HcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hc status {status}: {msg}")
        self.status = status


class hc_vq(C.Structure):
    _fields_ = [("d", C.c_int32), ("g", C.c_int32), ("c", C.c_int32), ("cbg", C.c_int32),
                ("lut_bits", C.c_int32), ("code_bits", C.c_int32)]


class hc_budget(C.Structure):
    _fields_ = [("tau", C.c_float), ("k_max", C.c_int64), ("renorm", C.c_int32),
                ("select_only", C.c_int32), ("shared_kv", C.c_int32)]


class hc_kcache(C.Structure):
    _fields_ = [("B", C.c_int32), ("L", C.c_int32), ("Hkv", C.c_int32), ("G", C.c_int32),
                ("vq", hc_vq), ("n_cap", C.c_int64), ("codes", C.c_void_p),
                ("codebook", C.c_void_p), ("cb_absmax", C.c_void_p), ("res_cap", C.c_int32), ("res_k", C.c_void_p),
                ("res_v", C.c_void_p), ("n_q", C.c_int64 * MAX_LAYERS),
                ("n_res", C.c_int32 * MAX_LAYERS)]


class hc_vstore(C.Structure):
    _fields_ = [("placement", C.c_int32), ("base", C.c_void_p), ("n_cap", C.c_int64)]


class hc_decode_debug(C.Structure):
    _fields_ = [("z", C.c_void_p), ("e", C.c_void_p), ("S", C.c_void_p), ("M", C.c_void_p),
                ("kstar", C.c_void_p)]


_lib = None


def lib():
    """Load libhc.so; raise loudly if it was not built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2507_19823_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        p, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        L.hc_last_error.restype = C.c_char_p
        L.hc_version.restype = C.c_char_p
        L.hc_launch_count.restype = C.c_uint64
        L.hc_profile_scan_events.argtypes = [p, p]
        L.hc_profile_scan_events.restype = i32
        L.hc_profile_eq3_events.argtypes = [p, p]
        L.hc_profile_eq3_events.restype = i32
        L.hc_codebook_absmax.argtypes = [p, hc_vq, i32, p, p]
        L.hc_codebook_absmax.restype = i32
        L.hc_quantize_keys.argtypes = [p, i64, p, hc_vq, p, i64, p]
        L.hc_quantize_keys.restype = i32
        L.hc_append_kv.argtypes = [C.POINTER(hc_kcache), C.POINTER(hc_vstore), i32, p, p, p]
        L.hc_append_kv.restype = i32
        L.hc_decode_workspace_bytes.argtypes = [C.POINTER(hc_kcache), hc_budget]
        L.hc_decode_workspace_bytes.restype = C.c_size_t
        L.hc_decode_attention.argtypes = [p, C.POINTER(hc_kcache), C.POINTER(hc_vstore), i32,
                                          hc_budget, p, p, p, p, C.POINTER(hc_decode_debug), p,
                                          C.c_size_t, p]
        L.hc_decode_attention.restype = i32
        L.hc_append_decode_attention.argtypes = [p, C.POINTER(hc_kcache), C.POINTER(hc_vstore), i32, p, p,
                                                 hc_budget, p, p, p, p, p, C.c_size_t, p]
        L.hc_append_decode_attention.restype = i32
        L.hc_select_workspace_bytes.argtypes = [i64, i64, hc_budget]
        L.hc_select_workspace_bytes.restype = C.c_size_t
        L.hc_select_topk.argtypes = [p, i64, i64, i32, hc_budget, p, p, p, p, C.c_size_t, p]
        L.hc_select_topk.restype = i32
        hw = [p, p, p, i64, i64, p, i64, i64, i64, i32, i32, i32, p, i32]
        L.hc_host_weighted_sum.argtypes = hw
        L.hc_host_weighted_sum.restype = i32
        L.hc_enqueue_host_weighted_sum.argtypes = hw + [p]
        L.hc_enqueue_host_weighted_sum.restype = i32
        hr = [p, p, p, i64, i64, p, i64, i64, i64, i32, i32, i32, i64, i64, p, i32]
        L.hc_host_weighted_sum_range.argtypes = hr
        L.hc_host_weighted_sum_range.restype = i32
        L.hc_enqueue_host_weighted_sum_range.argtypes = hr + [p]
        L.hc_enqueue_host_weighted_sum_range.restype = i32
        L.hc_gather_values.argtypes = [C.POINTER(hc_kcache), C.POINTER(hc_vstore), i32, p, p, p, i64,
                                       i64, i64, p, p, C.c_size_t, p]
        L.hc_gather_values.restype = i32
        L.hc_add_partial.argtypes = [p, p, i64, p]
        L.hc_add_partial.restype = i32
        L.hc_host_register.argtypes = [p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.hc_host_register.restype = i32
        L.hc_host_unregister.argtypes = [p]
        L.hc_host_unregister.restype = i32
        L.hc_host_worker_create.argtypes = [i32, i32, C.c_double, C.POINTER(C.c_void_p)]
        L.hc_host_worker_destroy.argtypes = [p]
        L.hc_host_worker_add_job.argtypes = [p, i64, i64, p, i64, i64, i32, i32, i32, p, C.POINTER(i32)]
        L.hc_host_worker_submit.argtypes = [p, i32, p, p, p, i64, i64, i64, p]
        L.hc_host_worker_wait.argtypes = [p, i32, p]
        L.hc_host_worker_status.argtypes = [p]
        L.hc_host_worker_pause.argtypes = [p, i32]
        for f in ("hc_host_worker_create", "hc_host_worker_destroy", "hc_host_worker_add_job",
                  "hc_host_worker_submit", "hc_host_worker_wait", "hc_host_worker_status",
                  "hc_host_worker_pause"):
            getattr(L, f).restype = i32
        L.hc_nccl_get_unique_id.argtypes = [p]
        L.hc_nccl_get_unique_id.restype = i32
        L.hc_nccl_comm_init.argtypes = [C.POINTER(C.c_void_p), i32, p, i32]
        L.hc_nccl_comm_init.restype = i32
        L.hc_nccl_comm_destroy.argtypes = [p]
        L.hc_nccl_comm_destroy.restype = i32
        L.hc_decode_sharded_workspace_bytes.argtypes = [C.POINTER(hc_kcache), hc_budget, i32]
        L.hc_decode_sharded_workspace_bytes.restype = C.c_size_t
        L.hc_decode_attention_sharded.argtypes = [p, C.POINTER(hc_kcache), C.POINTER(hc_vstore), i32,
                                                  hc_budget, p, p, p, p, i32, i32, i64, p, p,
                                                  C.c_size_t, p]
        L.hc_decode_attention_sharded.restype = i32
        L.hc_blockwise_attention.argtypes = [p, p, p, i64, i32, i32, i32, i64, p, p]
        L.hc_blockwise_attention.restype = i32
        L.hc_prefill_append.argtypes = [C.POINTER(hc_kcache), C.POINTER(hc_vstore), i32, p, p, i64, p]
        L.hc_prefill_append.restype = i32
        L.hc_pack_codes13.argtypes = [p, i64, i64, i64, p, i64, p]
        L.hc_pack_codes13.restype = i32
        L.hc_kmeans_workspace_bytes.argtypes = [hc_vq, i64]
        L.hc_kmeans_workspace_bytes.restype = C.c_size_t
        L.hc_kmeans_step.argtypes = [p, i64, p, i64, hc_vq, p, p, p, p, C.c_size_t, p]
        L.hc_kmeans_step.restype = i32
        KC, VS = C.POINTER(hc_kcache), C.POINTER(hc_vstore)
        L.hc_shard_workspace_bytes.argtypes = [KC, hc_budget]
        L.hc_shard_workspace_bytes.restype = C.c_size_t
        L.hc_shard_begin.argtypes = [p, KC, VS, i32, hc_budget, p, p, C.c_size_t, p]
        L.hc_shard_hist1.argtypes = [KC, VS, i32, hc_budget, p, p, p, C.c_size_t, p]
        L.hc_shard_hist2.argtypes = [KC, VS, i32, hc_budget, p, p, p, p, C.c_size_t, p]
        L.hc_shard_counts.argtypes = [KC, VS, i32, hc_budget, p, p, p, C.c_size_t, p]
        L.hc_shard_finish.argtypes = [KC, VS, i32, hc_budget, p, i32, i32, i64, p, p, p, p, p,
                                      C.c_size_t, p]
        for f in ("hc_shard_begin", "hc_shard_hist1", "hc_shard_hist2", "hc_shard_counts",
                  "hc_shard_finish"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _check(st: int):
    if st != HC_OK:
        raise HcError(st, lib().hc_last_error().decode())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def version() -> str:
    return lib().hc_version().decode()


def launch_count() -> int:
    """Kernels enqueued/captured by libhc so far (bench.py's gpu_launches)."""
    return int(lib().hc_launch_count())


def profile_scan_events(begin, end):
    """Record torch.cuda.Event's around the next scan launch (one-shot)."""
    _check(lib().hc_profile_scan_events(C.c_void_p(begin.cuda_event) if begin is not None else None,
                                        C.c_void_p(end.cuda_event) if end is not None else None))


def profile_eq3_events(begin, end):
    """Record torch.cuda.Event's around the next decode call's Eq. 3 stage (table + scan)."""
    _check(lib().hc_profile_eq3_events(C.c_void_p(begin.cuda_event) if begin is not None else None,
                                       C.c_void_p(end.cuda_event) if end is not None else None))


def budget(tau: float, k_max: int, renorm: bool = False, select_only: bool = False,
           shared_kv: bool = False) -> hc_budget:
    """R5 budget; shared_kv=True -> one selection per KV head (R8, include/hc.h)."""
    return hc_budget(float(tau), int(k_max), int(bool(renorm)), int(bool(select_only)),
                     int(bool(shared_kv)))


# ----------------------------------------------------------------------------- encode
def quantize_keys(keys, codebook, g: int, codes=None, stream=None):
    """R1: keys fp16 [rows][d] (cuda), codebook fp32 [cbg][c][d/g]
    -> codes int16-view-of-u16 [g][rows] (group-major)."""
    import torch
    rows, d = keys.shape
    cbg, c, dbar = codebook.shape
    if codes is None:
        codes = torch.empty((g, max(rows, 1)), dtype=torch.int16, device=keys.device)
    st = lib().hc_quantize_keys(_ptr(keys), rows, _ptr(codebook), hc_vq(d, g, c, cbg), _ptr(codes),
                                codes.shape[1], _stream(stream))
    _check(st)
    return codes


def kmeans_step(keys, sample, codebook, counts, g: int, labels=None, ws=None, stream=None):
    """f4: one MiniBatchKMeans step on the GPU (include/hc.h hc_kmeans_step).
    keys fp16 [n_keys][d], sample int64 [b] (cuda), codebook fp32 [cbg][c][d/g] and counts
    int64 [cbg][c] updated in place; labels int16-view-of-u16 [g][b] (optional)."""
    import torch
    n_keys, d = keys.shape
    cbg, c, dbar = codebook.shape
    b = sample.shape[0]
    vq = hc_vq(d, g, c, cbg)
    if ws is None:
        ws = Workspace(int(lib().hc_kmeans_workspace_bytes(vq, b)), keys.device)
    st = lib().hc_kmeans_step(_ptr(keys), n_keys, _ptr(sample), b, vq, _ptr(codebook),
                              _ptr(counts), _ptr(labels) if labels is not None else None,
                              _ptr(ws.t), ws.nbytes, _stream(stream))
    _check(st)
    return codebook, counts


def blockwise_attention(q, k, v, bs: int, out=None, stream=None):
    """f4 (iii), App. B: q [n][Hq][d], k, v [n][Hkv][d] fp16 (cuda) -> out [n][Hq][d] fp32."""
    import torch
    n, Hq, d = q.shape
    Hkv = k.shape[1]
    if out is None:
        out = torch.empty((n, Hq, d), dtype=torch.float32, device=q.device)
    _check(lib().hc_blockwise_attention(_ptr(q), _ptr(k), _ptr(v), n, Hq, Hkv, d, bs, _ptr(out),
                                        _stream(stream)))
    return out


def pack_codes13(codes16, n: int, n_cap: int, out=None, stream=None):
    """f3(ii): u16 codes [..., >= n] (int16 view, cuda) -> packed strips [..., 13 n_cap / 8] u8."""
    import torch
    lead = codes16.shape[:-1]
    strips = 1
    for x in lead:
        strips *= x
    if out is None:
        out = torch.zeros(tuple(lead) + (n_cap * 13 // 8,), dtype=torch.uint8, device=codes16.device)
    if not (out.is_contiguous() and codes16.is_contiguous()):
        raise ValueError("pack_codes13 needs contiguous tensors (strips back to back)")
    _check(lib().hc_pack_codes13(_ptr(codes16), strips, n, codes16.shape[-1], _ptr(out), n_cap,
                                 _stream(stream)))
    return out


def train_codebook(keys, g: int, c: int, iters: int = 200, batch: int = 10000, seed: int = 0,
                   cbg=None, init=None):
    """MiniBatchKMeans codebook training (max 200 iterations, batch 10,000) from the
    key matrix keys fp16 [N][d] (cuda).  init: fp32 [cbg][c][d/g] (default: the sub-vectors
    of c seeded distinct key rows).  Batches are seeded splitmix64 draws (synth)."""
    import numpy as np
    import torch

    import synth
    N, d = keys.shape
    cbg = g if cbg is None else cbg
    dbar = d // g
    if init is None:
        rows = synth.sample_rows(seed, 0, N, c)
        k0 = keys[torch.from_numpy(rows).to(keys.device)].float().view(c, g, dbar)
        init = (k0.permute(1, 0, 2).contiguous() if cbg == g else k0[:, 0, :].unsqueeze(0).contiguous())
    C_ = init.clone().float().contiguous()
    counts = torch.zeros((cbg, c), dtype=torch.int64, device=keys.device)
    ws = Workspace(int(lib().hc_kmeans_workspace_bytes(hc_vq(d, g, c, cbg), batch)), keys.device)
    for it in range(iters):
        sample = torch.from_numpy(synth.sample_rows(seed, 1 + it, N, batch).astype(np.int64)).to(keys.device)
        kmeans_step(keys, sample, C_, counts, g, ws=ws)
    return C_, counts


# ----------------------------------------------------------------------------- caches
class HostBuffer:
    """Page-locked, device-mapped host memory for the offloaded value store (A8):
    an anonymous mapping aligned to and advised for 2 MiB transparent huge pages
    (madvise MADV_HUGEPAGE), first-touched by parallel threads, then registered with
    hc_host_register.  Random 256-byte row reads by host threads and by the GPU then walk
    one page-table entry per 2 MiB instead of per 4 KiB (a 34 GB store has 8.4 M 4-KiB PTEs,
    67 MB of page tables -- a DRAM miss per row on top of the row itself)."""

    HUGE = 2 << 20

    def __init__(self, nbytes: int, huge: bool = True, threads: int = 16):
        import concurrent.futures as cf
        import mmap
        HP = self.HUGE
        self.size = max(HP, (int(nbytes) + HP - 1) // HP * HP)
        self.mm = mmap.mmap(-1, self.size + HP, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        self._anchor = C.c_char.from_buffer(self.mm)
        base = C.addressof(self._anchor)
        self.offset = (base + HP - 1) // HP * HP - base
        self.addr = base + self.offset
        self.huge = False
        if huge:
            libc = C.CDLL(None, use_errno=True)
            libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
            self.huge = libc.madvise(self.addr, self.size, 14) == 0  # MADV_HUGEPAGE
        step = max(HP, (self.size // max(1, threads)) // HP * HP)
        with cf.ThreadPoolExecutor(max_workers=threads) as ex:  # first touch (ctypes drops the GIL)
            list(ex.map(lambda o: C.memset(self.addr + o, 0, min(step, self.size - o)),
                        range(0, self.size, step)))
        dev = C.c_void_p()
        _check(lib().hc_host_register(self.addr, self.size, C.byref(dev)))
        self.dev = int(dev.value)
        self.registered = True

    def tensor(self, shape, dtype):
        import torch
        n = 1
        for x in shape:
            n *= int(x)
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        mv = memoryview(self.mm)[self.offset:self.offset + nbytes]
        return torch.frombuffer(mv, dtype=dtype).view(*shape)

    def device_pointer(self, host_ptr: int) -> int:
        return self.dev + (int(host_ptr) - self.addr)

    def close(self):
        if getattr(self, "registered", False):
            lib().hc_host_unregister(self.addr)
            self.registered = False

    def __del__(self):  # unregister before the mapping goes (its addresses get reused)
        try:
            self.close()
        except Exception:
            pass


@dataclass
class VStore:
    """Value store [B][L][Hkv][n_cap][d] fp16, in HBM or host-pinned mapped memory."""
    tensor: object           # torch fp16 tensor (cuda, or pinned cpu)
    placement: int
    n_cap: int
    host: HostBuffer | None = None

    @staticmethod
    def allocate(B, L, Hkv, n_cap, d, placement=HC_V_DEVICE, device="cuda", huge=True):
        """placement HC_V_HOST_MAPPED: a HostBuffer (2 MiB THP-advised, registered) unless
        huge=False (torch pinned memory, 4 KiB pages)."""
        import torch
        if placement == HC_V_DEVICE:
            t = torch.empty((B, L, Hkv, n_cap, d), dtype=torch.float16, device=device)
            return VStore(t, placement, n_cap)
        if huge:
            hb = HostBuffer(B * L * Hkv * n_cap * d * 2)
            if hb.dev == hb.addr:  # UVA: host and device addresses coincide (callers rely on it)
                return VStore(hb.tensor((B, L, Hkv, n_cap, d), torch.float16), placement, n_cap, hb)
            hb.close()
        t = torch.empty((B, L, Hkv, n_cap, d), dtype=torch.float16, pin_memory=True)
        return VStore(t, placement, n_cap)

    def batch_view(self, b0: int, nb: int) -> "VStore":
        """Sequences [b0, b0+nb) of the store (same memory)."""
        return VStore(self.tensor[b0:b0 + nb], self.placement, self.n_cap, self.host)

    def struct(self) -> hc_vstore:
        ptr = self.tensor.data_ptr()
        if self.placement == HC_V_HOST_MAPPED:
            ptr = self.host.device_pointer(ptr) if self.host is not None else host_device_pointer(ptr)
        return hc_vstore(self.placement, ptr, self.n_cap)


def host_device_pointer(host_ptr: int) -> int:
    """Device-accessible alias of pinned host memory.  With unified virtual addressing
    (always on for 64-bit Linux + sm_100), memory from cudaHostAlloc / pin_memory is
    mapped into every device's address space at the same address."""
    return host_ptr


class KCache:
    """Quantized key cache of all layers (hc_kcache).  Device tensors:
    codes [B][L][Hkv][g][n_cap] (u16 as int16), codebook [L][cbg][c][d/g] fp32,
    optional recent window res_k/res_v [B][L][Hkv][W][d] fp16."""

    def __init__(self, B, L, Hkv, G, d, g, c, n_cap, codebook, cbg=None, res_cap=0,
                 codes=None, device="cuda", lut_bits=16, code_bits=16):
        import torch
        cbg = g if cbg is None else cbg
        self.B, self.L, self.Hkv, self.G, self.d, self.g, self.c, self.cbg = B, L, Hkv, G, d, g, c, cbg
        self.n_cap, self.res_cap = n_cap, res_cap
        self.code_bits = code_bits
        self.codebook = codebook
        if code_bits == 13:  # packed strips (include/hc.h HC_STRIP13_BYTES)
            self.codes = codes if codes is not None else torch.zeros(
                (B, L, Hkv, g, n_cap * 13 // 8), dtype=torch.uint8, device=device)
        else:
            self.codes = codes if codes is not None else torch.zeros(
                (B, L, Hkv, g, n_cap), dtype=torch.int16, device=device)
        if res_cap > 0:
            self.res_k = torch.zeros((B, L, Hkv, res_cap, d), dtype=torch.float16, device=device)
            self.res_v = torch.zeros((B, L, Hkv, res_cap, d), dtype=torch.float16, device=device)
        else:
            self.res_k = self.res_v = None
        s = hc_kcache()
        s.B, s.L, s.Hkv, s.G = B, L, Hkv, G
        s.vq = hc_vq(d, g, c, cbg, lut_bits, code_bits)
        s.n_cap = n_cap
        s.codes = self.codes.data_ptr()
        s.codebook = codebook.data_ptr()
        # R2's codebook constant max_m |C[l][ci][m][e]|, computed once on the device
        self.cb_absmax = torch.empty((L, cbg, d // g), dtype=torch.float32, device=codebook.device)
        _check(lib().hc_codebook_absmax(_ptr(codebook), hc_vq(d, g, c, cbg), L,
                                        _ptr(self.cb_absmax), _stream()))
        s.cb_absmax = self.cb_absmax.data_ptr()
        s.res_cap = res_cap
        s.res_k = self.res_k.data_ptr() if self.res_k is not None else None
        s.res_v = self.res_v.data_ptr() if self.res_v is not None else None
        self.s = s

    @property
    def Hq(self):
        return self.G * self.Hkv

    def n_q(self, layer):
        return self.s.n_q[layer]

    def n_res(self, layer):
        return self.s.n_res[layer]

    def load_codes16(self, codes16, n: int, stream=None):
        """Fill the cache's codes from u16 codes [B][L][Hkv][g][>= n] (int16 view, cuda): a
        copy for 16-bit caches, hc_pack_codes13 for packed ones."""
        if self.code_bits != 13:
            self.codes[..., :n] = codes16[..., :n]
            return
        strips = self.B * self.L * self.Hkv * self.g
        _check(lib().hc_pack_codes13(_ptr(codes16), strips, n, codes16.shape[-1], _ptr(self.codes),
                                     self.n_cap, _stream(stream)))

    def prefill_append(self, layer, k, v, vstore, stream=None):
        """hc_prefill_append: k, v [B][n][Hkv][d] fp16 (cuda) -> codes / values at
        positions [n_q, n_q + n) of `layer` (bulk R1 encode)."""
        vs = vstore.struct()
        _check(lib().hc_prefill_append(C.byref(self.s), C.byref(vs), layer, _ptr(k), _ptr(v),
                                       k.shape[1], _stream(stream)))

    def set_counts(self, layer, n_q, n_res=0):
        self.s.n_q[layer] = n_q
        self.s.n_res[layer] = n_res

    def append(self, layer, k_new, v_new, vstore: VStore, stream=None):
        """hc_append_kv: k_new, v_new fp16 [B][Hkv][d] (cuda)."""
        vs = vstore.struct()
        _check(lib().hc_append_kv(C.byref(self.s), C.byref(vs), layer, _ptr(k_new), _ptr(v_new),
                                  _stream(stream)))

    def workspace_bytes(self, bud: hc_budget) -> int:
        return int(lib().hc_decode_workspace_bytes(C.byref(self.s), bud))

    def batch_view(self, b0: int, nb: int) -> "KCache":
        """The sequences [b0, b0+nb) as a cache of their own (same memory; pointers offset
        along the batch-major layouts).  Token counts are copied and advance separately, so
        every view of a batch must see the same appends (e.g. micro-batch pipelining)."""
        if not (0 <= b0 and nb >= 1 and b0 + nb <= self.B):
            raise ValueError("batch view out of range")
        v = object.__new__(KCache)
        v.__dict__.update(self.__dict__)
        v.B = nb
        v.codes = self.codes[b0:b0 + nb]
        v.res_k = self.res_k[b0:b0 + nb] if self.res_k is not None else None
        v.res_v = self.res_v[b0:b0 + nb] if self.res_v is not None else None
        s = hc_kcache()
        C.memmove(C.addressof(s), C.addressof(self.s), C.sizeof(hc_kcache))
        s.B = nb
        s.codes = v.codes.data_ptr()
        s.res_k = v.res_k.data_ptr() if v.res_k is not None else None
        s.res_v = v.res_v.data_ptr() if v.res_v is not None else None
        v.s = s
        return v


class Workspace:
    def __init__(self, nbytes, device="cuda"):
        import torch
        self.t = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)

    @property
    def nbytes(self):
        return self.t.numel()


def decode_attention(q, kc: KCache, vstore: VStore, layer: int, bud: hc_budget, out=None,
                     sel_idx=None, sel_w=None, sel_k=None, ws: Workspace | None = None,
                     debug: dict | None = None, stream=None):
    """hc_decode_attention for one layer: q fp16 [B][Hq][d] -> out fp32 [B][Hq][d]."""
    import torch
    if out is None:
        out = torch.empty((kc.B, kc.Hq, kc.d), dtype=torch.float32, device=q.device)
    if ws is None:
        ws = Workspace(kc.workspace_bytes(bud), device=q.device)
    vs = vstore.struct()
    dbg = None
    if debug is not None:
        dbg = hc_decode_debug(*(debug[k].data_ptr() if debug.get(k) is not None else None
                                for k in ("z", "e", "S", "M", "kstar")))
    st = lib().hc_decode_attention(_ptr(q), C.byref(kc.s), C.byref(vs), layer, bud, _ptr(out),
                                   _ptr(sel_idx), _ptr(sel_w), _ptr(sel_k),
                                   C.byref(dbg) if dbg is not None else None,
                                   _ptr(ws.t), ws.nbytes, _stream(stream))
    _check(st)
    return out


def append_decode_attention(q, kc: KCache, vstore: VStore, layer: int, k_new, v_new, bud: hc_budget,
                            out=None, sel_idx=None, sel_w=None, sel_k=None, ws: Workspace | None = None,
                            stream=None):
    """hc_append_decode_attention: kc.append(layer, k_new, v_new) then decode_attention, with
    the append overlapping the table build inside the library."""
    import torch
    if out is None:
        out = torch.empty((kc.B, kc.Hq, kc.d), dtype=torch.float32, device=q.device)
    if ws is None:
        ws = Workspace(kc.workspace_bytes(bud), device=q.device)
    vs = vstore.struct()
    _check(lib().hc_append_decode_attention(_ptr(q), C.byref(kc.s), C.byref(vs), layer, _ptr(k_new),
                                            _ptr(v_new), bud, _ptr(out), _ptr(sel_idx), _ptr(sel_w),
                                            _ptr(sel_k), _ptr(ws.t), ws.nbytes, _stream(stream)))
    return out


def select_topk(scores, d: int, bud: hc_budget, idx=None, w=None, k=None, ws=None, stream=None):
    """hc_select_topk: scores fp32 [rows][n] (cuda) -> (idx int32 [rows][k_max] ascending,
    w fp32 [rows][k_max], k int64 [rows])."""
    import torch
    rows, n = scores.shape
    km = int(bud.k_max)
    if idx is None:
        idx = torch.full((rows, km), -1, dtype=torch.int32, device=scores.device)
        w = torch.zeros((rows, km), dtype=torch.float32, device=scores.device)
        k = torch.zeros((rows,), dtype=torch.int64, device=scores.device)
    need = int(lib().hc_select_workspace_bytes(rows, n, bud))
    if ws is None:
        ws = Workspace(need, device=scores.device)
    _check(lib().hc_select_topk(_ptr(scores), rows, n, d, bud, _ptr(idx), _ptr(w), _ptr(k),
                                _ptr(ws.t), ws.nbytes, _stream(stream)))
    return idx, w, k


# ----------------------------------------------------------------------------- heterogeneous Eq. 5
def gather_values(kc: KCache, vstore: VStore, layer: int, sel_idx, sel_w, sel_k, tok_begin: int,
                  tok_end: int, out, ws: Workspace, stream=None):
    """hc_gather_values: GPU Eq. 5 over a given selection, kept tokens in [tok_begin, tok_end)."""
    vs = vstore.struct()
    _check(lib().hc_gather_values(C.byref(kc.s), C.byref(vs), layer, _ptr(sel_idx), _ptr(sel_w),
                                  _ptr(sel_k), sel_idx.shape[-1], int(tok_begin), int(tok_end), _ptr(out),
                                  _ptr(ws.t), ws.nbytes, _stream(stream)))
    return out


def add_partial(out, part, stream=None):
    """hc_add_partial: out += part (fp32; part may be pinned host memory, read zero-copy)."""
    _check(lib().hc_add_partial(_ptr(out), C.c_void_p(host_device_pointer(part.data_ptr()))
                                if not part.is_cuda else _ptr(part), out.numel(), _stream(stream)))
    return out


def host_weighted_sum_range(idx, w, k, vstore: VStore, layer: int, G: int, tok_begin: int, tok_end: int,
                            out, threads: int = 0, stream=None, *, n_valid: int):
    """hc_(enqueue_)host_weighted_sum_range on HOST tensors: idx/w [rows][k_stride], k [rows],
    out [rows][d]; V = the pinned value store's layer, rows [0, n_valid) valid (the layer's
    n_q; tok_end > n_valid raises HC_ERR_RANGE).  stream=None runs synchronously, else the work
    is enqueued as a host node on `stream` (graph-capturable)."""
    B, L, Hkv, n_cap, d = vstore.tensor.shape
    V = vstore.tensor[0, layer]
    rows, ks = idx.shape
    args = [_ptr(idx), _ptr(w), _ptr(k), rows, ks, _ptr(V), L * Hkv * n_cap * d, n_cap * d, int(n_valid),
            Hkv * G, G, d, int(tok_begin), int(tok_end), _ptr(out), int(threads)]
    if stream is None:
        _check(lib().hc_host_weighted_sum_range(*args))
    else:
        _check(lib().hc_enqueue_host_weighted_sum_range(*args, _stream(stream)))
    return out


class HostWorker:
    """hc_host_worker_*: persistent host thread running host shares of Eq. 5 on doorbells
    rung by GPU kernels (no graph host nodes).  See include/hc.h."""

    def __init__(self, threads: int = 0, max_jobs: int = 64, timeout_s: float = 10.0):
        h = C.c_void_p()
        _check(lib().hc_host_worker_create(int(threads), int(max_jobs), float(timeout_s), C.byref(h)))
        self.h = h

    def add_job(self, rows: int, k_stride: int, vstore: "VStore", G: int, out) -> int:
        B, L, Hkv, n_cap, d = vstore.tensor.shape
        j = C.c_int32()
        _check(lib().hc_host_worker_add_job(self.h, rows, k_stride, C.c_void_p(vstore.tensor.data_ptr()),
                                            L * Hkv * n_cap * d, n_cap * d, Hkv * G, G, d,
                                            _ptr(out), C.byref(j)))
        return int(j.value)

    def submit(self, job: int, sel_idx, sel_w, sel_k, t_split: int, v_off: int, stream=None, *,
               n_valid: int):
        """n_valid = the layer's n_q (t_split > n_valid raises HC_ERR_RANGE)."""
        _check(lib().hc_host_worker_submit(self.h, job, _ptr(sel_idx), _ptr(sel_w), _ptr(sel_k),
                                           int(t_split), int(n_valid), int(v_off), _stream(stream)))

    def wait(self, job: int, stream=None):
        _check(lib().hc_host_worker_wait(self.h, job, _stream(stream)))

    def status(self) -> int:
        return int(lib().hc_host_worker_status(self.h))

    def pause(self, paused: bool = True):
        _check(lib().hc_host_worker_pause(self.h, int(bool(paused))))

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().hc_host_worker_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- NCCL (sharded decode)
NCCL_UNIQUE_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """hc_nccl_get_unique_id: a fresh NCCL unique id (rank 0 makes it, the others receive it)."""
    buf = (C.c_char * NCCL_UNIQUE_ID_BYTES)()
    _check(lib().hc_nccl_get_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """An NCCL communicator of `world` ranks made by hc_nccl_comm_init (the library's
    libnccl.so.2 -- inside a PyTorch process, the one torch loaded)."""

    def __init__(self, world: int, rank: int, uid: bytes):
        if len(uid) != NCCL_UNIQUE_ID_BYTES:
            raise ValueError("uid must be NCCL_UNIQUE_ID_BYTES long")
        h = C.c_void_p()
        buf = (C.c_char * NCCL_UNIQUE_ID_BYTES).from_buffer_copy(uid)
        _check(lib().hc_nccl_comm_init(C.byref(h), int(world), buf, int(rank)))
        self.h, self.world, self.rank = h, int(world), int(rank)

    @staticmethod
    def from_process_group(group=None) -> "NcclComm":
        """Rank 0 makes the unique id; torch.distributed broadcasts it (plumbing only)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return NcclComm(world, rank, obj[0])

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().hc_nccl_comm_destroy(self.h)
            self.h = None
