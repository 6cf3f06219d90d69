// hc_nccl.cu -- the sequence-sharded decode behind ONE C-ABI call (SURVEY §8(b)/(e),
// include/hc.h hc_decode_attention_sharded): the five phase kernels of hc_shard.cu with the
// four exchanges between them issued by the library itself as NCCL collectives on the
// caller's stream (NVLink / NVSwitch on B200 boxes), so a C caller runs the global Eq. 4
// selection and Eq. 5 across R GPUs with no Python in
// between.  Everything is stream-ordered, so the whole layer is CUDA-graph capturable.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: inside a PyTorch process the library
// torch already loaded is reused, so communicators made by either side are the same objects;
// HC_NCCL_LIB overrides the path).  libhc.so therefore has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "../../include/hc.h"
#include "hc_internal.h"

namespace {

// the subset of nccl.h this file uses (values from NCCL's public header)
struct NcclId { char internal[HC_NCCL_UNIQUE_ID_BYTES]; };
enum { kNcclSuccess = 0 };
enum { kNcclSum = 0, kNcclMax = 2 };
enum { kNcclInt32 = 2, kNcclUint64 = 5, kNcclFloat32 = 7 };

struct NcclApi {
  void *h = nullptr;
  int (*get_unique_id)(NcclId *) = nullptr;
  int (*comm_init_rank)(ncclComm_t *, int, NcclId, int) = nullptr;
  int (*comm_destroy)(ncclComm_t) = nullptr;
  int (*all_reduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*all_gather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*error_string)(int) = nullptr;
  const char *why = "not loaded";
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

void nccl_load() {
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
  if (!h) {
    const char *p = getenv("HC_NCCL_LIB");
    h = dlopen(p && *p ? p : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) { g_nccl.why = "dlopen(libnccl.so.2) failed (set HC_NCCL_LIB)"; return; }
  NcclApi a;
  a.h = h;
  a.get_unique_id = (int (*)(NcclId *))dlsym(h, "ncclGetUniqueId");
  a.comm_init_rank = (int (*)(ncclComm_t *, int, NcclId, int))dlsym(h, "ncclCommInitRank");
  a.comm_destroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
  a.all_reduce = (int (*)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
  a.all_gather = (int (*)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclAllGather");
  a.error_string = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
  if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce || !a.all_gather) {
    g_nccl.why = "libnccl.so.2 lacks a collective symbol";
    return;
  }
  a.why = nullptr;
  g_nccl = a;
}

const NcclApi *nccl() {
  std::call_once(g_nccl_once, nccl_load);
  return g_nccl.why ? nullptr : &g_nccl;
}

hc_status nfail(hc_status st, const char *fmt, ...) {
  char buf[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return (hc_status)hc::set_error(st, buf);  // hc_last_error()
}

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// exchange buffers after the phase workspace: stats | h1 | h2 | cnt | allcnt
struct XLayout {
  size_t o_stats, o_h1, o_h2, o_cnt, o_all, total;
};
XLayout xlayout(size_t base, int64_t rows, int32_t world) {
  XLayout x{};
  size_t o = al256(base);
  x.o_stats = o; o += al256((size_t)rows * 2 * 4);
  x.o_h1 = o; o += al256((size_t)rows * hc::kNB * 2 * 8);
  x.o_h2 = o; o += al256((size_t)rows * hc::kNB * 8);
  x.o_cnt = o; o += al256((size_t)rows * 2 * 8);
  x.o_all = o; o += al256((size_t)world * rows * 2 * 8);
  x.total = o;
  return x;
}

}  // namespace

extern "C" {

hc_status hc_nccl_get_unique_id(void *id) {
  if (!id) return nfail(HC_ERR_ARG, "id NULL");
  const NcclApi *n = nccl();
  if (!n) return nfail(HC_ERR_NCCL, "%s", g_nccl.why);
  const int r = n->get_unique_id(reinterpret_cast<NcclId *>(id));
  return r == kNcclSuccess ? HC_OK : nfail(HC_ERR_NCCL, "ncclGetUniqueId: %d", r);
}

hc_status hc_nccl_comm_init(ncclComm_t *comm, int32_t world, const void *id, int32_t rank) {
  if (!comm || !id) return nfail(HC_ERR_ARG, "comm/id NULL");
  if (world < 1 || rank < 0 || rank >= world) return nfail(HC_ERR_RANGE, "rank/world");
  const NcclApi *n = nccl();
  if (!n) return nfail(HC_ERR_NCCL, "%s", g_nccl.why);
  NcclId uid;
  memcpy(&uid, id, sizeof(uid));
  const int r = n->comm_init_rank(comm, world, uid, rank);
  return r == kNcclSuccess ? HC_OK
                           : nfail(HC_ERR_NCCL, "ncclCommInitRank: %s", n->error_string ? n->error_string(r) : "?");
}

hc_status hc_nccl_comm_destroy(ncclComm_t comm) {
  if (!comm) return HC_OK;
  const NcclApi *n = nccl();
  if (!n) return nfail(HC_ERR_NCCL, "%s", g_nccl.why);
  return n->comm_destroy(comm) == kNcclSuccess ? HC_OK : nfail(HC_ERR_NCCL, "ncclCommDestroy");
}

size_t hc_decode_sharded_workspace_bytes(const hc_kcache *kc, hc_budget budget, int32_t world) {
  const size_t base = hc_shard_workspace_bytes(kc, budget);
  if (!base || world < 1) return 0;
  return xlayout(base, (int64_t)kc->B * kc->G * kc->Hkv, world).total;
}

hc_status hc_decode_attention_sharded(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs,
                                      int32_t layer, hc_budget budget, float *out, int32_t *sel_idx,
                                      float *sel_w, int64_t *sel_k, int32_t rank, int32_t world,
                                      int64_t shard_base, ncclComm_t comm, void *ws, size_t ws_bytes,
                                      hc_stream_t stream) {
  if (!kc || !vs || !q || !out || !sel_idx || !sel_w) return nfail(HC_ERR_ARG, "NULL pointer");
  if (world < 1 || rank < 0 || rank >= world) return nfail(HC_ERR_RANGE, "rank/world");
  if (world > 1 && !comm) return nfail(HC_ERR_ARG, "world > 1 needs an NCCL communicator");
  const size_t base = hc_shard_workspace_bytes(kc, budget);
  if (!base) return nfail(HC_ERR_SHAPE, "bad kcache");
  const int64_t rows = (int64_t)kc->B * kc->G * kc->Hkv;
  const XLayout x = xlayout(base, rows, world);
  if (!ws || ws_bytes < x.total) return nfail(HC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, x.total);
  const NcclApi *n = nullptr;
  if (comm) {
    n = nccl();
    if (!n) return nfail(HC_ERR_NCCL, "%s", g_nccl.why);
  }
  uint8_t *w8 = (uint8_t *)ws;
  int32_t *stats = (int32_t *)(w8 + x.o_stats);
  uint64_t *h1 = (uint64_t *)(w8 + x.o_h1), *h2 = (uint64_t *)(w8 + x.o_h2);
  uint64_t *cnt = (uint64_t *)(w8 + x.o_cnt), *allcnt = (uint64_t *)(w8 + x.o_all);
  cudaStream_t s = (cudaStream_t)stream;
  const int d = kc->vq.d;
  auto coll = [&](int r, const char *what) -> hc_status {
    if (r == kNcclSuccess) return HC_OK;
    return nfail(HC_ERR_NCCL, "%s: %s", what, n->error_string ? n->error_string(r) : "?");
  };
  hc_status st;
  // C1: {max z, -min z} all-reduce MAX
  if ((st = hc_shard_begin(q, kc, vs, layer, budget, stats, ws, base, stream))) return st;
  if (n && (st = coll(n->all_reduce(stats, stats, (size_t)rows * 2, kNcclInt32, kNcclMax, comm, s), "C1 max")))
    return st;
  // C2: coarse (count, mass) histograms all-reduce SUM (exact u64)
  if ((st = hc_shard_hist1(kc, vs, layer, budget, stats, h1, ws, base, stream))) return st;
  if (n && (st = coll(n->all_reduce(h1, h1, (size_t)rows * hc::kNB * 2, kNcclUint64, kNcclSum, comm, s), "C2 hist1")))
    return st;
  // C3: fine counts of the boundary bucket all-reduce SUM
  if ((st = hc_shard_hist2(kc, vs, layer, budget, stats, h1, h2, ws, base, stream))) return st;
  if (n && (st = coll(n->all_reduce(h2, h2, (size_t)rows * hc::kNB, kNcclUint64, kNcclSum, comm, s), "C3 hist2")))
    return st;
  // C4: per-rank (strict, tie) counts all-gather -> global positions in rank order
  if ((st = hc_shard_counts(kc, vs, layer, budget, h2, cnt, ws, base, stream))) return st;
  if (n) {
    if ((st = coll(n->all_gather(cnt, allcnt, (size_t)rows * 2, kNcclUint64, comm, s), "C4 counts"))) return st;
  } else if (cudaMemcpyAsync(allcnt, cnt, (size_t)rows * 2 * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
    return nfail(HC_ERR_CUDA, "counts copy");
  }
  // compaction at global positions + this rank's Eq. 5 numerator; C5: all-reduce SUM
  if ((st = hc_shard_finish(kc, vs, layer, budget, allcnt, rank, world, shard_base, out, sel_idx, sel_w, sel_k,
                            ws, base, stream)))
    return st;
  if (n && (st = coll(n->all_reduce(out, out, (size_t)rows * d, kNcclFloat32, kNcclSum, comm, s), "C5 out")))
    return st;
  return HC_OK;
}

}  // extern "C"
