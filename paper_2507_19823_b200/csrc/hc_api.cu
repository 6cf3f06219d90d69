// hc_api.cu -- the C ABI of include/hc.h: argument validation, workspace layout,
// and the stream-ordered launch sequence of one decode step.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>

#include "../../include/hc.h"
#include "hc_internal.h"

using namespace hc;

namespace hc {
static std::atomic<unsigned long long> g_launches{0};
static thread_local cudaEvent_t g_scan_ev[2] = {nullptr, nullptr};
static thread_local cudaEvent_t g_eq3_ev[2] = {nullptr, nullptr};
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    // measured: no gain in the graph-captured step, and up to 15 % slower for
    // eager layer calls (early-launched dependents crowd the SMs) -> off unless HC_PDL=1
    const char *ev = getenv("HC_PDL");
    v = (ev && !strcmp(ev, "1")) ? 1 : 0;
  }
  return v == 1;
}

void note_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
void scan_events(cudaEvent_t *begin, cudaEvent_t *end) {
  *begin = g_scan_ev[0];
  *end = g_scan_ev[1];
  g_scan_ev[0] = g_scan_ev[1] = nullptr;  // one-shot
}
}  // namespace hc

namespace {

thread_local char g_err[512] = "";

hc_status fail(hc_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

}  // namespace

int hc::set_error(int st, const char *msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return st;
}

namespace {

hc_status cuda_check(cudaError_t e, const char *what) {
  if (e != cudaSuccess) return fail(HC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return HC_OK;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
int next_pow2(int c) {
  int p = 1;
  while (p < c) p <<= 1;
  return p;
}


// Scan decomposition: choose tokens-per-thread (tile = 512*TPT tokens) and
// the group split so the work fills the SMs with the least shared-memory time, modelled
// per SM as  lookups/5.2 + slice_bytes_streamed/100  cycles (+ partial write/reduce).
bool scan_sk_enabled() {
  static int v = -1;
  if (v < 0) {
    const char *ev = getenv("HC_SCAN_SK");
    v = (ev && !strcmp(ev, "0")) ? 0 : 1;
  }
  return v != 0;
}

void choose_scan(int64_t units, int64_t n, int g, int cpow2, int G, int sms, int *tpt, int *split,
                 int lut8) {
  // per-SM shared-memory cycles: lookups * wavefronts/32 + (table slice + code strip) / 128 B
  const double wf = lut8 ? 3.53 : 6.15;            // measured wavefronts per warp lookup
  const double entry = lut8 ? 4.0 : 2.0 * G;       // table entry bytes
  double best = 1e300;
  *tpt = lut8 ? 32 : 16; *split = 1;
  const int tpts16[2] = {8, 16}, tpts8[1] = {32};
  const int *tl = lut8 ? tpts8 : tpts16;
  const int nt = lut8 ? 1 : 2;
  for (int ti = 0; ti < nt; ++ti) {
    const int t = tl[ti];
    const int64_t tile = 512LL * t;
    const int64_t tiles = units * ((n + tile - 1) / tile);
    for (int sp : {1, 2, 4}) {
      if (sp > g) continue;
      const int64_t items = tiles * sp;
      // unsplit + >= 2 tiles per CTA: the stream-K scan balances steps exactly (k_scan_sk)
      const bool sk = sp == 1 && !lut8 && tiles >= 2 * (int64_t)(sms < kSkMaxCtas ? sms : kSkMaxCtas) &&
                      scan_sk_enabled();
      const double waves = sk ? (double)items / sms : (double)((items + sms - 1) / sms);
      const double gper = (double)((g + sp - 1) / sp);
      // slice + code ingress arrives by bulk copy (TMA) at ~2x the LSU wavefront rate; a split
      // item's exact partial is added to z with float atomics (~4x a store) -- weights fitted to
      // config 2 (TPT 8 / 2 splits measured 383.6 vs 374.2 steps/s for TPT 16 / 4 splits)
      double item = tile * gper * wf / 32.0 + gper * (cpow2 * entry + tile * 4.0) / 256.0;
      if (sp > 1) item += tile * G * 4.0 / 16.0;  // partial atomics
      double cost = waves * item;
      if (sp > 1) cost += (double)units * n * G * 4.0 * (sp + 1) / (sms * 64.0);  // reduce pass
      if (cost < best * 0.999) { best = cost; *tpt = t; *split = sp; }
    }
  }
}

struct Layout {
  int cpow2;
  int64_t z_stride;
  int64_t k_eff;
  size_t o_hs, o_T, o_cbabs, o_z, o_zpart, o_idx, o_w, o_chunk, o_part, o_upart, o_udone, o_rpart,
      o_rdone, o_wpart, o_grp, o_ghist, o_gchunk, o_gkey, o_grange, o_skpart, o_skctr, o_sgh, o_sfc,
      o_scl, o_spre, o_slist, total;
  int64_t snch, scap;
  int skctr_n;
  int nch_max;  // sharded compaction chunks
};

Layout make_layout(const hc_kcache *kc, int64_t k_max, int shared = 0) {
  Layout L{};
  const int64_t B = kc->B, Hkv = kc->Hkv, G = kc->G, Hq = G * Hkv;
  const int64_t rows = B * Hq;
  const int g = kc->vq.g, d = kc->vq.d;
  L.cpow2 = next_pow2(kc->vq.c);
  if (L.cpow2 < 256) L.cpow2 = 256;
  const int64_t ncand_max = kc->n_cap + kc->res_cap;
  L.z_stride = round_up(ncand_max > 0 ? ncand_max : 1, 64);
  L.k_eff = k_max < ncand_max ? k_max : ncand_max;
  if (L.k_eff < 1) L.k_eff = 1;
  size_t o = 0;
  L.o_hs = o; o += align256((size_t)rows * sizeof(HeadState));
  L.o_T = o; o += align256((size_t)B * Hkv * g * L.cpow2 * G * 2);
  L.o_cbabs = o; o += align256((size_t)kc->vq.cbg * (d / g) * 4);
  L.o_z = o; o += align256((size_t)rows * L.z_stride * 4);
  L.o_zpart = o;  // (no partial planes: split scans accumulate exactly into z)
  // selection passes (hc_select_pass.cu): coarse / fine histograms, per-chunk counters and
  // prefixes, the in-range token lists
  L.snch = select_chunks(ncand_max > 0 ? ncand_max : 1);
  L.scap = select_list_cap(ncand_max > 0 ? ncand_max : 1);
  L.o_sgh = o; o += align256((size_t)rows * kNB * 12);  // ghist u32 then gmass u64
  L.o_sfc = o; o += align256((size_t)rows * kNB * 4);
  L.o_scl = o; o += align256((size_t)rows * L.snch * 4);
  L.o_spre = o; o += align256((size_t)rows * L.snch * 8);
  L.o_slist = o; o += align256((size_t)rows * L.scap * 8);
  L.o_idx = o; o += align256((size_t)rows * L.k_eff * 4);
  L.o_w = o; o += align256((size_t)rows * L.k_eff * 4);
  L.nch_max = shard_chunks(ncand_max > 0 ? ncand_max : 1);
  L.o_chunk = o; o += align256((size_t)rows * L.nch_max * 8);
  L.o_part = o; o += align256((size_t)rows * L.nch_max * d * 4);
  {
    const int64_t units = B * Hkv;
    const int64_t nchu = gather_union_chunks(ncand_max > 0 ? ncand_max : 1);
    L.o_upart = o; o += align256((size_t)units * nchu * G * d * 4);
    L.o_udone = o; o += align256((size_t)units * 4);
    const int64_t nchr = gather_rows_chunks(L.k_eff);
    L.o_rpart = o; o += align256((size_t)rows * nchr * 128 * 4);
    L.o_rdone = o; o += align256((size_t)rows * 4);
    // K3 fused with Eq. 5 (k_sel_write_gather): one partial per (row, contributor CTA)
    L.o_wpart = o; o += align256((size_t)rows * (select_chunks(ncand_max > 0 ? ncand_max : 1) + 1) * 128 * 4);
    L.o_grange = o; o += align256((size_t)rows * 16);  // sharded finish: list slice per row
    // stream-K scan (16-bit table): 2 partial tiles (8192 tokens x G int32) per CTA, one
    // counter per (tile, warp)
    L.o_skpart = o; o += align256((size_t)kSkMaxCtas * 2 * 8192 * G * 4);
    L.skctr_n = (int)(units * ((ncand_max + 4095) / 4096) * 16);  // per (tile, warp)
    L.o_skctr = o; o += align256((size_t)L.skctr_n * 4);
    if (shared) {  // R8 shared selection state, 4-level histograms, chunk counts
      L.o_grp = o; o += align256((size_t)units * sizeof(GroupState));
      L.o_ghist = o; o += align256((size_t)units * 4 * kNB * 16);
      L.o_gchunk = o; o += align256((size_t)units * grp_chunks(ncand_max > 0 ? ncand_max : 1) * 8);
      L.o_gkey = o; o += align256((size_t)units * L.z_stride * 8);
    }
  }
  L.total = o;
  return L;
}

hc_status check_vq(const hc_vq &vq) {
  if (vq.d <= 0 || vq.g <= 0 || vq.c <= 0) return fail(HC_ERR_SHAPE, "d, g, c must be positive");
  if (vq.d % vq.g) return fail(HC_ERR_SHAPE, "g=%d does not divide d=%d", vq.g, vq.d);
  const int dbar = vq.d / vq.g;
  if (!(dbar == 1 || dbar == 2 || dbar == 4 || dbar == 8 || dbar == 16))
    return fail(HC_ERR_UNSUPPORTED, "dbar=%d not in {1,2,4,8,16}", dbar);
  if (vq.c > 65536) return fail(HC_ERR_RANGE, "c=%d exceeds the 16-bit index range", vq.c);
  if (!(vq.cbg == 1 || vq.cbg == vq.g)) return fail(HC_ERR_SHAPE, "cbg must be 1 or g");
  if (!(vq.code_bits == 0 || vq.code_bits == 16 || vq.code_bits == 13))
    return fail(HC_ERR_UNSUPPORTED, "code_bits=%d not in {16, 13}", vq.code_bits);
  if (vq.code_bits == 13 && (vq.c > 8192 || vq.lut_bits == 8))
    return fail(HC_ERR_UNSUPPORTED, "13-bit codes need c <= 8192 and the 16-bit table");
  if (vq.g > 128) return fail(HC_ERR_UNSUPPORTED, "g=%d > 128 (|z~| must stay below 2^22)", vq.g);
  if (vq.d % 8 || vq.d > 256 || (32 % (vq.d / 8)))
    return fail(HC_ERR_UNSUPPORTED, "d=%d not in {64,128,256}", vq.d);
  return HC_OK;
}

hc_status check_kcache(const hc_kcache *kc) {
  if (!kc) return fail(HC_ERR_ARG, "kcache is NULL");
  hc_status st = check_vq(kc->vq);
  if (st) return st;
  if (kc->B <= 0 || kc->L <= 0 || kc->Hkv <= 0 || kc->L > HC_MAX_LAYERS)
    return fail(HC_ERR_SHAPE, "bad B/L/Hkv");
  if (!(kc->G == 1 || kc->G == 2 || kc->G == 4)) return fail(HC_ERR_UNSUPPORTED, "G=%d not in {1,2,4}", kc->G);
  if (kc->n_cap < 0 || kc->n_cap % 64) return fail(HC_ERR_SHAPE, "n_cap must be a multiple of 64");
  if (kc->res_cap < 0) return fail(HC_ERR_SHAPE, "res_cap < 0");
  if (kc->vq.c > 8192) return fail(HC_ERR_UNSUPPORTED, "c=%d > 8192 (shared-memory table slices)", kc->vq.c);
  if (kc->n_cap > 0 && !kc->codes) return fail(HC_ERR_ARG, "codes is NULL");
  if (!kc->codebook) return fail(HC_ERR_ARG, "codebook is NULL");
  if (kc->res_cap > 0 && (!kc->res_k || !kc->res_v)) return fail(HC_ERR_ARG, "res_k/res_v NULL");
  if ((int64_t)kc->B * kc->G * kc->Hkv > 65535) return fail(HC_ERR_UNSUPPORTED, "B*Hq > 65535");
  return HC_OK;
}

__global__ void k_z_to_int(const float *z, int64_t zs, int32_t *out, int64_t n) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[(int64_t)blockIdx.y * n + j] = __float2int_rn(z[(int64_t)blockIdx.y * zs + j]);
}

}  // namespace

extern "C" {

const char *hc_last_error(void) { return g_err; }
const char *hc_version(void) { return "hcattn-b200 0.1 (sm_100a)"; }

uint64_t hc_launch_count(void) { return g_launches.load(); }

hc_status hc_codebook_absmax(const float *codebook, hc_vq vq, int32_t L, float *out,
                             hc_stream_t stream) {
  hc_status st = check_vq(vq);
  if (st) return st;
  if (L <= 0) return fail(HC_ERR_ARG, "L <= 0");
  if (!codebook || !out) return fail(HC_ERR_ARG, "NULL pointer");
  return cuda_check(launch_cbabs(codebook, (int64_t)L * vq.cbg, vq.c, vq.d / vq.g, out,
                                 (cudaStream_t)stream), "hc_codebook_absmax");
}

hc_status hc_profile_scan_events(void *begin_event, void *end_event) {
  hc::g_scan_ev[0] = (cudaEvent_t)begin_event;
  hc::g_scan_ev[1] = (cudaEvent_t)end_event;
  return HC_OK;
}

hc_status hc_profile_eq3_events(void *begin_event, void *end_event) {
  hc::g_eq3_ev[0] = (cudaEvent_t)begin_event;
  hc::g_eq3_ev[1] = (cudaEvent_t)end_event;
  return HC_OK;
}

hc_status hc_host_register(void *host, size_t bytes, void **dev_ptr) {
  if (!host || !bytes || !dev_ptr) return fail(HC_ERR_ARG, "host/bytes/dev_ptr");
  cudaError_t e = cudaHostRegister(host, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) return cuda_check(e, "cudaHostRegister");
  e = cudaHostGetDevicePointer(dev_ptr, host, 0);
  return e != cudaSuccess ? cuda_check(e, "cudaHostGetDevicePointer") : HC_OK;
}

hc_status hc_host_unregister(void *host) {
  cudaError_t e = cudaHostUnregister(host);
  return e != cudaSuccess ? cuda_check(e, "cudaHostUnregister") : HC_OK;
}

hc_status hc_quantize_keys(const uint16_t *keys, int64_t rows, const float *codebook, hc_vq vq,
                           uint16_t *codes, int64_t code_stride, hc_stream_t stream) {
  hc_status st = check_vq(vq);
  if (st) return st;
  if (rows < 0) return fail(HC_ERR_ARG, "rows < 0");
  if (rows == 0) return HC_OK;
  if (!keys || !codebook || !codes) return fail(HC_ERR_ARG, "NULL pointer");
  if (code_stride < rows) return fail(HC_ERR_SHAPE, "code_stride < rows");
  if (rows > 0x7fffffff) return fail(HC_ERR_UNSUPPORTED, "rows > 2^31-1");
  EncodeArgs a{};
  a.keys = keys;
  a.kmap = RowMap{1, vq.d, 0, 0};
  a.rows = rows;
  a.C = codebook;
  a.d = vq.d; a.g = vq.g; a.c = vq.c; a.cbg = vq.cbg;
  a.codes = codes;
  a.omap = RowMap{1, 1, 0, 0};
  a.gstride = code_stride;
  // many rows (prefill): shared-memory-staged bulk kernel; few rows (decode): k_encode
  return cuda_check(rows >= 1024 ? launch_encode_bulk(a, (cudaStream_t)stream)
                                 : launch_encode(a, (cudaStream_t)stream),
                    "hc_quantize_keys");
}

hc_status hc_blockwise_attention(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t n,
                                 int32_t Hq, int32_t Hkv, int32_t d, int64_t bs, float *out,
                                 hc_stream_t stream) {
  if (n < 0 || bs <= 0 || Hq <= 0 || Hkv <= 0) return fail(HC_ERR_ARG, "bad n / bs / heads");
  if (d != 128) return fail(HC_ERR_UNSUPPORTED, "blockwise attention is built for d = 128");
  if (bs % 64) return fail(HC_ERR_SHAPE, "bs must be a multiple of 64");
  if (Hq % Hkv) return fail(HC_ERR_SHAPE, "Hq %% Hkv != 0");
  if (n == 0) return HC_OK;
  if (!q || !k || !v || !out) return fail(HC_ERR_ARG, "NULL pointer");
  return cuda_check(launch_blockwise_attn(q, k, v, n, Hq, Hkv, bs, out, (cudaStream_t)stream),
                    "hc_blockwise_attention");
}

hc_status hc_prefill_append(hc_kcache *kc, const hc_vstore *vs, int32_t layer, const uint16_t *k,
                            const uint16_t *v, int64_t n, hc_stream_t stream) {
  hc_status st = check_kcache(kc);
  if (st) return st;
  if (!vs || !vs->base) return fail(HC_ERR_ARG, "vstore is NULL");
  if (vs->n_cap != kc->n_cap) return fail(HC_ERR_SHAPE, "vstore.n_cap != kcache.n_cap");
  if (layer < 0 || layer >= kc->L) return fail(HC_ERR_RANGE, "layer %d out of range", layer);
  if (n < 0) return fail(HC_ERR_ARG, "n < 0");
  if (n == 0) return HC_OK;
  if (!k || !v) return fail(HC_ERR_ARG, "k/v NULL");
  if (kc->vq.code_bits == 13) return fail(HC_ERR_UNSUPPORTED, "prefill append writes 16-bit codes");
  if (kc->n_res[layer] != 0) return fail(HC_ERR_UNSUPPORTED, "prefill append with a non-empty window");
  const int64_t B = kc->B, L = kc->L, H = kc->Hkv, d = kc->vq.d, g = kc->vq.g, ncap = kc->n_cap;
  const int64_t nq = kc->n_q[layer];
  if (nq + n > ncap) return fail(HC_ERR_CAPACITY, "layer %d: %lld + %lld > n_cap", layer, (long long)nq, (long long)n);
  cudaStream_t s = (cudaStream_t)stream;
  for (int64_t b = 0; b < B; ++b) {  // rows r = t * Hkv + kv of sequence b
    EncodeArgs a{};
    a.keys = k;
    a.kmap = RowMap{1, d, 0, b * n * H * d};
    a.rows = n * H;
    a.C = kc->codebook + (int64_t)layer * kc->vq.cbg * kc->vq.c * (d / g);
    a.d = (int)d; a.g = (int)g; a.c = kc->vq.c; a.cbg = kc->vq.cbg;
    a.codes = kc->codes;
    a.omap = RowMap{H, 1, g * ncap, ((b * L + layer) * H) * g * ncap + nq};
    a.gstride = ncap;
    cudaError_t e = a.rows >= 1024 ? launch_encode_bulk(a, s) : launch_encode(a, s);
    if (e != cudaSuccess) return cuda_check(e, "hc_prefill_append encode");
    RowCopyArgs c{v, RowMap{1, d, 0, b * n * H * d}, vs->base,
                  RowMap{H, d, ncap * d, ((b * L + layer) * H * ncap + nq) * d}, n * H, (int)d};
    if ((e = launch_rowcopy(c, s)) != cudaSuccess) return cuda_check(e, "hc_prefill_append values");
  }
  kc->n_q[layer] = nq + n;
  return HC_OK;
}

hc_status hc_pack_codes13(const uint16_t *src, int64_t strips, int64_t n, int64_t src_stride,
                          uint8_t *dst, int64_t n_cap, hc_stream_t stream) {
  if (strips < 0 || n < 0) return fail(HC_ERR_ARG, "strips/n < 0");
  if (n_cap % 64 || n > n_cap) return fail(HC_ERR_SHAPE, "need n <= n_cap and n_cap %% 64 == 0");
  if (src_stride < n) return fail(HC_ERR_SHAPE, "src_stride < n");
  if (strips == 0 || n == 0) return HC_OK;
  if (!src || !dst) return fail(HC_ERR_ARG, "NULL pointer");
  return cuda_check(launch_pack13(src, strips, n, src_stride, dst, n_cap, (cudaStream_t)stream),
                    "hc_pack_codes13");
}

size_t hc_kmeans_workspace_bytes(hc_vq vq, int64_t b) {
  if (check_vq(vq) != HC_OK || b < 0) return 0;
  const size_t cc = (size_t)vq.cbg * vq.c, dbar = (size_t)(vq.d / vq.g);
  return align256(cc * 8) + align256(cc * dbar * 8) + align256((size_t)vq.g * (size_t)(b > 0 ? b : 1) * 2);
}

hc_status hc_kmeans_step(const uint16_t *keys, int64_t n_keys, const int64_t *sample, int64_t b,
                         hc_vq vq, float *codebook, int64_t *counts, uint16_t *labels, void *ws,
                         size_t ws_bytes, hc_stream_t stream) {
  hc_status st = check_vq(vq);
  if (st) return st;
  if (b < 0 || n_keys < 0) return fail(HC_ERR_ARG, "b < 0 or n_keys < 0");
  if (b == 0) return HC_OK;
  if (!keys || !sample || !codebook || !counts) return fail(HC_ERR_ARG, "NULL pointer");
  if (b > 0x7fffffff) return fail(HC_ERR_UNSUPPORTED, "b > 2^31-1");
  const size_t need = hc_kmeans_workspace_bytes(vq, b);
  if (!ws || ws_bytes < need) return fail(HC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
  const size_t cc = (size_t)vq.cbg * vq.c, dbar = (size_t)(vq.d / vq.g);
  uint8_t *w8 = (uint8_t *)ws;
  unsigned long long *n = (unsigned long long *)w8;
  unsigned long long *S = (unsigned long long *)(w8 + align256(cc * 8));
  uint16_t *lab = labels ? labels : (uint16_t *)(w8 + align256(cc * 8) + align256(cc * dbar * 8));
  EncodeArgs a{};
  a.keys = keys;
  a.kmap = RowMap{1, vq.d, 0, 0};
  a.rows = b;
  a.C = codebook;
  a.d = vq.d; a.g = vq.g; a.c = vq.c; a.cbg = vq.cbg;
  a.codes = lab;
  a.omap = RowMap{1, 1, 0, 0};
  a.gstride = b;
  a.kidx = sample;
  a.n_keys = n_keys;
  return cuda_check(launch_kmeans_step(a, sample, b, codebook, counts, n, S, (cudaStream_t)stream),
                    "hc_kmeans_step");
}

hc_status hc_append_kv(hc_kcache *kc, const hc_vstore *vs, int32_t layer, const uint16_t *k_new,
                       const uint16_t *v_new, hc_stream_t stream) {
  hc_status st = check_kcache(kc);
  if (st) return st;
  if (!vs || !vs->base) return fail(HC_ERR_ARG, "vstore is NULL");
  if (vs->n_cap != kc->n_cap) return fail(HC_ERR_SHAPE, "vstore.n_cap != kcache.n_cap");
  if (layer < 0 || layer >= kc->L) return fail(HC_ERR_RANGE, "layer %d out of range", layer);
  if (!k_new || !v_new) return fail(HC_ERR_ARG, "k_new/v_new NULL");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = kc->B, L = kc->L, H = kc->Hkv, d = kc->vq.d, g = kc->vq.g, W = kc->res_cap;
  const int64_t ncap = kc->n_cap;
  const int64_t nq = kc->n_q[layer];
  const int64_t nr = kc->n_res[layer];
  const int64_t rows = B * H;
  const RowMap codes_at = {H, L * H * g * ncap, g * ncap, (int64_t)layer * H * g * ncap + nq};
  const RowMap vstore_at = {H, L * H * ncap * d, ncap * d, ((int64_t)layer * H * ncap + nq) * d};
  const RowMap flat = {1, d, 0, 0};
  auto encode_from = [&](const uint16_t *src, RowMap km, const uint16_t *vsrc = nullptr,
                         RowMap vsm = RowMap{1, 0, 0, 0}, uint16_t *vdst = nullptr,
                         RowMap vdm = RowMap{1, 0, 0, 0}) -> cudaError_t {
    EncodeArgs a{};
    a.keys = src; a.kmap = km; a.rows = rows;
    a.vsrc = vsrc; a.vsmap = vsm; a.vdst = vdst; a.vdmap = vdm;
    a.C = kc->codebook + (int64_t)layer * kc->vq.cbg * kc->vq.c * (d / g);
    a.d = (int)d; a.g = (int)g; a.c = kc->vq.c; a.cbg = kc->vq.cbg;
    a.codes = kc->codes; a.omap = codes_at; a.gstride = ncap;
    if (kc->vq.code_bits == 13) {  // packed strips: strip of (b, layer, kv, group 0)
      a.pcodes = reinterpret_cast<uint8_t *>(kc->codes);
      a.psmap = RowMap{H, L * H * g, g, (int64_t)layer * H * g};
      a.strip_bytes = HC_STRIP13_BYTES(ncap);
      a.pn_cap = ncap;
      a.ptok = nq;
    }
    return launch_encode(a, s);
  };
  auto copy = [&](const uint16_t *src, RowMap sm, uint16_t *dst, RowMap dm) -> cudaError_t {
    RowCopyArgs a{src, sm, dst, dm, rows, (int)d};
    return launch_rowcopy(a, s);
  };
  cudaError_t e = cudaSuccess;
  if (W == 0) {
    if (nq >= ncap) return fail(HC_ERR_CAPACITY, "layer %d full (n_cap=%lld)", layer, (long long)ncap);
    e = encode_from(k_new, flat, v_new, flat, vs->base, vstore_at);
    if (e != cudaSuccess) return cuda_check(e, "hc_append_kv");
    kc->n_q[layer] = nq + 1;
    return HC_OK;
  }
  const int64_t p = nq + nr;
  if (nr < W) {
    const int64_t slot = p % W;
    const RowMap res_at = {H, L * H * W * d, W * d, ((int64_t)layer * H * W + slot) * d};
    e = copy(k_new, flat, kc->res_k, res_at);
    if (e == cudaSuccess) e = copy(v_new, flat, kc->res_v, res_at);
    if (e != cudaSuccess) return cuda_check(e, "hc_append_kv");
    kc->n_res[layer] = (int32_t)(nr + 1);
    return HC_OK;
  }
  if (nq >= ncap) return fail(HC_ERR_CAPACITY, "layer %d full (n_cap=%lld)", layer, (long long)ncap);
  const int64_t slot = nq % W;  // the oldest resident token (position nq)
  const RowMap res_at = {H, L * H * W * d, W * d, ((int64_t)layer * H * W + slot) * d};
  e = encode_from(kc->res_k, res_at, kc->res_v, res_at, vs->base, vstore_at);
  if (e == cudaSuccess) e = copy(k_new, flat, kc->res_k, res_at);
  if (e == cudaSuccess) e = copy(v_new, flat, kc->res_v, res_at);
  if (e != cudaSuccess) return cuda_check(e, "hc_append_kv");
  kc->n_q[layer] = nq + 1;
  return HC_OK;
}

size_t hc_decode_workspace_bytes(const hc_kcache *kc, hc_budget budget) {
  if (check_kcache(kc) != HC_OK) return 0;
  return make_layout(kc, budget.k_max, budget.shared_kv).total;
}

// validation + LayerArgs of one layer call (decode or a sharded phase)
static hc_status prepare_layer(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs,
                               int32_t layer, hc_budget budget, float *out, int32_t *sel_idx,
                               float *sel_w, int64_t *sel_k, void *ws, size_t ws_bytes,
                               cudaStream_t s, bool need_q, LayerArgs &a, Layout &Lw) {
  hc_status st = check_kcache(kc);
  if (st) return st;
  if (!vs || !vs->base) return fail(HC_ERR_ARG, "vstore is NULL");
  if (vs->n_cap != kc->n_cap) return fail(HC_ERR_SHAPE, "vstore.n_cap != kcache.n_cap");
  if (!(vs->placement == HC_V_DEVICE || vs->placement == HC_V_HOST_MAPPED))
    return fail(HC_ERR_ARG, "bad vstore placement");
  if (layer < 0 || layer >= kc->L) return fail(HC_ERR_RANGE, "layer %d out of range", layer);
  if (need_q && (!q || (!out && !budget.select_only))) return fail(HC_ERR_ARG, "q/out NULL");
  if (budget.select_only && (!sel_idx || !sel_w || !sel_k))
    return fail(HC_ERR_ARG, "select_only needs sel_idx, sel_w and sel_k");
  if (!(budget.tau > 0.0f && budget.tau <= 1.0f)) return fail(HC_ERR_ARG, "tau=%g not in (0,1]", budget.tau);
  if (budget.k_max < 1) return fail(HC_ERR_ARG, "k_max < 1");
  if (!!sel_idx != !!sel_w) return fail(HC_ERR_ARG, "pass both sel_idx and sel_w, or neither");
  const int64_t n_q = kc->n_q[layer], n_res = kc->n_res[layer];
  if (n_q < 0 || n_q > kc->n_cap || n_res < 0 || n_res > kc->res_cap)
    return fail(HC_ERR_RANGE, "cache counts out of range");
  const int64_t n_cand = n_q + n_res;
  if (n_cand == 0) return fail(HC_ERR_EMPTY, "layer %d has no tokens", layer);
  if (budget.shared_kv && budget.renorm)
    return fail(HC_ERR_UNSUPPORTED, "shared_kv selection takes renorm = 0");
  Lw = make_layout(kc, budget.k_max, budget.shared_kv);
  if (!ws || ws_bytes < Lw.total)
    return fail(HC_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, Lw.total);
  uint8_t *w8 = (uint8_t *)ws;
  const int64_t B = kc->B, H = kc->Hkv, G = kc->G, Hq = G * H, d = kc->vq.d, g = kc->vq.g;
  const int64_t L = kc->L, W = kc->res_cap, ncap = kc->n_cap;
  a = LayerArgs{};
  a.B = (int)B; a.Hkv = (int)H; a.G = (int)G; a.Hq = (int)Hq; a.d = (int)d; a.g = (int)g;
  a.c = kc->vq.c; a.cbg = kc->vq.cbg; a.dbar = (int)(d / g); a.cpow2 = Lw.cpow2;
  a.lut8 = kc->vq.lut_bits == 8 ? 1 : 0;
  a.n_q = n_q; a.n_res = n_res; a.n_cand = n_cand; a.n_cap = ncap; a.res_cap = W > 0 ? W : 1;
  a.gtok_lo = 0; a.gtok_hi = n_cand;
  a.q = q;
  a.C = kc->codebook + (int64_t)layer * kc->vq.cbg * kc->vq.c * (d / g);
  a.codes = kc->codes + (int64_t)layer * H * g * ncap;
  a.code_b_stride = L * H * g * ncap;
  if (kc->vq.code_bits == 13) {
    a.strip_bytes = HC_STRIP13_BYTES(ncap);
    a.pcodes = reinterpret_cast<const uint8_t *>(kc->codes) + (int64_t)layer * H * g * a.strip_bytes;
    a.pc_b_stride = L * H * g * a.strip_bytes;
  }
  a.res_k = W > 0 ? kc->res_k + (int64_t)layer * H * W * d : nullptr;
  a.res_v = W > 0 ? kc->res_v + (int64_t)layer * H * W * d : nullptr;
  a.res_b_stride = L * H * (W > 0 ? W : 1) * d;
  a.res_slot0 = W > 0 ? n_q % W : 0;
  a.V = vs->base + (int64_t)layer * H * ncap * d;
  a.v_placement = vs->placement == HC_V_DEVICE ? 0 : 1;
  a.v_b_stride = L * H * ncap * d;
  a.v_kv_stride = ncap * d;
  a.tau_q = (uint32_t)rint((double)budget.tau * 16777216.0);
  a.renorm = budget.renorm ? 1 : 0;
  a.kappa0 = (float)(1.4426950408889634 / sqrt((double)d));
  a.hs = (HeadState *)(w8 + Lw.o_hs);
  a.T = (int16_t *)(w8 + Lw.o_T);
  if (kc->cb_absmax) {
    a.cb_absmax = kc->cb_absmax + (int64_t)layer * kc->vq.cbg * (d / g);
  } else if (need_q) {
    float *cba = (float *)(w8 + Lw.o_cbabs);
    cudaError_t e0 = launch_cbabs(a.C, kc->vq.cbg, kc->vq.c, (int)(d / g), cba, s);
    if (e0 != cudaSuccess) return cuda_check(e0, "codebook absmax");
    a.cb_absmax = cba;
  }
  {  // table grid: chunks of 2 units (each codebook row loaded once per chunk; measured
     // 2 > 4 > 8 > 1 units at configs 2-4, profiles/r02_table_sweep.md), about 4 resident CTAs
     // per SM, at least a full batch of rows per thread
    const int64_t units = B * H, E = g * Lw.cpow2;
    int64_t tu = std::min<int64_t>({units, (int64_t)2, std::max<int64_t>(1, kTableQ / (d * G))});
    const int64_t chunks = (units + tu - 1) / tu;
    int64_t ts = (4 * (int64_t)num_sms() + chunks - 1) / chunks;
    ts = std::max<int64_t>(1, std::min<int64_t>(ts, E / 1024));
    static int ts_env = -1;  // dev override (HC_TSPLIT)
    if (ts_env < 0) { const char *ev = getenv("HC_TSPLIT"); ts_env = ev ? atoi(ev) : 0; }
    if (ts_env > 0) ts = std::min<int64_t>(ts_env, std::max<int64_t>(1, E / 32));
    static int tu_env = -1;  // dev override (HC_TUNITS)
    if (tu_env < 0) { const char *ev = getenv("HC_TUNITS"); tu_env = ev ? atoi(ev) : 0; }
    if (tu_env > 0 && tu_env <= std::min<int64_t>({units, (int64_t)kTableU, std::max<int64_t>(1, kTableQ / (d * G))})) {
      tu = tu_env;
      if (ts_env <= 0) ts = std::max<int64_t>(1, std::min<int64_t>((4 * (int64_t)num_sms() * tu + units - 1) / units, E / 1024));
    }
    a.tsplit = (int)ts;
    a.tunits = (int)tu;
  }
  a.z = (float *)(w8 + Lw.o_z);
  a.z_stride = Lw.z_stride;
  a.sel_ghist = (uint32_t *)(w8 + Lw.o_sgh);
  const int64_t k_cap = sel_idx ? budget.k_max : Lw.k_eff;  // row stride of idx / w
  a.k_max = k_cap;
  a.sel_idx = sel_idx ? sel_idx : (int32_t *)(w8 + Lw.o_idx);
  a.sel_w = sel_w ? sel_w : (float *)(w8 + Lw.o_w);
  a.sel_k = sel_k;
  a.out = out;
  a.num_sms = num_sms();
  choose_scan(B * H, n_q, (int)g, Lw.cpow2, (int)G, a.num_sms, &a.scan_tpt, &a.scan_split, a.lut8);
  {  // dev overrides (HC_SCAN_SPLIT, HC_SCAN_TPT) for cost-model checks
    static int sp_env = -1, tpt_env = -1;
    if (sp_env < 0) { const char *ev = getenv("HC_SCAN_SPLIT"); sp_env = ev ? atoi(ev) : 0; }
    if (tpt_env < 0) { const char *ev = getenv("HC_SCAN_TPT"); tpt_env = ev ? atoi(ev) : 0; }
    if (sp_env > 0 && sp_env <= g) a.scan_split = sp_env;
    if ((tpt_env == 8 || tpt_env == 16) && !a.lut8) a.scan_tpt = tpt_env;
  }
  a.zpart = (float *)(w8 + Lw.o_zpart);
  a.skpart = (int *)(w8 + Lw.o_skpart);
  a.skctr = (uint32_t *)(w8 + Lw.o_skctr);
  a.skctr_n = Lw.skctr_n;
  if (budget.shared_kv) {
    a.grp = (GroupState *)(w8 + Lw.o_grp);
    a.grp_hist = (unsigned long long *)(w8 + Lw.o_ghist);
    a.grp_chunk = (uint32_t *)(w8 + Lw.o_gchunk);
    a.grp_key = (unsigned long long *)(w8 + Lw.o_gkey);
  }

  return HC_OK;
}

static hc_status decode_impl(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs, int32_t layer,
                             hc_budget budget, float *out, int32_t *sel_idx, float *sel_w, int64_t *sel_k,
                             const hc_decode_debug *dbg, void *ws, size_t ws_bytes, cudaStream_t s,
                             cudaEvent_t join_before_scan);

hc_status hc_decode_attention(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs,
                              int32_t layer, hc_budget budget, float *out, int32_t *sel_idx,
                              float *sel_w, int64_t *sel_k, const hc_decode_debug *dbg, void *ws,
                              size_t ws_bytes, hc_stream_t stream) {
  return decode_impl(q, kc, vs, layer, budget, out, sel_idx, sel_w, sel_k, dbg, ws, ws_bytes,
                     (cudaStream_t)stream, nullptr);
}

// hc_append_decode_attention: the append's encode / value copy runs on a library side stream
// forked from `stream`, concurrently with the table build (both only read the layer's inputs
// and the codebook); the scan waits for it.  Fork / join are event edges, so the call is
// CUDA-graph capturable like the two calls it replaces.
namespace {
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  ~SideStream() {  // thread exit (errors ignored: the context may already be gone at process exit)
    if (join) cudaEventDestroy(join);
    if (fork) cudaEventDestroy(fork);
    if (st) cudaStreamDestroy(st);
  }
};
SideStream *side_stream() {
  thread_local SideStream ss[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  SideStream &x = ss[dev];
  if (!x.st) {
    if (cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming);
  }
  return &x;
}
}  // namespace

hc_status hc_append_decode_attention(const uint16_t *q, hc_kcache *kc, const hc_vstore *vs, int32_t layer,
                                     const uint16_t *k_new, const uint16_t *v_new, hc_budget budget, float *out,
                                     int32_t *sel_idx, float *sel_w, int64_t *sel_k, void *ws, size_t ws_bytes,
                                     hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  SideStream *ss = side_stream();
  if (!ss) return fail(HC_ERR_CUDA, "side stream");
  if (cudaEventRecord(ss->fork, s) != cudaSuccess || cudaStreamWaitEvent(ss->st, ss->fork, 0) != cudaSuccess)
    return fail(HC_ERR_CUDA, "fork");
  hc_status st = hc_append_kv(kc, vs, layer, k_new, v_new, (hc_stream_t)ss->st);
  if (cudaEventRecord(ss->join, ss->st) != cudaSuccess) return fail(HC_ERR_CUDA, "join record");
  if (st) {  // still join the side stream before returning the error
    cudaStreamWaitEvent(s, ss->join, 0);
    return st;
  }
  return decode_impl(q, kc, vs, layer, budget, out, sel_idx, sel_w, sel_k, nullptr, ws, ws_bytes, s, ss->join);
}

static hc_status decode_impl(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs, int32_t layer,
                             hc_budget budget, float *out, int32_t *sel_idx, float *sel_w, int64_t *sel_k,
                             const hc_decode_debug *dbg, void *ws, size_t ws_bytes, cudaStream_t s,
                             cudaEvent_t join_before_scan) {
  LayerArgs a;
  Layout Lw;
  hc_status st = prepare_layer(q, kc, vs, layer, budget, out, sel_idx, sel_w, sel_k, ws, ws_bytes, s,
                               true, a, Lw);
  if (st) return st;
  const int rows = a.B * a.Hq;
  const int64_t n_q = a.n_q, n_cand = a.n_cand;
  cudaError_t e;
  // Eq. 5 placement policy (measured): host-mapped values -> the GQA union
  // de-duplicated gather kernel (fewer host-link bytes: +18 % steps/s at config 3); HBM
  // values -> the high-occupancy per-head row gather (many rows in flight per SM).
  // HC_GATHER=fused|union|rows overrides; "fused" runs Eq. 5 inside the select kernel.
  static int gather_mode = -1;  // 0 fused, 1 union, 3 rows, 2 by placement
  if (gather_mode < 0) {
    const char *ev = getenv("HC_GATHER");
    gather_mode = (ev && !strcmp(ev, "fused")) ? 0
                  : (ev && !strcmp(ev, "union")) ? 1
                  : (ev && !strcmp(ev, "rows")) ? 3 : 2;
  }
  const bool want_union = gather_mode == 1 || (gather_mode == 2 && a.v_placement == 1);
  // shared per-KV-head selection (R8): the G rows keep one list -> always the union gather
  const bool shared = budget.shared_kv != 0;
  const bool union_gather = !budget.select_only && (want_union || shared) && a.G > 1;
  const bool want_rows = gather_mode == 3 || (gather_mode == 2 && a.v_placement == 0);
  bool rows_gather = !budget.select_only && !union_gather && (want_rows || shared) && a.d == 128;
  if (shared && !budget.select_only && !union_gather && !rows_gather)
    return fail(HC_ERR_UNSUPPORTED, "shared_kv with G = 1 needs d = 128");
  // the gather's completion counters are zeroed by k_table (no memset between chain kernels)
  if (union_gather) { a.gdone = (uint32_t *)((uint8_t *)ws + Lw.o_udone); a.gdone_n = a.B * a.Hkv; }
  if (rows_gather) { a.gdone = (uint32_t *)((uint8_t *)ws + Lw.o_rdone); a.gdone_n = rows; }
  // Eq. 3 stage profiling hook (one-shot): events around table + resident + scan
  cudaEvent_t e3b = g_eq3_ev[0], e3e = g_eq3_ev[1];
  g_eq3_ev[0] = g_eq3_ev[1] = nullptr;
  unsigned e3flag = 0u;
  if (e3b || e3e) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    e3flag = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  }
  if (e3b) cudaEventRecordWithFlags(e3b, s, e3flag);
  if ((e = launch_table(a, s)) != cudaSuccess) return cuda_check(e, "table");
  if (join_before_scan && cudaStreamWaitEvent(s, join_before_scan, 0) != cudaSuccess)
    return fail(HC_ERR_CUDA, "join");  // the append (side stream) wrote the new token
  if ((e = launch_resident(a, s)) != cudaSuccess) return cuda_check(e, "resident");
  if (n_q > 0 && (e = launch_scan(a, s)) != cudaSuccess) return cuda_check(e, "scan");
  if (e3e) cudaEventRecordWithFlags(e3e, s, e3flag);
  SelArgs sa{};
  sa.hs = a.hs; sa.z = a.z; sa.z_stride = a.z_stride; sa.rows = rows; sa.n = n_cand;
  sa.tau_q = a.tau_q; sa.k_max = a.k_max; sa.renorm = a.renorm;
  sa.sel_idx = a.sel_idx; sa.sel_w = a.sel_w; sa.sel_k = sel_k;
  sa.ghist = (uint32_t *)((uint8_t *)ws + Lw.o_sgh);
  sa.gmass = (unsigned long long *)(sa.ghist + rows * kNB);
  sa.fcnt = (uint32_t *)((uint8_t *)ws + Lw.o_sfc);
  sa.cntlo = (uint32_t *)((uint8_t *)ws + Lw.o_scl);
  sa.pre = (unsigned long long *)((uint8_t *)ws + Lw.o_spre);
  sa.list = (unsigned long long *)((uint8_t *)ws + Lw.o_slist);
  sa.nch = select_chunks(n_cand);
  sa.cap = Lw.scap;
  // the round-1 fused select kernel stays reachable for A/B measurements (HC_SELECT=fused) and
  // for Eq. 5 inside the select kernel (HC_GATHER=fused)
  // Selection kernel (hc_select_pass.cu): rows up to 64K candidates in one cluster
  // kernel (k_sel_small: scores in registers, latency-bound short rows, configs 1-2), longer
  // rows in three bandwidth-shaped passes (configs 3-5).  HC_SELECT=pass forces the passes,
  // HC_SELECT=fused the round-1 cluster kernel (read per call: the tests run all of them).
  const char *sel_env = getenv("HC_SELECT");
  const bool sel_old = sel_env && !strcmp(sel_env, "fused");
  const int sel_force = (sel_env && !strcmp(sel_env, "pass")) ? 1 : 0;
  const bool fused_gather = !(budget.select_only || union_gather || rows_gather);
  if (shared) {
    if ((e = launch_group_select(a, n_q > 0 ? a.scan_split : 1, s)) != cudaSuccess)
      return cuda_check(e, "shared select");
  } else if (sel_old || fused_gather) {
    if ((e = launch_select_fused(sa, a, n_q > 0 ? a.scan_split : 1, fused_gather ? 1 : 0, a.num_sms, s)) !=
        cudaSuccess)
      return cuda_check(e, "select");
  } else {
    // HBM values, per-head rows gather: the long-row passes fuse Eq. 5 into their K3
    // (k_sel_write_gather) unless HC_K3G=0
    const char *k3g_ev = getenv("HC_K3G");  // read per call (the tests run both)
    const int k3g_env = (k3g_ev && !strcmp(k3g_ev, "0")) ? 0 : 1;
    SelGather wg{&a, (float *)((uint8_t *)ws + Lw.o_wpart), (uint32_t *)((uint8_t *)ws + Lw.o_rdone), 0};
    const bool try_wg = k3g_env && rows_gather && a.d == 128 && !a.g_cnt;
    if ((e = launch_select(sa, n_q > 0 ? a.scan_split : 1, a.num_sms, s, sel_force, try_wg ? &wg : nullptr)) !=
        cudaSuccess)
      return cuda_check(e, "select");
    if (wg.used) rows_gather = false;  // Eq. 5 done inside K3
  }
  if (rows_gather) {
    uint32_t *done = (uint32_t *)((uint8_t *)ws + Lw.o_rdone);
    const int64_t kc2 = a.k_max < n_cand ? a.k_max : n_cand;
    if ((e = launch_gather_rows(a, kc2, (float *)((uint8_t *)ws + Lw.o_rpart), done, s)) != cudaSuccess)
      return cuda_check(e, "gather");
  }
  if (union_gather) {
    uint32_t *done = (uint32_t *)((uint8_t *)ws + Lw.o_udone);
    if ((e = launch_gather_union(a, (float *)((uint8_t *)ws + Lw.o_upart), done, s)) != cudaSuccess)
      return cuda_check(e, "gather");
  }
  if (dbg) {
    if (dbg->z) {
      dim3 gz((unsigned)((n_cand + 255) / 256), (unsigned)rows);
      k_z_to_int<<<gz, 256, 0, s>>>(a.z, a.z_stride, dbg->z, n_cand);
      note_launch();
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_check(e, "debug z");
    }
    if (dbg->e || dbg->S || dbg->M || dbg->kstar) {
      // strided fields of HeadState -> dense arrays
      if (dbg->e) cudaMemcpy2DAsync(dbg->e, 4, &a.hs->e, sizeof(HeadState), 4, rows, cudaMemcpyDeviceToDevice, s);
      if (dbg->S) cudaMemcpy2DAsync(dbg->S, 8, &a.hs->S, sizeof(HeadState), 8, rows, cudaMemcpyDeviceToDevice, s);
      if (dbg->M) cudaMemcpy2DAsync(dbg->M, 4, &a.hs->M, sizeof(HeadState), 4, rows, cudaMemcpyDeviceToDevice, s);
      if (dbg->kstar) cudaMemcpy2DAsync(dbg->kstar, 8, &a.hs->kstar, sizeof(HeadState), 8, rows, cudaMemcpyDeviceToDevice, s);
      if ((e = cudaGetLastError()) != cudaSuccess) return cuda_check(e, "debug");
    }
  }
  return HC_OK;
}

hc_status hc_gather_values(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, const int32_t *sel_idx,
                           const float *sel_w, const int64_t *sel_k, int64_t k_stride, int64_t tok_begin,
                           int64_t tok_end, float *out, void *ws, size_t ws_bytes, hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!sel_idx || !sel_w || !sel_k || !out) return fail(HC_ERR_ARG, "sel_idx/sel_w/sel_k/out NULL");
  if (k_stride < 1) return fail(HC_ERR_ARG, "k_stride < 1");
  if (tok_begin < 0 || tok_end < tok_begin) return fail(HC_ERR_RANGE, "bad token range [%lld, %lld)",
                                                        (long long)tok_begin, (long long)tok_end);
  LayerArgs a;
  Layout Lw;
  hc_budget bud{1.0f, k_stride, 0, 0, 0};
  hc_status st = prepare_layer(nullptr, kc, vs, layer, bud, out, const_cast<int32_t *>(sel_idx),
                               const_cast<float *>(sel_w), const_cast<int64_t *>(sel_k), ws, ws_bytes, s,
                               false, a, Lw);
  if (st) return st;
  a.k_in = sel_k;
  a.gtok_lo = tok_begin < a.n_cand ? tok_begin : a.n_cand;
  a.gtok_hi = tok_end < a.n_cand ? tok_end : a.n_cand;
  uint32_t *done = (uint32_t *)((uint8_t *)ws + Lw.o_udone);
  cudaError_t e = cudaMemsetAsync(done, 0, (size_t)a.B * a.Hkv * 4, s);
  if (e != cudaSuccess) return cuda_check(e, "gather counters");
  if (a.gtok_hi <= a.gtok_lo) {  // nothing in range: the GPU share is zero
    e = cudaMemsetAsync(out, 0, (size_t)a.B * a.Hq * a.d * 4, s);
    return e != cudaSuccess ? cuda_check(e, "gather zero") : HC_OK;
  }
  if ((e = launch_gather_union(a, (float *)((uint8_t *)ws + Lw.o_upart), done, s)) != cudaSuccess)
    return cuda_check(e, "gather");
  return HC_OK;
}

hc_status hc_add_partial(float *out, const float *part, int64_t n, hc_stream_t stream) {
  if (!out || !part) return fail(HC_ERR_ARG, "out/part NULL");
  if (n < 0) return fail(HC_ERR_ARG, "n < 0");
  cudaError_t e = launch_add_partial(out, part, n, (cudaStream_t)stream);
  return e != cudaSuccess ? cuda_check(e, "add partial") : HC_OK;
}

// ---------------------------------------------------------------- sequence-sharded decode
static hc_status shard_prepare(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs,
                               int32_t layer, hc_budget budget, void *ws, size_t ws_bytes,
                               cudaStream_t s, bool need_q, LayerArgs &a, Layout &Lw, SelArgs &sa,
                               int32_t *sel_idx = nullptr, float *sel_w = nullptr,
                               int64_t *sel_k = nullptr) {
  if (budget.shared_kv) return fail(HC_ERR_UNSUPPORTED, "sharded decode selects per query head (shared_kv = 0)");
  if (kc && kc->res_cap > 0 && kc->n_res[layer < 0 || layer >= HC_MAX_LAYERS ? 0 : layer] > 0)
    return fail(HC_ERR_UNSUPPORTED, "sharded decode does not take a resident window (n_res must be 0)");
  float dummy_out = 0.0f;
  hc_status st = prepare_layer(q, kc, vs, layer, budget, need_q ? &dummy_out : &dummy_out, sel_idx,
                               sel_w, sel_k, ws, ws_bytes, s, need_q, a, Lw);
  if (st) return st;
  a.out = nullptr;
  sa = SelArgs{};
  sa.hs = a.hs; sa.z = a.z; sa.z_stride = a.z_stride; sa.rows = a.B * a.Hq; sa.n = a.n_cand;
  // the cap is GLOBAL: a shard's own candidate count may be below k_max (k_eff clamps only
  // the workspace list stride of the unsharded path); the kept lists are written with the
  // caller's stride budget.k_max in the finish phase
  sa.tau_q = a.tau_q; sa.k_max = budget.k_max; sa.renorm = a.renorm;
  sa.sel_idx = a.sel_idx; sa.sel_w = a.sel_w; sa.sel_k = sel_k;
  return HC_OK;
}

size_t hc_shard_workspace_bytes(const hc_kcache *kc, hc_budget budget) {
  return hc_decode_workspace_bytes(kc, budget);
}

hc_status hc_shard_begin(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs, int32_t layer,
                         hc_budget budget, int32_t *stats, void *ws, size_t ws_bytes,
                         hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  LayerArgs a; Layout Lw; SelArgs sa;
  hc_status st = shard_prepare(q, kc, vs, layer, budget, ws, ws_bytes, s, true, a, Lw, sa);
  if (st) return st;
  if (!stats) return fail(HC_ERR_ARG, "stats NULL");
  cudaError_t e;
  if ((e = launch_table(a, s)) != cudaSuccess) return cuda_check(e, "table");
  if (a.n_q > 0 && (e = launch_scan(a, s)) != cudaSuccess) return cuda_check(e, "scan");
  return cuda_check(launch_shard_stats(a, a.n_q > 0 ? a.scan_split : 1, stats, s), "shard stats");
}

hc_status hc_shard_hist1(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                         const int32_t *gstats, uint64_t *h1, void *ws, size_t ws_bytes,
                         hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  LayerArgs a; Layout Lw; SelArgs sa;
  hc_status st = shard_prepare(nullptr, kc, vs, layer, budget, ws, ws_bytes, s, false, a, Lw, sa);
  if (st) return st;
  if (!gstats || !h1) return fail(HC_ERR_ARG, "NULL pointer");
  return cuda_check(launch_shard_hist1(a, gstats, (unsigned long long *)h1, s), "shard hist1");
}

hc_status hc_shard_hist2(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                         const int32_t *gstats, const uint64_t *h1, uint64_t *h2, void *ws,
                         size_t ws_bytes, hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  LayerArgs a; Layout Lw; SelArgs sa;
  hc_status st = shard_prepare(nullptr, kc, vs, layer, budget, ws, ws_bytes, s, false, a, Lw, sa);
  if (st) return st;
  if (!gstats || !h1 || !h2) return fail(HC_ERR_ARG, "NULL pointer");
  return cuda_check(launch_shard_hist2(a, sa, gstats, (const unsigned long long *)h1,
                                       (unsigned long long *)h2, s), "shard hist2");
}

hc_status hc_shard_counts(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                          const uint64_t *h2, uint64_t *cnt, void *ws, size_t ws_bytes,
                          hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  LayerArgs a; Layout Lw; SelArgs sa;
  hc_status st = shard_prepare(nullptr, kc, vs, layer, budget, ws, ws_bytes, s, false, a, Lw, sa);
  if (st) return st;
  if (!h2 || !cnt) return fail(HC_ERR_ARG, "NULL pointer");
  return cuda_check(launch_shard_counts(a, sa, (const unsigned long long *)h2,
                                        (uint32_t *)((uint8_t *)ws + Lw.o_chunk),
                                        (unsigned long long *)cnt, s), "shard counts");
}

hc_status hc_shard_finish(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                          const uint64_t *allcnt, int32_t rank, int32_t world, int64_t shard_base,
                          float *out, int32_t *sel_idx, float *sel_w, int64_t *sel_k, void *ws,
                          size_t ws_bytes, hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (rank < 0 || world < 1 || rank >= world) return fail(HC_ERR_RANGE, "rank/world");
  if (!allcnt || !out || !sel_idx || !sel_w) return fail(HC_ERR_ARG, "NULL pointer");
  if (shard_base < 0) return fail(HC_ERR_RANGE, "shard_base < 0");
  LayerArgs a; Layout Lw; SelArgs sa;
  hc_status st = shard_prepare(nullptr, kc, vs, layer, budget, ws, ws_bytes, s, false, a, Lw, sa,
                               sel_idx, sel_w, sel_k);
  if (st) return st;
  if (shard_base + a.n_cand > 0x7fffffffLL) return fail(HC_ERR_UNSUPPORTED, "global index >= 2^31");
  uint8_t *w8 = (uint8_t *)ws;
  cudaError_t e = launch_shard_finish(a, sa, (const uint32_t *)(w8 + Lw.o_chunk),
                                      (const unsigned long long *)allcnt, rank, shard_base,
                                      (float *)(w8 + Lw.o_part), out, s, (int64_t *)(w8 + Lw.o_grange),
                                      (float *)(w8 + Lw.o_rpart), (uint32_t *)(w8 + Lw.o_rdone),
                                      (float *)(w8 + Lw.o_upart), (uint32_t *)(w8 + Lw.o_udone),
                                      (unsigned long long *)(w8 + Lw.o_spre), (float *)(w8 + Lw.o_wpart));
  if (e != cudaSuccess) return cuda_check(e, "shard finish");
  if (sel_k) {
    const int rows = a.B * a.Hq;
    e = cudaMemcpy2DAsync(sel_k, 8, &a.hs->ksel, sizeof(HeadState), 8, rows,
                          cudaMemcpyDeviceToDevice, s);
  }
  return cuda_check(e, "shard finish");
}

size_t hc_select_workspace_bytes(int64_t rows, int64_t n, hc_budget budget) {
  (void)budget;
  if (rows <= 0 || n <= 0) return 0;
  const int64_t zs = round_up(n, 64);
  return align256((size_t)rows * sizeof(HeadState)) + align256((size_t)rows * zs * 4) +
         align256((size_t)rows * kNB * 4) * 2 + align256((size_t)rows * kNB * 8) +
         align256((size_t)rows * select_chunks(n) * 4) + align256((size_t)rows * select_chunks(n) * 8) +
         align256((size_t)rows * select_list_cap(n) * 8);
}

hc_status hc_select_topk(const float *scores, int64_t rows, int64_t n, int32_t d, hc_budget budget,
                         int32_t *idx, float *w, int64_t *k, void *ws, size_t ws_bytes,
                         hc_stream_t stream) {
  if (rows <= 0 || rows > 65535) return fail(HC_ERR_ARG, "rows must be in [1, 65535]");
  if (n <= 0) return fail(HC_ERR_EMPTY, "n == 0");
  if (n > (1ll << 27)) return fail(HC_ERR_UNSUPPORTED, "n > 2^27 (per-chunk selection state)");
  if (d <= 0) return fail(HC_ERR_ARG, "d <= 0");
  if (!scores || !idx || !w) return fail(HC_ERR_ARG, "NULL pointer");
  if (!(budget.tau > 0.0f && budget.tau <= 1.0f)) return fail(HC_ERR_ARG, "tau=%g not in (0,1]", budget.tau);
  if (budget.k_max < 1) return fail(HC_ERR_ARG, "k_max < 1");
  const size_t need = hc_select_workspace_bytes(rows, n, budget);
  if (!ws || ws_bytes < need) return fail(HC_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t *w8 = (uint8_t *)ws;
  const int64_t zs = round_up(n, 64);
  size_t o = 0;
  HeadState *hs = (HeadState *)(w8 + o); o += align256((size_t)rows * sizeof(HeadState));
  float *z = (float *)(w8 + o); o += align256((size_t)rows * zs * 4);
  SelArgs sa{};
  sa.ghist = (uint32_t *)(w8 + o); o += align256((size_t)rows * kNB * 4);
  sa.gmass = (unsigned long long *)(w8 + o); o += align256((size_t)rows * kNB * 8);
  sa.fcnt = (uint32_t *)(w8 + o); o += align256((size_t)rows * kNB * 4);
  sa.cntlo = (uint32_t *)(w8 + o); o += align256((size_t)rows * select_chunks(n) * 4);
  sa.pre = (unsigned long long *)(w8 + o); o += align256((size_t)rows * select_chunks(n) * 8);
  sa.list = (unsigned long long *)(w8 + o);
  sa.nch = select_chunks(n);
  sa.cap = select_list_cap(n);
  cudaError_t e;
  const float kappa0 = (float)(1.4426950408889634 / sqrt((double)d));
  if ((e = launch_select_float_prep(scores, rows, n, z, zs, hs, kappa0, s, sa.ghist, sa.gmass)) != cudaSuccess)
    return cuda_check(e, "prep");
  sa.hs = hs; sa.z = z; sa.z_stride = zs; sa.rows = (int)rows; sa.n = n;
  sa.tau_q = (uint32_t)rint((double)budget.tau * 16777216.0);
  sa.k_max = budget.k_max; sa.renorm = budget.renorm ? 1 : 0;
  sa.sel_idx = idx; sa.sel_w = w; sa.sel_k = k;
  return cuda_check(launch_select(sa, 1, num_sms(), s), "hc_select_topk");
}

}  // extern "C"
