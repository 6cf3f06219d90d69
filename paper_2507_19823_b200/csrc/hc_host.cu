// hc_host.cu -- the paper's "CPU part" of Eq. 2 (§3.2):
// Eq. 5's sparse weighted sum over the offloaded values, executed on host threads from
// the selection the GPU produced.  fp16 -> fp32 through a 64K-entry table; each thread
// owns whole rows (query heads), accumulates in fp32 in index order.
#include <cuda_runtime.h>
#include <omp.h>
#include <stdint.h>
#include <string.h>

#include <atomic>

#include "../../include/hc.h"

namespace {

float g_h2f[65536];
std::atomic<int> g_h2f_ready{0};

float half_bits_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h >> 15) << 31, exp = (h >> 10) & 0x1f, man = h & 0x3ff;
  uint32_t bits;
  if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else {
      float v = (float)man * 5.9604644775390625e-08f;  // man * 2^-24
      memcpy(&bits, &v, 4);
      bits |= sign;
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | (man << 13);
  } else {
    bits = sign | ((exp + 112u) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

void init_table() {
  if (g_h2f_ready.load(std::memory_order_acquire)) return;
  for (uint32_t h = 0; h < 65536; ++h) g_h2f[h] = half_bits_to_float((uint16_t)h);
  g_h2f_ready.store(1, std::memory_order_release);
}

struct HostArgs {
  const int32_t *idx;
  const float *w;
  const int64_t *k;
  int64_t rows, k_stride;
  const uint16_t *V;
  int64_t v_b_stride, v_kv_stride;
  int32_t Hq, G, d;
  float *out;
  int32_t threads;
  bool owned_once;
};

void run(const HostArgs &a) {
  init_table();
  const int nt = a.threads > 0 ? a.threads : omp_get_max_threads();
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1)
  for (int64_t row = 0; row < a.rows; ++row) {
    const int64_t b = row / a.Hq, hq = row % a.Hq, kv = hq / a.G;
    const uint16_t *Vb = a.V + b * a.v_b_stride + kv * a.v_kv_stride;
    float acc[256];
    for (int e = 0; e < a.d; ++e) acc[e] = 0.0f;
    const int64_t kk = a.k[row];
    const int32_t *ix = a.idx + row * a.k_stride;
    const float *wt = a.w + row * a.k_stride;
    for (int64_t r = 0; r < kk; ++r) {
      const uint16_t *vr = Vb + (int64_t)ix[r] * a.d;
      const float wr = wt[r];
      if (r + 4 < kk) __builtin_prefetch(Vb + (int64_t)ix[r + 4] * a.d, 0, 0);
      for (int e = 0; e < a.d; ++e) acc[e] += wr * g_h2f[vr[e]];
    }
    for (int e = 0; e < a.d; ++e) a.out[row * a.d + e] = acc[e];
  }
}

void CUDART_CB host_cb(void *p) {
  HostArgs *a = static_cast<HostArgs *>(p);
  run(*a);
  if (a->owned_once) delete a;
}

}  // namespace

extern "C" {

hc_status hc_host_weighted_sum(const int32_t *idx, const float *w, const int64_t *k, int64_t rows,
                               int64_t k_stride, const uint16_t *V, int64_t v_b_stride,
                               int64_t v_kv_stride, int32_t Hq, int32_t G, int32_t d, float *out,
                               int32_t threads) {
  if (!idx || !w || !k || !V || !out) return HC_ERR_ARG;
  if (rows < 0 || Hq <= 0 || G <= 0 || d <= 0 || d > 256 || Hq % G) return HC_ERR_SHAPE;
  HostArgs a{idx, w, k, rows, k_stride, V, v_b_stride, v_kv_stride, Hq, G, d, out, threads, false};
  run(a);
  return HC_OK;
}

hc_status hc_enqueue_host_weighted_sum(const int32_t *idx, const float *w, const int64_t *k,
                                       int64_t rows, int64_t k_stride, const uint16_t *V,
                                       int64_t v_b_stride, int64_t v_kv_stride, int32_t Hq,
                                       int32_t G, int32_t d, float *out, int32_t threads,
                                       hc_stream_t stream) {
  if (!idx || !w || !k || !V || !out) return HC_ERR_ARG;
  if (rows < 0 || Hq <= 0 || G <= 0 || d <= 0 || d > 256 || Hq % G) return HC_ERR_SHAPE;
  cudaStream_t s = (cudaStream_t)stream;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  // a captured host node may run many times: its argument block lives as long as the library
  HostArgs *a = new HostArgs{idx, w, k, rows, k_stride, V, v_b_stride, v_kv_stride, Hq, G, d,
                             out, threads, cap != cudaStreamCaptureStatusActive};
  if (cudaLaunchHostFunc(s, host_cb, a) != cudaSuccess) {
    delete a;
    return HC_ERR_CUDA;
  }
  return HC_OK;
}

}  // extern "C"
