// hc_kmeans.cu -- NEXT f4: the prefill side.
//
// (1) Bulk key encoding (R1) for many rows: the group's codebook slice is staged in
//     shared memory chunk by chunk and every thread scores its rows against the centroids
//     in ascending order (broadcast shared-memory reads; the first strict minimum is the
//     lowest-index argmin, so no cross-thread tie handling is needed).  The decode-time
//     k_encode (hc_encode.cu) instead spreads ONE row's centroids over a CTA (latency).
//     Bound: FP32 issue, (2·dbar + 3) lane-ops per (row, centroid).
// (2) One MiniBatchKMeans step (Sculley 2010 Alg. 1 in its batched form, DESIGN F4):
//     labels = bulk encode of the sampled rows with the step's starting centres; exact
//     per-centre sums in int64 units of 2^-24 (every fp16 value is such a multiple) via
//     global 64-bit atomics (order-free); update C <- (C·v + s)/(v + n) in double with
//     the oracle's operation order, v <- v + n.
#include "hc_internal.h"

namespace hc {

constexpr int kBT = 256;          // threads per CTA
constexpr int kBChunkBytes = 32768;

template <int DBAR> struct BulkCfg {
  static constexpr int kR = DBAR <= 4 ? 8 : (DBAR == 8 ? 4 : 2);  // rows per thread
  static constexpr int kCh = kBChunkBytes / (DBAR * 4);           // centroids per chunk
};

__device__ __forceinline__ int64_t bulk_rowoff(const EncodeArgs &a, int64_t r) {
  const int64_t kr = a.kidx ? a.kidx[r] : r;
  return (kr / a.kmap.R1) * a.kmap.s1 + (kr % a.kmap.R1) * a.kmap.s2 + a.kmap.s0;
}

template <int DBAR>
__global__ void __launch_bounds__(kBT) k_encode_bulk(EncodeArgs a) {
  constexpr int kR = BulkCfg<DBAR>::kR, kCh = BulkCfg<DBAR>::kCh;
  __shared__ __align__(16) float cs[kCh * DBAR];
  const int i = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kBT * kR;
  float kb[kR][DBAR];
  bool ok[kR];
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    const int64_t r = r0 + k * kBT + threadIdx.x;
    ok[k] = r < a.rows && (!a.kidx || (a.kidx[r] >= 0 && a.kidx[r] < a.n_keys));
    const uint16_t *kp = a.keys + (ok[k] ? bulk_rowoff(a, r) : 0) + (int64_t)i * DBAR;
#pragma unroll
    for (int e = 0; e < DBAR; ++e) kb[k][e] = ok[k] ? h2f(kp[e]) : 0.0f;
  }
  float best[kR];
  int bm[kR];
#pragma unroll
  for (int k = 0; k < kR; ++k) { best[k] = INFINITY; bm[k] = 0; }
  const float *Ci = a.C + (int64_t)(a.cbg == 1 ? 0 : i) * a.c * DBAR;
  for (int m0 = 0; m0 < a.c; m0 += kCh) {
    const int nc = a.c - m0 < kCh ? a.c - m0 : kCh;
    __syncthreads();
    const float *src = Ci + (int64_t)m0 * DBAR;
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      for (int q = threadIdx.x * 4; q < nc * DBAR; q += kBT * 4) {
        if (q + 4 <= nc * DBAR) {
          *reinterpret_cast<float4 *>(cs + q) = __ldg(reinterpret_cast<const float4 *>(src + q));
        } else {
          for (int u = q; u < nc * DBAR; ++u) cs[u] = src[u];
        }
      }
    } else {  // slice not 16-B aligned (c·dbar not a multiple of 4)
      for (int q = threadIdx.x; q < nc * DBAR; q += kBT) cs[q] = src[q];
    }
    __syncthreads();
#pragma unroll 2
    for (int m = 0; m < nc; ++m) {
      float cm[DBAR];
#pragma unroll
      for (int e = 0; e < DBAR; ++e) cm[e] = cs[m * DBAR + e];
#pragma unroll
      for (int k = 0; k < kR; ++k) {
        float dist = 0.0f;
#pragma unroll
        for (int e = 0; e < DBAR; ++e) {
          const float diff = __fsub_rn(kb[k][e], cm[e]);
          dist = __fmaf_rn(diff, diff, dist);
        }
        if (dist < best[k]) { best[k] = dist; bm[k] = m0 + m; }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    const int64_t r = r0 + k * kBT + threadIdx.x;
    if (r < a.rows) {
      a.codes[(r / a.omap.R1) * a.omap.s1 + (r % a.omap.R1) * a.omap.s2 + a.omap.s0 + (int64_t)i * a.gstride] =
          ok[k] ? (uint16_t)bm[k] : (uint16_t)0xFFFF;
    }
  }
}

cudaError_t launch_encode_bulk(const EncodeArgs &a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  const int dbar = a.d / a.g;
#define HC_BULK(D)                                                                           \
  {                                                                                          \
    const int64_t per = (int64_t)kBT * BulkCfg<D>::kR;                                       \
    dim3 grid((unsigned)((a.rows + per - 1) / per), (unsigned)a.g);                          \
    k_encode_bulk<D><<<grid, kBT, 0, s>>>(a);                                                \
    note_launch();                                                                           \
    break;                                                                                   \
  }
  switch (dbar) {
    case 1: HC_BULK(1)
    case 2: HC_BULK(2)
    case 4: HC_BULK(4)
    case 8: HC_BULK(8)
    case 16: HC_BULK(16)
    default: return cudaErrorInvalidValue;
  }
#undef HC_BULK
  return cudaGetLastError();
}

// ---------------------------------------------------------------- MiniBatchKMeans step
// one thread per (sample s, group i): n[ci][m] += 1, S[ci][m][e] += key·2^24 (exact int64)
__global__ void __launch_bounds__(256) k_km_accum(const uint16_t *keys, int64_t n_keys,
                                                  const int64_t *sample, int64_t b, int d, int g,
                                                  int c, int cbg, const uint16_t *labels,
                                                  unsigned long long *n, unsigned long long *S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= b * g) return;
  const int64_t s = t / g;
  const int i = (int)(t - s * g);
  const int64_t j = sample[s];
  if (j < 0 || j >= n_keys) return;
  const int dbar = d / g, ci = cbg == 1 ? 0 : i;
  const int m = labels[(int64_t)i * b + s];
  const int64_t cm = (int64_t)ci * c + m;
  atomicAdd(&n[cm], 1ull);
  for (int e = 0; e < dbar; ++e) {
    const float x = h2f(keys[j * d + (int64_t)i * dbar + e]);
    const long long fx = __float2ll_rn(__fmul_rn(x, 16777216.0f));  // exact: fp16 · 2^24
    atomicAdd(&S[cm * dbar + e], (unsigned long long)fx);            // two's complement sum
  }
}

// one thread per (ci, m): C <- (C·v + S·2^-24)/(v + n) in double (oracle order), v += n
__global__ void __launch_bounds__(256) k_km_update(int64_t cc, int dbar, float *C, int64_t *counts,
                                                   const unsigned long long *n,
                                                   const unsigned long long *S) {
  const int64_t cm = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cm >= cc) return;
  const long long nm = (long long)n[cm];
  if (!nm) return;
  const long long v = counts[cm];
  for (int e = 0; e < dbar; ++e) {
    const double num = __dadd_rn(__dmul_rn((double)C[cm * dbar + e], __ll2double_rn(v)),
                                 __dmul_rn(__ll2double_rn((long long)S[cm * dbar + e]), 0x1p-24));
    C[cm * dbar + e] = __double2float_rn(__ddiv_rn(num, __ll2double_rn(v + nm)));
  }
  counts[cm] = v + nm;
}

cudaError_t launch_kmeans_step(const EncodeArgs &enc, const int64_t *sample, int64_t b,
                               float *C, int64_t *counts, unsigned long long *n,
                               unsigned long long *S, cudaStream_t st) {
  const int dbar = enc.d / enc.g;
  const int64_t cc = (int64_t)enc.cbg * enc.c;
  cudaError_t e;
  if ((e = cudaMemsetAsync(n, 0, (size_t)cc * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(S, 0, (size_t)cc * dbar * 8, st)) != cudaSuccess) return e;
  if ((e = launch_encode_bulk(enc, st)) != cudaSuccess) return e;
  k_km_accum<<<(unsigned)((b * enc.g + 255) / 256), 256, 0, st>>>(
      enc.keys, enc.n_keys, sample, b, enc.d, enc.g, enc.c, enc.cbg, enc.codes, n, S);
  k_km_update<<<(unsigned)((cc + 255) / 256), 256, 0, st>>>(cc, dbar, C, counts, n, S);
  note_launch(2);
  return cudaGetLastError();
}

}  // namespace hc
