// hc_table.cu -- row a1: the query/codebook table T = q̄·C (§3.2 P:229,
// "yields an intermediate hash table T ∈ R^{g×c}. The computational cost is O(dc),
// constant with respect to sequence length n"), in the R2 fixed-point form, and the
// exact scores of the resident recent-window tokens (R3).
//
// Layout of T in the workspace: [unit = b*Hkv+kv][group i][m < cpow2][G heads] int16,
// i.e. one 8-byte entry per centroid serving the G = 4 GQA heads of the KV head, so
// the scan does ONE shared-memory lookup per (token, group) for all G heads.
// Entries m >= c are zero (the scan masks codes to cpow2-1).
#include <float.h>

#include "hc_internal.h"

namespace hc {

constexpr int kTB = 256;  // centroids per CTA

template <int G, int DBAR>
__device__ __forceinline__ void table_entry(const float (&qs)[G][DBAR], const float *Ci, int m,
                                            int c, float (&t)[G]) {
#pragma unroll
  for (int h = 0; h < G; ++h) t[h] = 0.0f;
  if (m < c) {
    float cm[DBAR];
#pragma unroll
    for (int e = 0; e < DBAR; ++e) cm[e] = __ldg(Ci + (int64_t)m * DBAR + e);
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float acc = __fmul_rn(qs[h][0], cm[0]);
#pragma unroll
      for (int e = 1; e < DBAR; ++e) acc = __fmaf_rn(qs[h][e], cm[e], acc);
      t[h] = acc;
    }
  }
}

// PHASE 0: per-head max |t| (atomicMax on non-negative float bits).
// PHASE 1: quantise with e_h and store the packed G x int16 entries.
template <int G, int DBAR, int PHASE>
__global__ void __launch_bounds__(kTB) k_table(LayerArgs a) {
  const int u = blockIdx.z;
  const int b = u / a.Hkv, kv = u - b * a.Hkv;
  const int i = blockIdx.y;
  const int m = blockIdx.x * kTB + threadIdx.x;
  const int hq0 = kv * G;
  float qs[G][DBAR];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < DBAR; ++e)
      qs[h][e] = h2f(__ldg(a.q + ((int64_t)b * a.Hq + hq0 + h) * a.d + i * DBAR + e));
  const float *Ci = a.C + (int64_t)(a.cbg == 1 ? 0 : i) * a.c * DBAR;
  float t[G];
  table_entry<G, DBAR>(qs, Ci, m, a.c, t);
  HeadState *hs = a.hs + (int64_t)b * a.Hq + hq0;
  if (PHASE == 0) {
    __shared__ float red[G][kTB / 32];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float v = fabsf(t[h]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
      if ((threadIdx.x & 31) == 0) red[h][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < G) {
      float v = 0.0f;
#pragma unroll
      for (int w = 0; w < kTB / 32; ++w) v = fmaxf(v, red[threadIdx.x][w]);
      atomicMax(&hs[threadIdx.x].amax, __float_as_uint(v));
    }
  } else {
    int16_t packed[G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const int e = scale_exponent(__uint_as_float(hs[h].amax));
      packed[h] = (int16_t)quant_t(t[h], pow2f(e));
    }
    int16_t *dst = a.T + (((int64_t)u * a.g + i) * a.cpow2 + m) * G;
    if constexpr (G == 4) {
      uint2 v;
      v.x = (uint32_t)(uint16_t)packed[0] | ((uint32_t)(uint16_t)packed[1] << 16);
      v.y = (uint32_t)(uint16_t)packed[2] | ((uint32_t)(uint16_t)packed[3] << 16);
      *reinterpret_cast<uint2 *>(dst) = v;
    } else if constexpr (G == 2) {
      *reinterpret_cast<uint32_t *>(dst) =
          (uint32_t)(uint16_t)packed[0] | ((uint32_t)(uint16_t)packed[1] << 16);
    } else {
#pragma unroll
      for (int h = 0; h < G; ++h) dst[h] = packed[h];
    }
    if (blockIdx.x == 0 && i == 0 && threadIdx.x < G) {
      const int e = scale_exponent(__uint_as_float(hs[threadIdx.x].amax));
      hs[threadIdx.x].e = e;
      hs[threadIdx.x].kappa = __fmul_rn(a.kappa0, pow2f(-e));
    }
  }
}

template <int G, int DBAR>
static cudaError_t table_g_d(const LayerArgs &a, cudaStream_t s) {
  dim3 grid((unsigned)(a.cpow2 / kTB), (unsigned)a.g, (unsigned)(a.B * a.Hkv));
  k_table<G, DBAR, 0><<<grid, kTB, 0, s>>>(a);
  k_table<G, DBAR, 1><<<grid, kTB, 0, s>>>(a);
  return cudaGetLastError();
}

template <int G>
static cudaError_t table_g(const LayerArgs &a, cudaStream_t s) {
  switch (a.dbar) {
    case 1: return table_g_d<G, 1>(a, s);
    case 2: return table_g_d<G, 2>(a, s);
    case 4: return table_g_d<G, 4>(a, s);
    case 8: return table_g_d<G, 8>(a, s);
    case 16: return table_g_d<G, 16>(a, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_table(const LayerArgs &a, cudaStream_t s) {
  switch (a.G) {
    case 1: return table_g<1>(a, s);
    case 2: return table_g<2>(a, s);
    case 4: return table_g<4>(a, s);
  }
  return cudaErrorInvalidValue;
}

// Resident tokens: one thread per (token, query head); exact fp32 FMA chain over d
// (R3), mapped onto the head's 2^-e grid; writes z and folds into M / zmin.
__global__ void __launch_bounds__(128) k_resident(LayerArgs a) {
  const int u = blockIdx.y;
  const int b = u / a.Hkv, kv = u - b * a.Hkv;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int h = (int)(idx % a.G);
  const int64_t r = idx / a.G;
  if (r >= a.n_res) return;
  const int hq = kv * a.G + h;
  const int64_t slot = (a.res_slot0 + r) % a.res_cap;
  const uint16_t *krow = a.res_k + (int64_t)b * a.res_b_stride + ((int64_t)kv * a.res_cap + slot) * a.d;
  const uint16_t *qrow = a.q + ((int64_t)b * a.Hq + hq) * a.d;
  float acc = 0.0f;
  for (int e = 0; e < a.d; ++e) acc = __fmaf_rn(h2f(__ldg(qrow + e)), h2f(__ldg(krow + e)), acc);
  HeadState *hs = a.hs + (int64_t)b * a.Hq + hq;
  const int ex = scale_exponent(__uint_as_float(hs->amax));
  const int zq = quant_res(acc, pow2f(ex));
  a.z[((int64_t)b * a.Hq + hq) * a.z_stride + a.n_q + r] = (float)zq;
  atomicMax(&hs->M, zq);
  atomicMin(&hs->zmin, zq);
}

cudaError_t launch_resident(const LayerArgs &a, cudaStream_t s) {
  if (a.n_res <= 0) return cudaSuccess;
  const int64_t work = a.n_res * a.G;
  dim3 grid((unsigned)((work + 127) / 128), (unsigned)(a.B * a.Hkv));
  k_resident<<<grid, 128, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace hc
