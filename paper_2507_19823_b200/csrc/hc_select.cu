// hc_select.cu -- standalone hc_select_topk front end (R5b): real-valued scores are
// mapped onto a per-row 2^-e fixed-point grid (|z| < 2^22), then the Eq. 4 selection
// passes (hc_select_pass.cu) run on them.
#include <float.h>

#include "hc_internal.h"

namespace hc {

constexpr int kSelThreads = 256;

// ---------------------------------------------------------------- standalone prep (R5b)
__global__ void __launch_bounds__(kSelThreads) k_float_prep(const float *sc, int64_t n, float *z,
                                                             int64_t zs, HeadState *hs,
                                                             float kappa0, uint32_t *ghist,
                                                             unsigned long long *gmass) {
  const int row = blockIdx.x;
  const float *src = sc + (int64_t)row * n;
  float A = 0.0f;
  for (int64_t j = threadIdx.x; j < n; j += kSelThreads) A = fmaxf(A, fabsf(src[j]));
  __shared__ float sA[kSelThreads / 32];
  __shared__ int smx[kSelThreads / 32], smn[kSelThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) A = fmaxf(A, __shfl_xor_sync(0xffffffffu, A, off));
  if ((threadIdx.x & 31) == 0) sA[threadIdx.x >> 5] = A;
  __syncthreads();
  A = 0.0f;
  for (int w = 0; w < kSelThreads / 32; ++w) A = fmaxf(A, sA[w]);
  int e = 100;
  if (A >= 0x1p-100f) {
    const int ex = ((__float_as_int(A) >> 23) & 0xff) - 127;
    e = 21 - ex;
    e = e < -100 ? -100 : (e > 100 ? 100 : e);
  }
  const float sc2 = pow2f(e);
  int mx = INT_MIN, mn = INT_MAX;
  for (int64_t j = threadIdx.x; j < n; j += kSelThreads) {
    const int v = quant_res(src[j], sc2);
    z[(int64_t)row * zs + j] = (float)v;
    mx = max(mx, v);
    mn = min(mn, v);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  mn = __reduce_min_sync(0xffffffffu, mn);
  if ((threadIdx.x & 31) == 0) { smx[threadIdx.x >> 5] = mx; smn[threadIdx.x >> 5] = mn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < kSelThreads / 32; ++w) { mx = max(mx, smx[w]); mn = min(mn, smn[w]); }
    hs[row].M = mx;
    hs[row].zmin = mn;
    hs[row].e = e;
    hs[row].kappa = __fmul_rn(kappa0, pow2f(-e));
    hs[row].S = 0ull;
    hs[row].mass_before = 0ull;
    hs[row].c1_done = 0u;
    hs[row].c2_done = 0u;
    hs[row].ticket = 0u;
    hs[row].state = 0u;
  }
  if (ghist)
    for (int i = threadIdx.x; i < kNB; i += kSelThreads) ghist[(int64_t)row * kNB + i] = 0u;
  if (gmass)
    for (int i = threadIdx.x; i < kNB; i += kSelThreads) gmass[(int64_t)row * kNB + i] = 0ull;
}

cudaError_t launch_select_float_prep(const float *scores, int64_t rows, int64_t n, float *z,
                                     int64_t z_stride, HeadState *hs, float kappa0,
                                     cudaStream_t s, uint32_t *ghist,
                                     unsigned long long *gmass) {
  k_float_prep<<<(unsigned)rows, kSelThreads, 0, s>>>(scores, n, z, z_stride, hs, kappa0, ghist, gmass);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
