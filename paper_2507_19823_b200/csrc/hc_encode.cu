// hc_encode.cu -- row a0: key encoding (R1, "Each sub-group is
// represented as nearest neighbor of the centroids in the codebook") and the
// row copies of the append protocol (value store / resident window).
#include <float.h>

#include "hc_internal.h"

namespace hc {

__device__ __forceinline__ int64_t rowoff(const RowMap &m, int64_t r) {
  return (r / m.R1) * m.s1 + (r % m.R1) * m.s2 + m.s0;
}

template <int DBAR>
__device__ __forceinline__ void load_centroid(const float *p, float (&c)[DBAR]) {
  if constexpr (DBAR % 4 == 0) {
#pragma unroll
    for (int e = 0; e < DBAR; e += 4) {
      float4 v = __ldg(reinterpret_cast<const float4 *>(p + e));
      c[e] = v.x; c[e + 1] = v.y; c[e + 2] = v.z; c[e + 3] = v.w;
    }
  } else if constexpr (DBAR == 2) {
    float2 v = __ldg(reinterpret_cast<const float2 *>(p));
    c[0] = v.x; c[1] = v.y;
  } else {
#pragma unroll
    for (int e = 0; e < DBAR; ++e) c[e] = __ldg(p + e);
  }
}

// One CTA per (key row, group).  Thread t owns the contiguous centroid block
// [t*per, (t+1)*per) and scans it in ascending m keeping the first strict minimum
// (loads unrolled by 8 so they are all in flight together); the CTA then reduces
// (dist, m) lexicographically.  Result: argmin with ties to the lowest index --
// identical to a sequential scan (R1).
template <int DBAR>
__global__ void __launch_bounds__(256) k_encode(EncodeArgs a) {
  const int64_t r = blockIdx.x;
  const int i = blockIdx.y;
  const uint16_t *krow = a.keys + rowoff(a.kmap, r) + (int64_t)i * DBAR;
  float kb[DBAR];
#pragma unroll
  for (int e = 0; e < DBAR; ++e) kb[e] = h2f(krow[e]);
  const float *Ci = a.C + (int64_t)(a.cbg == 1 ? 0 : i) * a.c * DBAR;
  const int per = (a.c + blockDim.x - 1) / blockDim.x;
  const int m0 = threadIdx.x * per;
  const int m1 = min(a.c, m0 + per);
  float best = INFINITY;
  int bm = 0x7fffffff;
  for (int mb = m0; mb < m1; mb += 8) {
    float cm[8][DBAR];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (mb + u < m1) load_centroid<DBAR>(Ci + (int64_t)(mb + u) * DBAR, cm[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (mb + u < m1) {
        float dist = 0.0f;
#pragma unroll
        for (int e = 0; e < DBAR; ++e) {
          const float diff = __fsub_rn(kb[e], cm[u][e]);
          dist = __fmaf_rn(diff, diff, dist);
        }
        if (dist < best) { best = dist; bm = mb + u; }
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    float ob = __shfl_xor_sync(0xffffffffu, best, off);
    int om = __shfl_xor_sync(0xffffffffu, bm, off);
    if (ob < best || (ob == best && om < bm)) { best = ob; bm = om; }
  }
  __shared__ float sb[8];
  __shared__ int sm[8];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sb[w] = best; sm[w] = bm; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    best = l < nw ? sb[l] : INFINITY;
    bm = l < nw ? sm[l] : 0x7fffffff;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      float ob = __shfl_xor_sync(0xffffffffu, best, off);
      int om = __shfl_xor_sync(0xffffffffu, bm, off);
      if (ob < best || (ob == best && om < bm)) { best = ob; bm = om; }
    }
    if (l == 0) a.codes[rowoff(a.omap, r) + (int64_t)i * a.gstride] = (uint16_t)bm;
  }
}

cudaError_t launch_encode(const EncodeArgs &a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  dim3 grid((unsigned)a.rows, (unsigned)a.g);
  const int dbar = a.d / a.g;
  switch (dbar) {
    case 1: k_encode<1><<<grid, 256, 0, s>>>(a); note_launch(); break;
    case 2: k_encode<2><<<grid, 256, 0, s>>>(a); note_launch(); break;
    case 4: k_encode<4><<<grid, 256, 0, s>>>(a); note_launch(); break;
    case 8: k_encode<8><<<grid, 256, 0, s>>>(a); note_launch(); break;
    case 16: k_encode<16><<<grid, 256, 0, s>>>(a); note_launch(); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// copy `rows` fp16 rows of d elements; one warp per row, 16 B per lane
__global__ void __launch_bounds__(256) k_rowcopy(RowCopyArgs a) {
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= a.rows) return;
  const int l = threadIdx.x & 31;
  const uint16_t *src = a.src + rowoff(a.smap, r);
  uint16_t *dst = a.dst + rowoff(a.dmap, r);
  for (int e = l * 8; e < a.d; e += 256) {
    *reinterpret_cast<uint4 *>(dst + e) = *reinterpret_cast<const uint4 *>(src + e);
  }
}

cudaError_t launch_rowcopy(const RowCopyArgs &a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  k_rowcopy<<<(unsigned)((a.rows + 7) / 8), 256, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
