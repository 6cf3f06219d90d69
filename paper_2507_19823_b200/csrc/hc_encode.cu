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

// One CTA (1024 threads) per (chunk of up to kER key rows, group i): the group's
// codebook slice is read ONCE per CTA (coalesced: thread t takes centroids
// t, t+1024, ...; loads unrolled so they are all in flight) and scored against all
// rows of the chunk.  Each thread keeps, per row, the first strict minimum over its
// centroids (ascending m); the CTA reduces (dist, m) lexicographically -> argmin
// with ties to the lowest index, identical to a sequential scan (R1).
constexpr int kEThreads = 512;
template <int DBAR> struct EncCfg {
  static constexpr int kER = 2;                                     // key rows per CTA
  static constexpr int kU = DBAR <= 2 ? 8 : (DBAR == 4 ? 4 : 2);   // centroid loads in flight
};

template <int DBAR>
__global__ void __launch_bounds__(kEThreads) k_encode(EncodeArgs a) {
  constexpr int kER = EncCfg<DBAR>::kER;
  constexpr int kU = EncCfg<DBAR>::kU;
  pdl_trigger();
  pdl_wait();
  const int64_t r0 = (int64_t)blockIdx.x * kER;
  const int64_t left = a.rows - r0;
  const int nr = left < kER ? (int)left : kER;
  const int i = blockIdx.y;
  float kb[kER][DBAR];
#pragma unroll
  for (int r = 0; r < kER; ++r) {
    const uint16_t *krow = a.keys + rowoff(a.kmap, r0 + (r < nr ? r : 0)) + (int64_t)i * DBAR;
#pragma unroll
    for (int e = 0; e < DBAR; ++e) kb[r][e] = h2f(krow[e]);
  }
  const float *Ci = a.C + (int64_t)(a.cbg == 1 ? 0 : i) * a.c * DBAR;
  float best[kER];
  int bm[kER];
#pragma unroll
  for (int r = 0; r < kER; ++r) { best[r] = INFINITY; bm[r] = 0x7fffffff; }
  for (int mb = threadIdx.x; mb < a.c; mb += kEThreads * kU) {
    float cm[kU][DBAR];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int m = mb + u * kEThreads;
      if (m < a.c) load_centroid<DBAR>(Ci + (int64_t)m * DBAR, cm[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int m = mb + u * kEThreads;
      if (m < a.c) {
#pragma unroll
        for (int r = 0; r < kER; ++r) {
          float dist = 0.0f;
#pragma unroll
          for (int e = 0; e < DBAR; ++e) {
            const float diff = __fsub_rn(kb[r][e], cm[u][e]);
            dist = __fmaf_rn(diff, diff, dist);
          }
          if (dist < best[r]) { best[r] = dist; bm[r] = m; }
        }
      }
    }
  }
  __shared__ float sb[kER][kEThreads / 32];
  __shared__ int sm[kER][kEThreads / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < kER; ++r) {
    float b_ = best[r];
    int m_ = bm[r];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, b_, off);
      const int om = __shfl_xor_sync(0xffffffffu, m_, off);
      if (ob < b_ || (ob == b_ && om < m_)) { b_ = ob; m_ = om; }
    }
    if (l == 0) { sb[r][w] = b_; sm[r][w] = m_; }
  }
  __syncthreads();
  if (w < nr) {  // warp r reduces row r
    const int r = w;
    float b_ = l < kEThreads / 32 ? sb[r][l] : INFINITY;
    int m_ = l < kEThreads / 32 ? sm[r][l] : 0x7fffffff;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, b_, off);
      const int om = __shfl_xor_sync(0xffffffffu, m_, off);
      if (ob < b_ || (ob == b_ && om < m_)) { b_ = ob; m_ = om; }
    }
    if (l == 0) {
      if (a.pcodes)  // packed 13-bit strip (f3(ii))
        put_code13(a.pcodes + (rowoff(a.psmap, r0 + r) + i) * a.strip_bytes, a.pn_cap, a.ptok, (uint32_t)m_);
      else
        a.codes[rowoff(a.omap, r0 + r) + (int64_t)i * a.gstride] = (uint16_t)m_;
    }
  }
  // fused append of the rows' values (hc_append_kv): group-0 CTAs copy 16 B per thread
  if (a.vsrc && i == 0) {
    const int per_row = a.d / 8;
    if ((int)threadIdx.x < nr * per_row) {
      const int r = threadIdx.x / per_row, q = threadIdx.x % per_row;
      const uint4 v = *reinterpret_cast<const uint4 *>(a.vsrc + rowoff(a.vsmap, r0 + r) + q * 8);
      *reinterpret_cast<uint4 *>(a.vdst + rowoff(a.vdmap, r0 + r) + q * 8) = v;
    }
  }
}

cudaError_t launch_encode(const EncodeArgs &a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  const int dbar = a.d / a.g;
#define HC_ENC(D)                                                                        \
  {                                                                                      \
    dim3 grid((unsigned)((a.rows + EncCfg<D>::kER - 1) / EncCfg<D>::kER), (unsigned)a.g); \
    launch_chain(k_encode<D>, grid, dim3(kEThreads), 0, s, a);                           \
    note_launch();                                                                       \
    break;                                                                               \
  }
  switch (dbar) {
    case 1: HC_ENC(1)
    case 2: HC_ENC(2)
    case 4: HC_ENC(4)
    case 8: HC_ENC(8)
    case 16: HC_ENC(16)
    default: return cudaErrorInvalidValue;
  }
#undef HC_ENC
  return cudaGetLastError();
}

// copy `rows` fp16 rows of d elements; one warp per row, 16 B per lane
__global__ void __launch_bounds__(256) k_rowcopy(RowCopyArgs a) {
  pdl_trigger();
  pdl_wait();
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
  launch_chain(k_rowcopy, dim3((unsigned)((a.rows + 7) / 8)), dim3(256), 0, s, a);
  note_launch();
  return cudaGetLastError();
}

// u16 strips -> packed 13-bit strips: one thread per (strip, 8 consecutive tokens); full
// groups are plain stores (8 B lo, 4 B nibbles, 1 B bits), a ragged last group read-
// modify-writes only its tokens
__global__ void __launch_bounds__(256) k_pack13(const uint16_t *src, int64_t strips, int64_t n,
                                                int64_t src_stride, uint8_t *dst, int64_t n_cap) {
  const int64_t groups = (n + 7) / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= strips * groups) return;
  const int64_t s = idx / groups, t0 = (idx - s * groups) * 8;
  const uint16_t *sp = src + s * src_stride + t0;
  uint8_t *strip = dst + s * (n_cap * 13 / 8);
  if (t0 + 8 <= n) {
    uint32_t lo0 = 0, lo1 = 0, nib = 0, bit = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t c = sp[u];
      if (u < 4) lo0 |= (c & 0xffu) << (8 * u); else lo1 |= (c & 0xffu) << (8 * (u - 4));
      nib |= ((c >> 8) & 15u) << (4 * u);
      bit |= ((c >> 12) & 1u) << u;
    }
    *reinterpret_cast<uint2 *>(strip + t0) = make_uint2(lo0, lo1);
    *reinterpret_cast<uint32_t *>(strip + n_cap + t0 / 2) = nib;
    strip[n_cap + n_cap / 2 + t0 / 8] = (uint8_t)bit;
  } else {
    for (int64_t t = t0; t < n; ++t) put_code13(strip, n_cap, t, sp[t - t0]);
  }
}

cudaError_t launch_pack13(const uint16_t *src, int64_t strips, int64_t n, int64_t src_stride,
                          uint8_t *dst, int64_t n_cap, cudaStream_t s) {
  const int64_t tot = strips * ((n + 7) / 8);
  if (tot <= 0) return cudaSuccess;
  k_pack13<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(src, strips, n, src_stride, dst, n_cap);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
