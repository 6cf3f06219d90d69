// hc_gather.cu -- row a5: the sparse weighted sum of Eq. 5,
//   ỹ = Σ_{i∈Π_k*} ã*_i V_i,
// over the selected rows of the offloaded value store (HBM, or pinned host memory
// mapped into the device address space -> zero-copy PCIe reads of ONLY the selected
// rows), merged with the resident recent-window rows (HBM).
//
// Grid (row = (b, query head), chunk of kRows selected rows).  Each half-warp reads
// one 256-byte V row (16 lanes × 16 B, coalesced, L1-bypassing) and accumulates 8
// fp32 lanes; 4 rows per half-warp are in flight per iteration.  Partials go to the
// workspace; the last CTA of a row (completion counter) sums them in chunk order,
// so the result is deterministic.
#include "hc_internal.h"

namespace hc {

constexpr int kGThreads = 256;
constexpr int kGUnroll = 8;

__device__ __forceinline__ uint4 ld_nc(const uint16_t *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void fma8(float (&acc)[8], float w, const uint4 &v) {
  const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&u[q]));
    acc[2 * q] = fmaf(w, f.x, acc[2 * q]);
    acc[2 * q + 1] = fmaf(w, f.y, acc[2 * q + 1]);
  }
}

__global__ void __launch_bounds__(kGThreads) k_gather(LayerArgs a) {
  const int row = blockIdx.y;          // b * Hq + hq
  const int ch = blockIdx.x;
  const int b = row / a.Hq, hq = row - b * a.Hq, kv = hq / a.G;
  HeadState *hs = a.hs + row;
  const int64_t k = hs->ksel;
  const int lpr = a.d >> 3;            // lanes per row (16 at d = 128)
  const int rpw = 32 / lpr;            // rows per warp
  const int slots = (kGThreads / 32) * rpw;
  const int lane = threadIdx.x & 31;
  const int slot = (threadIdx.x >> 5) * rpw + lane / lpr;
  const int sub = lane % lpr;          // which 8 dims
  const int64_t r0 = (int64_t)ch * a.grows;
  const int64_t r1 = min(k, r0 + a.grows);
  const int32_t *idx = a.sel_idx + (int64_t)row * a.k_max;
  const float *wt = a.sel_w + (int64_t)row * a.k_max;
  const uint16_t *Vb = a.V + (int64_t)b * a.v_b_stride + (int64_t)kv * a.v_kv_stride;
  const uint16_t *Rb = a.res_v + (int64_t)b * a.res_b_stride + (int64_t)kv * a.res_cap * a.d;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
  for (int64_t r = r0 + slot; r < r1; r += (int64_t)slots * kGUnroll) {
    uint4 v[kGUnroll];
    float w[kGUnroll];
#pragma unroll
    for (int u = 0; u < kGUnroll; ++u) {
      const int64_t rr = r + (int64_t)u * slots;
      if (rr < r1) {
        const int64_t j = idx[rr];
        w[u] = wt[rr];
        const uint16_t *src = j < a.n_q
                                  ? Vb + j * a.d
                                  : Rb + ((a.res_slot0 + (j - a.n_q)) % a.res_cap) * a.d;
        v[u] = ld_nc(src + sub * 8);
      } else {
        w[u] = 0.0f;
        v[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < kGUnroll; ++u) fma8(acc, w[u], v[u]);
  }
  // reduce the `slots` partial rows of this CTA: smem [slots][d]
  extern __shared__ float sred[];
#pragma unroll
  for (int e = 0; e < 8; ++e) sred[slot * a.d + sub * 8 + e] = acc[e];
  __syncthreads();
  float *part = a.partial + ((int64_t)row * a.gchunks + ch) * a.d;
  for (int e = threadIdx.x; e < a.d; e += kGThreads) {
    float s = 0.0f;
    for (int q = 0; q < slots; ++q) s += sred[q * a.d + e];
    part[e] = s;
  }
  // last CTA of this row sums the chunk partials in order
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&hs->gather_done, 1u);
    last = (prev == (unsigned)a.gchunks - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // deterministic parallel sum of the chunk partials: thread -> (dim e, part p);
  // part p sums chunks p, p+np, ... with 4 independent accumulators, then the parts
  // are added in order.
  const float *p0 = a.partial + (int64_t)row * a.gchunks * a.d;
  const int np = kGThreads / a.d;  // >= 1 since d <= 256
  const int e = threadIdx.x % a.d, pp = threadIdx.x / a.d;
  float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  if (pp < np) {
    int c = pp;
    for (; c + 3 * np < a.gchunks; c += 4 * np) {
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] += __ldcg(p0 + (int64_t)(c + q * np) * a.d + e);
    }
    for (; c < a.gchunks; c += np) s4[0] += __ldcg(p0 + (int64_t)c * a.d + e);
  }
  __syncthreads();
  if (pp < np) sred[pp * a.d + e] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  __syncthreads();
  if (threadIdx.x < a.d) {
    float s = 0.0f;
    for (int q = 0; q < np; ++q) s += sred[q * a.d + threadIdx.x];
    a.out[(int64_t)row * a.d + threadIdx.x] = s;
  }
  if (threadIdx.x == 0) hs->gather_done = 0;
}

cudaError_t launch_gather(const LayerArgs &a, cudaStream_t s) {
  dim3 grid((unsigned)a.gchunks, (unsigned)(a.B * a.Hq));
  const int lpr = a.d >> 3;
  const int slots = (kGThreads / 32) * (32 / lpr);
  const size_t smem = (size_t)slots * a.d * sizeof(float);
  k_gather<<<grid, kGThreads, smem, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
