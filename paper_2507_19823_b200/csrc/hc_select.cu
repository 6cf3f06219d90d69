// hc_select.cu -- rows a3 + a4: normalisation ã = softmax(z̃/√d)
// as exact fixed-point mass (R4) and the cumulative-magnitude eviction of Eq. 4
// with the k_max cap (R5), for many independent rows (query heads).
//
// No sort.  Keys are the integers Δ_j = M − z_j (< 2^24) and W is a function of Δ
// alone, so the τ cut and the cap cut are found with a two-level (12 + 12 bit)
// radix select on (count, mass) histograms in shared memory:
//   hist1  : coarse histogram of Δ >> shift (count u32, mass u64)      [pass 1 over z]
//   bound1 : per row: S, Θ = ⌈τ_q·S/2^24⌉, first coarse bucket b* where the
//            cumulative mass reaches Θ or the count reaches k_max
//   hist2  : fine histogram of Δ inside b*                              [pass 2]
//   bound2 : exact Δ* and r = #ties at Δ* kept (lowest indices first), k_sel
//   count  : per chunk (#Δ<Δ*, #Δ==Δ*)                                  [pass 3]
//   write  : ordered compaction -> ascending indices + weights W_j/S     [pass 4]
// All sums are integers, so the result is bit-exact and independent of the CTA
// decomposition (and of sequence sharding).
#include <float.h>

#include "hc_internal.h"

namespace hc {

constexpr int kSelThreads = 256;
constexpr int kBinsPerThread = kNB / kSelThreads;  // 16

__device__ __forceinline__ int row_shift(const HeadState &h) {
  const uint32_t dmax = (uint32_t)(h.M - h.zmin);
  const int bits = 32 - __clz(dmax);
  return bits > kNBBits ? bits - kNBBits : 0;
}

__device__ __forceinline__ uint32_t delta_of(const HeadState &h, float zf) {
  return (uint32_t)(h.M - __float2int_rn(zf));
}

__device__ void bound1_row(const SelArgs &a, int row);
__device__ void bound2_row(const SelArgs &a, int row);

// "last CTA done" for per-row multi-CTA passes: every CTA fences its global atomics,
// bumps the row counter, and the CTA that completes it runs the row's bound step.
__device__ __forceinline__ bool last_cta(uint32_t *counter, unsigned nctas) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == nctas - 1);
    if (s_last) *counter = 0;  // reset for the next use of the workspace
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// ---------------------------------------------------------------- pass 1
__global__ void __launch_bounds__(kSelThreads) k_hist1(SelArgs a, int64_t per_cta) {
  extern __shared__ __align__(16) uint8_t hsm[];  // 48 KiB dynamic: mass u64[kNB], count u32[kNB]
  unsigned long long *ms = reinterpret_cast<unsigned long long *>(hsm);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(hsm + kNB * 8);
  const int row = blockIdx.y;
  const HeadState h = a.hs[row];
  const int shift = row_shift(h);
  for (int i = threadIdx.x; i < kNB; i += kSelThreads) { cnt[i] = 0; ms[i] = 0ull; }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hs[row].shift = shift;
  __syncthreads();
  const float *z = a.z + (int64_t)row * a.z_stride;
  const int64_t j0 = (int64_t)blockIdx.x * per_cta;
  const int64_t j1 = min(a.n, j0 + per_cta);
  for (int64_t j = j0 + threadIdx.x * 4; j < j1; j += kSelThreads * 4) {
    float zv[4];
    if (j + 4 <= j1) {
      const float4 v = *reinterpret_cast<const float4 *>(z + j);
      zv[0] = v.x; zv[1] = v.y; zv[2] = v.z; zv[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) zv[u] = (j + u < j1) ? z[j + u] : NAN;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j + u >= j1) break;
      const uint32_t dl = delta_of(h, zv[u]);
      const uint32_t bk = dl >> shift;
      atomicAdd(&cnt[bk], 1u);
      const uint64_t W = mass(dl, h.kappa);
      if (W) atomicAdd(&ms[bk], (unsigned long long)W);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kNB; i += kSelThreads) {
    if (cnt[i]) {
      atomicAdd(&a.h1c[(int64_t)row * kNB + i], cnt[i]);
      if (ms[i]) atomicAdd(&a.h1m[(int64_t)row * kNB + i], ms[i]);
    }
  }
  if (last_cta(&a.hs[row].h1_done, gridDim.x)) bound1_row(a, row);
}

// block-wide exclusive scan of (uint64, uint64) pairs, returns totals
template <typename T>
__device__ __forceinline__ void block_scan2(T &x, T &y, T &tx, T &ty) {
  __shared__ T sx[kSelThreads / 32], sy[kSelThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T ix = x, iy = y;  // inclusive within warp
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    T ox = __shfl_up_sync(0xffffffffu, ix, off);
    T oy = __shfl_up_sync(0xffffffffu, iy, off);
    if (lane >= off) { ix += ox; iy += oy; }
  }
  if (lane == 31) { sx[w] = ix; sy[w] = iy; }
  __syncthreads();
  T bx = 0, by = 0;
  tx = 0; ty = 0;
#pragma unroll
  for (int k = 0; k < kSelThreads / 32; ++k) {
    if (k < w) { bx += sx[k]; by += sy[k]; }
    tx += sx[k]; ty += sy[k];
  }
  x = bx + ix - x;
  y = by + iy - y;
  __syncthreads();
}

// ---------------------------------------------------------------- bound 1
__device__ void bound1_row(const SelArgs &a, int row) {
  HeadState *hs = a.hs + row;
  const uint32_t *hc = a.h1c + (int64_t)row * kNB + threadIdx.x * kBinsPerThread;
  const unsigned long long *hm = a.h1m + (int64_t)row * kNB + threadIdx.x * kBinsPerThread;
  uint64_t c[kBinsPerThread], m[kBinsPerThread];
  uint64_t lc = 0, lm = 0;
#pragma unroll
  for (int k = 0; k < kBinsPerThread; ++k) {
    c[k] = __ldcg(hc + k);
    m[k] = __ldcg(hm + k);
    lc += c[k];
    lm += m[k];
  }
  uint64_t pc = lc, pm = lm, tc, tm;
  block_scan2<uint64_t>(pc, pm, tc, tm);  // pc, pm: exclusive prefix of this thread's bins
  const uint64_t S = tm;
  const bool tau_all = a.tau_q >= (1u << 24);
  const uint64_t theta = tau_all ? 0 : threshold(a.tau_q, S);
  const bool cap_all = (uint64_t)a.k_max >= tc;
  __shared__ int s_b;
  if (threadIdx.x == 0) s_b = kNB;
  __syncthreads();
  int found = kNB;
  uint64_t cc = pc, cm = pm;
#pragma unroll
  for (int k = 0; k < kBinsPerThread; ++k) {
    cc += c[k];
    cm += m[k];
    // a crossing can only happen at a non-empty bucket (Θ = 0 -> the first one)
    const bool trig = c[k] && ((!tau_all && cm >= theta) || (!cap_all && cc >= (uint64_t)a.k_max));
    if (trig && found == kNB) found = threadIdx.x * kBinsPerThread + k;
  }
  if (found < kNB) atomicMin(&s_b, found);
  __syncthreads();
  const int bstar = s_b;
  if (threadIdx.x == 0) {
    hs->S = S;
    hs->theta = theta;
    hs->bstar = bstar;
    if (bstar == kNB) {  // τ = 1 and n <= k_max: keep everything
      hs->delta_star = 0xffffffffu;
      hs->r_ties = 0;
      hs->ksel = (int64_t)tc;
      hs->kstar = (int64_t)tc;
      hs->sel_mass = S;
    }
  }
  if (bstar < kNB && bstar / kBinsPerThread == (int)threadIdx.x) {
    uint64_t bc = pc, bm = pm;
    for (int k = 0; k < bstar % kBinsPerThread; ++k) { bc += c[k]; bm += m[k]; }
    hs->cnt_before = (uint32_t)bc;
    hs->mass_before = bm;
  }
}

// ---------------------------------------------------------------- pass 2
__global__ void __launch_bounds__(kSelThreads) k_hist2(SelArgs a, int64_t per_cta) {
  __shared__ uint32_t cnt[kNB];
  const int row = blockIdx.y;
  const HeadState h = a.hs[row];
  if (h.bstar >= kNB) return;
  for (int i = threadIdx.x; i < kNB; i += kSelThreads) cnt[i] = 0;
  __syncthreads();
  const float *z = a.z + (int64_t)row * a.z_stride;
  const int64_t j0 = (int64_t)blockIdx.x * per_cta;
  const int64_t j1 = min(a.n, j0 + per_cta);
  const uint32_t fmask = (1u << h.shift) - 1u;
  for (int64_t j = j0 + threadIdx.x * 4; j < j1; j += kSelThreads * 4) {
    float zv[4];
    if (j + 4 <= j1) {
      const float4 v = *reinterpret_cast<const float4 *>(z + j);
      zv[0] = v.x; zv[1] = v.y; zv[2] = v.z; zv[3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) zv[u] = (j + u < j1) ? z[j + u] : NAN;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j + u >= j1) break;
      const uint32_t dl = delta_of(h, zv[u]);
      if ((int)(dl >> h.shift) == h.bstar) atomicAdd(&cnt[dl & fmask], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kNB; i += kSelThreads)
    if (cnt[i]) atomicAdd(&a.h2c[(int64_t)row * kNB + i], cnt[i]);
  if (last_cta(&a.hs[row].h2_done, gridDim.x)) bound2_row(a, row);
}

// ---------------------------------------------------------------- bound 2
__device__ void bound2_row(const SelArgs &a, int row) {
  HeadState *hs = a.hs + row;
  HeadState h;
  h.bstar = __ldcg(&hs->bstar);
  h.shift = __ldcg(&hs->shift);
  h.kappa = __ldcg(&hs->kappa);
  h.cnt_before = __ldcg(&hs->cnt_before);
  h.mass_before = __ldcg(&hs->mass_before);
  h.theta = __ldcg(&hs->theta);
  if (h.bstar >= kNB) return;
  const uint32_t dbase = (uint32_t)h.bstar << h.shift;
  const int v0 = threadIdx.x * kBinsPerThread;
  const uint32_t *hc = a.h2c + (int64_t)row * kNB + v0;
  uint64_t c[kBinsPerThread], w[kBinsPerThread];
  uint64_t lc = 0, lm = 0;
#pragma unroll
  for (int k = 0; k < kBinsPerThread; ++k) {
    c[k] = __ldcg(hc + k);
    w[k] = c[k] ? mass(dbase | (uint32_t)(v0 + k), h.kappa) : 0ull;
    lc += c[k];
    lm += c[k] * w[k];
  }
  uint64_t pc = lc, pm = lm, tc, tm;
  block_scan2<uint64_t>(pc, pm, tc, tm);
  const bool tau_all = a.tau_q >= (1u << 24);
  __shared__ int s_v;
  if (threadIdx.x == 0) s_v = kNB;
  __syncthreads();
  uint64_t cc = h.cnt_before + pc, cm = h.mass_before + pm;
  int found = kNB;
  uint64_t f_cc = 0, f_cm = 0;
#pragma unroll
  for (int k = 0; k < kBinsPerThread; ++k) {
    if (c[k] && found == kNB) {
      const bool tt = !tau_all && w[k] && (cm + c[k] * w[k] >= h.theta);
      const bool tk = cc + c[k] >= (uint64_t)a.k_max;
      if (tt || tk) { found = v0 + k; f_cc = cc; f_cm = cm; }
    }
    cc += c[k];
    cm += c[k] * w[k];
  }
  if (found < kNB) atomicMin(&s_v, found);
  __syncthreads();
  if (found < kNB && found == s_v) {
    const int k = found - v0;
    const uint64_t ck = c[k], wk = w[k];
    uint64_t r_tau = ~0ull, r_cap = ~0ull;
    if (!tau_all && wk && f_cm + ck * wk >= h.theta) r_tau = (h.theta - f_cm + wk - 1) / wk;
    if (f_cc + ck >= (uint64_t)a.k_max) r_cap = (uint64_t)a.k_max - f_cc;
    if (r_tau == 0) r_tau = 1;  // Eq. 4: k >= 1 (Θ may already be reached: impossible, guard)
    const uint64_t r = r_tau < r_cap ? r_tau : r_cap;
    hs->delta_star = dbase | (uint32_t)found;
    hs->r_ties = (uint32_t)r;
    hs->ksel = (int64_t)(f_cc + r);
    hs->kstar = (r_tau <= r_cap) ? (int64_t)(f_cc + r_tau) : -1;
    hs->sel_mass = f_cm + r * wk;
  }
}

// ---------------------------------------------------------------- pass 3 / 4
constexpr int kChunkTPT = 16;                              // tokens per thread
constexpr int kChunkTokens = kSelThreads * kChunkTPT;      // 4096

__device__ __forceinline__ void load16(const float *z, int64_t j, int64_t n, float (&zv)[16]) {
  if (j + 16 <= n) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = *reinterpret_cast<const float4 *>(z + j + 4 * q);
      zv[4 * q] = v.x; zv[4 * q + 1] = v.y; zv[4 * q + 2] = v.z; zv[4 * q + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < 16; ++u) zv[u] = (j + u < n) ? z[j + u] : NAN;
  }
}

__global__ void __launch_bounds__(kSelThreads) k_count(SelArgs a) {
  const int row = blockIdx.y, ch = blockIdx.x;
  const HeadState h = a.hs[row];
  const float *z = a.z + (int64_t)row * a.z_stride;
  const int64_t j = (int64_t)ch * kChunkTokens + threadIdx.x * kChunkTPT;
  uint32_t ns = 0, nt = 0;
  if (j < a.n) {
    float zv[16];
    load16(z, j, a.n, zv);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (j + u < a.n) {
        const uint32_t dl = delta_of(h, zv[u]);
        ns += dl < h.delta_star;
        nt += dl == h.delta_star;
      }
    }
  }
  ns = __reduce_add_sync(0xffffffffu, ns);
  nt = __reduce_add_sync(0xffffffffu, nt);
  __shared__ uint32_t s[2][kSelThreads / 32];
  if ((threadIdx.x & 31) == 0) { s[0][threadIdx.x >> 5] = ns; s[1][threadIdx.x >> 5] = nt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a0 = 0, a1 = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) { a0 += s[0][w]; a1 += s[1][w]; }
    a.chunk_cnt[((int64_t)row * a.nchunks + ch) * 2] = a0;
    a.chunk_cnt[((int64_t)row * a.nchunks + ch) * 2 + 1] = a1;
  }
}

__global__ void __launch_bounds__(kSelThreads) k_write(SelArgs a) {
  const int row = blockIdx.y, ch = blockIdx.x;
  const HeadState h = a.hs[row];
  // prefix over preceding chunks (strict, ties)
  __shared__ uint64_t s_pre[2];
  if (threadIdx.x < 32) {
    uint64_t ps = 0, pt = 0;
    const uint32_t *cc = a.chunk_cnt + (int64_t)row * a.nchunks * 2;
    for (int k = threadIdx.x; k < ch; k += 32) { ps += cc[2 * k]; pt += cc[2 * k + 1]; }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ps += __shfl_xor_sync(0xffffffffu, ps, off);
      pt += __shfl_xor_sync(0xffffffffu, pt, off);
    }
    if (threadIdx.x == 0) { s_pre[0] = ps; s_pre[1] = pt; }
  }
  __syncthreads();
  const uint64_t strict_before = s_pre[0], ties_before = s_pre[1];
  const float *z = a.z + (int64_t)row * a.z_stride;
  const int64_t j = (int64_t)ch * kChunkTokens + threadIdx.x * kChunkTPT;
  float zv[16];
  uint32_t dl[16];
  uint64_t ns = 0, nt = 0;
  if (j < a.n) load16(z, j, a.n, zv);
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const bool v = j + u < a.n;
    dl[u] = v ? delta_of(h, zv[u]) : 0xffffffffu;
    ns += v && dl[u] < h.delta_star;
    nt += v && dl[u] == h.delta_star;
  }
  uint64_t ps = ns, pt = nt, ts, tt;
  block_scan2<uint64_t>(ps, pt, ts, tt);
  const uint64_t r = h.r_ties;
  const uint64_t rem = r > ties_before ? r - ties_before : 0;  // ties still to take
  uint64_t tie_rank = pt;                                       // ties of this chunk before me
  uint64_t pos = strict_before + min(ties_before, r) + ps + min(rem, pt);
  const double denom = a.renorm ? (double)h.sel_mass : (double)h.S;
  int32_t *oi = a.sel_idx + (int64_t)row * a.k_max;
  float *ow = a.sel_w + (int64_t)row * a.k_max;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    bool take = false;
    if (dl[u] < h.delta_star) take = true;
    else if (dl[u] == h.delta_star && j + u < a.n) {
      take = tie_rank < rem;
      ++tie_rank;
    }
    if (take) {
      oi[pos] = (int32_t)(j + u);
      ow[pos] = (float)((double)mass(dl[u], h.kappa) / denom);
      ++pos;
    }
  }
  if (ch == 0 && threadIdx.x == 0 && a.sel_k) a.sel_k[row] = h.ksel;
}

cudaError_t launch_select(const SelArgs &a, cudaStream_t s) {
  // pass-1/2 decomposition: about 4 CTAs per SM in total, >= 4096 tokens each
  int64_t ctas_per_row = (int64_t)(4 * 148 + a.rows - 1) / a.rows;
  int64_t per_cta = (a.n + ctas_per_row - 1) / ctas_per_row;
  if (per_cta < 4096) per_cta = 4096;
  per_cta = (per_cta + 3) / 4 * 4;
  ctas_per_row = (a.n + per_cta - 1) / per_cta;
  dim3 g12((unsigned)ctas_per_row, (unsigned)a.rows);
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_hist1, cudaFuncAttributeMaxDynamicSharedMemorySize, kNB * 12);
    if (e != cudaSuccess) return e;
    configured[dev] = 1;
  }
  k_hist1<<<g12, kSelThreads, kNB * 12, s>>>(a, per_cta);  // + bound1 in each row's last CTA
  note_launch();
  k_hist2<<<g12, kSelThreads, 0, s>>>(a, per_cta);  // + bound2 in each row's last CTA
  note_launch();
  dim3 g34((unsigned)a.nchunks, (unsigned)a.rows);
  k_count<<<g34, kSelThreads, 0, s>>>(a);
  note_launch();
  k_write<<<g34, kSelThreads, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- standalone prep (R5b)
__global__ void __launch_bounds__(kSelThreads) k_float_prep(const float *sc, int64_t n, float *z,
                                                             int64_t zs, HeadState *hs,
                                                             float kappa0) {
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
  }
}

cudaError_t launch_select_float_prep(const float *scores, int64_t rows, int64_t n, float *z,
                                     int64_t z_stride, HeadState *hs, float kappa0,
                                     cudaStream_t s) {
  k_float_prep<<<(unsigned)rows, kSelThreads, 0, s>>>(scores, n, z, z_stride, hs, kappa0);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
