// hc_gather.cu -- row a5, Eq. 5 with GQA union de-duplication:
//   ỹ_h = Σ_{j ∈ Π_h} ã*_{h,j} V_j   for the G query heads h of one KV head.
// The G heads select from the SAME value rows V[b][l][kv]; a row kept by several heads
// is read once and accumulated with each head's weight.  Reads are the union of the G
// kept sets instead of their sum (fewer host-link / HBM bytes; results identical up to
// fp32 summation order).
//
// Grid (token chunk of kGC tokens, unit = (b, kv)).  Per CTA: each head's ascending kept
// list is cut to the chunk by binary search, the weights are scattered into a
// [G][kGC] shared table, the union of kept tokens is compacted in index order, and
// half-warps gather 256-byte rows (16 x 16-B L1-bypassing loads, zero-copy when V is
// host-mapped).  The unit's last CTA (completion counter) adds the chunk partials in
// chunk order -> deterministic.
#include "hc_internal.h"

namespace hc {

constexpr int kGC = 2048;     // tokens per chunk
constexpr int kGT = 256;      // threads
constexpr int kGUn = 4;       // rows in flight per half-warp

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int G>
__global__ void __launch_bounds__(kGT) k_gather_union(LayerArgs a, int nchunks, float *part,
                                                      uint32_t *done) {
  __shared__ float wtab[G][kGC];
  __shared__ uint16_t ulist[kGC];
  __shared__ int s_lo[G], s_hi[G], s_cnt;
  __shared__ int s_wc[kGT / 32];
  pdl_trigger();
  pdl_wait();
  const int ch = blockIdx.x, u = blockIdx.y;
  const int b = u / a.Hkv, kv = u - b * a.Hkv;
  // chunk ch covers [cb + ch*kGC, +kGC) ∩ [gtok_lo, gtok_hi), cb = gtok_lo rounded down
  const int64_t cb = a.gtok_lo / kGC * kGC;
  const int64_t j0 = cb + (int64_t)ch * kGC;  // slot t of wtab / ulist = token j0 + t
  const int64_t jlo = j0 > a.gtok_lo ? j0 : a.gtok_lo;
  const int64_t j1 = j0 + kGC < a.gtok_hi ? j0 + kGC : a.gtok_hi;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < G * kGC; i += kGT) (&wtab[0][0])[i] = 0.0f;
  // a row's list: its whole kept list (decode), or this rank's slice of it (sequence-sharded
  // finish: entries [g_off, g_off + g_cnt) hold GLOBAL indices, local token = index - g_base)
  if (tid < G) {
    const int row = b * a.Hq + kv * G + tid;
    const int64_t off = a.g_cnt ? a.g_off[row] : 0;
    const int64_t k = a.g_cnt ? a.g_cnt[row] : (a.k_in ? a.k_in[row] : a.hs[row].ksel);
    const int32_t *li = a.sel_idx + (int64_t)row * a.k_max + off;
    s_lo[tid] = (int)lower_bound_i32(li, k, jlo + a.g_base);
    s_hi[tid] = (int)lower_bound_i32(li, k, (j1 > jlo ? j1 : jlo) + a.g_base);
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const int row = b * a.Hq + kv * G + h;
    const int64_t off = a.g_cnt ? a.g_off[row] : 0;
    const int32_t *li = a.sel_idx + (int64_t)row * a.k_max + off;
    const float *lw = a.sel_w + (int64_t)row * a.k_max + off;
    const int64_t jb = j0 + a.g_base;
    for (int e = s_lo[h] + tid; e < s_hi[h]; e += kGT) wtab[h][li[e] - jb] = lw[e];
  }
  __syncthreads();
  // ordered compaction of the union (a token is kept by some head iff a weight slot is set;
  // a kept token with weight exactly 0 contributes nothing and may be skipped)
  const int per_w = kGC / (kGT / 32);  // tokens per warp
  int cnt = 0;
  for (int t = warp * per_w + lane; t < (warp + 1) * per_w; t += 32) {
    bool any = false;
#pragma unroll
    for (int h = 0; h < G; ++h) any |= wtab[h][t] != 0.0f;
    cnt += __popc(__ballot_sync(0xffffffffu, any));
  }
  if (lane == 0) s_wc[warp] = cnt;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += s_wc[w];
  if (tid == kGT - 1) {
    int tot = 0;
    for (int w = 0; w < kGT / 32; ++w) tot += s_wc[w];
    s_cnt = tot;
  }
  for (int t = warp * per_w + lane; t < (warp + 1) * per_w; t += 32) {
    bool any = false;
#pragma unroll
    for (int h = 0; h < G; ++h) any |= wtab[h][t] != 0.0f;
    const unsigned m = __ballot_sync(0xffffffffu, any);
    if (any) ulist[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)t;
    base += __popc(m);
  }
  __syncthreads();
  const int U = s_cnt;
  // gather: half-warp (16 lanes x 8 dims) per row, kGUn rows in flight per half-warp
  const int lpr = a.d >> 3;
  const int rpw = 32 / lpr;
  const int nsl = (kGT / 32) * rpw;
  const int slot = warp * rpw + lane / lpr, sub = lane % lpr;
  const uint16_t *Vb = a.V + (int64_t)b * a.v_b_stride + (int64_t)kv * a.v_kv_stride;
  const uint16_t *Rb = a.res_v + (int64_t)b * a.res_b_stride + (int64_t)kv * a.res_cap * a.d;
  float acc[G][8];
#pragma unroll
  for (int h = 0; h < G; ++h)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[h][e] = 0.0f;
  for (int r = slot; r < U; r += nsl * kGUn) {
    uint4 v[kGUn];
    int tt[kGUn];
#pragma unroll
    for (int q = 0; q < kGUn; ++q) {
      const int rr = r + q * nsl;
      tt[q] = rr < U ? ulist[rr] : -1;
      if (tt[q] >= 0) {
        const int64_t j = j0 + tt[q];
        const uint16_t *src;
        if (j < a.n_q) {
          src = Vb + j * a.d;
        } else {
          const uint32_t sl = (uint32_t)(a.res_slot0 + (j - a.n_q)) % (uint32_t)a.res_cap;
          src = Rb + (int64_t)sl * a.d;
        }
        v[q] = ldg_nc16(src + sub * 8);
      } else {
        v[q] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int q = 0; q < kGUn; ++q) {
      if (tt[q] < 0) continue;
      const uint32_t uu[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
      float f[8];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 f2 = __half22float2(*reinterpret_cast<const __half2 *>(&uu[p]));
        f[2 * p] = f2.x;
        f[2 * p + 1] = f2.y;
      }
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float w = wtab[h][tt[q]];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[h][e] = fmaf(w, f[e], acc[h][e]);
      }
    }
  }
  // CTA partial [G][d]: reduce the nsl slots through shared memory (reuse wtab)
  __syncthreads();
  float *red = &wtab[0][0];  // needs nsl * d floats per head pass: 16 * 128 = 2048 <= G*kGC
  float *pp = part + ((int64_t)u * nchunks + ch) * G * a.d;
#pragma unroll
  for (int h = 0; h < G; ++h) {
#pragma unroll
    for (int e = 0; e < 8; ++e) red[slot * a.d + sub * 8 + e] = acc[h][e];
    __syncthreads();
    for (int e = tid; e < a.d; e += kGT) {
      float s = 0.0f;
      for (int q = 0; q < nsl; ++q) s += red[q * a.d + e];
      pp[h * a.d + e] = s;
    }
    __syncthreads();
  }
  // the unit's last CTA sums the chunk partials in order
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(&done[u], 1u);
    last = prev == (unsigned)nchunks - 1;
    if (last) done[u] = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const float *p0 = part + (int64_t)u * nchunks * G * a.d;
  for (int i = tid; i < G * a.d; i += kGT) {
    float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int c = 0;
    for (; c + 3 < nchunks; c += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] += __ldcg(p0 + (int64_t)(c + q) * G * a.d + i);
    }
    for (; c < nchunks; ++c) s4[0] += __ldcg(p0 + (int64_t)c * G * a.d + i);
    const int h = i / a.d, e = i % a.d;
    a.out[((int64_t)b * a.Hq + kv * G + h) * a.d + e] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
}

int gather_union_chunks(int64_t n_cand) { return (int)((n_cand + kGC - 1) / kGC); }

__global__ void k_add_partial(float *out, const float *part, int64_t n) {
  pdl_trigger();
  pdl_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += part[i];
}

cudaError_t launch_add_partial(float *out, const float *part, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  launch_chain(k_add_partial, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, out, part, n);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// High-occupancy per-head gather (HBM values): CTA = (query head, chunk of kRC kept
// entries).  The chunk's (index, weight) pairs are staged in shared memory; each
// half-warp owns kRC/16 rows and issues all of their 16-B loads before the first FMA
// (16 rows x 16 B in flight per thread, ~2 CTAs per SM), which is what a random 256-B
// row gather needs to approach the HBM rate.  Chunk partials are added in chunk order by
// the row's last CTA.
constexpr int kRT = 256;   // threads
constexpr int kRU = 16;    // rows in flight per half-warp per round
constexpr int kRR = 8;     // max rounds per CTA (fewer CTAs -> fewer partials / fences)
constexpr int kRS = kRU * (kRT / 16);        // kept rows per round (256)
constexpr int kRC = kRS * kRR;               // max kept rows per CTA

__global__ void __launch_bounds__(kRT) k_gather_rows(LayerArgs a, int nch, float *part,
                                                     uint32_t *done, int rounds) {
  __shared__ int32_t sj[kRC];
  __shared__ float sw[kRC];
  __shared__ float red[(kRT / 32) * 2 * 128];
  pdl_trigger();
  pdl_wait();
  // grid (G, chunk, unit): the G heads of a KV head read their c-th kept chunks back to back
  // -- those cover about the same token range, so rows kept by several heads hit in L2
  const int u = blockIdx.z, ch = blockIdx.y, tid = threadIdx.x;
  const int b = u / a.Hkv, kv = u - b * a.Hkv;
  const int row = b * a.Hq + kv * a.G + blockIdx.x;
  const int64_t k = a.g_cnt ? a.g_cnt[row] : a.hs[row].ksel;
  const int64_t per = (int64_t)kRS * rounds;  // kept rows of this CTA
  const int64_t e0 = (int64_t)ch * per;
  if (k == 0) {  // nothing kept (a shard's slice can be empty): the row's share is zero
    if (ch == 0 && tid < 128) a.out[(int64_t)row * 128 + tid] = 0.0f;
    return;
  }
  if (e0 >= k) return;  // only the ceil(k/per) CTAs holding kept rows take part
  const int64_t off = a.g_cnt ? a.g_off[row] : 0;
  const int32_t *li = a.sel_idx + (int64_t)row * a.k_max + off;
  const float *lw = a.sel_w + (int64_t)row * a.k_max + off;
  for (int i = tid; i < per; i += kRT) {
    const bool v = e0 + i < k;
    sj[i] = v ? (int32_t)(li[e0 + i] - a.g_base) : -1;
    sw[i] = v ? lw[e0 + i] : 0.0f;
  }
  __syncthreads();
  const int lane = tid & 31, hw = tid >> 4;   // half-warp id (0..15)
  const int sub = lane & 15;                  // 8-dim slice (d = 128)
  const uint16_t *Vb = a.V + (int64_t)b * a.v_b_stride + (int64_t)kv * a.v_kv_stride;
  const uint16_t *Rb = a.res_v + (int64_t)b * a.res_b_stride + (int64_t)kv * a.res_cap * a.d;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
  const int nround = (int)((k - e0 + kRS - 1) / kRS);
  for (int rd = 0; rd < rounds && rd < nround; ++rd) {
    const int base = rd * kRS + hw * kRU;
    uint4 v[kRU];
#pragma unroll
    for (int q = 0; q < kRU; ++q) {
      const int j = sj[base + q];
      if (j >= 0) {
        const uint16_t *src;
        if (j < a.n_q) {
          src = Vb + (int64_t)j * a.d;
        } else {
          const uint32_t sl = (uint32_t)(a.res_slot0 + (j - a.n_q)) % (uint32_t)a.res_cap;
          src = Rb + (int64_t)sl * a.d;
        }
        v[q] = ldg_nc16(src + sub * 8);
      } else {
        v[q] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int q = 0; q < kRU; ++q) {
      const float w = sw[base + q];
      const uint32_t uu[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float2 f2 = __half22float2(*reinterpret_cast<const __half2 *>(&uu[p]));
        acc[2 * p] = fmaf(w, f2.x, acc[2 * p]);
        acc[2 * p + 1] = fmaf(w, f2.y, acc[2 * p + 1]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[hw * 128 + sub * 8 + e] = acc[e];
  __syncthreads();
  float *pp = part + ((int64_t)row * nch + ch) * 128;
  if (tid < 128) {
    float s = 0.0f;
    for (int q = 0; q < (kRT / 32) * 2; ++q) s += red[q * 128 + tid];
    pp[tid] = s;
    __threadfence();  // only the writers of the partial publish it
  }
  __shared__ bool last;
  __syncthreads();
  if (tid == 0) {
    const int nact = (int)((k + per - 1) / per);  // CTAs of this row that hold kept rows
    const unsigned prev = atomicAdd(&done[row], 1u);
    last = prev == (unsigned)(nact > 0 ? nact : 1) - 1;
    if (last) done[row] = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nact = (int)((k + per - 1) / per);
  if (tid < 128) {
    const float *p0 = part + (int64_t)row * nch * 128 + tid;
    float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int c = 0;
    for (; c + 3 < nact; c += 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) s4[q] += __ldcg(p0 + (int64_t)(c + q) * 128);
    }
    for (; c < nact; ++c) s4[0] += __ldcg(p0 + (int64_t)c * 128);
    a.out[(int64_t)row * 128 + tid] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
}

int gather_rows_chunks(int64_t k_cap) { return (int)((k_cap + kRS - 1) / kRS); }  // rounds = 1

cudaError_t launch_gather_rows(const LayerArgs &a, int64_t k_cap, float *part, uint32_t *done,
                               cudaStream_t s) {
  // rounds per CTA: as many as keep >= 4 CTAs per SM (fewer partials and fences per row)
  const int rows = a.B * a.Hq;
  int rounds = 1;
  while (rounds < kRR && (int64_t)rows * ((k_cap + (int64_t)kRS * rounds * 2 - 1) / ((int64_t)kRS * rounds * 2)) >=
                             (int64_t)a.num_sms * 4)
    rounds *= 2;
  const int nch = (int)((k_cap + (int64_t)kRS * rounds - 1) / ((int64_t)kRS * rounds));
  if (nch == 0) return cudaSuccess;
  // CTAs beyond a row's k_sel exit at once (they only count if they hold kept rows)
  dim3 grid((unsigned)a.G, (unsigned)nch, (unsigned)(a.B * a.Hkv));
  launch_chain(k_gather_rows, grid, dim3(kRT), 0, s, a, nch, part, done, rounds);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_gather_union(const LayerArgs &a, float *part, uint32_t *done, cudaStream_t s) {
  const int64_t cb = a.gtok_lo / kGC * kGC;
  const int nch = a.gtok_hi > a.gtok_lo ? gather_union_chunks(a.gtok_hi - cb) : 0;
  if (nch == 0) return cudaSuccess;
  dim3 grid((unsigned)nch, (unsigned)(a.B * a.Hkv));
  switch (a.G) {
    case 1: launch_chain(k_gather_union<1>, grid, dim3(kGT), 0, s, a, nch, part, done); break;
    case 2: launch_chain(k_gather_union<2>, grid, dim3(kGT), 0, s, a, nch, part, done); break;
    case 4: launch_chain(k_gather_union<4>, grid, dim3(kGT), 0, s, a, nch, part, done); break;
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
