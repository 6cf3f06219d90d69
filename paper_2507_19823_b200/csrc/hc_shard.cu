// hc_shard.cu -- SURVEY §8(e): sequence-sharded decode across R GPUs.
//
// Rank r holds the contiguous global token range [base, base + n_q) of every
// (b, layer, kv) unit (its own P codes and V rows).  Because the scores are exact
// integers (R2/R3) and the softmax mass W is a function of Δ = M - z alone (R4), the
// global selection (R5) can be assembled from integer all-reductions only:
//   stats  : local max / min of z                 -> all-reduce MAX       (C1)
//   hist1  : coarse (count, mass) histogram of Δ   -> all-reduce SUM u64   (C2)
//   hist2  : fine histogram inside the global b*   -> all-reduce SUM u64   (C3)
//   counts : local (#Δ<Δ*, #Δ==Δ*) per chunk       -> all-gather row totals (C4)
//   finish : ordered compaction with global offsets + local Eq. 5 partial sums
//                                                  -> all-reduce SUM fp32  (C5)
// Every rank evaluates bound1 / bound2 on the same reduced integers, so all ranks
// agree on (b*, Δ*, r) bit for bit: the index set is R-invariant.
#include <stdlib.h>
#include <string.h>

#include "hc_internal.h"

namespace hc {

constexpr int kShT = 256;
constexpr int kShChunk = 4096;  // tokens per compaction chunk (16 per thread)

__device__ __forceinline__ float sh_z(const LayerArgs &a, int row, int64_t j, int) {
  return a.z[(int64_t)row * a.z_stride + j];  // final after the scan (split scans add into z)
}

// visit tokens j of a row with 4 consecutive tokens per thread per round (16-B loads; z rows
// are 64-float aligned), grid-stride over the row's CTAs
template <typename F>
__device__ __forceinline__ void sh_tokens(const float *zr, int64_t n, F &&f) {
  const int64_t n4 = n & ~(int64_t)3;
  for (int64_t t = ((int64_t)blockIdx.x * kShT + threadIdx.x) * 4; t < n4; t += (int64_t)gridDim.x * kShT * 4) {
    const float4 v = *reinterpret_cast<const float4 *>(zr + t);
    f(t, v.x); f(t + 1, v.y); f(t + 2, v.z); f(t + 3, v.w);
  }
  if (blockIdx.x == 0)
    for (int64_t t = n4 + threadIdx.x; t < n; t += kShT) f(t, zr[t]);
}

// z <- sum of split partials; stats[row] = {max z, -min z} (atomic max)
__global__ void __launch_bounds__(kShT) k_sh_stats(LayerArgs a, int nsplit, int32_t *stats) {
  const int row = blockIdx.y;
  int mx = INT_MIN, mn = INT_MAX;
  sh_tokens(a.z + (int64_t)row * a.z_stride, a.n_cand, [&](int64_t, float zf) {
    const int zi = zint(zf);
    mx = max(mx, zi);
    mn = min(mn, zi);
  });
  mx = __reduce_max_sync(0xffffffffu, mx);
  mn = __reduce_min_sync(0xffffffffu, mn);
  if ((threadIdx.x & 31) == 0 && mx != INT_MIN) {
    atomicMax(&stats[2 * row], mx);
    atomicMax(&stats[2 * row + 1], -mn);
  }
}

// unsplit scan: the scan epilogue already folded max / min into hs -> no pass over z
__global__ void k_sh_stats_folded(const HeadState *hs, int32_t *stats, int rows) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) { stats[2 * r] = hs[r].M; stats[2 * r + 1] = -hs[r].zmin; }
}

__global__ void k_sh_init_stats(int32_t *stats, int rows) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) { stats[2 * r] = INT_MIN; stats[2 * r + 1] = INT_MIN; }
}

__device__ __forceinline__ int sh_shift(int M, int zmin) {
  const uint32_t dmax = (uint32_t)(M - zmin);
  const int bits = 32 - __clz(dmax);
  return bits > kNBBits ? bits - kNBBits : 0;
}

// coarse histogram (count, mass) of the local tokens with the GLOBAL M, zmin -> h1 (u64 atomics)
__global__ void __launch_bounds__(kShT) k_sh_hist1(LayerArgs a, const int32_t *gstats,
                                                   unsigned long long *h1) {
  __shared__ uint32_t cnt[kNB], mlo[kNB], mhi[kNB];
  const int row = blockIdx.y;
  const int M = gstats[2 * row], zmin = -gstats[2 * row + 1];
  const int shift = sh_shift(M, zmin);
  const float kappa = a.hs[row].kappa;
  for (int i = threadIdx.x; i < kNB; i += kShT) { cnt[i] = 0; mlo[i] = 0; mhi[i] = 0; }
  __syncthreads();
  sh_tokens(a.z + (int64_t)row * a.z_stride, a.n_cand, [&](int64_t, float zf) {
    const uint32_t dl = (uint32_t)(M - zint(zf));
    const uint32_t bk = dl >> shift;
    atomicAdd(&cnt[bk], 1u);
    const unsigned long long w = wmass(dl, kappa);  // conversion-pipe form of mass_d (bit-exact)
    const uint32_t wl = (uint32_t)w;
    uint32_t wh = (uint32_t)(w >> 32);
    const uint32_t old = atomicAdd(&mlo[bk], wl);
    wh += (old + wl < old) ? 1u : 0u;
    if (wh) atomicAdd(&mhi[bk], wh);
  });
  __syncthreads();
  unsigned long long *hr = h1 + (int64_t)row * kNB * 2;
  for (int i = threadIdx.x; i < kNB; i += kShT) {
    if (cnt[i]) {
      atomicAdd(&hr[2 * i], (unsigned long long)cnt[i]);
      atomicAdd(&hr[2 * i + 1], ((unsigned long long)mhi[i] << 32) + mlo[i]);
    }
  }
}

// block exclusive scan of pairs (kShT threads)
__device__ __forceinline__ void sh_scan2(unsigned long long &x, unsigned long long &y,
                                         unsigned long long &tx, unsigned long long &ty) {
  __shared__ unsigned long long sx[kShT / 32], sy[kShT / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long ix = x, iy = y;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long ox = __shfl_up_sync(0xffffffffu, ix, off);
    const unsigned long long oy = __shfl_up_sync(0xffffffffu, iy, off);
    if (lane >= off) { ix += ox; iy += oy; }
  }
  __syncthreads();
  if (lane == 31) { sx[w] = ix; sy[w] = iy; }
  __syncthreads();
  unsigned long long bx = 0, by = 0;
  tx = 0; ty = 0;
  for (int k = 0; k < kShT / 32; ++k) {
    if (k < w) { bx += sx[k]; by += sy[k]; }
    tx += sx[k]; ty += sy[k];
  }
  x = bx + ix - x;
  y = by + iy - y;
}

// bound1 on the GLOBAL coarse histogram (identical on every rank) -> hs
__global__ void __launch_bounds__(kShT) k_sh_bound1(SelArgs s, const int32_t *gstats,
                                                    const unsigned long long *h1, unsigned long long *h2z) {
  const int row = blockIdx.x;
  HeadState *hs = s.hs + row;
  // the next phase's fine histogram row, zeroed here (no memset node between the kernels)
  for (int i = threadIdx.x; i < kNB; i += kShT) h2z[(int64_t)row * kNB + i] = 0ull;
  constexpr int kB = kNB / kShT;
  const unsigned long long *hr = h1 + (int64_t)row * kNB * 2;
  unsigned long long c[kB], m[kB], lc = 0, lm = 0;
#pragma unroll
  for (int k = 0; k < kB; ++k) {
    const int bi = threadIdx.x * kB + k;
    c[k] = hr[2 * bi];
    m[k] = hr[2 * bi + 1];
    lc += c[k];
    lm += m[k];
  }
  unsigned long long pc = lc, pm = lm, tc, tm;
  sh_scan2(pc, pm, tc, tm);
  const unsigned long long S = tm, ntot = tc;
  const bool tau_all = s.tau_q >= (1u << 24);
  const unsigned long long theta = tau_all ? 0ull : threshold(s.tau_q, S);
  const bool cap_all = (unsigned long long)s.k_max >= ntot;
  __shared__ int sb;
  if (threadIdx.x == 0) sb = kNB;
  __syncthreads();
  int found = kNB;
  unsigned long long fcb = 0, fmb = 0, cc = pc, cm = pm;
#pragma unroll
  for (int k = 0; k < kB; ++k) {
    const bool trig = c[k] && ((!tau_all && cm + m[k] >= theta) ||
                               (!cap_all && cc + c[k] >= (unsigned long long)s.k_max));
    if (trig && found == kNB) { found = threadIdx.x * kB + k; fcb = cc; fmb = cm; }
    cc += c[k];
    cm += m[k];
  }
  if (found < kNB) atomicMin(&sb, found);
  __syncthreads();
  const int M = gstats[2 * row], zmin = -gstats[2 * row + 1];
  if (threadIdx.x == 0) {
    hs->M = M;
    hs->zmin = zmin;
    hs->shift = sh_shift(M, zmin);
    hs->S = S;
    hs->theta = theta;
    hs->bstar = sb;
    hs->ksel = (int64_t)ntot;
    hs->kstar = (int64_t)ntot;
    hs->delta_star = 0xffffffffu;
    hs->r_ties = 0;
    hs->sel_mass = S;
  }
  if (found < kNB && found == sb) { hs->cnt_before = (uint32_t)fcb; hs->mass_before = fmb; }
}

// fine histogram of local tokens inside the global b*
__global__ void __launch_bounds__(kShT) k_sh_hist2(LayerArgs a, unsigned long long *h2) {
  __shared__ uint32_t cnt[kNB];
  const int row = blockIdx.y;
  const HeadState h = a.hs[row];
  if (h.bstar >= kNB) return;
  for (int i = threadIdx.x; i < kNB; i += kShT) cnt[i] = 0;
  __syncthreads();
  const uint32_t fmask = (1u << h.shift) - 1u;
  sh_tokens(a.z + (int64_t)row * a.z_stride, a.n_cand, [&](int64_t, float zf) {
    const uint32_t dl = (uint32_t)(h.M - zint(zf));
    if ((int)(dl >> h.shift) == h.bstar) atomicAdd(&cnt[dl & fmask], 1u);
  });
  __syncthreads();
  for (int i = threadIdx.x; i < kNB; i += kShT)
    if (cnt[i]) atomicAdd(&h2[(int64_t)row * kNB + i], (unsigned long long)cnt[i]);
}

// bound2 on the GLOBAL fine histogram -> Δ*, r, k_sel (identical on every rank)
__global__ void __launch_bounds__(kShT) k_sh_bound2(SelArgs s, const unsigned long long *h2,
                                                    unsigned long long *cntz) {
  const int row = blockIdx.x;
  HeadState *hs = s.hs + row;
  if (threadIdx.x < 2) cntz[(int64_t)row * 2 + threadIdx.x] = 0ull;  // the counts phase's totals
  const HeadState h = *hs;
  if (h.bstar >= kNB) return;
  constexpr int kB = kNB / kShT;
  const uint32_t dbase = (uint32_t)h.bstar << h.shift;
  const unsigned long long *hr = h2 + (int64_t)row * kNB;
  unsigned long long c[kB], w[kB], lc = 0, lm = 0;
#pragma unroll
  for (int k = 0; k < kB; ++k) {
    const int bi = threadIdx.x * kB + k;
    c[k] = hr[bi];
    w[k] = c[k] ? mass_d(dbase | (uint32_t)bi, h.kappa) : 0ull;
    lc += c[k];
    lm += c[k] * w[k];
  }
  unsigned long long pc = lc, pm = lm, tc, tm;
  sh_scan2(pc, pm, tc, tm);
  const bool tau_all = s.tau_q >= (1u << 24);
  __shared__ int sv;
  if (threadIdx.x == 0) sv = kNB;
  __syncthreads();
  unsigned long long cc = h.cnt_before + pc, cm = h.mass_before + pm;
  int found = kNB;
  unsigned long long f_cc = 0, f_cm = 0, f_w = 0, f_c = 0;
#pragma unroll
  for (int k = 0; k < kB; ++k) {
    if (c[k] && found == kNB) {
      const bool tt = !tau_all && w[k] && (cm + c[k] * w[k] >= h.theta);
      const bool tk = cc + c[k] >= (unsigned long long)s.k_max;
      if (tt || tk) { found = threadIdx.x * kB + k; f_cc = cc; f_cm = cm; f_w = w[k]; f_c = c[k]; }
    }
    cc += c[k];
    cm += c[k] * w[k];
  }
  if (found < kNB) atomicMin(&sv, found);
  __syncthreads();
  if (found < kNB && found == sv) {
    unsigned long long r_tau = ~0ull, r_cap = ~0ull;
    if (!tau_all && f_w && f_cm + f_c * f_w >= h.theta) r_tau = (h.theta - f_cm + f_w - 1) / f_w;
    if (f_cc + f_c >= (unsigned long long)s.k_max) r_cap = (unsigned long long)s.k_max - f_cc;
    if (r_tau == 0) r_tau = 1;
    const unsigned long long r = r_tau < r_cap ? r_tau : r_cap;
    hs->delta_star = dbase | (uint32_t)found;
    hs->r_ties = (uint32_t)r;
    hs->ksel = (int64_t)(f_cc + r);
    hs->kstar = (r_tau <= r_cap) ? (int64_t)(f_cc + r_tau) : -1;
    hs->sel_mass = f_cm + r * f_w;
  }
}

// per-chunk local (strict, tie) counts -> chunk [rows][nch][2]; row totals -> cnt [rows][2]
__global__ void __launch_bounds__(kShT) k_sh_counts(LayerArgs a, int nch, uint32_t *chunk,
                                                    unsigned long long *cnt) {
  const int row = blockIdx.y, ch = blockIdx.x;
  const HeadState h = a.hs[row];
  const int64_t j0 = (int64_t)ch * kShChunk;
  unsigned ns = 0, nt = 0;
  const float *zr = a.z + (int64_t)row * a.z_stride;
#pragma unroll
  for (int k = 0; k < kShChunk / (kShT * 4); ++k) {  // 4 x 16-B loads per thread
    const int64_t t = j0 + ((int64_t)k * kShT + threadIdx.x) * 4;
    if (t + 4 <= a.n_cand) {
      const float4 v = *reinterpret_cast<const float4 *>(zr + t);
      const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t dl = (uint32_t)(h.M - zint(f[u]));
        ns += dl < h.delta_star;
        nt += dl == h.delta_star;
      }
    } else {
      for (int64_t j = t; j < t + 4 && j < a.n_cand; ++j) {
        const uint32_t dl = (uint32_t)(h.M - zint(zr[j]));
        ns += dl < h.delta_star;
        nt += dl == h.delta_star;
      }
    }
  }
  ns = __reduce_add_sync(0xffffffffu, ns);
  nt = __reduce_add_sync(0xffffffffu, nt);
  __shared__ unsigned s0[kShT / 32], s1[kShT / 32];
  if ((threadIdx.x & 31) == 0) { s0[threadIdx.x >> 5] = ns; s1[threadIdx.x >> 5] = nt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned a0 = 0, a1 = 0;
    for (int w = 0; w < kShT / 32; ++w) { a0 += s0[w]; a1 += s1[w]; }
    chunk[((int64_t)row * nch + ch) * 2] = a0;
    chunk[((int64_t)row * nch + ch) * 2 + 1] = a1;
    atomicAdd(&cnt[2 * row], (unsigned long long)a0);
    atomicAdd(&cnt[2 * row + 1], (unsigned long long)a1);
  }
}

// ordered compaction with the offsets of lower ranks + local Eq. 5 partial numerators.
// allcnt [R][rows][2] (all-gathered row totals).  Writes the rank's kept tokens (GLOBAL
// indices base + j) at their GLOBAL positions of sel_idx / sel_w, and part [rows][nch][d].
__global__ void __launch_bounds__(kShT) k_sh_write(LayerArgs a, SelArgs s, int nch,
                                                   const uint32_t *chunk,
                                                   const unsigned long long *allcnt, int rank,
                                                   int64_t base, float *part, int64_t *grange) {
  const int row = blockIdx.y, ch = blockIdx.x;
  const HeadState h = a.hs[row];
  if (grange && ch == 0 && threadIdx.x == 0) {  // this rank's slice of the row's kept list
    unsigned long long sb = 0, tb = 0;
    for (int r = 0; r < rank; ++r) {
      sb += allcnt[((int64_t)r * s.rows + row) * 2];
      tb += allcnt[((int64_t)r * s.rows + row) * 2 + 1];
    }
    const unsigned long long sr = allcnt[((int64_t)rank * s.rows + row) * 2];
    const unsigned long long tr = allcnt[((int64_t)rank * s.rows + row) * 2 + 1];
    const unsigned long long rt = h.r_ties;
    const unsigned long long tk = tb >= rt ? 0ull : (rt - tb < tr ? rt - tb : tr);
    grange[row] = (int64_t)(sb + (tb < rt ? tb : rt));  // [2][rows]: offsets, then counts
    grange[s.rows + row] = (int64_t)(sr + tk);
  }
  __shared__ unsigned long long sp[2];
  if (threadIdx.x == 0) {
    unsigned long long ps = 0, pt = 0;
    for (int r = 0; r < rank; ++r) {
      ps += allcnt[((int64_t)r * s.rows + row) * 2];
      pt += allcnt[((int64_t)r * s.rows + row) * 2 + 1];
    }
    for (int k = 0; k < ch; ++k) {
      ps += chunk[((int64_t)row * nch + k) * 2];
      pt += chunk[((int64_t)row * nch + k) * 2 + 1];
    }
    sp[0] = ps;
    sp[1] = pt;
  }
  __syncthreads();
  const unsigned long long s_before = sp[0], t_before = sp[1], r = h.r_ties;
  const int64_t j0 = (int64_t)ch * kShChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp w owns tokens [j0 + w*512, +512) of the chunk; ballots keep index order
  const int64_t w0 = j0 + (int64_t)warp * (kShChunk / (kShT / 32));
  const int64_t w1 = w0 + kShChunk / (kShT / 32);
  __shared__ unsigned long long ws_[kShT / 32], wt_[kShT / 32];
  unsigned ns = 0, nt = 0;
  for (int64_t j = w0 + lane; j < w1 && j < a.n_cand; j += 32) {
    const uint32_t dl = (uint32_t)(h.M - zint(a.z[(int64_t)row * a.z_stride + j]));
    ns += dl < h.delta_star;
    nt += dl == h.delta_star;
  }
  ns = __reduce_add_sync(0xffffffffu, ns);
  nt = __reduce_add_sync(0xffffffffu, nt);
  if (lane == 0) { ws_[warp] = ns; wt_[warp] = nt; }
  __syncthreads();
  unsigned long long s_w = s_before, t_w = t_before;
  for (int k = 0; k < warp; ++k) { s_w += ws_[k]; t_w += wt_[k]; }
  const double denom = s.renorm ? (double)h.sel_mass : (double)h.S;
  int32_t *oi = s.sel_idx + (int64_t)row * s.k_max;
  float *ow = s.sel_w + (int64_t)row * s.k_max;
  unsigned long long pos = s_w + (t_w < r ? t_w : r), t_run = t_w;
  const unsigned lt = (1u << lane) - 1u;
  // gather: each lane handles 4 dims of d = 128 (dpl = d / 32)
  const int dpl = a.d >> 5;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
  const int b = row / a.Hq, hq = row - b * a.Hq, kv = hq / a.G;
  const uint16_t *Vb = a.V + (int64_t)b * a.v_b_stride + (int64_t)kv * a.v_kv_stride;
  for (int64_t jb = w0; jb < w1 && jb < a.n_cand; jb += 32) {
    const int64_t j = jb + lane;
    const bool v = j < w1 && j < a.n_cand;
    const uint32_t dl = v ? (uint32_t)(h.M - zint(a.z[(int64_t)row * a.z_stride + j])) : 0xffffffffu;
    const bool st = v && dl < h.delta_star;
    const bool ti = v && dl == h.delta_star;
    const unsigned bt = __ballot_sync(0xffffffffu, ti);
    const bool take = st || (ti && t_run + __popc(bt & lt) < r);
    const unsigned bs = __ballot_sync(0xffffffffu, take);
    float wv = 0.0f;
    if (take) {
      const unsigned long long p = pos + __popc(bs & lt);
      wv = (float)((double)mass_d(dl, h.kappa) / denom);
      if ((int64_t)p < s.k_max) {
        oi[p] = (int32_t)(base + j);
        ow[p] = wv;
      }
    }
    // Eq. 5 partial: the warp walks its kept rows (lane-order), all lanes read each row
    unsigned m = grange ? 0u : bs;  // grange: k_gather_rows does Eq. 5 afterwards
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const float w_ = __shfl_sync(0xffffffffu, wv, src);
      const int64_t jj = jb + src;
      const uint16_t *row_p = Vb + jj * a.d + lane * dpl;
      for (int e = 0; e < dpl; ++e) acc[e] = fmaf(w_, __half2float(__ushort_as_half(row_p[e])), acc[e]);
    }
    pos += __popc(bs);
    t_run += __popc(bt);
  }
  if (grange) return;
  __shared__ float red[kShT / 32][256];
  for (int e = 0; e < dpl; ++e) red[warp][lane * dpl + e] = acc[e];
  __syncthreads();
  for (int e = threadIdx.x; e < a.d; e += kShT) {
    float sum = 0.0f;
    for (int w = 0; w < kShT / 32; ++w) sum += red[w][e];
    part[((int64_t)row * nch + ch) * a.d + e] = sum;
  }
}

// Ordered compaction only (Eq. 5 follows in k_gather_rows over the rank's list slice):
// warp w of the CTA owns tokens [j0 + 512 w, +512), walked 256 per step (8 per lane, two
// 16-B loads), warp scans of the lanes' (tie, kept) counts give in-order positions, kept
// (Δ, token) pairs are staged in shared memory and written lane-parallel.  Also records
// this rank's slice [off, off + cnt) of every row's kept list (grange [2][rows]).
constexpr int kShWT = kShChunk / (kShT / 32);  // tokens per warp (512)
__global__ void __launch_bounds__(kShT) k_sh_compact(LayerArgs a, SelArgs s, int nch,
                                                     const uint32_t *chunk,
                                                     const unsigned long long *allcnt, int rank,
                                                     int64_t base, int64_t *grange) {
  const int row = blockIdx.y, ch = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const HeadState h = a.hs[row];
  __shared__ unsigned long long sp[2];
  __shared__ unsigned s_ws[kShT / 32], s_wt[kShT / 32];
  __shared__ uint32_t stg_d[kShT / 32][256], stg_t[kShT / 32][256];
  if (tid == 0) {
    unsigned long long ps = 0, pt = 0;
    for (int r = 0; r < rank; ++r) {
      ps += allcnt[((int64_t)r * s.rows + row) * 2];
      pt += allcnt[((int64_t)r * s.rows + row) * 2 + 1];
    }
    if (ch == 0) {
      const unsigned long long sr = allcnt[((int64_t)rank * s.rows + row) * 2];
      const unsigned long long tr = allcnt[((int64_t)rank * s.rows + row) * 2 + 1];
      const unsigned long long rt = h.r_ties;
      const unsigned long long tk = pt >= rt ? 0ull : (rt - pt < tr ? rt - pt : tr);
      grange[row] = (int64_t)(ps + (pt < rt ? pt : rt));
      grange[s.rows + row] = (int64_t)(sr + tk);
    }
    for (int k = 0; k < ch; ++k) {
      ps += chunk[((int64_t)row * nch + k) * 2];
      pt += chunk[((int64_t)row * nch + k) * 2 + 1];
    }
    sp[0] = ps;
    sp[1] = pt;
  }
  const float *zr = a.z + (int64_t)row * a.z_stride;
  const int64_t w_lo = (int64_t)ch * kShChunk + (int64_t)warp * kShWT;
  const int64_t w_hi = w_lo + kShWT < a.n_cand ? w_lo + kShWT : a.n_cand;
  auto load8 = [&](int64_t t, uint32_t (&dl)[8]) {
    float v[8];
    if (t + 8 <= w_hi) {
      const float4 a4 = *reinterpret_cast<const float4 *>(zr + t);
      const float4 b4 = *reinterpret_cast<const float4 *>(zr + t + 4);
      v[0] = a4.x; v[1] = a4.y; v[2] = a4.z; v[3] = a4.w; v[4] = b4.x; v[5] = b4.y; v[6] = b4.z; v[7] = b4.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = t + u < w_hi ? zr[t + u] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) dl[u] = t + u < w_hi ? (uint32_t)(h.M - zint(v[u])) : 0xffffffffu;
  };
  {  // per-warp totals
    unsigned ns = 0, nt = 0;
    for (int64_t tb = w_lo; tb < w_hi; tb += 256) {
      uint32_t dl[8];
      load8(tb + lane * 8, dl);
#pragma unroll
      for (int u = 0; u < 8; ++u) { ns += dl[u] < h.delta_star; nt += dl[u] == h.delta_star; }
    }
    ns = __reduce_add_sync(0xffffffffu, ns);
    nt = __reduce_add_sync(0xffffffffu, nt);
    if (lane == 0) { s_ws[warp] = ns; s_wt[warp] = nt; }
  }
  __syncthreads();
  unsigned long long s_w = sp[0], t_run = sp[1];
  for (int k = 0; k < warp; ++k) { s_w += s_ws[k]; t_run += s_wt[k]; }
  const unsigned long long r_ties = h.r_ties;
  unsigned long long pos = s_w + (t_run < r_ties ? t_run : r_ties);
  const double den_d = s.renorm ? (double)h.sel_mass : (double)h.S;
  const float inv_den = (float)(1.0 / den_d);
  int32_t *oi = s.sel_idx + (int64_t)row * s.k_max;
  float *ow = s.sel_w + (int64_t)row * s.k_max;
  for (int64_t tb = w_lo; tb < w_hi; tb += 256) {
    const int64_t t0 = tb + lane * 8;
    uint32_t dl[8];
    load8(t0, dl);
    unsigned nst = 0, ntie = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) { nst += dl[u] < h.delta_star; ntie += dl[u] == h.delta_star; }
    unsigned tie_pre = ntie;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned o = __shfl_up_sync(0xffffffffu, tie_pre, off);
      if (lane >= off) tie_pre += o;
    }
    const unsigned tie_tot = __shfl_sync(0xffffffffu, tie_pre, 31);
    tie_pre -= ntie;
    const unsigned long long my_t0 = t_run + tie_pre;
    const unsigned taken = my_t0 >= r_ties ? 0u : (unsigned)((r_ties - my_t0) < ntie ? (r_ties - my_t0) : ntie);
    unsigned kpre = nst + taken;
    const unsigned kept = kpre;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned o = __shfl_up_sync(0xffffffffu, kpre, off);
      if (lane >= off) kpre += o;
    }
    const unsigned kept_tot = __shfl_sync(0xffffffffu, kpre, 31);
    unsigned q = kpre - kept, seen = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      bool take = dl[u] < h.delta_star;
      if (dl[u] == h.delta_star) { take = seen < taken; ++seen; }
      if (take) { stg_d[warp][q] = dl[u]; stg_t[warp][q] = (uint32_t)(t0 + u - w_lo); ++q; }
    }
    __syncwarp();
    for (unsigned i = lane; i < kept_tot; i += 32) {
      const unsigned long long p = pos + i;
      if ((int64_t)p < s.k_max) {
        oi[p] = (int32_t)(base + w_lo + stg_t[warp][i]);
        ow[p] = __fmul_rn((float)mass_d(stg_d[warp][i], h.kappa), inv_den);
      }
    }
    __syncwarp();
    pos += kept_tot;
    t_run += tie_tot;
  }
}

// The fused finish's chunk prefixes (K3G, hc_select_pass.cu): per row, the GLOBAL (strict, tie)
// counts before each of this rank's chunks -- the lower ranks' totals (all-gathered) plus this
// rank's earlier chunks -- as (strict << 32 | ties); and the row marked resolved for K3G.
__global__ void __launch_bounds__(256) k_sh_pre(SelArgs s, int nch, const uint32_t *chunk,
                                                const unsigned long long *allcnt, int rank, uint32_t *rdonez) {
  const int row = blockIdx.x, t = threadIdx.x;
  if (t == 0) rdonez[row] = 0u;  // K3G's per-row completion counter (no memset node)
  __shared__ unsigned long long base2[2];
  __shared__ unsigned long long wsum[2][8];
  if (t == 0) {
    unsigned long long ps = 0, pt = 0;
    for (int r = 0; r < rank; ++r) {
      ps += allcnt[((int64_t)r * s.rows + row) * 2];
      pt += allcnt[((int64_t)r * s.rows + row) * 2 + 1];
    }
    base2[0] = ps;
    base2[1] = pt;
    s.hs[row].state = kStDone;
  }
  // thread-contiguous runs of chunks, then a block scan of the run totals
  const int per = (nch + 255) / 256;
  const int c0 = min(nch, t * per), c1 = min(nch, c0 + per);
  unsigned long long xs = 0, xt = 0;
  for (int c = c0; c < c1; ++c) {
    xs += chunk[((int64_t)row * nch + c) * 2];
    xt += chunk[((int64_t)row * nch + c) * 2 + 1];
  }
  unsigned long long is = xs, it = xt;
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long os = __shfl_up_sync(0xffffffffu, is, off);
    const unsigned long long ot = __shfl_up_sync(0xffffffffu, it, off);
    if (lane >= off) { is += os; it += ot; }
  }
  if (lane == 31) { wsum[0][w] = is; wsum[1][w] = it; }
  __syncthreads();
  unsigned long long bs = base2[0], bt = base2[1];
  for (int q = 0; q < w; ++q) { bs += wsum[0][q]; bt += wsum[1][q]; }
  bs += is - xs;
  bt += it - xt;
  for (int c = c0; c < c1; ++c) {
    s.pre[(int64_t)row * nch + c] = (bs << 32) | bt;
    bs += chunk[((int64_t)row * nch + c) * 2];
    bt += chunk[((int64_t)row * nch + c) * 2 + 1];
  }
}

// deterministic sum of the chunk partials -> out [rows][d] (this rank's numerator share)
__global__ void k_sh_reduce(int rows, int nch, int d, const float *part, float *out) {
  const int row = blockIdx.x;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float sum = 0.0f;
    for (int c = 0; c < nch; ++c) sum += part[((int64_t)row * nch + c) * d + e];
    out[(int64_t)row * d + e] = sum;
  }
}

static int sh_grid(int64_t n) {
  int64_t g = (n + kShT * 16 - 1) / (kShT * 16);
  return (int)(g < 1 ? 1 : (g > 64 ? 64 : g));
}

cudaError_t launch_shard_stats(const LayerArgs &a, int nsplit, int32_t *stats, cudaStream_t st) {
  const int rows = a.B * a.Hq;
  if (nsplit <= 1 && a.n_res == 0 && a.n_q > 0) {
    k_sh_stats_folded<<<(rows + 127) / 128, 128, 0, st>>>(a.hs, stats, rows);
    note_launch();
    return cudaGetLastError();
  }
  k_sh_init_stats<<<(rows + 127) / 128, 128, 0, st>>>(stats, rows);
  note_launch();
  k_sh_stats<<<dim3(sh_grid(a.n_cand), rows), kShT, 0, st>>>(a, nsplit, stats);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_hist1(const LayerArgs &a, const int32_t *gstats, unsigned long long *h1,
                               cudaStream_t st) {
  const int rows = a.B * a.Hq;
  cudaMemsetAsync(h1, 0, (size_t)rows * kNB * 16, st);
  k_sh_hist1<<<dim3(sh_grid(a.n_cand), rows), kShT, 0, st>>>(a, gstats, h1);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_shard_hist2(const LayerArgs &a, const SelArgs &s, const int32_t *gstats,
                               const unsigned long long *h1, unsigned long long *h2, cudaStream_t st) {
  const int rows = a.B * a.Hq;
  k_sh_bound1<<<rows, kShT, 0, st>>>(s, gstats, h1, h2);
  note_launch();
  k_sh_hist2<<<dim3(sh_grid(a.n_cand), rows), kShT, 0, st>>>(a, h2);
  note_launch();
  return cudaGetLastError();
}

int shard_chunks(int64_t n) { return (int)((n + kShChunk - 1) / kShChunk); }

cudaError_t launch_shard_counts(const LayerArgs &a, const SelArgs &s, const unsigned long long *h2,
                                uint32_t *chunk, unsigned long long *cnt, cudaStream_t st) {
  const int rows = a.B * a.Hq;
  k_sh_bound2<<<rows, kShT, 0, st>>>(s, h2, cnt);
  note_launch();
  const int nch = shard_chunks(a.n_cand);
  if (nch > 0) {
    k_sh_counts<<<dim3(nch, rows), kShT, 0, st>>>(a, nch, chunk, cnt);
    note_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_shard_finish(const LayerArgs &a, const SelArgs &s, const uint32_t *chunk,
                                const unsigned long long *allcnt, int rank, int64_t base,
                                float *part, float *out, cudaStream_t st, int64_t *grange,
                                float *rpart, uint32_t *rdone, float *upart, uint32_t *udone,
                                unsigned long long *pre, float *wpart) {
  const int rows = a.B * a.Hq;
  const int nch = shard_chunks(a.n_cand);
  const char *k3g_ev = getenv("HC_K3G");
  if (nch > 0 && pre && wpart && rdone && a.d == 128 && a.v_placement == 0 && !(k3g_ev && !strcmp(k3g_ev, "0")) &&
      nch == select_chunks(a.n_cand)) {
    // values in HBM: this rank's ordered compaction fused with its Eq. 5 share (K3G) over the
    // chunk prefixes of the global order
    SelArgs s2 = s;
    s2.pre = pre;
    s2.nch = nch;
    s2.n = a.n_cand;
    k_sh_pre<<<rows, 256, 0, st>>>(s2, nch, chunk, allcnt, rank, rdone);
    note_launch();
    LayerArgs g = a;
    g.out = out;
    return launch_select_write_gather(s2, g, wpart, rdone, a.num_sms, st, base);
  }
  if (nch > 0 && grange && a.v_placement == 1 && a.G > 1 && upart && udone) {
    // host-resident values (config 5): the GQA union of this rank's kept rows is read once
    // over the host link (as in the unsharded decode), not once per head
    k_sh_compact<<<dim3(nch, rows), kShT, 0, st>>>(a, s, nch, chunk, allcnt, rank, base, grange);
    note_launch();
    cudaError_t e = cudaMemsetAsync(udone, 0, (size_t)a.B * a.Hkv * 4, st);
    if (e != cudaSuccess) return e;
    LayerArgs g = a;
    g.g_off = grange;
    g.g_cnt = grange + rows;
    g.g_base = base;
    g.out = out;
    g.gtok_lo = 0;
    g.gtok_hi = a.n_cand;
    return launch_gather_union(g, upart, udone, st);
  }
  if (nch > 0 && grange && a.d == 128) {
    // compaction only, then the many-rows-in-flight gather over this rank's list slice
    k_sh_compact<<<dim3(nch, rows), kShT, 0, st>>>(a, s, nch, chunk, allcnt, rank, base, grange);
    note_launch();
    cudaError_t e = cudaMemsetAsync(rdone, 0, (size_t)rows * 4, st);
    if (e != cudaSuccess) return e;
    LayerArgs g = a;
    g.g_off = grange;
    g.g_cnt = grange + rows;
    g.g_base = base;
    g.out = out;
    const int64_t kc2 = a.k_max < a.n_cand ? a.k_max : a.n_cand;
    return launch_gather_rows(g, kc2, rpart, rdone, st);
  } else if (nch > 0) {
    k_sh_write<<<dim3(nch, rows), kShT, 0, st>>>(a, s, nch, chunk, allcnt, rank, base, part, nullptr);
    note_launch();
    k_sh_reduce<<<rows, 128, 0, st>>>(rows, nch, a.d, part, out);
    note_launch();
  } else {
    cudaMemsetAsync(out, 0, (size_t)rows * a.d * 4, st);
  }
  return cudaGetLastError();
}

}  // namespace hc
