// hc_select_fused.cu -- rows a3, a4, a5 in ONE kernel per layer:
//   normalisation ã = softmax(z̃/√d) as exact fixed-point mass (R4),
//   Eq. 4 cumulative-mass eviction with the k_max cap (R5),
//   Eq. 5 weighted sum of the kept value rows (R6).
//
// One thread-block CLUSTER of `cs` CTAs per row (= query head).  Each CTA owns a
// contiguous token range of the row; the row-wide reductions go through distributed
// shared memory (DSMEM) instead of global atomics and extra launches:
//   P0  z (final after the scan) -> SMEM cache; M, zmin (cluster max/min) unless folded
//   P1  coarse (count, mass) histogram of Δ = M - z >> shift   [SMEM atomics]
//       cluster reduce: CTA r owns bins [r*NB/cs, (r+1)*NB/cs) and sums them over peers;
//       bound1: S, Θ = ⌈τ_q·S/2^24⌉, first bucket b* where mass reaches Θ or count k_max
//   P2  fine count histogram inside b* -> cluster reduce -> bound2: exact Δ*, #ties r
//   P3  ordered compaction: per-warp (strict, tie) counts -> prefixes over warps and
//       cluster ranks; each warp walks its chunk 256 tokens per step (8 per lane), warp
//       scans give in-order positions, kept (Δ, token) are staged in shared memory and
//       written lane-parallel: ascending indices and weights W_j/S -> sel_idx / sel_w
//   P4  (HC_GATHER=fused only) gather: every CTA sums ã_j·V_j over ITS kept rows; the
//       default path runs Eq. 5 in hc_gather.cu (k_gather_rows / k_gather_union).
// Two instantiations: with P4 (1 CTA/SM) and selection-only (64 registers, 2 CTAs/SM
// for long rows).
// All sums that decide indices are integers: bit-exact and decomposition-invariant.
#include <cooperative_groups.h>
#include <stdlib.h>

#include "hc_internal.h"

namespace cg = cooperative_groups;

namespace hc {

constexpr int kFT = 512;                 // threads per CTA
constexpr int kZCacheMax = 24576;        // tokens whose z a CTA keeps in shared memory
constexpr int kGU = 8;                   // gathered rows in flight per half-warp

struct Slot {  // per-CTA values published to the cluster through DSMEM
  int M, zmin;
  unsigned long long c, m;      // totals of the owned bins
  int cand;                     // first triggering bin in the owned range (kNB: none)
  unsigned long long cb, mb;    // count / mass before `cand`
  unsigned long long ns, nt;    // strict / tie counts of the token range
  unsigned long long r_tau, r_cap, w;  // bound2 details at the fine candidate
};

template <typename T>
__device__ __forceinline__ void bscan2(T &x, T &y, T &tx, T &ty, T *sx, T *sy) {
  // block-wide exclusive scan of pairs over kFT threads; tx, ty = totals
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T ix = x, iy = y;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T ox = __shfl_up_sync(0xffffffffu, ix, off);
    const T oy = __shfl_up_sync(0xffffffffu, iy, off);
    if (lane >= off) { ix += ox; iy += oy; }
  }
  __syncthreads();
  if (lane == 31) { sx[w] = ix; sy[w] = iy; }
  __syncthreads();
  T bx = 0, by = 0;
  tx = 0; ty = 0;
#pragma unroll
  for (int k = 0; k < kFT / 32; ++k) {
    if (k < w) { bx += sx[k]; by += sy[k]; }
    tx += sx[k]; ty += sy[k];
  }
  x = bx + ix - x;
  y = by + iy - y;
}


// visit every token t in [0, nt) of the CTA once (any order) with 16 tokens per thread in
// flight: 4 x 16-B loads issued before use (zsrc is 16-B aligned: the z cache or the z row)
template <typename F>
__device__ __forceinline__ void for_tokens_pos(const float *zsrc, int64_t nt, F &&f) {
  const int64_t nt4 = nt & ~(int64_t)3;
  for (int64_t base = (int64_t)threadIdx.x * 4; base < nt4; base += (int64_t)kFT * 16) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + (int64_t)u * kFT * 4;
      v[u] = t < nt4 ? *reinterpret_cast<const float4 *>(zsrc + t) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + (int64_t)u * kFT * 4;
      if (t < nt4) { f(t, v[u].x); f(t + 1, v[u].y); f(t + 2, v[u].z); f(t + 3, v[u].w); }
    }
  }
  for (int64_t t = nt4 + threadIdx.x; t < nt; t += kFT) f(t, zsrc[t]);
}

template <typename F>
__device__ __forceinline__ void for_tokens(const float *zsrc, int64_t nt, F &&f) {
  const int64_t nt4 = nt & ~(int64_t)3;
  for (int64_t base = (int64_t)threadIdx.x * 4; base < nt4; base += (int64_t)kFT * 16) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + (int64_t)u * kFT * 4;
      v[u] = t < nt4 ? *reinterpret_cast<const float4 *>(zsrc + t) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (base + (int64_t)u * kFT * 4 < nt4) {
        f(v[u].x); f(v[u].y); f(v[u].z); f(v[u].w);
      }
    }
  }
  for (int64_t t = nt4 + threadIdx.x; t < nt; t += kFT) f(zsrc[t]);
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

__device__ __forceinline__ uint4 ld_nc16(const uint16_t *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// kG = false: selection only (P0-P3; the gather runs as its own kernel or not at all) --
// lighter on registers, two CTAs per SM
template <bool kG, int kOcc>
__global__ void __launch_bounds__(kFT, kOcc)
    k_select_fused(SelArgs s, LayerArgs la, int cs, int nsplit, int zcache, int do_gather,
                   int stop) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.x / cs;
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) uint8_t smem[];
  // per-bin mass as two u32 words (native 32-bit shared atomics; a 64-bit shared
  // atomicAdd compiles to a CAS spin loop): mass = mhi * 2^32 + mlo
  uint32_t *mlo = reinterpret_cast<uint32_t *>(smem);                            // [kNB]
  uint32_t *mhi = reinterpret_cast<uint32_t *>(smem + kNB * 4);                  // [kNB]
  uint32_t *cnt = reinterpret_cast<uint32_t *>(smem + kNB * 8);                  // [kNB]
  float *zc = reinterpret_cast<float *>(smem + kNB * 12);                        // token cache
  __shared__ Slot slot;
  __shared__ unsigned long long sx[kFT / 32], sy[kFT / 32];
  __shared__ float s_red[(kFT / 32) * 32 * 8];  // gather partials [nslots][d] (nslots*d == 4096)

  pdl_trigger();
  pdl_wait();
  HeadState *hs = s.hs + row;
  const float kappa = hs->kappa;
  const int64_t n = s.n;
  const int64_t per = ((n + cs - 1) / cs + 15) / 16 * 16;
  const int64_t j0 = (int64_t)rank * per;
  const int64_t j1 = j0 + per < n ? j0 + per : n;
  const int64_t nt = j1 > j0 ? j1 - j0 : 0;  // tokens of this CTA
  const float *zsrc = zcache ? zc : s.z + (int64_t)row * s.z_stride + j0;  // token t at zsrc[t]

  // ---------------------------------------------------------------- P0: z, M, zmin
  // 4 consecutive tokens per thread per round, all split planes loaded before use.
  int mx = INT_MIN, mn = INT_MAX;
  // z final and not cached: M / zmin were folded into hs by the scan / resident / prep
  // epilogues -> no pass over z here
  const bool skip_p0 = nsplit <= 1 && !zcache;
  if (skip_p0) {
    if (tid == 0) {
      const int m0 = hs->M, z0 = hs->zmin;
      mx = m0;
      mn = z0;
    }
  } else {  // stream z once (final after the scan: split scans accumulate exactly into z)
    for_tokens_pos(s.z + (int64_t)row * s.z_stride + j0, nt, [&](int64_t t, float zf) {
      if (zcache) zc[t] = zf;
      const int zi = zint(zf);
      mx = max(mx, zi);
      mn = min(mn, zi);
    });
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  mn = __reduce_min_sync(0xffffffffu, mn);
  {
    __shared__ int wmx[kFT / 32], wmn[kFT / 32];
    if ((tid & 31) == 0) { wmx[tid >> 5] = mx; wmn[tid >> 5] = mn; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kFT / 32; ++w) { mx = max(mx, wmx[w]); mn = min(mn, wmn[w]); }
      slot.M = mx;
      slot.zmin = mn;
    }
  }
  cl.sync();
  int M = INT_MIN, zmin = INT_MAX;
  for (int r = 0; r < cs; ++r) {
    const Slot *o = cl.map_shared_rank(&slot, r);
    M = max(M, o->M);
    zmin = min(zmin, o->zmin);
  }
  const uint32_t dmax = (uint32_t)(M - zmin);
  const int bits = 32 - __clz(dmax);
  const int shift = bits > kNBBits ? bits - kNBBits : 0;
  if (stop == 1) { cl.sync(); return; }
  const int nbo = kNB / cs;                 // owned bins per CTA
  const int b_lo = rank * nbo;

  // ---------------------------------------------------------------- P1: coarse histogram
  for (int i = tid; i < kNB; i += kFT) { cnt[i] = 0; mlo[i] = 0u; mhi[i] = 0u; }
  __syncthreads();
  for_tokens(zsrc, nt, [&](float zf) {
    const uint32_t dl = (uint32_t)(M - zint(zf));
    const uint32_t bk = dl >> shift;
    atomicAdd(&cnt[bk], 1u);
    uint32_t wl, wh;
    mass_parts(dl, kappa, wl, wh);
    const uint32_t old = atomicAdd(&mlo[bk], wl);
    wh += (old + wl < old) ? 1u : 0u;  // carry out of the low word
    if (wh) atomicAdd(&mhi[bk], wh);
  });
  cl.sync();
  for (int i = tid; i < nbo; i += kFT) {  // sum my owned bins over the peers
    uint32_t c = cnt[b_lo + i];
    unsigned long long m = ((unsigned long long)mhi[b_lo + i] << 32) + mlo[b_lo + i];
    for (int r = 0; r < cs; ++r) {
      if (r == rank) continue;
      c += cl.map_shared_rank(cnt, r)[b_lo + i];
      m += ((unsigned long long)cl.map_shared_rank(mhi, r)[b_lo + i] << 32) +
           cl.map_shared_rank(mlo, r)[b_lo + i];
    }
    cnt[b_lo + i] = c;
    mlo[b_lo + i] = (uint32_t)m;
    mhi[b_lo + i] = (uint32_t)(m >> 32);
  }
  cl.sync();
  // bound1 over the owned bins: thread owns bins [b_lo + tid*bpt, +bpt)
  const int bpt = (nbo + kFT - 1) / kFT;
  unsigned long long lc = 0, lm = 0;
  for (int k = 0; k < bpt; ++k) {
    const int bi = tid * bpt + k;
    if (bi < nbo) { lc += cnt[b_lo + bi]; lm += ((unsigned long long)mhi[b_lo + bi] << 32) + mlo[b_lo + bi]; }
  }
  unsigned long long pc = lc, pm = lm, tc, tm;
  bscan2<unsigned long long>(pc, pm, tc, tm, sx, sy);
  if (tid == 0) { slot.c = tc; slot.m = tm; slot.cand = kNB; }
  cl.sync();
  unsigned long long before_c = 0, before_m = 0, S = 0, ntot = 0;
  for (int r = 0; r < cs; ++r) {
    const Slot *o = cl.map_shared_rank(&slot, r);
    if (r < rank) { before_c += o->c; before_m += o->m; }
    S += o->m;
    ntot += o->c;
  }
  const bool tau_all = s.tau_q >= (1u << 24);
  const unsigned long long theta = tau_all ? 0ull : threshold(s.tau_q, S);
  const bool cap_all = (unsigned long long)s.k_max >= ntot;
  {
    unsigned long long cc = before_c + pc, cm = before_m + pm;
    int found = kNB;
    unsigned long long fcb = 0, fmb = 0;
    for (int k = 0; k < bpt; ++k) {
      const int bi = tid * bpt + k;
      if (bi >= nbo) break;
      const unsigned long long c = cnt[b_lo + bi];
      const unsigned long long m = ((unsigned long long)mhi[b_lo + bi] << 32) + mlo[b_lo + bi];
      const bool trig = c && ((!tau_all && cm + m >= theta) || (!cap_all && cc + c >= (unsigned long long)s.k_max));
      if (trig && found == kNB) { found = b_lo + bi; fcb = cc; fmb = cm; }
      cc += c;
      cm += m;
    }
    if (found < kNB) atomicMin(&slot.cand, found);
    __syncthreads();
    if (found < kNB && found == slot.cand) { slot.cb = fcb; slot.mb = fmb; }
  }
  cl.sync();
  int bstar = kNB, owner = -1;
  for (int r = 0; r < cs; ++r) {
    const int c = cl.map_shared_rank(&slot, r)->cand;
    if (c < bstar) { bstar = c; owner = r; }
  }
  if (stop == 2) { cl.sync(); return; }
  unsigned long long cnt_before = 0, mass_before = 0;
  if (owner >= 0) {
    cnt_before = cl.map_shared_rank(&slot, owner)->cb;
    mass_before = cl.map_shared_rank(&slot, owner)->mb;
  }
  // ---------------------------------------------------------------- P2: fine histogram
  uint32_t delta_star = 0xffffffffu;
  unsigned long long r_ties = 0, ksel = ntot, selmass = S;
  long long kstar = (long long)ntot;
  if (bstar < kNB) {
    cl.sync();  // every peer finished reading my slot / bins
    for (int i = tid; i < kNB; i += kFT) cnt[i] = 0;
    __syncthreads();
    const uint32_t fmask = (1u << shift) - 1u;
    for_tokens(zsrc, nt, [&](float zf) {
      const uint32_t dl = (uint32_t)(M - zint(zf));
      if ((int)(dl >> shift) == bstar) atomicAdd(&cnt[dl & fmask], 1u);
    });
    cl.sync();
    for (int i = tid; i < nbo; i += kFT) {
      uint32_t c = cnt[b_lo + i];
      for (int r = 0; r < cs; ++r)
        if (r != rank) c += cl.map_shared_rank(cnt, r)[b_lo + i];
      cnt[b_lo + i] = c;
    }
    cl.sync();
    const uint32_t dbase = (uint32_t)bstar << shift;
    lc = 0; lm = 0;
    for (int k = 0; k < bpt; ++k) {
      const int bi = tid * bpt + k;
      if (bi < nbo && cnt[b_lo + bi]) {
        lc += cnt[b_lo + bi];
        lm += (unsigned long long)cnt[b_lo + bi] * mass_d(dbase | (uint32_t)(b_lo + bi), kappa);
      }
    }
    pc = lc; pm = lm;
    bscan2<unsigned long long>(pc, pm, tc, tm, sx, sy);
    if (tid == 0) { slot.c = tc; slot.m = tm; slot.cand = kNB; }
    cl.sync();
    unsigned long long bc = cnt_before, bm = mass_before;
    for (int r = 0; r < rank; ++r) {
      const Slot *o = cl.map_shared_rank(&slot, r);
      bc += o->c;
      bm += o->m;
    }
    {
      unsigned long long cc = bc + pc, cm = bm + pm;
      int found = kNB;
      unsigned long long f_cc = 0, f_cm = 0, f_w = 0, f_c = 0;
      for (int k = 0; k < bpt; ++k) {
        const int bi = tid * bpt + k;
        if (bi >= nbo) break;
        const unsigned long long c = cnt[b_lo + bi];
        if (!c) continue;
        const unsigned long long w = mass_d(dbase | (uint32_t)(b_lo + bi), kappa);
        const bool tt = !tau_all && w && (cm + c * w >= theta);
        const bool tk = cc + c >= (unsigned long long)s.k_max;
        if ((tt || tk) && found == kNB) { found = b_lo + bi; f_cc = cc; f_cm = cm; f_w = w; f_c = c; }
        cc += c;
        cm += c * w;
      }
      if (found < kNB) atomicMin(&slot.cand, found);
      __syncthreads();
      if (found < kNB && found == slot.cand) {
        unsigned long long r_tau = ~0ull, r_cap = ~0ull;
        if (!tau_all && f_w && f_cm + f_c * f_w >= theta) r_tau = (theta - f_cm + f_w - 1) / f_w;
        if (f_cc + f_c >= (unsigned long long)s.k_max) r_cap = (unsigned long long)s.k_max - f_cc;
        if (r_tau == 0) r_tau = 1;
        slot.cb = f_cc;
        slot.mb = f_cm;
        slot.r_tau = r_tau;
        slot.r_cap = r_cap;
        slot.w = f_w;
      }
    }
    cl.sync();
    int fbin = kNB, fown = -1;
    for (int r = 0; r < cs; ++r) {
      const int c = cl.map_shared_rank(&slot, r)->cand;
      if (c < fbin) { fbin = c; fown = r; }
    }
    const Slot *o = cl.map_shared_rank(&slot, fown < 0 ? 0 : fown);
    const unsigned long long r_tau = o->r_tau, r_cap = o->r_cap, f_cc = o->cb, f_cm = o->mb, f_w = o->w;
    const unsigned long long r = r_tau < r_cap ? r_tau : r_cap;
    delta_star = dbase | (uint32_t)fbin;
    r_ties = r;
    ksel = f_cc + r;
    kstar = (r_tau <= r_cap) ? (long long)(f_cc + r_tau) : -1;
    selmass = f_cm + r * f_w;
  }
  // ---------------------------------------------------------------- P3: compaction
  cl.sync();  // peers done with my slot
  if (stop == 3) return;
  // warp-chunked ordered compaction: warp w owns tokens [w*wc, (w+1)*wc) of this CTA and
  // walks it 256 tokens per step, 8 consecutive tokens per lane (two 16-B loads); warp
  // scans of the lanes' (tie, kept) counts give in-order positions.
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t wc = ((nt + kFT / 32 - 1) / (kFT / 32) + 255) / 256 * 256;
  const int64_t w_lo = (int64_t)warp * wc < nt ? (int64_t)warp * wc : nt;
  const int64_t w_hi = w_lo + wc < nt ? w_lo + wc : nt;
  auto load8 = [&](int64_t t, float (&v)[8]) {  // tokens t..t+7 (t % 8 == 0), 0 past w_hi
    if (t + 8 <= w_hi) {
      const float4 a4 = *reinterpret_cast<const float4 *>(zsrc + t);
      const float4 b4 = *reinterpret_cast<const float4 *>(zsrc + t + 4);
      v[0] = a4.x; v[1] = a4.y; v[2] = a4.z; v[3] = a4.w;
      v[4] = b4.x; v[5] = b4.y; v[6] = b4.z; v[7] = b4.w;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = t + u < w_hi ? zsrc[t + u] : 0.0f;
    }
  };
  __shared__ unsigned long long s_ws[kFT / 32], s_wt[kFT / 32];
  {
    unsigned int ns = 0, ntie = 0;
    constexpr int kCU = kOcc == 1 ? 4 : 2;  // steps in flight (2 x 16-B loads each)
    for (int64_t tb = w_lo; tb < w_hi; tb += kCU * 256) {
      float v[kCU][8];
#pragma unroll
      for (int k = 0; k < kCU; ++k) load8(tb + k * 256 + lane * 8, v[k]);
#pragma unroll
      for (int k = 0; k < kCU; ++k)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (tb + k * 256 + lane * 8 + u < w_hi) {
            const uint32_t dl = (uint32_t)(M - zint(v[k][u]));
            ns += dl < delta_star;
            ntie += dl == delta_star;
          }
        }
    }
    ns = __reduce_add_sync(0xffffffffu, ns);
    ntie = __reduce_add_sync(0xffffffffu, ntie);
    if (lane == 0) { s_ws[warp] = ns; s_wt[warp] = ntie; }
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long a0 = 0, a1 = 0;
    for (int w = 0; w < kFT / 32; ++w) {
      const unsigned long long x0 = s_ws[w], x1 = s_wt[w];
      s_ws[w] = a0;  // exclusive prefix within the CTA
      s_wt[w] = a1;
      a0 += x0;
      a1 += x1;
    }
    slot.ns = a0;
    slot.nt = a1;
  }
  cl.sync();
  unsigned long long s_before = 0, t_before = 0;
  for (int r = 0; r < rank; ++r) {
    const Slot *o = cl.map_shared_rank(&slot, r);
    s_before += o->ns;
    t_before += o->nt;
  }
  const unsigned long long cta_s = slot.ns, cta_t = slot.nt;
  // weight W_j / denom in fp32: W has <= 24 significant bits (exact in fp32), one rounding
  // of 1/denom -> relative error < 2^-23
  const float inv_den = (float)(1.0 / (s.renorm ? (double)selmass : (double)S));
  int32_t *oi = s.sel_idx + (int64_t)row * s.k_max;
  float *ow = s.sel_w + (int64_t)row * s.k_max;
  const unsigned long long sel_begin = s_before + (t_before < r_ties ? t_before : r_ties);
  const unsigned long long sel_end =
      s_before + cta_s + (t_before + cta_t < r_ties ? t_before + cta_t : r_ties);
  const unsigned long long sel_count = sel_end - sel_begin;
  {
    unsigned long long t_run = t_before + s_wt[warp];                      // ties before
    unsigned long long pos = s_before + s_ws[warp] + (t_run < r_ties ? t_run : r_ties);
    // staging slice of this warp (in the P1 mass bins, free after P2): 256 x (Δ, offset in
    // the step) + one dump slot that absorbs the stores of tokens not kept (branch-free)
    uint32_t *stg_d = reinterpret_cast<uint32_t *>(smem) + warp * 257;
    uint16_t *stg_o = reinterpret_cast<uint16_t *>(reinterpret_cast<uint32_t *>(smem) + (kFT / 32) * 257) + warp * 257;
    float vn[8], vnn[8];  // two steps prefetched
    if (w_lo < w_hi) load8(w_lo + lane * 8, vn);
    if (w_lo + 256 < w_hi) load8(w_lo + 256 + lane * 8, vnn);
    for (int64_t tb = w_lo; tb < w_hi; tb += 256) {
      const int64_t t0 = tb + lane * 8;
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { v[u] = vn[u]; vn[u] = vnn[u]; }
      if (tb + 512 < w_hi) load8(t0 + 512, vnn);
      uint32_t dl[8];
      unsigned nst = 0, ntie = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = t0 + u < w_hi;
        dl[u] = ok ? (uint32_t)(M - zint(v[u])) : 0xffffffffu;
        nst += ok && dl[u] < delta_star;
        ntie += ok && dl[u] == delta_star;
      }
      // exclusive warp scans: ties before this lane, then kept before this lane
      unsigned tie_pre = ntie;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, tie_pre, off);
        if (lane >= off) tie_pre += o;
      }
      const unsigned tie_tot = __shfl_sync(0xffffffffu, tie_pre, 31);
      tie_pre -= ntie;
      const unsigned long long my_t0 = t_run + tie_pre;
      const unsigned taken = my_t0 >= r_ties ? 0u
                             : (unsigned)((r_ties - my_t0) < ntie ? (r_ties - my_t0) : ntie);
      unsigned kpre = nst + taken;
      const unsigned kept = kpre;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, kpre, off);
        if (lane >= off) kpre += o;
      }
      const unsigned kept_tot = __shfl_sync(0xffffffffu, kpre, 31);
      // stage the step's kept (Δ, token) in this warp's shared slice, then write them
      // lane-parallel: one weight per lane instead of 8 divergent ones, coalesced stores
      unsigned q = kpre - kept;
      unsigned ties_seen = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool is_tie = dl[u] == delta_star && t0 + u < w_hi;
        const bool take = dl[u] < delta_star || (is_tie && ties_seen < taken);
        ties_seen += is_tie ? 1u : 0u;
        const unsigned slot = take ? q : 256u;
        stg_d[slot] = dl[u];
        stg_o[slot] = (uint16_t)(lane * 8 + u);
        q += take ? 1u : 0u;
      }
      __syncwarp();
      for (unsigned i = lane; i < kept_tot; i += 32) {
        oi[pos + i] = (int32_t)(j0 + tb + stg_o[i]);
        ow[pos + i] = __fmul_rn((float)mass_d(stg_d[i], kappa), inv_den);
      }
      __syncwarp();
      pos += kept_tot;
      t_run += tie_tot;
    }
  }
  if (rank == 0 && tid == 0) {
    hs->M = M;
    hs->zmin = zmin;
    hs->shift = shift;
    hs->bstar = bstar;
    hs->S = S;
    hs->theta = theta;
    hs->delta_star = delta_star;
    hs->r_ties = (uint32_t)r_ties;
    hs->ksel = (int64_t)ksel;
    hs->kstar = kstar;
    hs->sel_mass = selmass;
    if (s.sel_k) s.sel_k[row] = (int64_t)ksel;
  }
  if (!kG || !do_gather || stop == 4) {
    cl.sync();  // peers may still read my slot (P3 prefix) through DSMEM
    return;
  }
  // ---------------------------------------------------------------- P4: gather (Eq. 5)
  __syncthreads();  // this CTA's sel_idx / sel_w writes are visible to its own threads
  const int b = row / la.Hq, hq = row - b * la.Hq, kv = hq / la.G;
  const int lpr = la.d >> 3;           // lanes per row (16 at d = 128)
  const int rpw = 32 / lpr;
  const int nslots = (kFT / 32) * rpw;
  const int gslot = (tid >> 5) * rpw + lane / lpr;
  const int sub = lane % lpr;
  const uint16_t *Vb = la.V + (int64_t)b * la.v_b_stride + (int64_t)kv * la.v_kv_stride;
  const uint16_t *Rb = la.res_v + (int64_t)b * la.res_b_stride + (int64_t)kv * la.res_cap * la.d;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
  const int64_t r0 = (int64_t)sel_begin, r1 = (int64_t)(sel_begin + sel_count);
  // HBM values: half-warp per 256-B row, 16-B cp.async (LDGSTS, L1-bypassing) into a
  // per-thread 2-stage shared-memory ring: stage k+1's kGU rows are in flight while stage k
  // is consumed (each thread reads back only its own copies: no barrier), doubling the rows
  // in flight per SM without registers.
  if (stop != 5 && la.v_placement == 0) {
    int32_t jn[kGU], jc[kGU];
    float wn[kGU], wc[kGU];
    const int64_t step = (int64_t)nslots * kGU;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem);
    auto src_of = [&](int64_t j) -> const uint16_t * {
      if (j < la.n_q) return Vb + j * la.d;
      const uint32_t sl = (uint32_t)(la.res_slot0 + (j - la.n_q)) % (uint32_t)la.res_cap;
      return Rb + (int64_t)sl * la.d;
    };
    auto issue = [&](int stage, const int32_t (&jj)[kGU]) {
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        if (jj[u] >= 0) {
          const uint32_t dst = ring + (uint32_t)(((stage * kGU + u) * kFT + tid) * 16);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                       "l"(src_of(jj[u]) + sub * 8)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    __syncthreads();  // the ring overwrites the histogram / z-cache space
    int64_t r = r0 + gslot;
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      const int64_t rr = r + (int64_t)u * nslots;
      jc[u] = rr < r1 ? oi[rr] : -1;
      wc[u] = rr < r1 ? ow[rr] : 0.0f;
    }
    issue(0, jc);
    int stage = 0;
    for (; r < r1; r += step) {
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        const int64_t rr = r + step + (int64_t)u * nslots;
        jn[u] = rr < r1 ? oi[rr] : -1;
        wn[u] = rr < r1 ? ow[rr] : 0.0f;
      }
      issue(stage ^ 1, jn);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        if (jc[u] >= 0) {
          const uint4 v = *reinterpret_cast<const uint4 *>(smem + ((stage * kGU + u) * kFT + tid) * 16);
          fma8(acc, wc[u], v);
        }
        jc[u] = jn[u];
        wc[u] = wn[u];
      }
      stage ^= 1;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  // host-mapped values: half-warp per 256-B row (16 x 16-B L1-bypassing zero-copy loads
  // over the host link), software-pipelined: the (index, weight) batch of round k+1 is
  // loaded while round k's rows are in flight
  if (stop != 5 && la.v_placement != 0) {
    int32_t jn[kGU];
    float wn[kGU];
    const int64_t step = (int64_t)nslots * kGU;
    int64_t r = r0 + gslot;
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      const int64_t rr = r + (int64_t)u * nslots;
      jn[u] = rr < r1 ? oi[rr] : -1;
      wn[u] = rr < r1 ? ow[rr] : 0.0f;
    }
    for (; r < r1; r += step) {
      uint4 v[kGU];
      float w[kGU];
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        const int64_t j = jn[u];
        w[u] = wn[u];
        if (j >= 0) {
          const uint16_t *src;
          if (j < la.n_q) {
            src = Vb + j * la.d;
          } else {  // resident window slot (rare): 32-bit modulo
            const uint32_t slot_ = (uint32_t)(la.res_slot0 + (j - la.n_q)) % (uint32_t)la.res_cap;
            src = Rb + (int64_t)slot_ * la.d;
          }
          v[u] = ld_nc16(src + sub * 8);
        } else {
          v[u] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        const int64_t rr = r + step + (int64_t)u * nslots;
        jn[u] = rr < r1 ? oi[rr] : -1;
        wn[u] = rr < r1 ? ow[rr] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kGU; ++u) fma8(acc, w[u], v[u]);
    }
  }
  // CTA partial: slots -> d floats (fixed order), kept in shared memory for the cluster
  float *part = reinterpret_cast<float *>(cnt);  // reuse the histogram space (>= d floats)
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 8; ++e) s_red[gslot * la.d + sub * 8 + e] = acc[e];
  __syncthreads();
  for (int e = tid; e < la.d; e += kFT) {
    float sum = 0.0f;
    for (int q = 0; q < nslots; ++q) sum += s_red[q * la.d + e];
    part[e] = sum;
  }
  cl.sync();
  if (rank == 0) {
    for (int e = tid; e < la.d; e += kFT) {
      float sum = 0.0f;
      for (int r = 0; r < cs; ++r) sum += cl.map_shared_rank(part, r)[e];
      la.out[(int64_t)row * la.d + e] = sum;
    }
  }
  cl.sync();  // keep peers' shared memory alive until rank 0 has read it
}

cudaError_t launch_select_fused(const SelArgs &s, const LayerArgs &la, int nsplit, int do_gather,
                                int num_sms, cudaStream_t st) {
  const size_t ring = (size_t)2 * kGU * kFT * 16;  // cp.async gather ring (HBM values)
  auto smem_of = [&](int cs_, int *zc) {
    const int64_t per = ((s.n + cs_ - 1) / cs_ + 15) / 16 * 16;
    *zc = per <= kZCacheMax ? 1 : 0;
    size_t sm = (size_t)kNB * 12 + (*zc ? (size_t)per * 4 : 0);
    if (do_gather && la.v_placement == 0 && sm < ring) sm = ring;
    return sm;
  };
  // CTAs resident per SM: 1 with the gather (128 registers), else 2 if shared memory allows
  auto occ_of = [&](size_t sm) { return (!do_gather && sm <= 110 * 1024) ? 2 : 1; };
  int cs = 1, zcache = 0, occ = 1;
  while (cs < 8 && s.n / (cs * 2) >= 1024) {
    int zc2 = 0;
    const size_t sm2 = smem_of(cs * 2, &zc2);
    // a second CTA per SM only pays for long rows (latency of the phase barriers otherwise)
    const int o2 = s.n / (cs * 2) >= 32768 ? occ_of(sm2) : 1;
    if ((int64_t)s.rows * cs * 2 > (int64_t)num_sms * o2) break;
    cs *= 2;
    occ = (int64_t)s.rows * cs > num_sms ? 2 : 1;
  }
  const size_t smem = smem_of(cs, &zcache);
  static int configured[64][3] = {{0}};
  int dev = 0;
  cudaGetDevice(&dev);
  const int vi = do_gather ? 0 : occ;  // 0: gather, 1: select 1 CTA/SM, 2: select 2 CTAs/SM
  auto fn = vi == 0 ? k_select_fused<true, 1> : vi == 1 ? k_select_fused<false, 1> : k_select_fused<false, 2>;
  if (dev >= 0 && dev < 64 && !configured[dev][vi]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kNB * 12 + kZCacheMax * 4));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    (void)e;
    configured[dev][vi] = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(s.rows * cs));
  cfg.blockDim = dim3(kFT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  static int stop_env = -1;
  if (stop_env < 0) {
    const char *ev = getenv("HC_SEL_STOP");
    stop_env = ev ? atoi(ev) : 0;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, s, la, cs, nsplit, zcache, do_gather, stop_env);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace hc
