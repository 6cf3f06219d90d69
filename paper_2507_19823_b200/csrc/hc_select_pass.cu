// hc_select_pass.cu -- rows a3 + a4 of the decode step: the softmax mass (R4, PAPER.md
// P:236 "ã = softmax(z̃/√d)") and Eq. 4's cumulative-mass cut with the k_max cap (R5,
// P:240-252), as three bandwidth-shaped passes over the scores z instead of one cluster of
// CTAs per row (the round-1 k_select_fused: 3-4 passes, 2-3 shared atomics per token).
//
//   K1 k_sel_mass    every token: W = mass(Δ), Δ = M - z (M folded by the scan epilogue)
//                    -> the exact total S (u64 in registers, one global atomic per CTA) and a
//                    COUNT-only coarse histogram of Δ >> shift (one shared atomic per token).
//                    The row's last CTA bounds the prefix mass of every coarse bin from the
//                    exact counts and W's monotonicity in Δ (W at the bin's two ends, widened
//                    by a slack that covers the exp2 polynomial's rounding), and keeps the
//                    range of bins the exact cut can fall in (plus the k_max cap's bin, from
//                    exact counts).  shift == 0 (bins = exact Δ values) resolves right there.
//   K2 k_sel_refine  the exact mass of every token above that range (P_above) and exact
//                    counts (exact masses too if the range spans more than kNB values) of
//                    the tokens inside it; the last CTA walks them to the exact Δ*, the
//                    number r of Δ* ties kept (lowest indices), k_sel, k*, the kept mass --
//                    or, for a wide range, narrows it to one fine bin for a second K2
//                    launch (a no-op when the first resolved).
//   K3 k_sel_compact single-pass ordered compaction: CTAs take per-row chunk tickets in
//                    order and chain (strict, tie) counts by decoupled look-back, so every
//                    kept token's output position (ascending index) is known in one pass;
//                    the kept (index, W/S) pairs are staged in shared memory and written
//                    coalesced.
//
// Every decision is integer arithmetic on exact quantities (counts, u64 masses, the
// 128-bit threshold Θ), so the kept set equals the oracle's bit for bit (or_select: sort by
// (Δ asc, index asc), prefix to Θ, cap) -- the bounds only choose WHERE to look.
#include "hc_internal.h"

namespace hc {

constexpr int kST = 512;             // threads per CTA (all three kernels)
constexpr int kBPT = kNB / kST;      // histogram bins per thread in the block-wide walks (8)
constexpr uint32_t kStRefine1 = 1, kStRefine2 = 2, kStDone = 3, kStError = 4;

__device__ __forceinline__ uint64_t wmass(uint32_t dl, float kappa) {
  uint32_t lo, hi;
  mass_parts(dl, kappa, lo, hi);  // == mass_d(dl, kappa), branch-free
  return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ int sel_shift(int M, int zmin) {
  const uint32_t dmax = (uint32_t)(M - zmin);
  const int bits = 32 - __clz(dmax);
  return bits > kNBBits ? bits - kNBBits : 0;
}

__device__ __forceinline__ unsigned long long shfl_u64_up(unsigned long long v, int off) {
  const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, off);
  const uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), off);
  return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, off);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), off);
    v += ((unsigned long long)hi << 32) | lo;
  }
  return v;
}

// block-wide exclusive scan of up to three u64 values per thread (kST threads); tot = totals
template <int K>
__device__ __forceinline__ void bscan(unsigned long long (&x)[K], unsigned long long (&tot)[K],
                                      unsigned long long (*sw)[kST / 32]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long inc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) inc[k] = x[k];
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const unsigned long long o = shfl_u64_up(inc[k], off);
      if (lane >= off) inc[k] += o;
    }
  }
  __syncthreads();
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < K; ++k) sw[k][w] = inc[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    unsigned long long before = 0, t = 0;
    for (int q = 0; q < kST / 32; ++q) {
      const unsigned long long v = sw[k][q];
      if (q < w) before += v;
      t += v;
    }
    tot[k] = t;
    x[k] = before + inc[k] - x[k];
  }
}

// visit the row's tokens [j0, j1) of this CTA, 4 consecutive per thread per round, 4 rounds
// of 16-B loads in flight (z rows are 64-float aligned, j0 % 4 == 0)
template <typename F>
__device__ __forceinline__ void sel_tokens(const float *zr, int64_t j0, int64_t j1, F &&f) {
  const int64_t j14 = j0 + ((j1 - j0) & ~(int64_t)3);
  for (int64_t base = j0 + (int64_t)threadIdx.x * 4; base < j14; base += (int64_t)kST * 16) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t t = base + (int64_t)u * kST * 4;
      v[u] = t < j14 ? *reinterpret_cast<const float4 *>(zr + t) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (base + (int64_t)u * kST * 4 < j14) { f(v[u].x); f(v[u].y); f(v[u].z); f(v[u].w); }
    }
  }
  for (int64_t t = j14 + threadIdx.x; t < j1; t += kST) f(zr[t]);
}

// Resolve the cut exactly over consecutive Δ values base .. base + kNB - 1 whose counts are
// cnt[] (shared) and whose per-token mass is W(base + b) -- or, if `mass` is given, whose
// per-bin exact masses are mass[] and bin b spans Δ in [base + (b << f), base + ((b+1) << f)).
// cc0 / cm0 = count / exact mass of every candidate with Δ below base.  Called by a whole CTA;
// the thread that finds the cut writes the row's state.
__device__ void resolve_bins(const uint32_t *cnt, const unsigned long long *mass, int f, uint32_t base,
                             uint32_t top, unsigned long long cc0, unsigned long long cm0,
                             const SelArgs &s, HeadState *hs, int row, float kappa,
                             unsigned long long theta, bool tau_all, bool cap_all,
                             unsigned long long S, int *s_found) {
  __shared__ unsigned long long sw[2][kST / 32];
  const int t = threadIdx.x;
  unsigned long long c8[kBPT], m8[kBPT];
  unsigned long long x[2] = {0, 0}, tot[2];
#pragma unroll
  for (int k = 0; k < kBPT; ++k) {
    const int b = t * kBPT + k;
    const uint32_t dl = base + ((uint32_t)b << f);
    c8[k] = dl <= top ? cnt[b] : 0u;
    m8[k] = mass ? mass[b] : (c8[k] ? c8[k] * wmass(dl, kappa) : 0ull);
    x[0] += c8[k];
    x[1] += m8[k];
  }
  if (t == 0) *s_found = kNB;
  bscan<2>(x, tot, sw);
  unsigned long long cc = cc0 + x[0], cm = cm0 + x[1];
  int found = kNB;
  unsigned long long fcc = 0, fcm = 0, fc = 0, fm = 0;
#pragma unroll
  for (int k = 0; k < kBPT; ++k) {
    const bool trig = c8[k] && ((!tau_all && cm + m8[k] >= theta) || (!cap_all && cc + c8[k] >= (unsigned long long)s.k_max));
    if (trig && found == kNB) { found = t * kBPT + k; fcc = cc; fcm = cm; fc = c8[k]; fm = m8[k]; }
    cc += c8[k];
    cm += m8[k];
  }
  if (found < kNB) atomicMin(s_found, found);
  __syncthreads();
  const int fb = *s_found;
  if (fb == kNB) {  // the bounds promised the cut in this range: never reached
    if (t == 0) hs->state = kStError;
    return;
  }
  if (found != fb) return;
  const uint32_t dlo = base + ((uint32_t)fb << f);
  if (f > 0) {  // narrow to this fine bin: exact counts / mass before it are known
    hs->r_lo = dlo;
    hs->r_hi = min(dlo + ((1u << f) - 1u), top);
    hs->fshift = 0;
    hs->cnt_before = (uint32_t)fcc;
    hs->mass_before = fcm;
    hs->state = kStRefine2;
    return;
  }
  const unsigned long long w = wmass(dlo, kappa);
  unsigned long long r_tau = ~0ull, r_cap = ~0ull;
  if (!tau_all && fcm + fm >= theta) r_tau = fcm >= theta ? 1ull : (theta - fcm + w - 1) / w;
  if (r_tau == 0) r_tau = 1;
  if (!cap_all && fcc + fc >= (unsigned long long)s.k_max) r_cap = (unsigned long long)s.k_max - fcc;
  const unsigned long long r = r_tau < r_cap ? r_tau : r_cap;
  hs->delta_star = dlo;
  hs->r_ties = (uint32_t)r;
  hs->ksel = (int64_t)(fcc + r);
  hs->kstar = r_tau <= r_cap ? (int64_t)(fcc + r_tau) : -1;
  hs->sel_mass = fcm + r * w;
  hs->theta = theta;
  if (s.sel_k) s.sel_k[row] = (int64_t)(fcc + r);
  __threadfence();
  hs->state = kStDone;
}

// ---------------------------------------------------------------------------- K0 (split scans)
// group-split scans accumulate z with atomics and fold no max / min: one pass for them
__global__ void __launch_bounds__(kST) k_sel_minmax(SelArgs s, int64_t per) {
  const int row = blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(s.n, j0 + per);
  int mx = INT_MIN, mn = INT_MAX;
  sel_tokens(s.z + (int64_t)row * s.z_stride, j0, j1, [&](float zf) {
    const int zi = zint(zf);
    mx = max(mx, zi);
    mn = min(mn, zi);
  });
  mx = __reduce_max_sync(0xffffffffu, mx);
  mn = __reduce_min_sync(0xffffffffu, mn);
  if ((threadIdx.x & 31) == 0 && mx != INT_MIN) {
    atomicMax(&s.hs[row].M, mx);
    atomicMin(&s.hs[row].zmin, mn);
  }
}

// ---------------------------------------------------------------------------- K1
__global__ void __launch_bounds__(kST, 2) k_sel_mass(SelArgs s, int64_t per) {
  __shared__ uint32_t hist[kNB];
  __shared__ unsigned long long s_red[kST / 32];
  __shared__ bool s_last;
  __shared__ int s_found;
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y, t = threadIdx.x;
  HeadState *hs = s.hs + row;
  const int M = hs->M, zmin = hs->zmin;
  const float kappa = hs->kappa;
  const int shift = sel_shift(M, zmin);
  const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(s.n, j0 + per);
  for (int i = t; i < kNB; i += kST) hist[i] = 0u;
  {  // this CTA's share of the row's refine histograms and look-back words (used by K2 / K3)
    const int64_t nf = (int64_t)kNB, nl = s.lb_n;
    const int64_t f0 = nf * blockIdx.x / gridDim.x, f1 = nf * (blockIdx.x + 1) / gridDim.x;
    for (int64_t i = f0 + t; i < f1; i += kST) {
      s.fcnt[(int64_t)row * kNB + i] = 0u;
      s.fmass[(int64_t)row * kNB + i] = 0ull;
    }
    const int64_t l0 = nl * blockIdx.x / gridDim.x, l1 = nl * (blockIdx.x + 1) / gridDim.x;
    for (int64_t i = l0 + t; i < l1; i += kST) s.lb[(int64_t)row * nl + i] = 0ull;
  }
  __syncthreads();
  unsigned long long S = 0;
  sel_tokens(s.z + (int64_t)row * s.z_stride, j0, j1, [&](float zf) {
    const uint32_t dl = (uint32_t)(M - zint(zf));
    S += wmass(dl, kappa);
    atomicAdd(&hist[dl >> shift], 1u);
  });
  S = warp_sum_u64(S);
  if ((t & 31) == 0) s_red[t >> 5] = S;
  __syncthreads();
  if (t == 0) {
    unsigned long long tot = 0;
    for (int w = 0; w < kST / 32; ++w) tot += s_red[w];
    if (tot) atomicAdd((unsigned long long *)&hs->S, tot);
  }
  uint32_t *gh = s.ghist + (int64_t)row * kNB;
  for (int i = t; i < kNB; i += kST) {
    const uint32_t c = hist[i];
    if (c) atomicAdd(&gh[i], c);
  }
  __threadfence();
  __syncthreads();
  if (t == 0) {
    const uint32_t prev = atomicAdd(&hs->c1_done, 1u);
    s_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // ---- the row's last CTA: exact counts, exact S, mass bounds per coarse bin
  const unsigned long long Sx = __ldcg((const unsigned long long *)&hs->S);
  const uint32_t dmax = (uint32_t)(M - zmin);
  const bool tau_all = s.tau_q >= (1u << 24);
  const unsigned long long theta = tau_all ? 0ull : threshold(s.tau_q, Sx);
  const unsigned long long ntot = (unsigned long long)s.n;
  const bool cap_all = (unsigned long long)s.k_max >= ntot;
  for (int i = t; i < kNB; i += kST) hist[i] = __ldcg(&gh[i]);
  if (t == 0) {
    hs->c1_done = 0u;
    hs->shift = shift;
    hs->theta = theta;
    hs->ticket = 0u;
  }
  __syncthreads();
  if (tau_all && cap_all) {  // everything is kept
    if (t == 0) {
      hs->delta_star = 0xffffffffu;
      hs->r_ties = 0u;
      hs->ksel = (int64_t)ntot;
      hs->kstar = (int64_t)ntot;
      hs->sel_mass = Sx;
      if (s.sel_k) s.sel_k[row] = (int64_t)ntot;
      __threadfence();
      hs->state = kStDone;
    }
    return;
  }
  if (shift == 0) {  // coarse bins are exact Δ values: exact masses from the counts
    if (t == 0) hs->mass_before = 0ull;
    resolve_bins(hist, nullptr, 0, 0u, dmax, 0ull, 0ull, s, hs, row, kappa, theta, tau_all, cap_all, Sx,
                 &s_found);
    return;
  }
  __shared__ unsigned long long sw[3][kST / 32];
  __shared__ int s_ba, s_bb, s_bcap;
  // per coarse bin b (Δ in [d0, d1]): count c and mass bounds c*W_lo <= mass <= c*W_hi.  W is
  // non-increasing in Δ up to the polynomial's rounding (rel. 2^-22) and the truncation: the
  // bounds are widened by 2^-20 relative + 2 so they hold for every Δ of the bin
  auto bin = [&](int k, uint32_t &c, unsigned long long &lo, unsigned long long &hi) {
    const uint32_t b = (uint32_t)(t * kBPT + k);
    const uint32_t d0 = b << shift;
    c = d0 <= dmax ? hist[b] : 0u;
    lo = hi = 0ull;
    if (c) {
      const uint32_t d1 = min(d0 + ((1u << shift) - 1u), dmax);
      const unsigned long long wh = wmass(d0, kappa), wl = wmass(d1, kappa);
      hi = c * (wh + (wh >> 20) + 2ull);
      lo = c * (wl > (wl >> 20) + 2ull ? wl - (wl >> 20) - 2ull : 0ull);
    }
  };
  unsigned long long x[3] = {0, 0, 0}, tot[3];
#pragma unroll 1
  for (int k = 0; k < kBPT; ++k) {
    uint32_t c;
    unsigned long long lo, hi;
    bin(k, c, lo, hi);
    x[0] += c;
    x[1] += lo;
    x[2] += hi;
  }
  if (t == 0) { s_ba = kNB; s_bb = -1; s_bcap = kNB; }
  bscan<3>(x, tot, sw);
  {
    unsigned long long C = x[0], Lm = x[1], Um = x[2];
    int ba = kNB, bb = -1, bcap = kNB;
#pragma unroll 1
    for (int k = 0; k < kBPT; ++k) {
      const int b = t * kBPT + k;
      uint32_t c;
      unsigned long long lo, hi;
      bin(k, c, lo, hi);
      if (c) {
        if (!tau_all && ba == kNB && Um + hi >= theta) ba = b;   // first bin the cut may end in
        if (!tau_all && Lm < theta) bb = b;                       // last bin it may end in
        if (!cap_all && bcap == kNB && C + c >= (unsigned long long)s.k_max) bcap = b;
      }
      C += c;
      Lm += lo;
      Um += hi;
    }
    if (ba < kNB) atomicMin(&s_ba, ba);
    if (bb >= 0) atomicMax(&s_bb, bb);
    if (bcap < kNB) atomicMin(&s_bcap, bcap);
  }
  __syncthreads();
  int lo_b, hi_b;
  if (tau_all) {
    lo_b = hi_b = s_bcap;
  } else if (s_bcap < s_ba) {  // the cap binds before the mass can reach Θ
    lo_b = hi_b = s_bcap;
  } else {
    lo_b = s_ba;
    hi_b = s_bb < lo_b ? lo_b : s_bb;
    if (s_bcap < hi_b) hi_b = s_bcap;
  }
  if (lo_b >= kNB) {  // cannot happen: Θ <= S and k_max < n are always reached
    if (t == 0) hs->state = kStError;
    return;
  }
  // the count before the range (exact): the owner of bin lo_b has it
  if (lo_b / kBPT == t) {
    unsigned long long C = x[0];
    for (int k = 0; k < lo_b % kBPT; ++k) C += hist[t * kBPT + k];
    const uint32_t rlo = (uint32_t)lo_b << shift;
    const uint32_t rhi = min(((uint32_t)(hi_b + 1) << shift) - 1u, dmax);
    int f = 0;
    while (((rhi - rlo) >> f) >= (uint32_t)kNB) ++f;
    hs->cnt_before = (uint32_t)C;
    hs->mass_before = 0ull;  // K2's first pass accumulates the exact mass above the range
    hs->r_lo = rlo;
    hs->r_hi = rhi;
    hs->fshift = f;
    __threadfence();
    hs->state = kStRefine1;
  }
}

// ---------------------------------------------------------------------------- K2
__global__ void __launch_bounds__(kST) k_sel_refine(SelArgs s, int64_t per, int pass) {
  extern __shared__ __align__(16) uint8_t sm2[];
  uint32_t *fc = reinterpret_cast<uint32_t *>(sm2);                 // [kNB] fine counts
  uint32_t *fml = reinterpret_cast<uint32_t *>(sm2 + kNB * 4);      // [kNB] fine mass, low word
  uint32_t *fmh = reinterpret_cast<uint32_t *>(sm2 + kNB * 8);      // [kNB] high word
  unsigned long long *s_mass = reinterpret_cast<unsigned long long *>(sm2 + kNB * 4);  // resolve: over fml/fmh
  __shared__ unsigned long long s_red[kST / 32];
  __shared__ bool s_last;
  __shared__ int s_found;
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y, t = threadIdx.x;
  HeadState *hs = s.hs + row;
  if (hs->state != (pass == 0 ? kStRefine1 : kStRefine2)) return;
  const int M = hs->M;
  const float kappa = hs->kappa;
  const uint32_t lo = hs->r_lo, hi = hs->r_hi;
  const int f = hs->fshift;
  const bool first = pass == 0;
  const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(s.n, j0 + per);
  for (int i = t; i < kNB; i += kST) { fc[i] = 0u; fml[i] = 0u; fmh[i] = 0u; }
  __syncthreads();
  unsigned long long P = 0;
  sel_tokens(s.z + (int64_t)row * s.z_stride, j0, j1, [&](float zf) {
    const uint32_t dl = (uint32_t)(M - zint(zf));
    if (dl < lo) {
      if (first) P += wmass(dl, kappa);
    } else if (dl <= hi) {
      const uint32_t fb = (dl - lo) >> f;
      atomicAdd(&fc[fb], 1u);
      if (f > 0) {  // fine bins of several Δ values: their exact mass too
        uint32_t wl, wh;
        mass_parts(dl, kappa, wl, wh);
        const uint32_t old = atomicAdd(&fml[fb], wl);
        wh += (old + wl < old) ? 1u : 0u;
        if (wh) atomicAdd(&fmh[fb], wh);
      }
    }
  });
  if (first) {
    P = warp_sum_u64(P);
    if ((t & 31) == 0) s_red[t >> 5] = P;
  }
  __syncthreads();
  if (first && t == 0) {
    unsigned long long tot = 0;
    for (int w = 0; w < kST / 32; ++w) tot += s_red[w];
    if (tot) atomicAdd((unsigned long long *)&hs->mass_before, tot);
  }
  uint32_t *gc = s.fcnt + (int64_t)row * kNB;
  unsigned long long *gm = s.fmass + (int64_t)row * kNB;
  for (int i = t; i < kNB; i += kST) {
    const uint32_t c = fc[i];
    if (c) {
      atomicAdd(&gc[i], c);
      if (f > 0) atomicAdd(&gm[i], ((unsigned long long)fmh[i] << 32) + fml[i]);
    }
  }
  __threadfence();
  __syncthreads();
  if (t == 0) {
    const uint32_t prev = atomicAdd(&hs->c2_done, 1u);
    s_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // ---- the row's last CTA: walk the fine bins to the exact cut
  __syncthreads();  // (s_mass overlays fml / fmh)
  for (int i = t; i < kNB; i += kST) {
    fc[i] = __ldcg(&gc[i]);
    s_mass[i] = f > 0 ? __ldcg(&gm[i]) : 0ull;
  }
  if (t == 0) hs->c2_done = 0u;
  __syncthreads();
  // the histograms are read: clear them for a second pass / the next call
  for (int i = t; i < kNB; i += kST) { gc[i] = 0u; gm[i] = 0ull; }
  const unsigned long long Sx = hs->S, theta = hs->theta;
  const bool tau_all = s.tau_q >= (1u << 24);
  const bool cap_all = (unsigned long long)s.k_max >= (unsigned long long)s.n;
  const unsigned long long cc0 = hs->cnt_before, cm0 = __ldcg((const unsigned long long *)&hs->mass_before);
  resolve_bins(fc, f > 0 ? s_mass : nullptr, f, lo, hi, cc0, cm0, s, hs, row, kappa, theta, tau_all,
               cap_all, Sx, &s_found);
}

// ---------------------------------------------------------------------------- K3
// look-back word: [flag 2 bits (1 aggregate, 2 inclusive prefix)][strict 31][ties 31]
__device__ __forceinline__ unsigned long long lb_pack(uint32_t flag, uint32_t ns, uint32_t nt) {
  return ((unsigned long long)flag << 62) | ((unsigned long long)ns << 31) | nt;
}

template <int TPT>
__global__ void __launch_bounds__(kST) k_sel_compact(SelArgs s) {
  constexpr int kChunk = kST * TPT;
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t *stg_d = reinterpret_cast<uint32_t *>(sm);                // [kChunk] Δ of kept tokens
  uint16_t *stg_o = reinterpret_cast<uint16_t *>(sm + kChunk * 4);   // [kChunk] offset in chunk
  __shared__ unsigned long long sw[2][kST / 32];
  __shared__ int s_ticket;
  __shared__ unsigned long long s_pre;
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y, t = threadIdx.x, lane = t & 31;
  HeadState *hs = s.hs + row;
  if (t == 0) s_ticket = (int)atomicAdd(&hs->ticket, 1u);
  __syncthreads();
  const int c = s_ticket;
  if (hs->state != kStDone) return;  // (an error state writes nothing: sel_k stays unset)
  const int M = hs->M;
  const float kappa = hs->kappa;
  const uint32_t dstar = hs->delta_star;
  const unsigned long long r = hs->r_ties;
  const int64_t j0 = (int64_t)c * kChunk, j1 = min(s.n, j0 + kChunk);
  const float *zr = s.z + (int64_t)row * s.z_stride;
  // my TPT consecutive tokens
  uint32_t dl[TPT];
  const int64_t tb = j0 + (int64_t)t * TPT;
#pragma unroll
  for (int q = 0; q < TPT; q += 4) {
    float4 v = make_float4(0, 0, 0, 0);
    if (tb + q + 4 <= j1) {
      v = __ldcs(reinterpret_cast<const float4 *>(zr + tb + q));
    } else {
      if (tb + q < j1) v.x = zr[tb + q];
      if (tb + q + 1 < j1) v.y = zr[tb + q + 1];
      if (tb + q + 2 < j1) v.z = zr[tb + q + 2];
    }
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      dl[q + u] = tb + q + u < j1 ? (uint32_t)(M - zint(vv[u])) : 0xffffffffu;
  }
  unsigned long long x[2] = {0, 0}, tot[2];
#pragma unroll
  for (int q = 0; q < TPT; ++q) {
    x[0] += dl[q] < dstar;
    x[1] += (dl[q] == dstar && dstar != 0xffffffffu) ? 1u : 0u;
  }
  const unsigned long long my_s = x[0], my_t = x[1];
  bscan<2>(x, tot, sw);
  // decoupled look-back: publish the aggregate, sum predecessors back to an inclusive prefix
  unsigned long long *lbr = s.lb + (int64_t)row * s.lb_n;
  if (t < 32) {
    if (t == 0)
      st_relaxed_u64(&lbr[c], c == 0 ? lb_pack(2u, (uint32_t)tot[0], (uint32_t)tot[1])
                                     : lb_pack(1u, (uint32_t)tot[0], (uint32_t)tot[1]));
    unsigned long long ps = 0, pt = 0;
    int p = c - 1;
    while (p >= 0) {  // 32 predecessors per round, newest first
      const int q = p - lane;
      unsigned long long wv = 0;
      if (q >= 0) {
        do { wv = ld_relaxed_u64(&lbr[q]); } while ((wv >> 62) == 0ull);
      } else {
        wv = lb_pack(2u, 0u, 0u);
      }
      const unsigned incl = __ballot_sync(0xffffffffu, (wv >> 62) == 2ull);
      const int stop = incl ? __ffs(incl) - 1 : 32;  // the newest inclusive prefix
      unsigned long long vs = lane <= stop ? ((wv >> 31) & 0x7fffffffull) : 0ull;
      unsigned long long vt = lane <= stop ? (wv & 0x7fffffffull) : 0ull;
      vs = warp_sum_u64(vs);
      vt = warp_sum_u64(vt);
      ps += vs;
      pt += vt;
      if (incl) break;
      p -= 32;
    }
    if (t == 0) {
      if (c > 0) st_relaxed_u64(&lbr[c], lb_pack(2u, (uint32_t)(ps + tot[0]), (uint32_t)(pt + tot[1])));
      s_pre = (ps << 32) | pt;
    }
  }
  __syncthreads();
  const unsigned long long Sb = s_pre >> 32, Tb = s_pre & 0xffffffffull;
  // in-chunk positions: strict tokens always, ties while fewer than r precede them globally
  unsigned long long sb = Sb + x[0], tcount = Tb + x[1];
  const unsigned long long pos0 = Sb + (Tb < r ? Tb : r);  // first output slot of this chunk
  const unsigned long long pos_end = Sb + tot[0] + (Tb + tot[1] < r ? Tb + tot[1] : r);
  unsigned long long pos = sb + (tcount < r ? tcount : r);
#pragma unroll
  for (int q = 0; q < TPT; ++q) {
    const bool strict = dl[q] < dstar;
    const bool tie = dl[q] == dstar && dstar != 0xffffffffu;
    const bool take = strict || (tie && tcount < r);
    if (take) {
      const unsigned long long ls = pos - pos0;
      stg_d[ls] = dl[q];
      stg_o[ls] = (uint16_t)(t * TPT + q);
      ++pos;
    }
    tcount += tie ? 1u : 0u;
  }
  (void)my_s;
  (void)my_t;
  __syncthreads();
  const int kept = (int)(pos_end - pos0);
  const float inv_den = (float)(1.0 / (s.renorm ? (double)hs->sel_mass : (double)hs->S));
  int32_t *oi = s.sel_idx + (int64_t)row * s.k_max + pos0;
  float *ow = s.sel_w + (int64_t)row * s.k_max + pos0;
  for (int i = t; i < kept; i += kST) {
    oi[i] = (int32_t)(j0 + stg_o[i]);
    ow[i] = __fmul_rn((float)wmass(stg_d[i], kappa), inv_den);
  }
}

// ---------------------------------------------------------------------------- launcher
int select_lb_chunks(int64_t n) { return (int)((n + kST * 4 - 1) / (kST * 4)); }  // smallest chunk

cudaError_t launch_select(SelArgs s, int nsplit, int num_sms, cudaStream_t st) {
  if (s.rows <= 0 || s.n <= 0) return cudaSuccess;
  // K1 / K2 work split: about 3 CTAs per SM over all rows, >= 4096 tokens per CTA
  int64_t cpr = ((int64_t)num_sms * 3 + s.rows - 1) / s.rows;
  const int64_t max_cpr = (s.n + 4095) / 4096;
  if (cpr > max_cpr) cpr = max_cpr;
  if (cpr < 1) cpr = 1;
  int64_t per = (s.n + cpr - 1) / cpr;
  per = (per + 63) / 64 * 64;
  cpr = (s.n + per - 1) / per;
  const dim3 g12((unsigned)cpr, (unsigned)s.rows);
  // K3 chunk: 8192 tokens for long rows, 2048 when the rows are short
  const int tpt3 = (int64_t)s.rows * ((s.n + 8191) / 8192) >= 2LL * num_sms ? 16 : 4;
  const int64_t chunk3 = (int64_t)kST * tpt3;
  const int64_t nch3 = (s.n + chunk3 - 1) / chunk3;
  if (nch3 > s.lb_n) return cudaErrorInvalidValue;
  if (nsplit > 1) {
    launch_chain(k_sel_minmax, g12, dim3(kST), 0, st, s, per);
    note_launch();
  }
  launch_chain(k_sel_mass, g12, dim3(kST), 0, st, s, per);
  note_launch();
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaFuncSetAttribute(k_sel_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_sel_compact<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_sel_compact<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    configured[dev] = 1;
  }
  const size_t smem2 = (size_t)kNB * 12;
  launch_chain(k_sel_refine, g12, dim3(kST), smem2, st, s, per, 0);
  note_launch();
  launch_chain(k_sel_refine, g12, dim3(kST), smem2, st, s, per, 1);
  note_launch();
  const size_t smem3 = (size_t)chunk3 * 6;
  if (tpt3 == 16)
    launch_chain(k_sel_compact<16>, dim3((unsigned)nch3, (unsigned)s.rows), dim3(kST), smem3, st, s);
  else
    launch_chain(k_sel_compact<4>, dim3((unsigned)nch3, (unsigned)s.rows), dim3(kST), smem3, st, s);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
