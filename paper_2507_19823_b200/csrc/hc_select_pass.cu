// hc_select_pass.cu -- rows a3 + a4 of the decode step: the softmax mass (R4, PAPER.md
// P:236 "ã = softmax(z̃/√d)") and Eq. 4's cumulative-mass cut with the k_max cap (R5,
// P:240-252), as three bandwidth-shaped passes over the scores z instead of one cluster of
// CTAs per row (the round-1 k_select_fused: 3-4 passes, 2-3 shared atomics per token).
//
//   K1 k_sel_mass    every token: Δ = M - z (M folded by the scan epilogue), its exact mass W
//                    (R4; token pairs on the fp32x2 pipe, wmass2) -> an EXACT (count, mass)
//                    histogram of Δ >> shift (count + the u64 mass as two u32 words: three
//                    shared atomics per token).  The row's last CTA scans the exact bins: S, Θ =
//                    ceil(τ_q S / 2^24) and the one coarse bin the cut falls in (the first
//                    whose cumulative mass reaches Θ or whose cumulative count reaches k_max),
//                    with the exact count and mass before it.
//   K2 k_sel_refine  every token: Δ; per K3-chunk counts of the tokens before the cut bin, and
//                    the cut bin's tokens themselves (exact per-Δ counts + (index, Δ) on a
//                    per-row list); the last CTA walks the bin's <= 2^11 Δ values to the exact
//                    Δ*, the number r of Δ* ties kept (lowest indices), k_sel, k*, the kept
//                    mass, then every chunk's (strict, tie) counts and their exclusive prefix.
//   K4 k_sel_prefix  (rows of more than kFinishInK2 chunks) that finish, one CTA per row.
//   K3 k_sel_write   persistent CTAs over the (row, chunk) items: the chunk's kept tokens at
//                    their global positions (prefix + in-chunk scan), staged in shared memory
//                    and written coalesced as (index, W/S).  With values in HBM, K3G
//                    (k_sel_write_gather) also sums Eq. 5 over the kept rows as it emits them.
//   k_sel_small      rows of <= 64K candidates: all of the above in one cluster kernel per row.
// A row whose in-range list overflowed its capacity (heavy ties) is finished from a pass over
// its z instead -- slower, equally exact.
//
// Every decision is integer arithmetic on exact quantities (counts, u64 masses, the
// 128-bit threshold Θ), so the kept set equals the oracle's bit for bit (or_select: sort by
// (Δ asc, index asc), prefix to Θ, cap).
#include <cooperative_groups.h>

#include <type_traits>

#include "hc_internal.h"

namespace cg = cooperative_groups;

namespace hc {

constexpr int kST = 512;             // threads per CTA (all three kernels)
constexpr int kBPT = kNB / kST;      // histogram bins per thread in the block-wide walks (8)

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

// TMA-staged stream of one z row's chunks (kSelChunk tokens = 16 KB each) through NB shared
// buffers: chunk k+NB is requested (cp.async.bulk, one mbarrier per buffer) as soon as every
// thread is done with chunk k, so the HBM reads run ahead of the per-token work without
// registers.  In a chunk thread t owns tokens 4t + 2048u .. +3 (u = 0, 1): each LDS.128 of a
// warp reads 512 contiguous bytes (conflict-free).
template <int NB>
struct ZStream {
  float *buf;      // [NB][kSelChunk]
  uint64_t *bar;   // [NB] "full" barriers
  uint32_t *done;  // [NB] warps finished with the slot's chunk
  const float *zr;
  int64_t n;
  uint32_t ph;
  __device__ void init(float *b, uint64_t *br, uint32_t *dn, const float *z, int64_t n_) {
    buf = b; bar = br; done = dn; zr = z; n = n_; ph = 0u;
    if (threadIdx.x == 0) {
      for (int i = 0; i < NB; ++i) { mbar_init(&bar[i], 1); done[i] = 0u; }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  __device__ void request(int64_t c, int slot) {  // one thread
    const int64_t j0 = c * kSelChunk;
    const int64_t cnt = min((int64_t)kSelChunk, n - j0);
    const uint32_t bytes = (uint32_t)((cnt * 4 + 15) & ~(int64_t)15);  // z rows are padded to 64
    mbar_expect_tx(&bar[slot], bytes);
    bulk_g2s(buf + (size_t)slot * kSelChunk, zr + j0, bytes, &bar[slot]);
  }
  __device__ const float *wait(int slot) {
    mbar_wait(&bar[slot], (ph >> slot) & 1u);
    ph ^= 1u << slot;
    return buf + (size_t)slot * kSelChunk;
  }
  // a warp is done with `slot` (every value it read from it has been consumed); the last warp
  // out refills the slot with chunk c (c < 0: nothing left) -- no CTA-wide barrier, so warps
  // drift up to NB chunks apart
  __device__ void release(int64_t c, int slot) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      const uint32_t old = atomicAdd(&done[slot], 1u);
      if (old == blockDim.x / 32 - 1) {
        done[slot] = 0u;
        if (c >= 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads -> async write
          request(c, slot);
        }
      }
    }
  }
};

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
  pdl_trigger();
  pdl_wait();  // z is the scan's output
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
constexpr int kZB = 3;  // z stream buffers per CTA
constexpr int kZB2 = 5;  // z stream buffers of K2 (no mass histograms there: room for more in flight)
constexpr int64_t kFinishInK2 = kZB2 * kSelChunk / 2;  // chunks whose counters fit K2's z buffers

__global__ void __launch_bounds__(kST, 2) k_sel_mass(SelArgs s, int64_t per) {
  extern __shared__ __align__(128) uint8_t sm1[];
  float *zbuf = reinterpret_cast<float *>(sm1);                                 // [kZB][kSelChunk]
  uint32_t *mlo = reinterpret_cast<uint32_t *>(sm1 + kZB * kSelChunk * 4);      // [kNB] mass, low word
  uint32_t *mhi = mlo + kNB;                                                    // [kNB] high word
  unsigned long long *bmass = reinterpret_cast<unsigned long long *>(mlo);     // last CTA: [kNB] (overlay)
  __shared__ uint32_t hist[kNB];
  __shared__ uint64_t zbar[kZB];
  __shared__ uint32_t zdone[kZB];
  __shared__ bool s_last;
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y, t = threadIdx.x;
  HeadState *hs = s.hs + row;
  const int M = hs->M, zmin = hs->zmin;
  const float kappa = hs->kappa;
  const int shift = sel_shift(M, zmin);
  const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(s.n, j0 + per);
  for (int i = t; i < kNB; i += kST) { hist[i] = 0u; mlo[i] = 0u; mhi[i] = 0u; }
  {  // this CTA's share of the row's refine histograms and chunk counters (used by K2 / K4)
    const int64_t nf = (int64_t)kNB, nl = s.nch;
    const int64_t f0 = nf * blockIdx.x / gridDim.x, f1 = nf * (blockIdx.x + 1) / gridDim.x;
    for (int64_t i = f0 + t; i < f1; i += kST) s.fcnt[(int64_t)row * kNB + i] = 0u;
    const int64_t l0 = nl * blockIdx.x / gridDim.x, l1 = nl * (blockIdx.x + 1) / gridDim.x;
    for (int64_t i = l0 + t; i < l1; i += kST) s.cntlo[(int64_t)row * nl + i] = 0u;
  }
  ZStream<kZB> zs;
  zs.init(zbuf, zbar, zdone, s.z + (int64_t)row * s.z_stride, s.n);  // (its __syncthreads also covers the zeroing)
  const int64_t c0 = j0 / kSelChunk, c1 = (j1 + kSelChunk - 1) / kSelChunk;
  if (t == 0)
    for (int i = 0; i < kZB && c0 + i < c1; ++i) zs.request(c0 + i, i);
  for (int64_t c = c0; c < c1; ++c) {
    const int slot = (int)((c - c0) % kZB);
    const float *zc = zs.wait(slot);
    const int nv = (int)min((int64_t)kSelChunk, s.n - c * kSelChunk);
    auto body = [&](auto full) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i0 = 4 * t + 2048 * u;
        const float4 v = *reinterpret_cast<const float4 *>(zc + i0);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; e += 2) {  // token pairs: the mass on the packed fp32x2 pipe
          const uint32_t d0 = (uint32_t)(M - zint(vv[e])), d1 = (uint32_t)(M - zint(vv[e + 1]));
          uint64_t wp[2];
          wmass2(d0, d1, kappa, wp[0], wp[1]);
          const uint32_t dd[2] = {d0, d1};
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (decltype(full)::value || i0 + e + q < nv) {
              const uint32_t b = dd[q] >> shift;
              const uint32_t wl = (uint32_t)wp[q];
              uint32_t wh = (uint32_t)(wp[q] >> 32);
              atomicAdd(&hist[b], 1u);
              const uint32_t old = atomicAdd(&mlo[b], wl);  // exact u64 per bin: low word + carry
              wh += (old + wl < old) ? 1u : 0u;
              if (wh) atomicAdd(&mhi[b], wh);
            }
          }
        }
      }
    };
    if (nv == kSelChunk) body(std::true_type{}); else body(std::false_type{});
    zs.release(c + kZB < c1 ? c + kZB : -1, slot);
  }
  __syncthreads();  // every token counted into hist / mlo / mhi
  uint32_t *gh = s.ghist + (int64_t)row * kNB;
  unsigned long long *gm = s.gmass + (int64_t)row * kNB;
  for (int i = t; i < kNB; i += kST) {
    const uint32_t c = hist[i];
    if (c) {
      atomicAdd(&gh[i], c);
      atomicAdd(&gm[i], ((unsigned long long)mhi[i] << 32) + mlo[i]);
    }
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
  // ---- the row's last CTA: exact (count, mass) per coarse bin -> exact S, Θ and the one
  // coarse bin the cut falls in (the first whose cumulative mass reaches Θ or cumulative
  // count reaches k_max); K2 resolves it to the exact Δ* over its 2^shift values
  const uint32_t dmax = (uint32_t)(M - zmin);
  const unsigned long long ntot = (unsigned long long)s.n;
  const bool tau_all = s.tau_q >= (1u << 24);
  const bool cap_all = (unsigned long long)s.k_max >= ntot;
  for (int i = t; i < kNB; i += kST) {
    hist[i] = __ldcg(&gh[i]);
    bmass[i] = __ldcg(&gm[i]);
  }
  if (t == 0) {
    hs->c1_done = 0u;
    hs->shift = shift;
    hs->ticket = 0u;
  }
  __syncthreads();
  __shared__ unsigned long long sw[2][kST / 32];
  __shared__ int s_found;
  uint32_t c8[kBPT];
  unsigned long long m8[kBPT], x[2] = {0, 0}, tot[2];
#pragma unroll
  for (int k = 0; k < kBPT; ++k) {
    const uint32_t b = (uint32_t)(t * kBPT + k);
    c8[k] = ((b << shift) <= dmax) ? hist[b] : 0u;
    m8[k] = c8[k] ? bmass[b] : 0ull;
    x[0] += c8[k];
    x[1] += m8[k];
  }
  if (t == 0) s_found = kNB;
  bscan<2>(x, tot, sw);
  const unsigned long long Sx = tot[1];  // exact: every token's W in exactly one bin
  const unsigned long long theta = tau_all ? 0ull : threshold(s.tau_q, Sx);
  if (tau_all && cap_all) {  // everything is kept
    for (int64_t c = t; c < s.nch; c += kST)  // chunk c: c*kSelChunk tokens before it, all strict
      s.pre[(int64_t)row * s.nch + c] = (unsigned long long)(c * kSelChunk) << 32;
    if (t == 0) {
      hs->S = Sx;
      hs->theta = 0ull;
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
  unsigned long long cc = x[0], cm = x[1];
  int found = kNB;
  unsigned long long fcc = 0, fcm = 0;
#pragma unroll
  for (int k = 0; k < kBPT; ++k) {
    const bool trig = c8[k] && ((!tau_all && cm + m8[k] >= theta) ||
                                (!cap_all && cc + c8[k] >= (unsigned long long)s.k_max));
    if (trig && found == kNB) { found = t * kBPT + k; fcc = cc; fcm = cm; }
    cc += c8[k];
    cm += m8[k];
  }
  if (found < kNB) atomicMin(&s_found, found);
  __syncthreads();
  const int fb = s_found;
  if (fb == kNB) {  // cannot happen: Θ <= S and k_max < n are always reached
    if (t == 0) hs->state = kStError;
    return;
  }
  if (found == fb) {
    const uint32_t rlo = (uint32_t)fb << shift;
    hs->S = Sx;
    hs->theta = theta;
    hs->cnt_before = (uint32_t)fcc;
    hs->mass_before = fcm;  // exact: the bins before the cut's
    hs->r_lo = rlo;
    hs->r_hi = min(rlo + ((1u << shift) - 1u), dmax);
    hs->fshift = 0;         // 2^shift <= kNB: K2's fine bins are exact Δ values
    __threadfence();
    hs->state = kStRefine1;
  }
}

// ---------------------------------------------------------------------------- K2
__device__ void finish_row(const SelArgs &s, int row, uint32_t *cs, uint32_t *ct, uint32_t *fc);

// The CTA's token range is whole chunks; per chunk every thread holds 16 consecutive tokens.
__global__ void __launch_bounds__(kST, 2) k_sel_refine(SelArgs s, int64_t per) {
  extern __shared__ __align__(16) uint8_t sm2[];
  uint32_t *fc = reinterpret_cast<uint32_t *>(sm2);                 // [kNB] exact counts per Δ
  float *zbuf = reinterpret_cast<float *>(sm2 + kNB * 4);           // [kZB2][kSelChunk]
  unsigned long long *lq_all =                                          // [kST/32][64] per-warp list queues
      reinterpret_cast<unsigned long long *>(sm2 + kNB * 4 + kZB2 * kSelChunk * 4);
  __shared__ uint64_t zbar[kZB2];
  __shared__ uint32_t zdone[kZB2];
  __shared__ bool s_last;
  __shared__ int s_found;
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  HeadState *hs = s.hs + row;
  if (hs->state != kStRefine1) return;
  const int M = hs->M;
  const float kappa = hs->kappa;
  const uint32_t lo = hs->r_lo, hi = hs->r_hi;
  // K1 leaves one coarse bin of at most 2^11 Δ values: the fine bins are exact Δ values
  if (hs->fshift != 0 || hi - lo >= (uint32_t)kNB) {
    if (t == 0) hs->state = kStError;
    return;
  }
  const int64_t j0 = (int64_t)blockIdx.x * per, j1 = min(s.n, j0 + per);
  for (int i = t; i < kNB; i += kST) fc[i] = 0u;
  ZStream<kZB2> zs;
  zs.init(zbuf, zbar, zdone, s.z + (int64_t)row * s.z_stride, s.n);
  const int64_t c0 = j0 / kSelChunk, c1 = (j1 + kSelChunk - 1) / kSelChunk;
  if (t == 0)
    for (int i = 0; i < kZB2 && c0 + i < c1; ++i) zs.request(c0 + i, i);
  unsigned long long *lq = lq_all + warp * 64;
  int lqn = 0;                // warp-uniform list-queue length (flushed 32 entries per global atomic)
  unsigned long long *lst = s.list + (int64_t)row * s.cap;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t c = c0; c < c1; ++c) {
    const int slot = (int)((c - c0) % kZB2);
    const float *zc = zs.wait(slot);
    const int64_t cb = c * kSelChunk;
    const int nv = (int)min((int64_t)kSelChunk, s.n - cb);
    uint32_t nlo = 0;
#pragma unroll
    for (int u2 = 0; u2 < 2; ++u2) {
      const int i0 = 4 * t + 2048 * u2;
      const float4 v4 = *reinterpret_cast<const float4 *>(zc + i0);
      const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool valid = i0 + e < nv;
        const uint32_t dl = (uint32_t)(M - zint(vv[e]));
        const bool above = valid && dl < lo;
        const bool inr = valid && dl >= lo && dl <= hi;
        nlo += above ? 1u : 0u;
        const unsigned mr = __ballot_sync(0xffffffffu, inr);
        if (mr) {  // in-range: fine histogram + the row's in-range list (via the warp's queue)
          if (inr) {
            atomicAdd(&fc[dl - lo], 1u);
            lq[lqn + __popc(mr & lt)] = ((unsigned long long)(cb + i0 + e) << 32) | dl;
          }
          lqn += __popc(mr);
          if (lqn >= 32) {  // one global atomic reserves 32 list slots for the warp
            __syncwarp();
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&hs->ticket, 32u);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base + lane < (unsigned)s.cap) lst[base + lane] = lq[lane];
            const unsigned long long rest = lane + 32 < lqn ? lq[lane + 32] : 0ull;
            __syncwarp();
            if (lane + 32 < lqn) lq[lane] = rest;
            lqn -= 32;
            __syncwarp();
          }
        }
      }
    }
    // the chunk's count of tokens above the range (K4 adds its in-range tokens below Δ*)
    nlo = __reduce_add_sync(0xffffffffu, nlo);
    if (lane == 0 && nlo) atomicAdd(&s.cntlo[(int64_t)row * s.nch + c], nlo);
    zs.release(c + kZB2 < c1 ? c + kZB2 : -1, slot);
  }
  __syncwarp();
  if (lqn > 0) {  // the warp's last list entries
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(&hs->ticket, (unsigned)lqn);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane < lqn && base + lane < (unsigned)s.cap) lst[base + lane] = lq[lane];
  }
  __syncthreads();  // every in-range token counted into fc
  uint32_t *gc = s.fcnt + (int64_t)row * kNB;
  for (int i = t; i < kNB; i += kST) {
    const uint32_t c = fc[i];
    if (c) atomicAdd(&gc[i], c);
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
  // ---- the row's last CTA: walk the bin's Δ values to the exact cut
  for (int i = t; i < kNB; i += kST) fc[i] = __ldcg(&gc[i]);
  if (t == 0) hs->c2_done = 0u;
  __syncthreads();
  const bool tau_all = s.tau_q >= (1u << 24);
  const bool cap_all = (unsigned long long)s.k_max >= (unsigned long long)s.n;
  const unsigned long long Sx = hs->S, theta = hs->theta;  // exact (K1)
  const unsigned long long cc0 = hs->cnt_before, cm0 = __ldcg((const unsigned long long *)&hs->mass_before);
  resolve_bins(fc, nullptr, 0, lo, hi, cc0, cm0, s, hs, row, kappa, theta, tau_all, cap_all, Sx, &s_found);
  if (s.nch <= kFinishInK2) {  // the row's finish here (no K4 launch): counters over the z buffers
    __syncthreads();
    finish_row(s, row, reinterpret_cast<uint32_t *>(zbuf), reinterpret_cast<uint32_t *>(zbuf) + s.nch, fc);
  }
}

// ---------------------------------------------------------------------------- K4
// One CTA per row.  Dynamic shared memory: strict / tie counts per chunk [2][nch] (+ the
// second refine's fine counts [kNB]).
// The row's finish, by one whole CTA: (if narrowed) the second refine; then per chunk the
// (strict, tie) counts and their exclusive prefix.  cs / ct: [nch] shared, fc: [kNB] shared.
__device__ void finish_row(const SelArgs &s, int row, uint32_t *cs, uint32_t *ct, uint32_t *fc) {
  __shared__ unsigned long long sw[2][kST / 32];
  __shared__ int s_found;
  const int t = threadIdx.x;
  HeadState *hs = s.hs + row;
  const float *zr = s.z + (int64_t)row * s.z_stride;
  const unsigned long long *lst = s.list + (int64_t)row * s.cap;
  const unsigned long long nl = hs->ticket;               // in-range tokens of K2 (may exceed cap)
  const bool complete = nl <= (unsigned long long)s.cap;
  const int M = hs->M;
  const float kappa = hs->kappa;
  if (hs->state == kStRefine2) {  // the boundary fine bin [r_lo, r_hi]: exact counts per Δ
    const uint32_t lo = hs->r_lo, hi = hs->r_hi;
    for (int i = t; i < kNB; i += kST) fc[i] = 0u;
    __syncthreads();
    if (complete) {
      for (unsigned long long e = t; e < nl; e += kST) {
        const uint32_t dl = (uint32_t)lst[e];
        if (dl >= lo && dl <= hi) atomicAdd(&fc[dl - lo], 1u);
      }
    } else {
      for (int64_t j = t; j < s.n; j += kST) {
        const uint32_t dl = (uint32_t)(M - zint(zr[j]));
        if (dl >= lo && dl <= hi) atomicAdd(&fc[dl - lo], 1u);
      }
    }
    __syncthreads();
    const bool tau_all = s.tau_q >= (1u << 24);
    const bool cap_all = (unsigned long long)s.k_max >= (unsigned long long)s.n;
    resolve_bins(fc, nullptr, 0, lo, hi, hs->cnt_before, hs->mass_before, s, hs, row, kappa, hs->theta,
                 tau_all, cap_all, hs->S, &s_found);
    __syncthreads();
  }
  if (hs->state != kStDone) return;
  const uint32_t dstar = hs->delta_star;
  const int64_t nch = s.nch;
  if (dstar == 0xffffffffu) {  // everything kept: the chunks' sizes
    for (int64_t c = t; c < nch; c += kST) {
      cs[c] = (uint32_t)(min(s.n, (c + 1) * kSelChunk) - c * kSelChunk);
      ct[c] = 0u;
    }
  } else if (complete) {  // above the range + the in-range tokens below / at Δ*
    for (int64_t c = t; c < nch; c += kST) { cs[c] = s.cntlo[(int64_t)row * nch + c]; ct[c] = 0u; }
    __syncthreads();
    for (unsigned long long e = t; e < nl; e += kST) {
      const unsigned long long w = lst[e];
      const uint32_t dl = (uint32_t)w;
      const int64_t c = (int64_t)(w >> 32) / kSelChunk;
      if (dl < dstar) atomicAdd(&cs[c], 1u);
      else if (dl == dstar) atomicAdd(&ct[c], 1u);
    }
  } else {  // the list overflowed: count from z (slow path, exact)
    for (int64_t c = t; c < nch; c += kST) { cs[c] = 0u; ct[c] = 0u; }
    __syncthreads();
    for (int64_t j = t; j < s.n; j += kST) {
      const uint32_t dl = (uint32_t)(M - zint(zr[j]));
      if (dl < dstar) atomicAdd(&cs[j / kSelChunk], 1u);
      else if (dl == dstar) atomicAdd(&ct[j / kSelChunk], 1u);
    }
  }
  __syncthreads();
  // exclusive prefix over the chunks (thread-contiguous runs, then a block scan)
  const int64_t per = (nch + kST - 1) / kST;
  const int64_t c0 = min(nch, (int64_t)t * per), c1 = min(nch, c0 + per);
  unsigned long long x[2] = {0, 0}, tot[2];
  for (int64_t c = c0; c < c1; ++c) { x[0] += cs[c]; x[1] += ct[c]; }
  bscan<2>(x, tot, sw);
  unsigned long long ps = x[0], pt = x[1];
  unsigned long long *pre = s.pre + (int64_t)row * nch;
  for (int64_t c = c0; c < c1; ++c) {
    pre[c] = (ps << 32) | pt;
    ps += cs[c];
    pt += ct[c];
  }
}

// K4 (only when a row's chunk counters do not fit K2's shared memory): one CTA per row
__global__ void __launch_bounds__(kST) k_sel_prefix(SelArgs s) {
  extern __shared__ __align__(16) uint8_t sm4[];
  uint32_t *cs = reinterpret_cast<uint32_t *>(sm4);       // [nch] strict
  uint32_t *ct = cs + s.nch;                               // [nch] ties
  uint32_t *fc = ct + s.nch;                               // [kNB] second-refine counts
  pdl_trigger();
  pdl_wait();
  finish_row(s, blockIdx.x, cs, ct, fc);
}

// ---------------------------------------------------------------------------- K3
// Persistent CTAs of kWT threads over the (row, chunk) items; the next item's z chunk streams
// into the other shared buffer (cp.async.bulk) while this one is compacted.  Thread t owns the
// 16 consecutive tokens 16t .. 16t+15 of the chunk, so one block scan of its (strict, tie)
// counts orders the chunk.
constexpr int kWT = 256;

__global__ void __launch_bounds__(kWT, 4) k_sel_write(SelArgs s) {
  extern __shared__ __align__(128) uint8_t sm3[];
  float *zbuf = reinterpret_cast<float *>(sm3);                                        // [2][kSelChunk]
  uint32_t *stg_d = reinterpret_cast<uint32_t *>(sm3 + 2 * kSelChunk * 4);            // [kSelChunk]
  uint16_t *stg_o = reinterpret_cast<uint16_t *>(sm3 + 3 * kSelChunk * 4);            // [kSelChunk]
  __shared__ uint64_t zbar[2];
  __shared__ uint32_t sw[kWT / 32];
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t items = (int64_t)s.rows * s.nch;
  if (t == 0) {
    mbar_init(&zbar[0], 1);
    mbar_init(&zbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto request = [&](int64_t it, int slot) {  // thread 0: the item's z chunk -> buffer `slot`
    const int64_t row = it / s.nch, c = it - row * s.nch;
    const int64_t j0 = c * kSelChunk;
    const int64_t cnt = min((int64_t)kSelChunk, s.n - j0);
    const uint32_t bytes = (uint32_t)((cnt * 4 + 15) & ~(int64_t)15);
    mbar_expect_tx(&zbar[slot], bytes);
    bulk_g2s(zbuf + (size_t)slot * kSelChunk, s.z + row * s.z_stride + j0, bytes, &zbar[slot]);
  };
  if (t == 0) {
    if ((int64_t)blockIdx.x < items) request(blockIdx.x, 0);
    if ((int64_t)blockIdx.x + gridDim.x < items) request((int64_t)blockIdx.x + gridDim.x, 1);
  }
  uint32_t ph = 0u;
  int slot = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x, slot ^= 1) {
    const int row = (int)(it / s.nch);
    const int64_t c = it - (int64_t)row * s.nch;
    const HeadState *hs = s.hs + row;
    const uint32_t state = hs->state;
    const int M = hs->M;
    const float kappa = hs->kappa;
    const uint32_t dstar = hs->delta_star;
    const unsigned long long r = hs->r_ties;
    const unsigned long long pw = s.pre[(int64_t)row * s.nch + c];
    const unsigned long long den = s.renorm ? hs->sel_mass : hs->S;
    const int64_t j0 = c * kSelChunk;
    const int nv = (int)min((int64_t)kSelChunk, s.n - j0);
    mbar_wait(&zbar[slot], (ph >> slot) & 1u);
    ph ^= 1u << slot;
    const float *zc = zbuf + (size_t)slot * kSelChunk + 16 * t;
    if (state == kStDone) {  // (an error state writes nothing: sel_k stays unset)
      uint32_t dl[16], my = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 v4 = *reinterpret_cast<const float4 *>(zc + 4 * k);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = 16 * t + 4 * k + e;
          dl[4 * k + e] = i < nv ? (uint32_t)(M - zint(vv[e])) : 0xffffffffu;
        }
      }
      const bool ties_on = dstar != 0xffffffffu;
      uint32_t ms = 0, mt = 0;  // my tokens' strict / tie bits
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        ms |= (dl[u] < dstar ? 1u : 0u) << u;
        mt |= ((ties_on && dl[u] == dstar) ? 1u : 0u) << u;
      }
      my = ((uint32_t)__popc(ms) << 16) | (uint32_t)__popc(mt);
      // block exclusive scan of the packed (strict << 16 | ties) counts (each <= kSelChunk)
      uint32_t inc = my;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
      }
      if (lane == 31) sw[warp] = inc;
      __syncthreads();
      uint32_t before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kWT / 32; ++w) {
        const uint32_t v = sw[w];
        before += w < warp ? v : 0u;
        total += v;
      }
      const uint32_t ex = before + inc - my;
      const unsigned long long Sb = pw >> 32, Tb = pw & 0xffffffffull;
      const unsigned long long pos0 = Sb + (Tb < r ? Tb : r);
      unsigned long long ts = Tb + (ex & 0xffffu);
      // kept tokens: the strict ones and, while fewer than r ties precede them, the ties
      uint32_t keep = ms;
      if (mt) {
        const unsigned long long room = ts < r ? r - ts : 0ull;  // ties this thread may keep
        uint32_t m = mt;
        for (unsigned long long k = 0; k < room && m; ++k) { keep |= m & (0u - m); m &= m - 1u; }
      }
      const unsigned base = (unsigned)(Sb + (ex >> 16) + (ts < r ? ts : r) - pos0);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (keep >> u & 1u) {
          const unsigned ls = base + __popc(keep & ((1u << u) - 1u));
          stg_d[ls] = dl[u];
          stg_o[ls] = (uint16_t)(16 * t + u);
        }
      }
      __syncthreads();
      const unsigned long long tt = Tb + (total & 0xffffu);
      const int kept = (int)(Sb + (total >> 16) + (tt < r ? tt : r) - pos0);
      const float inv_den = (float)(1.0 / (double)den);
      int32_t *oi = s.sel_idx + (int64_t)row * s.k_max + pos0;
      float *ow = s.sel_w + (int64_t)row * s.k_max + pos0;
      for (int i = t; i < kept; i += kWT) {
        oi[i] = (int32_t)(j0 + stg_o[i]);
        ow[i] = __fmul_rn((float)wmass(stg_d[i], kappa), inv_den);
      }
    }
    __syncthreads();  // every read of zc / the staging / sw retired
    if (t == 0 && it + 2 * (int64_t)gridDim.x < items) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      request(it + 2 * (int64_t)gridDim.x, slot);
    }
  }
}

// K3 + Eq. 5 for values in HBM (d = 128): "K3G".  Persistent CTAs over CONTIGUOUS ranges of
// the (row, chunk) items (row-major), 3 per SM: each item is compacted exactly as in K3 (the
// (index, W/S) lists are still written), then its kept value rows are gathered right away --
// half-warp per row, 8 rows (16-B loads) in flight per half-warp -- into fp32 accumulators
// that persist across the CTA's consecutive items of the same row.  When the row changes the
// CTA writes one partial (its contributor slot) and the row's last contributor adds the
// partials in CTA order (deterministic).  Concurrent CTAs sit at the same relative chunk of
// neighbouring rows, so the G heads of a KV head read the same token range at about the same
// time and shared kept rows hit in L2.  Replaces K3 + k_gather_rows (one pass over the kept
// rows overlapping the compaction's z stream).
template <int kGU, int kMinB>  // value rows in flight per half-warp, CTAs per SM
__global__ void __launch_bounds__(kWT, kMinB) k_sel_write_gather(SelArgs s, LayerArgs a, float *wpart,
                                                                 uint32_t *wdone, int64_t per, int maxc,
                                                                 int64_t idx_base) {
  extern __shared__ __align__(128) uint8_t sm3[];
  float *zbuf = reinterpret_cast<float *>(sm3);                                        // [2][kSelChunk]
  uint32_t *stg_d = reinterpret_cast<uint32_t *>(sm3 + 2 * kSelChunk * 4);            // [kSelChunk]
  float *stg_w = reinterpret_cast<float *>(stg_d);                                    // (weights, in place)
  uint16_t *stg_o = reinterpret_cast<uint16_t *>(sm3 + 3 * kSelChunk * 4);            // [kSelChunk]
  float *red = reinterpret_cast<float *>(sm3 + 3 * kSelChunk * 4 + kSelChunk * 2);    // [16][128]
  __shared__ uint64_t zbar[2];
  __shared__ uint32_t sw[kWT / 32];
  __shared__ bool s_last;
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int hw = t >> 4, sub = t & 15;  // half-warp, its 8-dim slice
  const int64_t items = (int64_t)s.rows * s.nch;
  const int64_t it0 = (int64_t)blockIdx.x * per, it1 = min(items, it0 + per);
  if (it0 >= it1) return;
  if (t == 0) {
    mbar_init(&zbar[0], 1);
    mbar_init(&zbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto request = [&](int64_t it, int slot) {  // thread 0: the item's z chunk -> buffer `slot`
    const int64_t row = it / s.nch, c = it - row * s.nch;
    const int64_t j0 = c * kSelChunk;
    const int64_t cnt = min((int64_t)kSelChunk, s.n - j0);
    const uint32_t bytes = (uint32_t)((cnt * 4 + 15) & ~(int64_t)15);
    mbar_expect_tx(&zbar[slot], bytes);
    bulk_g2s(zbuf + (size_t)slot * kSelChunk, s.z + row * s.z_stride + j0, bytes, &zbar[slot]);
  };
  if (t == 0) {
    request(it0, 0);
    if (it0 + 1 < it1) request(it0 + 1, 1);
  }
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
  // the row's partial -> my contributor slot; the row's last contributor sums them in order
  auto flush = [&](int row) {
#pragma unroll
    for (int e = 0; e < 8; ++e) red[hw * 128 + sub * 8 + e] = acc[e];
    __syncthreads();
    const int64_t first = ((int64_t)row * s.nch) / per;
    const int64_t lastc = ((int64_t)(row + 1) * s.nch - 1) / per;
    const int cnt = (int)(lastc - first + 1), me = (int)(blockIdx.x - first);
    if (t < 128) {
      float v = 0.0f;
#pragma unroll
      for (int q = 0; q < 16; ++q) v += red[q * 128 + t];
      wpart[((int64_t)row * maxc + me) * 128 + t] = v;
      __threadfence();
    }
    __syncthreads();
    if (t == 0) {
      const uint32_t prev = atomicAdd(&wdone[row], 1u);
      s_last = prev == (uint32_t)cnt - 1u;
      if (s_last) wdone[row] = 0u;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (t < 128) {
        const float *p0 = wpart + (int64_t)row * maxc * 128 + t;
        float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        int c = 0;
        for (; c + 3 < cnt; c += 4) {
#pragma unroll
          for (int q = 0; q < 4; ++q) s4[q] += __ldcg(p0 + (int64_t)(c + q) * 128);
        }
        for (; c < cnt; ++c) s4[0] += __ldcg(p0 + (int64_t)c * 128);
        a.out[(int64_t)row * 128 + t] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
  };
  uint32_t ph = 0u;
  int slot = 0;
  int cur_row = (int)(it0 / s.nch);
  for (int64_t it = it0; it < it1; ++it, slot ^= 1) {
    const int row = (int)(it / s.nch);
    if (row != cur_row) {
      flush(cur_row);
      cur_row = row;
    }
    const int64_t c = it - (int64_t)row * s.nch;
    const HeadState *hs = s.hs + row;
    const uint32_t state = hs->state;
    const int M = hs->M;
    const float kappa = hs->kappa;
    const uint32_t dstar = hs->delta_star;
    const unsigned long long r = hs->r_ties;
    const unsigned long long pw = s.pre[(int64_t)row * s.nch + c];
    const unsigned long long den = s.renorm ? hs->sel_mass : hs->S;
    const int64_t j0 = c * kSelChunk;
    const int nv = (int)min((int64_t)kSelChunk, s.n - j0);
    mbar_wait(&zbar[slot], (ph >> slot) & 1u);
    ph ^= 1u << slot;
    const float *zc = zbuf + (size_t)slot * kSelChunk + 16 * t;
    int kept = 0;
    if (state == kStDone) {
      uint32_t dl[16], my = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 v4 = *reinterpret_cast<const float4 *>(zc + 4 * k);
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = 16 * t + 4 * k + e;
          dl[4 * k + e] = i < nv ? (uint32_t)(M - zint(vv[e])) : 0xffffffffu;
        }
      }
      const bool ties_on = dstar != 0xffffffffu;
      uint32_t ms = 0, mt = 0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        ms |= (dl[u] < dstar ? 1u : 0u) << u;
        mt |= ((ties_on && dl[u] == dstar) ? 1u : 0u) << u;
      }
      my = ((uint32_t)__popc(ms) << 16) | (uint32_t)__popc(mt);
      uint32_t inc = my;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
      }
      if (lane == 31) sw[warp] = inc;
      __syncthreads();
      uint32_t before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kWT / 32; ++w) {
        const uint32_t v = sw[w];
        before += w < warp ? v : 0u;
        total += v;
      }
      const uint32_t ex = before + inc - my;
      const unsigned long long Sb = pw >> 32, Tb = pw & 0xffffffffull;
      const unsigned long long pos0 = Sb + (Tb < r ? Tb : r);
      unsigned long long ts = Tb + (ex & 0xffffu);
      uint32_t keep = ms;
      if (mt) {
        const unsigned long long room = ts < r ? r - ts : 0ull;
        uint32_t m = mt;
        for (unsigned long long k = 0; k < room && m; ++k) { keep |= m & (0u - m); m &= m - 1u; }
      }
      const unsigned base = (unsigned)(Sb + (ex >> 16) + (ts < r ? ts : r) - pos0);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        if (keep >> u & 1u) {
          const unsigned ls = base + __popc(keep & ((1u << u) - 1u));
          stg_d[ls] = dl[u];
          stg_o[ls] = (uint16_t)(16 * t + u);
        }
      }
      __syncthreads();
      const unsigned long long tt = Tb + (total & 0xffffu);
      kept = (int)(Sb + (total >> 16) + (tt < r ? tt : r) - pos0);
      const float inv_den = (float)(1.0 / (double)den);
      int32_t *oi = s.sel_idx + (int64_t)row * s.k_max + pos0;
      float *ow = s.sel_w + (int64_t)row * s.k_max + pos0;
      for (int i = t; i < kept; i += kWT) {
        const float w = __fmul_rn((float)wmass(stg_d[i], kappa), inv_den);
        oi[i] = (int32_t)(idx_base + j0 + stg_o[i]);  // global index (a shard's base + local)
        ow[i] = w;
        stg_w[i] = w;
      }
      __syncthreads();
    }
    // the chunk is consumed: refill its buffer with item it + 2 while the rows are gathered
    if (t == 0 && it + 2 < it1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      request(it + 2, slot);
    }
    if (kept > 0) {  // Eq. 5 over the chunk's kept rows (CTA-uniform)
      const int b = row / a.Hq, kv = (row - b * a.Hq) / a.G;
      const uint16_t *Vb = a.V + (int64_t)b * a.v_b_stride + (int64_t)kv * a.v_kv_stride;
      const uint16_t *Rb = a.res_v + (int64_t)b * a.res_b_stride + (int64_t)kv * a.res_cap * a.d;
      for (int i0 = hw * kGU; i0 < kept; i0 += 16 * kGU) {
        uint4 v[kGU];
#pragma unroll
        for (int q = 0; q < kGU; ++q) {
          const int i = i0 + q;
          if (i < kept) {
            const int64_t j = j0 + stg_o[i];
            const uint16_t *src;
            if (j < a.n_q) {
              src = Vb + j * 128;
            } else {
              const uint32_t sl = (uint32_t)(a.res_slot0 + (j - a.n_q)) % (uint32_t)a.res_cap;
              src = Rb + (int64_t)sl * 128;
            }
            v[q] = ldg_nc16(src + sub * 8);
          } else {
            v[q] = make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int q = 0; q < kGU; ++q) {
          const float w = i0 + q < kept ? stg_w[i0 + q] : 0.0f;
          const uint32_t uu[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
          for (int p2 = 0; p2 < 4; ++p2) {
            const float2 f2 = __half22float2(*reinterpret_cast<const __half2 *>(&uu[p2]));
            acc[2 * p2] = fmaf(w, f2.x, acc[2 * p2]);
            acc[2 * p2 + 1] = fmaf(w, f2.y, acc[2 * p2 + 1]);
          }
        }
      }
    }
    __syncthreads();  // every read of zc / the staging / sw retired
  }
  flush(cur_row);
}

template <int GU, int MB>
static cudaError_t k3g_launch(const SelArgs &s, const LayerArgs &a, float *wpart, uint32_t *wdone, int num_sms,
                              cudaStream_t st, int64_t idx_base) {
  const int64_t items = (int64_t)s.rows * s.nch;
  if (items <= 0) return cudaSuccess;
  int64_t grid = (int64_t)MB * num_sms;
  if (grid > items) grid = items;
  const int64_t per = (items + grid - 1) / grid;
  grid = (items + per - 1) / per;
  const int maxc = select_wg_maxc(s.nch, per);
  const size_t smem = (size_t)3 * kSelChunk * 4 + (size_t)kSelChunk * 2 + 16 * 128 * 4;
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaFuncSetAttribute(k_sel_write_gather<GU, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured[dev] = 1;
  }
  launch_chain(k_sel_write_gather<GU, MB>, dim3((unsigned)grid), dim3(kWT), smem, st, s, a, wpart, wdone, per, maxc,
               idx_base);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_select_write_gather(const SelArgs &s, const LayerArgs &a, float *wpart, uint32_t *wdone,
                                       int num_sms, cudaStream_t st, int64_t idx_base) {
  static int v = -1;  // dev override (HC_K3G_GU = 8 | 12 | 16): rows in flight per half-warp
  if (v < 0) { const char *ev = getenv("HC_K3G_GU"); v = ev ? atoi(ev) : 8; }
  if (v == 16) return k3g_launch<16, 2>(s, a, wpart, wdone, num_sms, st, idx_base);
  if (v == 12) return k3g_launch<12, 2>(s, a, wpart, wdone, num_sms, st, idx_base);
  if (v == 4) return k3g_launch<4, 3>(s, a, wpart, wdone, num_sms, st, idx_base);
  return k3g_launch<8, 3>(s, a, wpart, wdone, num_sms, st, idx_base);
}

// ---------------------------------------------------------------------------- short rows
// Rows of up to kSmallMaxN candidates (configs 1, 2): ONE kernel, a cluster of cs <= 8 CTAs per
// row, every CTA holding its <= 8192 scores in registers (16 per thread) for all passes.  The
// row-wide sums go through global atomics (histograms, L2-resident) and DSMEM (a few scalars per
// CTA); after each cluster barrier every CTA re-reads the row's histogram and derives the same
// bound / cut redundantly -- no single-CTA tail, no broadcast.  Same integer rules as the long-
// row passes, so the same bit-exact result.
constexpr int kSmTok = 8192;  // tokens per CTA
constexpr int64_t kSmallMaxN = 8LL * kSmTok;

struct CutResult {
  int bin;  // kNB: none
  unsigned long long cc, cm, c, m;  // count / mass before the bin, the bin's count / mass
};

// The cut over kNB consecutive bins (bin b covers Δ in [base + (b << f), ...); counts cnt[],
// masses from mass[] or c * W(base + (b << f)); cc0 / cm0 before base) -- by the whole CTA,
// result in *res (same on every CTA given the same inputs).
__device__ void find_cut(const uint32_t *cnt, const unsigned long long *mass, int f, uint32_t base,
                         uint32_t top, unsigned long long cc0, unsigned long long cm0, float kappa,
                         unsigned long long theta, bool tau_all, bool cap_all, int64_t k_max,
                         CutResult *res, unsigned long long (*sw)[kST / 32]) {
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
  if (t == 0) res->bin = kNB;
  bscan<2>(x, tot, sw);
  unsigned long long cc = cc0 + x[0], cm = cm0 + x[1];
  int found = kNB;
  unsigned long long fcc = 0, fcm = 0, fc = 0, fm = 0;
#pragma unroll
  for (int k = 0; k < kBPT; ++k) {
    const bool trig = c8[k] && ((!tau_all && cm + m8[k] >= theta) || (!cap_all && cc + c8[k] >= (unsigned long long)k_max));
    if (trig && found == kNB) { found = t * kBPT + k; fcc = cc; fcm = cm; fc = c8[k]; fm = m8[k]; }
    cc += c8[k];
    cm += m8[k];
  }
  if (found < kNB) atomicMin(&res->bin, found);
  __syncthreads();
  if (found < kNB && found == res->bin) { res->cc = fcc; res->cm = fcm; res->c = fc; res->m = fm; }
  __syncthreads();
}

template <bool GATHER>  // GATHER: Eq. 5 over HBM values (d = 128) inside the kernel (la.out)
__global__ void __launch_bounds__(kST) k_sel_small(SelArgs s, int cs, int folded, LayerArgs la) {
  extern __shared__ __align__(16) uint8_t sm5[];
  uint32_t *stg_d = reinterpret_cast<uint32_t *>(sm5);                         // [kSmTok]
  uint16_t *stg_o = reinterpret_cast<uint16_t *>(sm5 + kSmTok * 4);           // [kSmTok]
  uint32_t *mlo = reinterpret_cast<uint32_t *>(sm5 + kSmTok * 6);             // [kNB] mass, low word
  uint32_t *mhi = mlo + kNB;                                                  // [kNB] high word
  __shared__ uint32_t hist[kNB];
  __shared__ unsigned long long sw[2][kST / 32];
  __shared__ struct {
    int M, zmin;
    unsigned long long tc, tm;  // my slice's exact count / mass
    int cbin;                   // the cut's coarse bin (slice owner)
    unsigned long long ccc, ccm;
    uint32_t ns, nt;
  } slot;
  __shared__ CutResult cr;
  __shared__ int s_red_i[2][kST / 32];
  cg::cluster_group cl = cg::this_cluster();
  pdl_trigger();
  pdl_wait();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.x / cs;
  HeadState *hs = s.hs + row;
  const int64_t j0 = (int64_t)rank * kSmTok + 16 * t;  // my 16 consecutive tokens
  const float *zr = s.z + (int64_t)row * s.z_stride;
  float zv[16];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t p = j0 + 4 * k;
    if (p + 4 <= s.n) {
      const float4 v = *reinterpret_cast<const float4 *>(zr + p);
      zv[4 * k] = v.x; zv[4 * k + 1] = v.y; zv[4 * k + 2] = v.z; zv[4 * k + 3] = v.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) zv[4 * k + u] = p + u < s.n ? zr[p + u] : 0.0f;
    }
  }
  uint32_t vmask = 0;  // my valid tokens
#pragma unroll
  for (int u = 0; u < 16; ++u) vmask |= (j0 + u < s.n ? 1u : 0u) << u;
  // ---- M, zmin: folded by the scan epilogue, else a cluster reduction of my tokens' range
  int M, zmin;
  if (folded) {
    M = hs->M;
    zmin = hs->zmin;
  } else {
    int mx = INT_MIN, mn = INT_MAX;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (vmask >> u & 1u) { const int zi = zint(zv[u]); mx = max(mx, zi); mn = min(mn, zi); }
    mx = __reduce_max_sync(0xffffffffu, mx);
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (lane == 0) { s_red_i[0][warp] = mx; s_red_i[1][warp] = mn; }
    __syncthreads();
    if (t == 0) {
      for (int w = 1; w < kST / 32; ++w) { mx = max(mx, s_red_i[0][w]); mn = min(mn, s_red_i[1][w]); }
      slot.M = mx;
      slot.zmin = mn;
    }
    cl.sync();
    M = INT_MIN; zmin = INT_MAX;
    for (int r = 0; r < cs; ++r) {
      const auto *o = cl.map_shared_rank(&slot, r);
      M = max(M, o->M);
      zmin = min(zmin, o->zmin);
    }
  }
  const float kappa = hs->kappa;
  const int shift = sel_shift(M, zmin);
  const uint32_t dmax = (uint32_t)(M - zmin);
  uint32_t dl[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) dl[u] = (vmask >> u & 1u) ? (uint32_t)(M - zint(zv[u])) : 0xffffffffu;
  // ---- pass A: exact (count, mass) per coarse bin of my tokens (shared atomics, split words)
  for (int i = t; i < kNB; i += kST) { hist[i] = 0u; mlo[i] = 0u; mhi[i] = 0u; }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 16; u += 2) {  // token pairs: the mass on the packed fp32x2 pipe
    uint64_t wp[2];
    wmass2(dl[u], dl[u + 1], kappa, wp[0], wp[1]);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (vmask >> (u + q) & 1u) {
        const uint32_t bb = dl[u + q] >> shift;
        const uint32_t wl = (uint32_t)wp[q];
        uint32_t wh = (uint32_t)(wp[q] >> 32);
        atomicAdd(&hist[bb], 1u);
        const uint32_t old = atomicAdd(&mlo[bb], wl);
        wh += (old + wl < old) ? 1u : 0u;
        if (wh) atomicAdd(&mhi[bb], wh);
      }
    }
  }
  cl.sync();
  // ---- my slice of the bins, summed over the cluster (DSMEM), and its totals
  const int nbs = kNB / cs, b0 = rank * nbs, b1 = rank + 1 == cs ? kNB : b0 + nbs;
  uint32_t *red_c = reinterpret_cast<uint32_t *>(sm5);                          // [kNB] over the staging
  unsigned long long *red_m = reinterpret_cast<unsigned long long *>(sm5 + kNB * 4);  // [kNB]
  {
    unsigned long long tc = 0, tm = 0;
    for (int i = b0 + t; i < b1; i += kST) {
      uint32_t c = 0;
      unsigned long long m = 0;
      for (int rr = 0; rr < cs; ++rr) {
        c += cl.map_shared_rank(hist, rr)[i];
        m += ((unsigned long long)cl.map_shared_rank(mhi, rr)[i] << 32) + cl.map_shared_rank(mlo, rr)[i];
      }
      red_c[i - b0] = c;
      red_m[i - b0] = m;
      tc += c;
      tm += m;
    }
    tc = warp_sum_u64(tc);
    tm = warp_sum_u64(tm);
    if (lane == 0) { sw[0][warp] = tc; sw[1][warp] = tm; }
    __syncthreads();
    if (t == 0) {
      unsigned long long a0 = 0, a1 = 0;
      for (int w = 0; w < kST / 32; ++w) { a0 += sw[0][w]; a1 += sw[1][w]; }
      slot.tc = a0;
      slot.tm = a1;
    }
  }
  cl.sync();  // slice totals published; every peer is done reading my hist / mlo / mhi
  unsigned long long Sx = 0;
  for (int rr = 0; rr < cs; ++rr) Sx += cl.map_shared_rank(&slot, rr)->tm;  // exact
  const bool tau_all = s.tau_q >= (1u << 24);
  const unsigned long long theta = tau_all ? 0ull : threshold(s.tau_q, Sx);
  const unsigned long long ntot = (unsigned long long)s.n;
  const bool cap_all = (unsigned long long)s.k_max >= ntot;
  uint32_t dstar = 0xffffffffu;
  unsigned long long r = 0, ksel = ntot, selmass = Sx;
  long long kstar = (long long)ntot;
  if (!(tau_all && cap_all)) {
    // the slice the cut falls in (every CTA, same totals): first whose cumulative mass reaches Θ
    // or cumulative count reaches k_max
    int sc = cs;
    unsigned long long cc0 = 0, cm0 = 0;
    for (int rr = 0; rr < cs; ++rr) {
      const auto *o = cl.map_shared_rank(&slot, rr);
      if ((!tau_all && cm0 + o->tm >= theta) || (!cap_all && cc0 + o->tc >= (unsigned long long)s.k_max)) {
        sc = rr;
        break;
      }
      cc0 += o->tc;
      cm0 += o->tm;
    }
    if (sc == cs) {  // cannot happen: Θ <= S and k_max < n are always reached
      if (rank == 0 && t == 0) hs->state = kStError;
      if (GATHER && rank == 0 && t < 128) la.out[(int64_t)row * 128 + t] = 0.0f;
      cl.sync();
      return;
    }
    if (rank == sc) {  // the owner walks its slice's exact bins to the cut bin
      const int nb = (rank + 1 == cs ? kNB : b0 + nbs) - b0;
      for (int i = nb + t; i < kNB; i += kST) { red_c[i] = 0u; red_m[i] = 0ull; }
      __syncthreads();
      find_cut(red_c, red_m, shift, (uint32_t)b0 << shift, dmax, cc0, cm0, kappa, theta, tau_all, cap_all,
               s.k_max, &cr, sw);
      if (t == 0) { slot.cbin = cr.bin; slot.ccc = cr.cc; slot.ccm = cr.cm; }
    }
    cl.sync();
    const auto *oc = cl.map_shared_rank(&slot, sc);
    const int cbin = oc->cbin;
    const unsigned long long cc1 = oc->ccc, cm1 = oc->ccm;
    if (cbin >= kNB) {
      if (rank == 0 && t == 0) hs->state = kStError;
      if (GATHER && rank == 0 && t < 128) la.out[(int64_t)row * 128 + t] = 0.0f;
      cl.sync();
      return;
    }
    // ---- pass B: exact per-Δ counts over the cut bin's 2^shift values, summed over DSMEM
    const uint32_t base = (uint32_t)(sc * nbs + cbin) << shift;  // the cut bin (global index)
    const uint32_t top2 = min(base + ((1u << shift) - 1u), dmax);
    for (int i = t; i < kNB; i += kST) hist[i] = 0u;  // (peers finished reading it before the last syncs)
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if ((vmask >> u & 1u) && dl[u] >= base && dl[u] <= top2) atomicAdd(&hist[dl[u] - base], 1u);
    cl.sync();
    uint32_t *sum = red_c;  // [kNB] (the slice sums are no longer needed)
    for (int i = t; i < kNB; i += kST) {
      uint32_t c = 0;
      if (base + (uint32_t)i <= top2)
        for (int rr = 0; rr < cs; ++rr) c += cl.map_shared_rank(hist, rr)[i];
      sum[i] = c;
    }
    __syncthreads();
    find_cut(sum, nullptr, 0, base, top2, cc1, cm1, kappa, theta, tau_all, cap_all, s.k_max, &cr, sw);
    const int bin = cr.bin;
    if (bin >= kNB) {
      if (rank == 0 && t == 0) hs->state = kStError;
      if (GATHER && rank == 0 && t < 128) la.out[(int64_t)row * 128 + t] = 0.0f;
      cl.sync();
      return;
    }
    dstar = base + (uint32_t)bin;
    const unsigned long long w = wmass(dstar, kappa);
    unsigned long long r_tau = ~0ull, r_cap = ~0ull;
    if (!tau_all && cr.cm + cr.m >= theta) r_tau = cr.cm >= theta ? 1ull : (theta - cr.cm + w - 1) / w;
    if (r_tau == 0) r_tau = 1;
    if (!cap_all && cr.cc + cr.c >= (unsigned long long)s.k_max) r_cap = (unsigned long long)s.k_max - cr.cc;
    r = r_tau < r_cap ? r_tau : r_cap;
    ksel = cr.cc + r;
    kstar = r_tau <= r_cap ? (long long)(cr.cc + r_tau) : -1;
    selmass = cr.cm + r * w;
  }
  // ---- pass C: ordered compaction (my 16 consecutive tokens; CTAs in rank order)
  const bool ties_on = dstar != 0xffffffffu;
  uint32_t ms = 0, mt = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    ms |= ((vmask >> u & 1u) && dl[u] < dstar ? 1u : 0u) << u;
    mt |= ((vmask >> u & 1u) && ties_on && dl[u] == dstar ? 1u : 0u) << u;
  }
  const uint32_t my = ((uint32_t)__popc(ms) << 16) | (uint32_t)__popc(mt);
  uint32_t inc = my;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += o;
  }
  __shared__ uint32_t swc[kST / 32];
  if (lane == 31) swc[warp] = inc;
  __syncthreads();
  uint32_t before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kST / 32; ++w) { before += w < warp ? swc[w] : 0u; total += swc[w]; }
  if (t == 0) { slot.ns = total >> 16; slot.nt = total & 0xffffu; }
  cl.sync();
  unsigned long long Sb = 0, Tb = 0;
  for (int rr = 0; rr < rank; ++rr) {
    const auto *o = cl.map_shared_rank(&slot, rr);
    Sb += o->ns;
    Tb += o->nt;
  }
  const uint32_t ex = before + inc - my;
  const unsigned long long pos0 = Sb + (Tb < r ? Tb : r);
  unsigned long long ts = Tb + (ex & 0xffffu);
  uint32_t keep = ms;
  if (mt) {
    const unsigned long long room = ts < r ? r - ts : 0ull;
    uint32_t m = mt;
    for (unsigned long long k = 0; k < room && m; ++k) { keep |= m & (0u - m); m &= m - 1u; }
  }
  const unsigned lb = (unsigned)(Sb + (ex >> 16) + (ts < r ? ts : r) - pos0);
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    if (keep >> u & 1u) {
      const unsigned ls = lb + __popc(keep & ((1u << u) - 1u));
      stg_d[ls] = dl[u];
      stg_o[ls] = (uint16_t)(16 * t + u);
    }
  }
  __syncthreads();
  const unsigned long long tt = Tb + (total & 0xffffu);
  const int kept = (int)(Sb + (total >> 16) + (tt < r ? tt : r) - pos0);
  const float inv_den = (float)(1.0 / (s.renorm ? (double)selmass : (double)Sx));
  int32_t *oi = s.sel_idx + (int64_t)row * s.k_max + pos0;
  float *ow = s.sel_w + (int64_t)row * s.k_max + pos0;
  const int64_t cbase = (int64_t)rank * kSmTok;
  float *stg_w = reinterpret_cast<float *>(stg_d);  // weights in place of Δ (GATHER)
  for (int i = t; i < kept; i += kST) {
    const float w = __fmul_rn((float)wmass(stg_d[i], kappa), inv_den);
    oi[i] = (int32_t)(cbase + stg_o[i]);
    ow[i] = w;
    if (GATHER) stg_w[i] = w;
  }
  if constexpr (GATHER) {  // Eq. 5: my kept rows (half-warp per row, 8 in flight), cluster sum
    __shared__ float gpart[128];
    __syncthreads();
    const int hw = t >> 4, sub = t & 15;
    const int b = row / la.Hq, kv = (row - b * la.Hq) / la.G;
    const uint16_t *Vb = la.V + (int64_t)b * la.v_b_stride + (int64_t)kv * la.v_kv_stride;
    const uint16_t *Rb = la.res_v + (int64_t)b * la.res_b_stride + (int64_t)kv * la.res_cap * la.d;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
    for (int i0 = hw * 8; i0 < kept; i0 += (kST / 16) * 8) {
      uint4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = i0 + q;
        if (i < kept) {
          const int64_t j = cbase + stg_o[i];
          const uint16_t *src;
          if (j < la.n_q) {
            src = Vb + j * 128;
          } else {
            const uint32_t sl = (uint32_t)(la.res_slot0 + (j - la.n_q)) % (uint32_t)la.res_cap;
            src = Rb + (int64_t)sl * 128;
          }
          v[q] = ldg_nc16(src + sub * 8);
        } else {
          v[q] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float w = i0 + q < kept ? stg_w[i0 + q] : 0.0f;
        const uint32_t uu[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
        for (int p2 = 0; p2 < 4; ++p2) {
          const float2 f2 = __half22float2(*reinterpret_cast<const __half2 *>(&uu[p2]));
          acc[2 * p2] = fmaf(w, f2.x, acc[2 * p2]);
          acc[2 * p2 + 1] = fmaf(w, f2.y, acc[2 * p2 + 1]);
        }
      }
    }
    __syncthreads();  // the staging is read: [kST/16][128] partials over it
    float *red = reinterpret_cast<float *>(sm5);
#pragma unroll
    for (int e = 0; e < 8; ++e) red[hw * 128 + sub * 8 + e] = acc[e];
    __syncthreads();
    if (t < 128) {
      float v = 0.0f;
      for (int q = 0; q < kST / 16; ++q) v += red[q * 128 + t];
      gpart[t] = v;
    }
    cl.sync();
    if (rank == 0 && t < 128) {
      float o = 0.0f;
      for (int rr = 0; rr < cs; ++rr) o += cl.map_shared_rank(gpart, rr)[t];
      la.out[(int64_t)row * 128 + t] = o;
    }
  }
  if (rank == 0 && t == 0) {
    hs->M = M;
    hs->zmin = zmin;
    hs->shift = shift;
    hs->S = Sx;
    hs->theta = theta;
    hs->delta_star = dstar;
    hs->r_ties = (uint32_t)r;
    hs->ksel = (int64_t)ksel;
    hs->kstar = kstar;
    hs->sel_mass = selmass;
    hs->state = kStDone;
    if (s.sel_k) s.sel_k[row] = (int64_t)ksel;
  }
  cl.sync();  // peers may still read my slot through DSMEM
}

cudaError_t launch_select_small(const SelArgs &s, int folded, cudaStream_t st, const LayerArgs *ga) {
  const int cs = (int)((s.n + kSmTok - 1) / kSmTok);
  if (cs < 1 || cs > 8) return cudaErrorInvalidValue;
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaFuncSetAttribute(k_sel_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmTok * 6 + kNB * 8);
    cudaFuncSetAttribute(k_sel_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmTok * 6 + kNB * 8);
    configured[dev] = 1;
  }
  LayerArgs dummy{};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(s.rows * cs));
  cfg.blockDim = dim3(kST);
  cfg.dynamicSmemBytes = (size_t)kSmTok * 6 + (size_t)kNB * 8;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = ga ? cudaLaunchKernelEx(&cfg, k_sel_small<true>, s, cs, folded, *ga)
                     : cudaLaunchKernelEx(&cfg, k_sel_small<false>, s, cs, folded, dummy);
  note_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------------------- launcher

cudaError_t launch_select(SelArgs s, int nsplit, int num_sms, cudaStream_t st, int force, SelGather *wg) {
  if (s.rows <= 0 || s.n <= 0) return cudaSuccess;
  if (force != 1 && s.n <= kSmallMaxN) {
    if (wg) wg->used = 1;
    return launch_select_small(s, nsplit > 1 ? 0 : 1, st, wg ? wg->a : nullptr);
  }
  if (s.nch != select_chunks(s.n)) return cudaErrorInvalidValue;
  // K1 / K2: one wave of 2 CTAs per SM over all rows, whole chunks per CTA
  int64_t cpr = (2LL * num_sms) / s.rows;
  if (cpr < 1) cpr = 1;
  if (cpr > s.nch) cpr = s.nch;
  const int64_t per = (s.nch + cpr - 1) / cpr * kSelChunk;
  cpr = (s.n + per - 1) / per;
  const dim3 g12((unsigned)cpr, (unsigned)s.rows);
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaFuncSetAttribute(k_sel_mass, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(k_sel_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_sel_prefix, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_sel_write, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    configured[dev] = 1;
  }
  if (nsplit > 1) {
    launch_chain(k_sel_minmax, g12, dim3(kST), 0, st, s, per);
    note_launch();
  }
  const size_t smem1 = (size_t)kZB * kSelChunk * 4 + (size_t)kNB * 8;
  launch_chain(k_sel_mass, g12, dim3(kST), smem1, st, s, per);
  note_launch();
  const size_t smem2 = (size_t)kNB * 4 + (size_t)kZB2 * kSelChunk * 4 + (kST / 32) * 64 * 8;
  launch_chain(k_sel_refine, g12, dim3(kST), smem2, st, s, per);
  note_launch();
  if (s.nch > kFinishInK2) {  // rows too long for K2's in-place finish
    const size_t smem4 = (size_t)s.nch * 8 + (size_t)kNB * 4;
    if (smem4 > 200 * 1024) return cudaErrorInvalidValue;
    launch_chain(k_sel_prefix, dim3((unsigned)s.rows), dim3(kST), smem4, st, s);
    note_launch();
  }
  if (wg) {
    wg->used = 1;
    return launch_select_write_gather(s, *wg->a, wg->wpart, wg->wdone, num_sms, st, 0);
  }
  const int64_t items3 = (int64_t)s.rows * s.nch;
  const int64_t grid3 = items3 < 4LL * num_sms ? items3 : 4LL * num_sms;
  launch_chain(k_sel_write, dim3((unsigned)grid3), dim3(kWT), (size_t)kSelChunk * 14, st, s);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
