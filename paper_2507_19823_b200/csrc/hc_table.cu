// hc_table.cu -- row a1: the query/codebook table T = q̄·C (§3.2 P:229,
// "yields an intermediate hash table T ∈ R^{g×c}. The computational cost is O(dc),
// constant with respect to sequence length n"), in the R2 fixed-point form, and the
// exact scores of the resident recent-window tokens (R3).
//
// Layout of T in the workspace: [unit = b*Hkv+kv][group i][m < cpow2][G heads] int16,
// i.e. one 8-byte entry per centroid serving the G = 4 GQA heads of the KV head, so
// the scan does ONE shared-memory lookup per (token, group) for all G heads.
// Entries m >= c are zero (the scan masks codes to cpow2-1).
#include <float.h>
#include <stdlib.h>
#include <string.h>

#include "hc_internal.h"

namespace hc {

constexpr int kTB = 256;  // centroids per CTA

// One pass (R2).  CTA = (part, unit chunk): part p of the g * cpow2 entries (flattened
// e = i * cpow2 + m, contiguous 32-aligned ranges) for a chunk of up to 8 consecutive units
// u = b * Hkv + kv.  A unit's entries depend on its own query but the codebook rows are
// shared (C is [cbg][c][dbar], the same for every unit), so each codebook row is loaded once
// per CTA and serves every unit of the chunk: the L2 latency of a batch of rows is covered by
// units x rows entries of arithmetic.  The CTA stages its units' query heads in shared memory
// as floats [unit][i][e][h], issues its first batch of rows, derives each head's scale from
// the bound A_h = max_i fmaf-chain(|q̄_i,e|, Cabs[ci][e]) (one chain per (unit, group) per
// thread, shared-memory max -- the same value in every CTA), then computes every entry t (the
// oracle's FMA chain) and stores the packed G x int16 clamp(rint(t * 2^e_h)).
// quant_t_d in the magic-number domain ("magic quantizer"): y = fmaf(t, 2^e, 1.5 * 2^23) is
// 1.5 * 2^23 + rint(t * 2^e) (t * 2^e is exact, or below 2^-126 and rounds to 0 either way;
// the magic is even, so ties still go to even), clamped to +-32767 around the magic; the low
// 16 bits of y's encoding are then rint's two's complement.  Equal to quant_t_d for every
// finite t (a huge |t * 2^e| lands past the clamp, like quant_t_d's pre-clamp).  A magic of
// 1.5 * 2^23 + 32768 (also even) yields r + 32768, the scan's biased even-head field.

template <int DBAR>
struct TBatch {  // codebook rows in flight per thread (registers: kTBatch * DBAR floats)
  static constexpr int n = DBAR == 1 ? 16 : (DBAR == 2 ? 8 : (DBAR == 4 ? 4 : 2));
};

template <int DBAR>
__device__ __forceinline__ void load_centroid(const float *cp, bool ok, float (&cm)[DBAR]) {
  if (!ok) {
#pragma unroll
    for (int e = 0; e < DBAR; ++e) cm[e] = 0.0f;
    return;
  }
  if constexpr (DBAR % 4 == 0) {  // 16-B codebook loads (rows are DBAR*4-B aligned)
#pragma unroll
    for (int e = 0; e < DBAR; e += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(cp + e));
      cm[e] = v.x; cm[e + 1] = v.y; cm[e + 2] = v.z; cm[e + 3] = v.w;
    }
  } else if constexpr (DBAR == 2) {
    const float2 v = __ldg(reinterpret_cast<const float2 *>(cp));
    cm[0] = v.x; cm[1] = v.y;
  } else {
#pragma unroll
    for (int e = 0; e < DBAR; ++e) cm[e] = __ldg(cp + e);
  }
}

template <int G, int DBAR, bool L8>
__global__ void __launch_bounds__(kTB, DBAR <= 4 ? 4 : 2) k_table(LayerArgs a) {
  pdl_trigger();
  pdl_wait();
  const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int64_t nct = (int64_t)gridDim.x * gridDim.y;
  if (a.gdone && cta == 0)
    for (int t = threadIdx.x; t < a.gdone_n; t += blockDim.x) a.gdone[t] = 0u;
  if (a.skctr && cta == 1 % nct)
    for (int t = threadIdx.x; t < a.skctr_n; t += blockDim.x) a.skctr[t] = 0u;
  if (a.sel_ghist) {  // the selection's coarse (count u32, mass u64) histograms: every CTA clears its slice
    const int64_t nw = (int64_t)a.B * a.Hq * kNB * 3 / 4;  // uint4 words
    uint4 *gh = reinterpret_cast<uint4 *>(a.sel_ghist);
    for (int64_t t = nw * cta / nct + threadIdx.x; t < nw * (cta + 1) / nct; t += blockDim.x)
      gh[t] = make_uint4(0u, 0u, 0u, 0u);
  }
  const int units = a.B * a.Hkv;
  const int u0 = blockIdx.y * a.tunits, nu = min(a.tunits, units - u0);
  const int part = blockIdx.x, parts = gridDim.x;
  if (a.scan_split > 1 && a.n_q > 0) {  // the split scan accumulates into z: zero [0, n_q)
    const int64_t nz4 = (a.n_q + 3) / 4;  // float4s per row (rows are 64-float aligned)
    for (int r = 0; r < nu * G; ++r) {     // the chunk's rows b * Hq + kv * G + h = u * G + h
      float4 *zr = reinterpret_cast<float4 *>(a.z + ((int64_t)u0 * G + r) * a.z_stride);
      for (int64_t q = (int64_t)part * blockDim.x + threadIdx.x; q < nz4; q += (int64_t)parts * blockDim.x)
        zr[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  const int lg = 31 - __clz(a.cpow2);
  const int E = a.g << lg;  // <= 2^24 (g <= 256, cpow2 <= 2^16)
  const int e0 = (int)(((int64_t)E * part / parts) & ~(int64_t)31);
  const int e1 = part + 1 == parts ? E : (int)(((int64_t)E * (part + 1) / parts) & ~(int64_t)31);
  constexpr int NB = TBatch<DBAR>::n;
  // the CTA walks its groups i in [i_lo, i_hi]; in group i it owns centroids [mlo, mhi)
  const int i_lo = e0 >> lg, i_hi = e1 > e0 ? (e1 - 1) >> lg : i_lo - 1;
  float cmb[NB][DBAR];  // one batch of codebook rows: centroids m + ub * kTB
  auto load_batch = [&](int i, int m, int mc) {
    const float *Cg = a.C + (int64_t)(a.cbg == 1 ? 0 : i) * a.c * DBAR;
#pragma unroll
    for (int ub = 0; ub < NB; ++ub) {
      const int mm = m + ub * kTB;
      const bool ok = mm < mc;  // centroids m >= c are rows of zeros -> entries 0
      load_centroid<DBAR>(Cg + (int64_t)(ok ? mm : 0) * DBAR, ok, cmb[ub]);
    }
  };
  auto group_range = [&](int i, int &mlo, int &mhi) {
    const int gb = i << lg;
    mlo = max(e0 - gb, 0);
    mhi = min(e1 - gb, a.cpow2);
  };
  {  // the first batch: in flight while the scales are derived
    int mlo, mhi;
    group_range(i_lo, mlo, mhi);
    if (i_lo <= i_hi) load_batch(i_lo, mlo + (int)threadIdx.x, min(mhi, a.c));
  }
  // the chunk's query heads, [unit][d][G] floats (unit uu = u0 + uu: rows (u * G + h) of q)
  __shared__ __align__(16) float qsm[kTableQ];
  __shared__ int sA[kTableU][G];  // per-head bound A (non-negative floats order as ints)
  const int dG = a.d * G;
  for (int uu = 0; uu < nu; ++uu)  // consecutive threads write consecutive floats (no conflicts)
    for (int t = threadIdx.x; t < dG; t += kTB)
      qsm[uu * dG + t] = h2f(__ldg(a.q + ((int64_t)(u0 + uu) * G + t % G) * a.d + t / G));
  if (threadIdx.x < kTableU * G) sA[threadIdx.x / G][threadIdx.x % G] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < nu * a.g; t += kTB) {  // one (unit, group) chain per thread
    const int uu = t / a.g, gi = t - uu * a.g;
    const float *ca = a.cb_absmax + (int64_t)(a.cbg == 1 ? 0 : gi) * DBAR;
    const float *qg = qsm + uu * dG + gi * DBAR * G;
    // lanes of the same unit reduce first (bounds are non-negative: they order as unsigned)
    const unsigned grp = __match_any_sync(__activemask(), uu);
    const bool lead = (threadIdx.x & 31) == __ffs(grp) - 1;
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float bb = __fmul_rn(fabsf(qg[h]), __ldg(ca));
#pragma unroll
      for (int e = 1; e < DBAR; ++e) bb = __fmaf_rn(fabsf(qg[e * G + h]), __ldg(ca + e), bb);
      const unsigned mx = __reduce_max_sync(grp, __float_as_uint(bb));
      if (lead) atomicMax(&sA[uu][h], (int)mx);
    }
  }
  __syncthreads();
  __shared__ float2 ssc[kTableU][G >= 2 ? G / 2 : 1];  // (2^e_2p, 2^e_2p+1) per unit
  if (threadIdx.x < nu * G) {
    const int uu = threadIdx.x / G, h = threadIdx.x % G;
    const float A = __int_as_float(sA[uu][h]);
    const int e = L8 ? scale_exponent8(A) : scale_exponent(A);
    reinterpret_cast<float *>(&ssc[uu][0])[h] = pow2f(e);
    if (part == 0) {
      HeadState *hs = a.hs + (int64_t)(u0 + uu) * G + h;  // row b * Hq + kv * G + h
      hs->e = e;
      hs->kappa = __fmul_rn(a.kappa0, pow2f(-e));
      hs->amax = __float_as_uint(A);
      hs->M = INT_MIN;     // folded by the scan / resident epilogues (atomics)
      hs->zmin = INT_MAX;
      hs->S = 0ull;        // the selection's accumulators and counters (hc_select_pass.cu)
      hs->mass_before = 0ull;
      hs->c1_done = 0u;
      hs->c2_done = 0u;
      hs->ticket = 0u;
      hs->state = 0u;
    }
  }
  if (G == 1 && threadIdx.x < nu) ssc[threadIdx.x][0].y = 1.0f;
  __syncthreads();
  // heads in pairs for the packed fp32x2 FMA (every lane an IEEE fmaf, as the oracle's chain);
  // the magic quantizer: even heads' magic carries the +32768 bias
  constexpr int NP = G >= 2 ? G / 2 : 1;
  constexpr float kMe = G >= 2 ? 12582912.0f + 32768.0f : 12582912.0f;
  const float2 mg = make_float2(kMe, 12582912.0f);
  bool have = true;  // cmb holds the first batch of group i_lo
  for (int i = i_lo; i <= i_hi; ++i) {
    int mlo, mhi;
    group_range(i, mlo, mhi);
    const int mc = min(mhi, a.c);
    for (int m = mlo + (int)threadIdx.x; m < mhi; m += kTB * NB) {
      if (!have) load_batch(i, m, mc);
      have = false;
      for (int uu = 0; uu < nu; ++uu) {
        float2 qp[NP][DBAR];  // (q_2p, q_2p+1) of unit uu, group i, component k
        const float *qg = qsm + uu * dG + i * DBAR * G;
#pragma unroll
        for (int k = 0; k < DBAR; ++k)
#pragma unroll
          for (int p = 0; p < NP; ++p)
            qp[p][k] = G >= 2 ? make_float2(qg[k * G + 2 * p], qg[k * G + 2 * p + 1]) : make_float2(qg[k * G], 0.0f);
        float2 sp[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) sp[p] = ssc[uu][p];
        const int64_t u = u0 + uu;
        int16_t *Tg = a.T + ((int64_t)u * E + (i << lg)) * G;
#pragma unroll
        for (int ub = 0; ub < NB; ++ub) {
          const int mm = m + ub * kTB;
          if (mm >= mhi) break;
          float2 t[NP];  // the R2 FMA chain
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            t[p] = __fmul2_rn(qp[p][0], make_float2(cmb[ub][0], cmb[ub][0]));
#pragma unroll
            for (int k = 1; k < DBAR; ++k) t[p] = __ffma2_rn(qp[p][k], make_float2(cmb[ub][k], cmb[ub][k]), t[p]);
          }
          if constexpr (G == 4 && L8) {  // R2b: 4 x (int8 + 128) packed in one u32, head h at byte h
            const float th[4] = {t[0].x, t[0].y, t[NP - 1].x, t[NP - 1].y};
            const float sh[4] = {sp[0].x, sp[0].y, sp[NP - 1].x, sp[NP - 1].y};
            uint32_t wv = 0;
#pragma unroll
            for (int h = 0; h < 4; ++h) wv |= (uint32_t)(quant_t8_d(th[h], sh[h]) + 128) << (8 * h);
            reinterpret_cast<uint32_t *>(a.T)[u * E + (i << lg) + mm] = wv;
          } else {
            uint32_t w[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) {
              float2 y = __ffma2_rn(t[p], sp[p], mg);
              y.x = fminf(fmaxf(y.x, kMe - 32767.0f), kMe + 32767.0f);
              y.y = fminf(fmaxf(y.y, 12582912.0f - 32767.0f), 12582912.0f + 32767.0f);
              w[p] = __byte_perm(__float_as_uint(y.x), __float_as_uint(y.y), 0x5410);
            }
            // even heads are stored biased by +32768 (an unsigned 16-bit field under the odd
            // head's signed one), so the scan adds a whole 32-bit word per head pair (hc_scan.cu Lut)
            if constexpr (G == 4) {
              *reinterpret_cast<uint2 *>(Tg + mm * 4) = make_uint2(w[0], w[NP - 1]);
            } else if constexpr (G == 2) {
              *reinterpret_cast<uint32_t *>(Tg + mm * 2) = w[0];
            } else {
              Tg[mm] = (int16_t)(uint16_t)w[0];
            }
          }
        }
      }
    }
    have = false;
  }
}

template <int G, int DBAR>
static cudaError_t table_g_d(const LayerArgs &a, cudaStream_t s) {
  dim3 grid((unsigned)a.tsplit, (unsigned)((a.B * a.Hkv + a.tunits - 1) / a.tunits));
  if (G == 4 && a.lut8)
    launch_chain(k_table<G, DBAR, true>, grid, dim3(kTB), 0, s, a);
  else
    launch_chain(k_table<G, DBAR, false>, grid, dim3(kTB), 0, s, a);
  note_launch();
  return cudaGetLastError();
}

template <int G>
static cudaError_t table_g(const LayerArgs &a, cudaStream_t s) {
  switch (a.dbar) {
    case 1: return table_g_d<G, 1>(a, s);
    case 2: return table_g_d<G, 2>(a, s);
    case 4: return table_g_d<G, 4>(a, s);
    case 8: return table_g_d<G, 8>(a, s);
    case 16: return table_g_d<G, 16>(a, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_table(const LayerArgs &a, cudaStream_t s) {
  switch (a.G) {
    case 1: return table_g<1>(a, s);
    case 2: return table_g<2>(a, s);
    case 4: return table_g<4>(a, s);
  }
  return cudaErrorInvalidValue;
}

// Cabs[l][ci][e] = max_m |C[l][ci][m][e]| (R2's codebook constant); one CTA per (l, ci)
__global__ void __launch_bounds__(256) k_cbabs(const float *C, int c, int dbar, float *out) {
  const int64_t slice = (int64_t)blockIdx.x;  // l * cbg + ci
  const float *Cs = C + slice * c * dbar;
  float mx[16];
  for (int e = 0; e < 16; ++e) mx[e] = 0.0f;
  for (int m = threadIdx.x; m < c; m += 256)
    for (int e = 0; e < dbar; ++e) mx[e] = fmaxf(mx[e], fabsf(Cs[(int64_t)m * dbar + e]));
  __shared__ float red[16][8];
  for (int e = 0; e < dbar; ++e) {
    float v = mx[e];
    for (int off = 16; off > 0; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
    if ((threadIdx.x & 31) == 0) red[e][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < dbar) {
    float v = 0.0f;
    for (int w = 0; w < 8; ++w) v = fmaxf(v, red[threadIdx.x][w]);
    out[slice * dbar + threadIdx.x] = v;
  }
}

cudaError_t launch_cbabs(const float *C, int64_t slices, int c, int dbar, float *out, cudaStream_t s) {
  if (slices <= 0) return cudaSuccess;
  k_cbabs<<<(unsigned)slices, 256, 0, s>>>(C, c, dbar, out);
  note_launch();
  return cudaGetLastError();
}

// Resident (exact-key) tokens, R3: z = rint(clamp(fmaf-chain_e(q_e * k_e) * 2^e_h)).  Also the
// dense scan of the value-offload-only mode (every token resident, n_q = 0).
// CTA = (unit, tile of kRT tokens); the tile's key rows are staged in shared memory with
// coalesced 16-B loads (row stride padded by 4 B so the 8 tokens of a warp hit 8 banks),
// then thread (token, head) runs the FMA chain in ascending e over half2 pairs.
constexpr int kRT = 128;  // tokens per CTA (kRT * G threads for G = 4)

template <int G>
__global__ void __launch_bounds__(kRT * G) k_resident(LayerArgs a) {
  extern __shared__ __align__(16) uint8_t rsm[];
  pdl_trigger();
  pdl_wait();
  const int u = blockIdx.y;
  const int b = u / a.Hkv, kv = u - b * a.Hkv;
  const int d = a.d;
  const int rowb = d * 2 + 4;                   // padded row stride (bytes)
  float *qs = reinterpret_cast<float *>(rsm);   // [G][d]
  uint8_t *ks = rsm + G * d * 4;                // [kRT][rowb]
  const int64_t r0 = (int64_t)blockIdx.x * kRT;
  const int nthr = kRT * G;
  for (int i = threadIdx.x; i < G * d; i += nthr)
    qs[i] = h2f(a.q[((int64_t)b * a.Hq + kv * G + i / d) * d + i % d]);
  const int per_row = d / 8;  // 16-B pieces per row
  for (int i = threadIdx.x; i < kRT * per_row; i += nthr) {
    const int t = i / per_row, pc = i % per_row;
    const int64_t r = r0 + t;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < a.n_res) {
      const int64_t slot = (a.res_slot0 + r) % a.res_cap;
      v = *reinterpret_cast<const uint4 *>(a.res_k + (int64_t)b * a.res_b_stride +
                                           ((int64_t)kv * a.res_cap + slot) * d + pc * 8);
    }
    uint32_t *dst = reinterpret_cast<uint32_t *>(ks + t * rowb + pc * 16);
    dst[0] = v.x; dst[1] = v.y; dst[2] = v.z; dst[3] = v.w;  // 4-B aligned (padded rows)
  }
  __syncthreads();
  const int t = threadIdx.x / G, h = threadIdx.x % G;
  const int64_t r = r0 + t;
  if (r >= a.n_res) return;
  const __half2 *krow = reinterpret_cast<const __half2 *>(ks + t * rowb);
  const float *qh = qs + h * d;
  float acc = 0.0f;
  for (int e2 = 0; e2 < d / 2; ++e2) {
    const float2 kf = __half22float2(krow[e2]);
    acc = __fmaf_rn(qh[2 * e2], kf.x, acc);
    acc = __fmaf_rn(qh[2 * e2 + 1], kf.y, acc);
  }
  const int hq = kv * G + h;
  HeadState *hsr = a.hs + (int64_t)b * a.Hq + hq;
  const int zq = quant_res(acc, pow2f(hsr->e));
  a.z[((int64_t)b * a.Hq + hq) * a.z_stride + a.n_q + r] = (float)zq;
  atomicMax(&hsr->M, zq);
  atomicMin(&hsr->zmin, zq);
}

cudaError_t launch_resident(const LayerArgs &a, cudaStream_t s) {
  if (a.n_res <= 0) return cudaSuccess;
  // with no quantized tokens (value-offload-only mode) this IS the key scan: profile it
  cudaEvent_t eb = nullptr, ee = nullptr;
  unsigned evflag = 0;
  if (a.n_q == 0) {
    scan_events(&eb, &ee);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    evflag = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
    if (eb) cudaEventRecordWithFlags(eb, s, evflag);
  }
  dim3 grid((unsigned)((a.n_res + kRT - 1) / kRT), (unsigned)(a.B * a.Hkv));
  const size_t smem = (size_t)a.G * a.d * 4 + (size_t)kRT * (a.d * 2 + 4);
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {  // d = 256 needs > 48 KiB
    cudaFuncSetAttribute(k_resident<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(k_resident<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(k_resident<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    configured[dev] = 1;
  }
  switch (a.G) {
    case 1: launch_chain(k_resident<1>, grid, dim3(kRT * 1), smem, s, a); break;
    case 2: launch_chain(k_resident<2>, grid, dim3(kRT * 2), smem, s, a); break;
    case 4: launch_chain(k_resident<4>, grid, dim3(kRT * 4), smem, s, a); break;
    default: return cudaErrorInvalidValue;
  }
  note_launch();
  if (ee) cudaEventRecordWithFlags(ee, s, evflag);
  return cudaGetLastError();
}

}  // namespace hc
