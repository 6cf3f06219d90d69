// hc_group.cu -- NEXT f3(iii): ONE Eq. 4 selection per KV head, shared
// by its G query heads (DESIGN.md §2 R8).  The kept set is chosen on the head-averaged
// attention distribution ā_j = (1/G) Σ_h ã_{h,j} in exact integers:
//   W_{h,j} = R4 mass (own M_h, κ_h), S_h = Σ_j W_{h,j}, ρ_h = floor((2^104-1)/S_h),
//   A_j = Σ_h floor(W_{h,j}·ρ_h / 2^64)   (≈ G·2^40·ā_j, < 2^43),
//   order (A desc, j asc), Θ = ceil(τ_q·S_A/2^24), k_sel = min(k*, k_max);
// each head then sums its OWN weights W_{h,j}/S_h over the shared rows (Eq. 5),
// so one value row serves G heads: up to G x fewer gathered bytes.
//
// A is not a function of one score, so the Δ-space select of hc_select_fused does not
// apply.  The selection here is a 4-level radix select on the 48-bit order key
//   D = 2^48 - 1 - K(A),  K(A) = (e+1)·2^42 + (A - 2^e)·2^(42-e),  e = floor(log2 A)
// (K(0) = 0): D is injective and ascending in the kept order, so 4 x 12-bit levels resolve
// the exact boundary key D* -- each level a (count, mass) histogram pass over the G score
// rows plus a one-CTA bound, like bound1/bound2 of R5.  Then chunk counts, and an ordered
// compaction that writes the same index list to the G query-head rows.
#include "hc_internal.h"

namespace hc {

constexpr int kGrT = 256;        // threads of the pass kernels
constexpr int kGrChunk = 4096;   // tokens per count / compaction chunk (16 per thread)
constexpr int kGrLevels = 4;

__device__ __forceinline__ uint64_t grp_key(uint64_t A) {  // D: ascending = kept first
  uint64_t K = 0;
  if (A) {
    const int e = 63 - __clzll((long long)A);
    K = ((uint64_t)(e + 1) << 42) | ((A - (1ull << e)) << (42 - e));
  }
  return ((1ull << 48) - 1) - K;
}

__device__ __forceinline__ uint64_t grp_key_to_A(uint64_t D) {
  const uint64_t K = ((1ull << 48) - 1) - D;
  const int e1 = (int)(K >> 42);
  if (!e1) return 0;
  const int e = e1 - 1;
  return (1ull << e) + ((K & ((1ull << 42) - 1)) >> (42 - e));
}

// per-unit (b, kv) context loaded by every pass kernel
struct GrpCtx {
  const float *z[4];
  int32_t M[4];
  float kappa[4];
  uint64_t rho[4];
};

template <int G>
__device__ __forceinline__ void grp_ctx(const LayerArgs &a, int u, GrpCtx &c) {
  const int b = u / a.Hkv, kv = u - b * a.Hkv;
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const int row = b * a.Hq + kv * G + h;
    const HeadState &hs = a.hs[row];
    c.z[h] = a.z + (int64_t)row * a.z_stride;
    c.M[h] = hs.M;
    c.kappa[h] = hs.kappa;
    c.rho[h] = a.grp[u].rho[h];
  }
}

// split scans leave M unfolded: M = max z over the quantized tokens (atomicMax), z final
__global__ void __launch_bounds__(kGrT) k_grp_fin(LayerArgs a, int) {
  const int row = blockIdx.y;
  const float *zr = a.z + (int64_t)row * a.z_stride;
  const int64_t nq = a.n_q;
  int mx = INT_MIN;
  for (int64_t t = ((int64_t)blockIdx.x * kGrT + threadIdx.x) * 4; t < nq; t += (int64_t)gridDim.x * kGrT * 4) {
    if (t + 4 <= nq) {
      const float4 v = *reinterpret_cast<const float4 *>(zr + t);
      mx = max(max(mx, zint(v.x)), max(zint(v.y), max(zint(v.z), zint(v.w))));
    } else {
      for (int u = 0; u < 4 && t + u < nq; ++u) mx = max(mx, zint(zr[t + u]));
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx != INT_MIN) atomicMax(&a.hs[row].M, mx);
}

__device__ __forceinline__ void ld_z4(const float *zr, int64_t t, int64_t n, float (&v)[4]) {
  if (t + 4 <= n) {
    const float4 q = *reinterpret_cast<const float4 *>(zr + t);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = t + u < n ? zr[t + u] : 0.0f;
  }
}

// S_h = Σ_j W_{h,j} (u64 atomics; hs.S zeroed by k_grp_init)
__global__ void __launch_bounds__(kGrT) k_grp_mass(LayerArgs a) {
  const int row = blockIdx.y;
  const HeadState &hs = a.hs[row];
  const int M = hs.M;
  const float kappa = hs.kappa;
  const float *zr = a.z + (int64_t)row * a.z_stride;
  const int64_t n = a.n_cand;
  unsigned long long S = 0;
  for (int64_t t = ((int64_t)blockIdx.x * kGrT + threadIdx.x) * 4; t < n; t += (int64_t)gridDim.x * kGrT * 4) {
    float v[4];
    ld_z4(zr, t, n, v);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u < n) S += mass_d((uint32_t)(M - zint(v[u])), kappa);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
  if ((threadIdx.x & 31) == 0 && S) atomicAdd((unsigned long long *)&a.hs[row].S, S);
}

__global__ void k_grp_init(LayerArgs a, int units) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < units) {
    GroupState g{};
    a.grp[i] = g;
  }
  if (i < units * a.G) a.hs[i].S = 0;  // rows = units * G
}

// ρ_h = floor((2^104 - 1) / S_h), S_h >= 2^40 (the max token has W = 2^40)
__global__ void k_grp_rho(LayerArgs a, int units) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= units * a.G) return;
  const int u = i / a.G, h = i - u * a.G;
  const unsigned __int128 num = ((unsigned __int128)1 << 104) - 1;
  const uint64_t S = a.hs[i].S;
  a.grp[u].rho[h] = S ? (uint64_t)(num / S) : 0ull;
}

__device__ __forceinline__ void hist_add(uint32_t *cnt, uint32_t *mlo, uint32_t *mhi, int bk, uint64_t A) {
  atomicAdd(&cnt[bk], 1u);
  if (A) {
    const uint32_t wl = (uint32_t)A;
    uint32_t wh = (uint32_t)(A >> 32);
    const uint32_t old = atomicAdd(&mlo[bk], wl);
    wh += (old + wl < old) ? 1u : 0u;
    if (wh) atomicAdd(&mhi[bk], wh);
  }
}

__device__ __forceinline__ void hist_flush(const uint32_t *cnt, const uint32_t *mlo, const uint32_t *mhi,
                                           unsigned long long *hr) {
  for (int i = threadIdx.x; i < kNB; i += kGrT) {
    if (cnt[i]) {
      atomicAdd(&hr[2 * i], (unsigned long long)cnt[i]);
      atomicAdd(&hr[2 * i + 1], ((unsigned long long)mhi[i] << 32) + mlo[i]);
    }
  }
}

// level 0: A_j from the G score rows (4 consecutive tokens per thread), store the order key
// D_j for the later passes, (count, mass) histogram of D's top 12 bits
template <int G>
__global__ void __launch_bounds__(kGrT) k_grp_hist0(LayerArgs a) {
  __shared__ uint32_t cnt[kNB], mlo[kNB], mhi[kNB];
  const int u = blockIdx.y;
  GrpCtx c;
  grp_ctx<G>(a, u, c);
  for (int i = threadIdx.x; i < kNB; i += kGrT) { cnt[i] = 0; mlo[i] = 0; mhi[i] = 0; }
  __syncthreads();
  const int64_t n = a.n_cand;
  unsigned long long *key = a.grp_key + (int64_t)u * a.z_stride;
  for (int64_t t = ((int64_t)blockIdx.x * kGrT + threadIdx.x) * 4; t < n; t += (int64_t)gridDim.x * kGrT * 4) {
    float v[G][4];
#pragma unroll
    for (int h = 0; h < G; ++h) ld_z4(c.z[h], t, n, v[h]);
    uint64_t A[4], D[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      A[k] = 0;
#pragma unroll
      for (int h = 0; h < G; ++h)
        A[k] += __umul64hi(mass_d((uint32_t)(c.M[h] - zint(v[h][k])), c.kappa[h]), c.rho[h]);
      D[k] = t + k < n ? grp_key(A[k]) : ~0ull;
    }
    *reinterpret_cast<ulonglong2 *>(key + t) = make_ulonglong2(D[0], D[1]);
    *reinterpret_cast<ulonglong2 *>(key + t + 2) = make_ulonglong2(D[2], D[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (t + k < n) hist_add(cnt, mlo, mhi, (int)(D[k] >> 36), A[k]);
  }
  __syncthreads();
  hist_flush(cnt, mlo, mhi, a.grp_hist + (int64_t)u * kGrLevels * kNB * 2);
}

// levels 1..3: histogram of the next 12 key bits of the tokens inside the prefix bucket
__global__ void __launch_bounds__(kGrT) k_grp_hist(LayerArgs a, int lv) {
  __shared__ uint32_t cnt[kNB], mlo[kNB], mhi[kNB];
  const int u = blockIdx.y;
  const GroupState &gs = a.grp[u];
  if (gs.done) return;
  const int sh_bin = 36 - 12 * lv, sh_pre = 48 - 12 * lv;
  const uint64_t pre = gs.prefix >> sh_pre;
  for (int i = threadIdx.x; i < kNB; i += kGrT) { cnt[i] = 0; mlo[i] = 0; mhi[i] = 0; }
  __syncthreads();
  const int64_t n = a.n_cand;
  const unsigned long long *key = a.grp_key + (int64_t)u * a.z_stride;
  for (int64_t t = ((int64_t)blockIdx.x * kGrT + threadIdx.x) * 4; t < n; t += (int64_t)gridDim.x * kGrT * 4) {
    const ulonglong2 k01 = *reinterpret_cast<const ulonglong2 *>(key + t);
    const ulonglong2 k23 = *reinterpret_cast<const ulonglong2 *>(key + t + 2);
    const uint64_t D[4] = {k01.x, k01.y, k23.x, k23.y};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (t + k < n && (D[k] >> sh_pre) == pre)
        hist_add(cnt, mlo, mhi, (int)((D[k] >> sh_bin) & (kNB - 1)), grp_key_to_A(D[k]));
  }
  __syncthreads();
  hist_flush(cnt, mlo, mhi, a.grp_hist + ((int64_t)u * kGrLevels + lv) * kNB * 2);
}

// one CTA (1024 threads, 4 bins each) per unit: locate the boundary bin of level lv
constexpr int kGrB = 1024;
__global__ void __launch_bounds__(kGrB) k_grp_bound(LayerArgs a, int lv) {
  __shared__ unsigned long long sx[kGrB / 32], sy[kGrB / 32];
  __shared__ int s_found;
  const int u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  GroupState &gs = a.grp[u];
  if (gs.done) return;
  const unsigned long long *hr = a.grp_hist + ((int64_t)u * kGrLevels + lv) * kNB * 2;
  unsigned long long c[4], m[4], lc = 0, lm = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c[k] = hr[2 * (tid * 4 + k)];
    m[k] = hr[2 * (tid * 4 + k) + 1];
    lc += c[k];
    lm += m[k];
  }
  unsigned long long ic = lc, im = lm;  // inclusive warp scan
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long oc = __shfl_up_sync(0xffffffffu, ic, off);
    const unsigned long long om = __shfl_up_sync(0xffffffffu, im, off);
    if (lane >= off) { ic += oc; im += om; }
  }
  if (lane == 31) { sx[w] = ic; sy[w] = im; }
  if (tid == 0) s_found = kNB;
  __syncthreads();
  unsigned long long bc = 0, bm = 0, tc = 0, tm = 0;
  for (int k = 0; k < kGrB / 32; ++k) {
    if (k < w) { bc += sx[k]; bm += sy[k]; }
    tc += sx[k]; tm += sy[k];
  }
  bc += ic - lc;  // exclusive prefix of this thread's first bin
  bm += im - lm;
  const bool tau_all = a.tau_q >= (1u << 24);
  if (lv == 0) {  // totals over all candidates: S_A, Θ (all threads compute the same values)
    const unsigned long long theta = tau_all ? 0ull : threshold(a.tau_q, tm);
    if (tid == 0) { gs.SA = tm; gs.theta = theta; gs.ntot = tc; }
    __syncthreads();
  }
  const unsigned long long theta = lv == 0 ? (tau_all ? 0ull : threshold(a.tau_q, tm)) : gs.theta;
  const unsigned long long ntot = lv == 0 ? tc : gs.ntot;
  const bool cap_all = (unsigned long long)a.k_max >= ntot;
  const unsigned long long cb0 = gs.cb, mb0 = gs.mb;
  unsigned long long cc = cb0 + bc, cm = mb0 + bm;
  int found = kNB;
  unsigned long long f_cc = 0, f_cm = 0, f_c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool trig = c[k] && ((!tau_all && cm + m[k] >= theta) ||
                               (!cap_all && cc + c[k] >= (unsigned long long)a.k_max));
    if (trig && found == kNB) { found = tid * 4 + k; f_cc = cc; f_cm = cm; f_c = c[k]; }
    cc += c[k];
    cm += m[k];
  }
  if (found < kNB) atomicMin(&s_found, found);
  __syncthreads();
  if (lv == 0 && s_found == kNB) {  // no boundary: keep every candidate
    if (tid == 0) {
      gs.done = 1;
      gs.dstar = 1ull << 48;  // > every key
      gs.r_ties = 0;
      gs.ksel = (long long)ntot;
      gs.kstar = (long long)ntot;
    }
    return;
  }
  if (found < kNB && found == s_found) {
    const int sh_bin = 36 - 12 * lv;
    const uint64_t prefix = gs.prefix | ((uint64_t)found << sh_bin);
    if (lv < kGrLevels - 1) {
      gs.prefix = prefix;
      gs.cb = f_cc;
      gs.mb = f_cm;
    } else {  // exact key D* = prefix: every token in the bin has the same A*
      const uint64_t As = grp_key_to_A(prefix);
      unsigned long long r_tau = ~0ull, r_cap = ~0ull;
      if (!tau_all && As && f_cm + f_c * As >= theta) {
        r_tau = (theta - f_cm + As - 1) / As;
        if (r_tau == 0) r_tau = 1;
      }
      if (f_cc + f_c >= (unsigned long long)a.k_max) r_cap = (unsigned long long)a.k_max - f_cc;
      const unsigned long long r = r_tau < r_cap ? r_tau : r_cap;
      gs.dstar = prefix;
      gs.r_ties = r;
      gs.ksel = (long long)(f_cc + r);
      gs.kstar = r_tau <= r_cap ? (long long)(f_cc + r_tau) : -1;
      gs.done = 1;
    }
  }
}

// per chunk: (#D < D*, #D == D*)
__global__ void __launch_bounds__(kGrT) k_grp_count(LayerArgs a, int nch) {
  const int u = blockIdx.y, ch = blockIdx.x;
  const GroupState &gs = a.grp[u];
  const uint64_t ds = gs.dstar;
  const unsigned long long *key = a.grp_key + (int64_t)u * a.z_stride;
  const int64_t n = a.n_cand;
  unsigned ns = 0, nt = 0;
#pragma unroll
  for (int k = 0; k < kGrChunk / kGrT / 4; ++k) {
    const int64_t t = (int64_t)ch * kGrChunk + ((int64_t)k * kGrT + threadIdx.x) * 4;
    if (t < n) {
      const ulonglong2 k01 = *reinterpret_cast<const ulonglong2 *>(key + t);
      const ulonglong2 k23 = *reinterpret_cast<const ulonglong2 *>(key + t + 2);
      const uint64_t D[4] = {k01.x, k01.y, k23.x, k23.y};
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // tail keys are ~0: never < or == D* (< 2^48 + 1)
        ns += D[q] < ds;
        nt += D[q] == ds;
      }
    }
  }
  __shared__ unsigned s_s[kGrT / 32], s_t[kGrT / 32];
  ns = __reduce_add_sync(0xffffffffu, ns);
  nt = __reduce_add_sync(0xffffffffu, nt);
  if ((threadIdx.x & 31) == 0) { s_s[threadIdx.x >> 5] = ns; s_t[threadIdx.x >> 5] = nt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned S0 = 0, T0 = 0;
    for (int k = 0; k < kGrT / 32; ++k) { S0 += s_s[k]; T0 += s_t[k]; }
    a.grp_chunk[((int64_t)u * nch + ch) * 2] = S0;
    a.grp_chunk[((int64_t)u * nch + ch) * 2 + 1] = T0;
  }
}

// ordered compaction: thread t owns tokens j0 + 16t .. +15 (ascending); kept = D < D* or
// one of the first r_ties ties (lowest indices) -> the same index list for the G rows,
// each row with its own weight W_{h,j} / S_h
template <int G>
__global__ void __launch_bounds__(kGrT) k_grp_compact(LayerArgs a, int nch) {
  constexpr int kPT = kGrChunk / kGrT;
  const int u = blockIdx.y, ch = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const GroupState &gs = a.grp[u];
  const int b = u / a.Hkv, kv = u - b * a.Hkv;
  GrpCtx c;
  grp_ctx<G>(a, u, c);
  __shared__ unsigned long long s_pre[2];
  __shared__ unsigned s_ws[kGrT / 32], s_wt[kGrT / 32];
  if (tid < 32) {  // tokens of earlier chunks
    unsigned long long ps = 0, pt = 0;
    for (int k = tid; k < ch; k += 32) {
      ps += a.grp_chunk[((int64_t)u * nch + k) * 2];
      pt += a.grp_chunk[((int64_t)u * nch + k) * 2 + 1];
    }
    for (int off = 16; off; off >>= 1) {
      ps += __shfl_xor_sync(0xffffffffu, ps, off);
      pt += __shfl_xor_sync(0xffffffffu, pt, off);
    }
    if (tid == 0) { s_pre[0] = ps; s_pre[1] = pt; }
  }
  const int64_t j0 = (int64_t)ch * kGrChunk + (int64_t)tid * kPT;
  const unsigned long long *key = a.grp_key + (int64_t)u * a.z_stride;
  uint64_t D[kPT];
  unsigned ns = 0, nt = 0;
#pragma unroll
  for (int k = 0; k < kPT; k += 2) {
    ulonglong2 kk = make_ulonglong2(~0ull, ~0ull);
    if (j0 + k < a.n_cand) kk = *reinterpret_cast<const ulonglong2 *>(key + j0 + k);
    D[k] = kk.x;
    D[k + 1] = j0 + k + 1 < a.n_cand ? kk.y : ~0ull;
  }
#pragma unroll
  for (int k = 0; k < kPT; ++k) {
    ns += D[k] < gs.dstar;
    nt += D[k] == gs.dstar;
  }
  unsigned is = ns, it = nt;  // inclusive warp scans
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned os = __shfl_up_sync(0xffffffffu, is, off);
    const unsigned ot = __shfl_up_sync(0xffffffffu, it, off);
    if (lane >= off) { is += os; it += ot; }
  }
  if (lane == 31) { s_ws[w] = is; s_wt[w] = it; }
  __syncthreads();
  unsigned long long sb = s_pre[0], tb = s_pre[1];
  for (int k = 0; k < w; ++k) { sb += s_ws[k]; tb += s_wt[k]; }
  sb += is - ns;  // strict tokens before my first token
  tb += it - nt;  // ties before my first token
  const unsigned long long r = gs.r_ties;
  unsigned long long pos = sb + (tb < r ? tb : r);
  float inv[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const uint64_t S = a.hs[b * a.Hq + kv * G + h].S;
    inv[h] = (float)(1.0 / (double)(S ? S : 1));
  }
  // stage this warp's kept tokens (ascending) in shared memory, then write them
  // lane-parallel: coalesced row stores, one weight per lane instead of divergent ones
  __shared__ uint32_t s_stg[kGrT / 32][32 * kPT];
  const unsigned long long wpos = __shfl_sync(0xffffffffu, pos, 0);
  unsigned q = (unsigned)(pos - wpos);
#pragma unroll
  for (int k = 0; k < kPT; ++k) {
    bool take = D[k] < gs.dstar;
    if (D[k] == gs.dstar) { take = tb < r; ++tb; }
    if (take) s_stg[w][q++] = (uint32_t)(tid * kPT + k);
  }
  const unsigned wtot = __shfl_sync(0xffffffffu, q, 31);
  __syncwarp();
  const int64_t cj0 = (int64_t)ch * kGrChunk;
  for (unsigned i = lane; i < wtot; i += 32) {
    const int64_t j = cj0 + s_stg[w][i];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const int row = b * a.Hq + kv * G + h;
      const uint32_t dl = (uint32_t)(c.M[h] - zint(c.z[h][j]));
      a.sel_idx[(int64_t)row * a.k_max + wpos + i] = (int32_t)j;
      a.sel_w[(int64_t)row * a.k_max + wpos + i] = __fmul_rn((float)mass_d(dl, c.kappa[h]), inv[h]);
    }
  }
  if (ch == 0 && tid < G) {
    const int row = b * a.Hq + kv * G + tid;
    a.hs[row].ksel = gs.ksel;
    a.hs[row].kstar = gs.kstar;
    a.hs[row].theta = gs.theta;
    if (a.sel_k) a.sel_k[row] = gs.ksel;
  }
}

int grp_chunks(int64_t n) { return (int)((n + kGrChunk - 1) / kGrChunk); }

template <int G>
static cudaError_t grp_run(const LayerArgs &a, int nsplit, cudaStream_t st) {
  const int units = a.B * a.Hkv, rows = units * G;
  const int64_t n = a.n_cand;
  cudaError_t e;
  if ((e = cudaMemsetAsync(a.grp_hist, 0, (size_t)units * kGrLevels * kNB * 16, st)) != cudaSuccess) return e;
  k_grp_init<<<(rows + 255) / 256, 256, 0, st>>>(a, units);
  note_launch();
  // pass grids: ~4 CTAs per SM over all rows / units
  auto pgrid = [&](int nrow) {
    int64_t x = ((int64_t)a.num_sms * 4 + nrow - 1) / nrow;
    const int64_t need = (n + kGrT * 16 - 1) / (kGrT * 16);
    if (x > need) x = need;
    return (unsigned)(x < 1 ? 1 : x);
  };
  if (nsplit > 1 && a.n_q > 0) {
    k_grp_fin<<<dim3(pgrid(rows), rows), kGrT, 0, st>>>(a, nsplit);
    note_launch();
  }
  k_grp_mass<<<dim3(pgrid(rows), rows), kGrT, 0, st>>>(a);
  note_launch();
  k_grp_rho<<<(rows + 127) / 128, 128, 0, st>>>(a, units);
  note_launch();
  for (int lv = 0; lv < kGrLevels; ++lv) {
    if (lv == 0) k_grp_hist0<G><<<dim3(pgrid(units), units), kGrT, 0, st>>>(a);
    else k_grp_hist<<<dim3(pgrid(units), units), kGrT, 0, st>>>(a, lv);
    k_grp_bound<<<units, kGrB, 0, st>>>(a, lv);
    note_launch(2);
  }
  const int nch = grp_chunks(n);
  k_grp_count<<<dim3(nch, units), kGrT, 0, st>>>(a, nch);
  k_grp_compact<G><<<dim3(nch, units), kGrT, 0, st>>>(a, nch);
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_group_select(const LayerArgs &a, int nsplit, cudaStream_t st) {
  switch (a.G) {
    case 1: return grp_run<1>(a, nsplit, st);
    case 2: return grp_run<2>(a, nsplit, st);
    case 4: return grp_run<4>(a, nsplit, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hc
