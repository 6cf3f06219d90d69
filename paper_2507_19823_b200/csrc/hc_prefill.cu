// hc_prefill.cu -- NEXT f4 (iii): App. B "Enhanced prefilling with block-wise attention"
// (DESIGN F5): query i of block kb = i / bs attends to the anchor block
// (keys j < bs) and, causally, to its own block (kb*bs <= j <= i); block 0 is causal.
//
// Flash-attention-style kernel on the tensor cores with warp-level mma.sync
// (m16n8k16, fp16 inputs, fp32 accumulate): CTA = 64 queries of one query head (4 warps x
// 16 rows), key tiles of 64 double-buffered in shared memory by cp.async, online softmax
// in fp32 (exp2 with log2(e)/sqrt(d) folded into the scale), P rounded to fp16 for the PV
// product.  Only the anchor tiles and the own-block tiles up to the diagonal are visited,
// so the work is O(n * 2 bs) instead of O(n^2).  d = 128.
//
// Two kernels: k_blockwise_attn_tc (default, bs % 128 == 0): tcgen05.mma with operands in
// 128B-swizzled shared memory (UMMA descriptors), S and O accumulators in TMEM, lazy softmax
// rescaling; k_blockwise_attn (mma.sync m16n8k16) for bs % 128 != 0 or HC_PREFILL_TC=0.
#include <stdlib.h>
#include <string.h>

#include "hc_internal.h"

namespace hc {

constexpr int kPD = 128;          // head dim
constexpr int kPBM = 64;          // queries per CTA
constexpr int kPBN = 64;          // keys per tile
constexpr int kPRow = kPD + 8;    // padded smem row (halves): conflict-free ldmatrix
constexpr int kPT = 128;          // threads

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;  // zero-fill rows past n
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void *p) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(s));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void *p) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(s));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2 (2^-inf = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t *>(&h);
}

struct PrefillArgs {
  const uint16_t *q, *k, *v;  // [n][Hq][d], [n][Hkv][d], [n][Hkv][d] fp16
  float *out;                 // [n][Hq][d]
  int64_t n, bs;
  int Hq, Hkv;
  float scale_log2;           // log2(e) / sqrt(d)
};

__global__ void __launch_bounds__(kPT) k_blockwise_attn(PrefillArgs a) {
  extern __shared__ __align__(16) uint16_t psm[];
  uint16_t *sQ = psm;                          // [64][kPRow]
  uint16_t *sK = sQ + kPBM * kPRow;            // [2][64][kPRow]
  uint16_t *sV = sK + 2 * kPBN * kPRow;        // [2][64][kPRow]
  const int h = blockIdx.y, kvh = h / (a.Hq / a.Hkv);
  const int64_t i0 = (int64_t)blockIdx.x * kPBM;
  const int64_t kb = i0 / a.bs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t qs = (int64_t)a.Hq * kPD, ks = (int64_t)a.Hkv * kPD;

  // key tiles: anchor [0, bs) (kb >= 1), then the own block from kb*bs up to the diagonal
  const int64_t last = i0 + kPBM < a.n ? i0 + kPBM : a.n;  // keys < last
  const int n_anchor = kb == 0 ? 0 : (int)(a.bs / kPBN);
  const int64_t own0 = kb * a.bs;
  const int n_own = (int)((last - own0 + kPBN - 1) / kPBN);
  const int ntiles = n_anchor + n_own;
  auto tile_start = [&](int t) -> int64_t { return t < n_anchor ? (int64_t)t * kPBN : own0 + (int64_t)(t - n_anchor) * kPBN; };
  auto load_kv = [&](int t, int buf) {
    const int64_t k0 = tile_start(t);
    for (int c = tid; c < kPBN * (kPD / 8); c += kPT) {
      const int r = c / (kPD / 8), col = (c % (kPD / 8)) * 8;
      const int64_t j = k0 + r;
      const bool ok = j < a.n;
      const int64_t jj = ok ? j : 0;
      cp_async16(sK + (buf * kPBN + r) * kPRow + col, a.k + jj * ks + (int64_t)kvh * kPD + col, ok);
      cp_async16(sV + (buf * kPBN + r) * kPRow + col, a.v + jj * ks + (int64_t)kvh * kPD + col, ok);
    }
  };
  for (int c = tid; c < kPBM * (kPD / 8); c += kPT) {
    const int r = c / (kPD / 8), col = (c % (kPD / 8)) * 8;
    const int64_t i = i0 + r;
    const bool ok = i < a.n;
    cp_async16(sQ + r * kPRow + col, a.q + (ok ? i : 0) * qs + (int64_t)h * kPD + col, ok);
  }
  load_kv(0, 0);
  cp_async_commit();

  uint32_t qf[kPD / 16][4];  // this warp's 16 query rows as A fragments (8 k-steps of 16)
  float o[kPD / 8][4];       // output accumulators: 16 rows x 128 (16 n-blocks of 8)
#pragma unroll
  for (int nb = 0; nb < kPD / 8; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.0f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.0f, 0.0f};
  const int64_t qrow0 = i0 + warp * 16 + gid, qrow1 = qrow0 + 8;

  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    cp_async_wait_all();
    __syncthreads();
    if (t + 1 < ntiles) { load_kv(t + 1, buf ^ 1); }
    cp_async_commit();
    if (t == 0) {
#pragma unroll
      for (int ks16 = 0; ks16 < kPD / 16; ++ks16) {
        const int mi = lane >> 3, r = lane & 7;
        ldsm_x4(qf[ks16], sQ + (warp * 16 + (mi & 1) * 8 + r) * kPRow + ks16 * 16 + (mi >> 1) * 8);
      }
    }
    const int64_t k0 = tile_start(t);
    const uint16_t *Kt = sK + buf * kPBN * kPRow;
    const uint16_t *Vt = sV + buf * kPBN * kPRow;
    // S = Q K^T : 16 x 64 per warp (8 n-blocks of 8 keys)
    float s[kPBN / 8][4];
#pragma unroll
    for (int nb = 0; nb < kPBN / 8; ++nb) s[nb][0] = s[nb][1] = s[nb][2] = s[nb][3] = 0.0f;
#pragma unroll
    for (int ks16 = 0; ks16 < kPD / 16; ++ks16) {
#pragma unroll
      for (int nb2 = 0; nb2 < kPBN / 16; ++nb2) {  // two n-blocks per ldmatrix.x4
        uint32_t bf[4];
        const int mi = lane >> 3, r = lane & 7;
        // matrices: (keys nb2*16+0..7, d k0..k0+7), (same keys, d +8), (keys +8, d), (keys +8, d +8)
        ldsm_x4(bf, Kt + (nb2 * 16 + (mi >> 1) * 8 + r) * kPRow + ks16 * 16 + (mi & 1) * 8);
        mma16816(s[2 * nb2], qf[ks16], bf[0], bf[1]);
        mma16816(s[2 * nb2 + 1], qf[ks16], bf[2], bf[3]);
      }
    }
    // mask + online softmax (rows qrow0 / qrow1; keys k0 + nb*8 + tig*2 + {0,1})
    const bool diag = k0 + kPBN > i0 && (kb == 0 || k0 >= own0);  // tile may hold keys > i
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int nb = 0; nb < kPBN / 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t j = k0 + nb * 8 + tig * 2 + (e & 1);
        const int64_t i = (e < 2) ? qrow0 : qrow1;
        float x = s[nb][e] * a.scale_log2;
        if (j >= a.n || (diag && j > i)) x = -INFINITY;
        s[nb][e] = x;
        mnew[e >> 1] = fmaxf(mnew[e >> 1], x);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
    }
    float corr[2], rs[2] = {0.0f, 0.0f};
#pragma unroll
    for (int r = 0; r < 2; ++r) corr[r] = mnew[r] == -INFINITY ? 1.0f : exp2f(mrow[r] - mnew[r]);
#pragma unroll
    for (int nb = 0; nb < kPBN / 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mm = mnew[e >> 1];
        const float p = mm == -INFINITY ? 0.0f : exp2f(s[nb][e] - mm);
        s[nb][e] = p;
        rs[e >> 1] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      lrow[r] = lrow[r] * corr[r] + rs[r];
      mrow[r] = mnew[r];
    }
#pragma unroll
    for (int nb = 0; nb < kPD / 8; ++nb) {
      o[nb][0] *= corr[0]; o[nb][1] *= corr[0];
      o[nb][2] *= corr[1]; o[nb][3] *= corr[1];
    }
    // O += P V : P as A fragments (k-steps of 16 keys), V via ldmatrix.trans
#pragma unroll
    for (int kk = 0; kk < kPBN / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_h2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_h2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_h2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_h2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int nb2 = 0; nb2 < kPD / 16; ++nb2) {  // two 8-wide dv blocks per ldmatrix.x4.trans
        uint32_t vb[4];
        const int mi = lane >> 3, r = lane & 7;
        // matrices: (keys kk*16+0..7, dv nb2*16+0..7), (keys +8, same dv), (keys, dv +8), (keys +8, dv +8)
        ldsm_x4_t(vb, Vt + (kk * 16 + (mi & 1) * 8 + r) * kPRow + nb2 * 16 + (mi >> 1) * 8);
        mma16816(o[2 * nb2], pa, vb[0], vb[1]);
        mma16816(o[2 * nb2 + 1], pa, vb[2], vb[3]);
      }
    }
  }
  // normalise and store (rows past n are not written)
  const float inv0 = lrow[0] > 0.0f ? 1.0f / lrow[0] : 0.0f;
  const float inv1 = lrow[1] > 0.0f ? 1.0f / lrow[1] : 0.0f;
#pragma unroll
  for (int nb = 0; nb < kPD / 8; ++nb) {
    const int col = nb * 8 + tig * 2;
    if (qrow0 < a.n)
      *reinterpret_cast<float2 *>(a.out + qrow0 * qs + (int64_t)h * kPD + col) = make_float2(o[nb][0] * inv0, o[nb][1] * inv0);
    if (qrow1 < a.n)
      *reinterpret_cast<float2 *>(a.out + qrow1 * qs + (int64_t)h * kPD + col) = make_float2(o[nb][2] * inv1, o[nb][3] * inv1);
  }
}

// ---------------------------------------------------------------------------------------
// tcgen05 version: CTA = 128 queries of one head (4 warps, thread t owns query row t), key
// tiles of 128.  Per tile: S = Q K^T (tcgen05.mma kind::f16, M = N = 128, K = 16 x 8,
// fp32 accumulator in TMEM columns [0, 128)), each thread reads its S row from TMEM
// (tcgen05.ld 32x32b), does the online-softmax update for its own row (no shuffles), writes
// P (fp16) into shared memory, then O_tile = P V (second MMA into TMEM columns [128, 256))
// and O_reg = O_reg * corr + O_tile in registers.  Operands live in shared memory in the
// 128-byte-swizzled K-major layout the UMMA descriptors describe (8-row x 128-B atoms,
// 16-B chunk c of row r at c ^ (r & 7)); V is stored transposed (d-major) so both MMAs use
// K-major B operands.
constexpr int kTM = 128;  // queries per CTA / keys per tile
constexpr int kTThreads = 128;

__device__ __forceinline__ uint32_t sw128_off(int r, int cg) {  // 16-B chunk cg (0..15) of row r
  const int kc = cg >> 3, c = cg & 7;
  return (uint32_t)(kc * (kTM * 128) + r * 128 + ((c ^ (r & 7)) << 4));
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;            // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;  // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1u << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2u << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint64_t umma_desc_k(uint32_t tile_saddr, int ks) {  // K step of 16
  return umma_desc(tile_saddr + (uint32_t)((ks >> 2) * (kTM * 128) + (ks & 3) * 32));
}
// MN-major B (V as stored: key rows, dv contiguous): atoms of 8 keys x 64 dv (1024 B),
// 8-key groups at SBO = 1024 B, the two 64-dv halves at LBO = 16 KiB; K step (16 keys) = 2 KiB
__device__ __forceinline__ uint64_t umma_desc_mn(uint32_t tile_saddr, int ks) {
  uint64_t d = (uint64_t)(((tile_saddr + (uint32_t)ks * 2048u) >> 4) & 0x3FFFu);
  d |= (uint64_t)((kTM * 128) >> 4) << 16;  // leading byte offset: next 64-wide MN half
  d |= (uint64_t)(1024u >> 4) << 32;         // stride byte offset: next 8 K-rows
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
// f16 x f16 -> f32, M = N = 128, A K-major; B K-major (S = Q K^T) or MN-major (O = P V)
constexpr uint32_t kIdescF16 = (1u << 4) | ((uint32_t)(kTM >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
constexpr uint32_t kIdescF16BMN = kIdescF16 | (1u << 16);

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t acc,
                                         uint32_t idesc = kIdescF16) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
#define HC_TLD32(addr, r)                                                                          \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"\
               "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"     \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),  \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),           \
                 "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),        \
                 "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),        \
                 "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),        \
                 "=r"(r[31])                                                                        \
               : "r"(addr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__global__ void __launch_bounds__(kTThreads, 2) k_blockwise_attn_tc(PrefillArgs a) {
  extern __shared__ __align__(1024) uint8_t tsm_raw[];
  uint8_t *tsm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t *sQ = tsm;                   // [128 q][128 d]      K-major (A of S)
  uint8_t *sK = sQ + kTM * 256;        // [128 keys][128 d]   K-major (B of S)
  uint8_t *sVt = sK + kTM * 256;       // [128 keys][128 d]   MN-major (B of O), same layout as sK
  uint8_t *sP = sK;                    // [128 q][128 keys]   K-major (A of O): reuses sK once S is done
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int h = blockIdx.y, kvh = h / (a.Hq / a.Hkv);
  const int64_t i0 = (int64_t)blockIdx.x * kTM;
  const int64_t kb = i0 / a.bs;
  const int64_t qs = (int64_t)a.Hq * kPD, ks_ = (int64_t)a.Hkv * kPD;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Q tile -> swizzled smem (thread t: row t, 16 chunks of 16 B)
  {
    const int64_t i = i0 + tid;
    const uint16_t *src = a.q + (i < a.n ? i : 0) * qs + (int64_t)h * kPD;
#pragma unroll
    for (int cg = 0; cg < 16; ++cg) {
      uint4 v = i < a.n ? *reinterpret_cast<const uint4 *>(src + cg * 8) : make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4 *>(sQ + sw128_off(tid, cg)) = v;
    }
  }
  fence_async_smem();  // generic smem writes -> visible to the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_sel = (uint32_t)(warp * 32) << 16;
  const uint32_t aQ = (uint32_t)__cvta_generic_to_shared(sQ), aK = (uint32_t)__cvta_generic_to_shared(sK);
  const uint32_t aVt = (uint32_t)__cvta_generic_to_shared(sVt), aP = (uint32_t)__cvta_generic_to_shared(sP);

  const int64_t last = i0 + kTM < a.n ? i0 + kTM : a.n;
  const int n_anchor = kb == 0 ? 0 : (int)(a.bs / kTM);
  const int64_t own0 = kb * a.bs;
  const int n_own = (int)((last - own0 + kTM - 1) / kTM);
  const int ntiles = n_anchor + n_own;
  const int64_t qi = i0 + tid;  // this thread's query
  // O accumulates in TMEM across tiles (PV MMAs with accumulate); the softmax reference
  // max m_ref is only raised when a tile's max exceeds it by more than 2^8 (then O and l are
  // rescaled in place), so P = 2^(s - m_ref) <= 2^8 stays well inside fp16
  float mref = -INFINITY, lrow = 0.0f;
  uint32_t phase = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int64_t k0 = t < n_anchor ? (int64_t)t * kTM : own0 + (int64_t)(t - n_anchor) * kTM;
    // K and V tiles (key rows), coalesced (16 consecutive threads per 256-B row), all 32
    // 16-B copies per thread in flight at once (cp.async, zero-fill past n)
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int idx = it * kTThreads + tid, r = idx >> 4, cg = idx & 15;
      const int64_t j = k0 + r;
      const bool ok = j < a.n;
      const int64_t off = (ok ? j : 0) * ks_ + (int64_t)kvh * kPD + cg * 8;
      cp_async16(sK + sw128_off(r, cg), a.k + off, ok);
      cp_async16(sVt + sw128_off(r, cg), a.v + off, ok);
    }
    cp_async_commit();
    cp_async_wait_all();
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < kPD / 16; ++kk) umma_f16(tS, umma_desc_k(aQ, kk), umma_desc_k(aK, kk), kk > 0);
      umma_commit(&mbar);
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    tc_fence_after();
    // this thread's S row (TMEM lane = row), raw scores; the log2(e)/sqrt(d) scale is folded
    // into the exponent's FMA.  Masking only on the diagonal / ragged tiles (CTA-uniform).
    const bool masked = (k0 + kTM > i0 && (kb == 0 || k0 >= own0)) || k0 + kTM > a.n;
    float sv[kTM];
    float mraw = -INFINITY;
    {
      uint32_t r[32];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        HC_TLD32(tS + lane_sel + c4 * 32, r);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) sv[c4 * 32 + u] = __uint_as_float(r[u]);
      }
    }
    if (masked) {
      const int lim = (int)min((int64_t)kTM, min(a.n, qi + 1) - k0);  // keys < k0 + lim are visible
#pragma unroll
      for (int u = 0; u < kTM; ++u)
        if (u >= lim) sv[u] = -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < kTM; ++u) mraw = fmaxf(mraw, sv[u]);
    const float mt = mraw * a.scale_log2;
    const bool raise = mt > mref + 8.0f;  // also true for the first finite max
    float corr = 1.0f;
    if (raise) {
      corr = mref == -INFINITY ? 0.0f : exp2f(mref - mt);
      mref = mt;
      lrow *= corr;
    }
    if (t > 0 && __any_sync(0xffffffffu, raise)) {  // rescale this warp's O rows in TMEM
      uint32_t r[32];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        HC_TLD32(tO + lane_sel + c4 * 32, r);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * corr);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%32], {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,"
                     "%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31};"
                     ::"r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                     "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
                     "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
                     "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
                     "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(tO + lane_sel + c4 * 32)
                     : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    float rs = 0.0f;
    const float nm = mref == -INFINITY ? 0.0f : -mref;  // all-masked rows: sv = -inf -> p = 0
#pragma unroll
    for (int cg = 0; cg < 16; ++cg) {  // P row (fp16, <= 2^8) -> swizzled smem (reuses sK)
      uint32_t w4[4];
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        const float p0 = ex2_approx(fmaf(sv[cg * 8 + 2 * e2], a.scale_log2, nm));
        const float p1 = ex2_approx(fmaf(sv[cg * 8 + 2 * e2 + 1], a.scale_log2, nm));
        rs += p0 + p1;
        w4[e2] = pack_h2(p0, p1);
      }
      *reinterpret_cast<uint4 *>(sP + sw128_off(tid, cg)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
    lrow += rs;
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < kTM / 16; ++kk)
        umma_f16(tO, umma_desc_k(aP, kk), umma_desc_mn(aVt, kk), (t > 0 || kk > 0) ? 1u : 0u, kIdescF16BMN);
      umma_commit(&mbar);
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    tc_fence_after();
  }
  {  // out = O / l
    const float inv = lrow > 0.0f ? 1.0f / lrow : 0.0f;
    float *op = a.out + qi * qs + (int64_t)h * kPD;
    uint32_t r[32];
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) {
      HC_TLD32(tO + lane_sel + c4 * 32, r);
      tmem_wait_ld();
      if (qi < a.n) {
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          *reinterpret_cast<float4 *>(op + c4 * 32 + e) =
              make_float4(__uint_as_float(r[e]) * inv, __uint_as_float(r[e + 1]) * inv,
                          __uint_as_float(r[e + 2]) * inv, __uint_as_float(r[e + 3]) * inv);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

static int prefill_tc() {
  static int v = -1;
  if (v < 0) {
    const char *ev = getenv("HC_PREFILL_TC");
    v = (ev && !strcmp(ev, "0")) ? 0 : 1;
  }
  return v;
}

cudaError_t launch_blockwise_attn(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t n,
                                  int Hq, int Hkv, int64_t bs, float *out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  PrefillArgs a{q, k, v, out, n, bs, Hq, Hkv, (float)(1.4426950408889634 / sqrt((double)kPD))};
  if (prefill_tc() && bs % kTM == 0) {
    const size_t smem = (size_t)3 * kTM * 256 + 1024;
    static int configured_tc[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !configured_tc[dev]) {
      cudaError_t e = cudaFuncSetAttribute(k_blockwise_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      configured_tc[dev] = 1;
    }
    dim3 grid((unsigned)((n + kTM - 1) / kTM), (unsigned)Hq);
    k_blockwise_attn_tc<<<grid, kTThreads, smem, s>>>(a);
    note_launch();
    return cudaGetLastError();
  }
  const size_t smem = (size_t)(kPBM + 4 * kPBN) * kPRow * 2;
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_blockwise_attn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[dev] = 1;
  }
  dim3 grid((unsigned)((n + kPBM - 1) / kPBM), (unsigned)Hq);
  k_blockwise_attn<<<grid, kPT, smem, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hc
