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
// This is the prefill side (not the decode hot path); mma.sync keeps it simple -- a
// tcgen05 / TMEM version is the next step if prefill throughput matters.
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

cudaError_t launch_blockwise_attn(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t n,
                                  int Hq, int Hkv, int64_t bs, float *out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  PrefillArgs a{q, k, v, out, n, bs, Hq, Hkv, (float)(1.4426950408889634 / sqrt((double)kPD))};
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
