// hc_device.cuh -- device-side arithmetic of the CUDA path (sm_100a).
// Implements DESIGN.md §2 readings R1-R6 with explicit IEEE intrinsics so the
// results are bit-identical to the independent CPU oracle (no code shared).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#ifndef HC_HD
#define HC_HD __device__ __forceinline__
#endif

namespace hc {

constexpr int kNB = 4096;        // buckets per histogram level (12 bits)
constexpr int kNBBits = 12;

HC_HD float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// exact 2^e for -126 <= e <= 127
HC_HD float pow2f(int e) { return __int_as_float((e + 127) << 23); }

// R2: e_h = 100 if A < 2^-100 else clamp(14 - floor(log2 A), -100, 100)
HC_HD int scale_exponent(float A) {
  if (!(A >= 0x1p-100f)) return 100;
  int ex = ((__float_as_int(A) >> 23) & 0xff) - 127;  // A is normal here
  int e = 14 - ex;
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}

// R2b (8-bit table): e = clamp(6 - floor(log2 A), -100, 100)
HC_HD int scale_exponent8(float A) {
  if (!(A >= 0x1p-100f)) return 100;
  int ex = ((__float_as_int(A) >> 23) & 0xff) - 127;
  int e = 6 - ex;
  return e < -100 ? -100 : (e > 100 ? 100 : e);
}

HC_HD int quant_t8(float t, float s) {
  float v = rintf(__fmul_rn(t, s));
  v = fminf(fmaxf(v, -127.0f), 127.0f);
  return (int)v;
}

// R2: T_fx = clamp(rint(t * 2^e), +-32767)
HC_HD int quant_t(float t, float s) {
  float v = rintf(__fmul_rn(t, s));
  v = fminf(fmaxf(v, -32767.0f), 32767.0f);
  return (int)v;
}

#ifdef __CUDACC__
// Device versions of quant_t / quant_t8 without conversion instructions (FRND and F2I issue
// at 1/8 rate): pre-clamping to +-2^16 does not change clamp(rint(x)), and for |x| <= 2^22
// adding 1.5*2^23 rounds to the nearest integer, ties to even, exactly like rintf.
__device__ __forceinline__ int rint_small(float x) {  // |x| <= 2^22
  return __float_as_int(__fadd_rn(x, 12582912.0f)) - 0x4B400000;
}
__device__ __forceinline__ int quant_t_d(float t, float s) {
  const int r = rint_small(fminf(fmaxf(__fmul_rn(t, s), -65536.0f), 65536.0f));
  return min(max(r, -32767), 32767);
}
__device__ __forceinline__ int quant_t8_d(float t, float s) {
  const int r = rint_small(fminf(fmaxf(__fmul_rn(t, s), -65536.0f), 65536.0f));
  return min(max(r, -127), 127);
}
#endif

// R3 resident: rint(clamp(acc * 2^e, +-2^22))
HC_HD int quant_res(float acc, float s) {
  float v = __fmul_rn(acc, s);
  v = fminf(fmaxf(v, -4194304.0f), 4194304.0f);
  return __float2int_rn(v);
}

// R4: exp2_det polynomial (degree 6 on [0,1))
HC_HD float exp2_poly(float f) {
  float p = 0x1.c6e292p-13f;
  p = __fmaf_rn(p, f, 0x1.46301cp-10f);
  p = __fmaf_rn(p, f, 0x1.3d24eap-7f);
  p = __fmaf_rn(p, f, 0x1.c68562p-5f);
  p = __fmaf_rn(p, f, 0x1.ebfd9ap-3f);
  p = __fmaf_rn(p, f, 0x1.62e42ap-1f);
  p = __fmaf_rn(p, f, 0x1.000000p+0f);
  return p;
}

// R4: W(Δ) = trunc(2^40 * exp2_det(-(Δ·κ)))
HC_HD uint64_t mass(uint32_t delta, float kappa) {
  float x = -__fmul_rn(__uint2float_rn(delta), kappa);
  if (x < -40.0f) return 0ull;
  float nf = floorf(x);
  float f = __fsub_rn(x, nf);
  float p = exp2_poly(f);
  float v = __fmul_rn(p, pow2f(40 + (int)nf));
  return __float2ull_rz(v);
}

#ifdef __CUDACC__
// Exact int of an integer-valued fp32 score with |z| <= 2^22 (every z̃ here: R3 with
// g <= 128, R3 resident clamp, R5b): one FADD + one integer op instead of a conversion
// (F2I issues at 1/8 of the FP32 rate).
__device__ __forceinline__ int zint(float z) {
  return __float_as_int(__fadd_rn(z, 12582912.0f)) - 0x4B400000;
}

// mass() without conversion instructions, bit-identical to it: every step below is exact
// (delta <= 2^23 -> float by exponent bias; floor of x in [-40, 0] by the 1.5*2^23 round
// trick; truncation of v in [1, 2^41) by exponent/mantissa shift).
__device__ __forceinline__ uint64_t mass_d(uint32_t delta, float kappa) {
  const float df = delta <= (1u << 23) ? __fsub_rn(__int_as_float(0x4B000000 + (int)delta), 8388608.0f)
                                       : __uint2float_rn(delta);
  const float x = -__fmul_rn(df, kappa);
  if (x < -40.0f) return 0ull;
  const float r = __fadd_rn(x, 12582912.0f);  // nearest integer to x
  int ni = __float_as_int(r) - 0x4B400000;
  float nf = __fsub_rn(r, 12582912.0f);
  if (nf > x) { nf = __fsub_rn(nf, 1.0f); ni -= 1; }
  const float f = __fsub_rn(x, nf);
  const float v = __fmul_rn(exp2_poly(f), pow2f(40 + ni));
  const uint32_t b = __float_as_uint(v);
  if (b < 0x3F800000u) return 0ull;  // v < 1
  const int e = (int)(b >> 23) - 127;
  const uint64_t m = (b & 0x7FFFFFu) | 0x800000u;
  return e >= 23 ? m << (e - 23) : m >> (23 - e);
}
#endif

#ifdef __CUDACC__
// ---- packed 13-bit codes (f3(ii), include/hc.h): strip = [lo n_cap B][nib n_cap/2 B][bit n_cap/8 B]
__device__ __forceinline__ void rmw_bits(uint8_t *byte_addr, int bit_in_byte, uint32_t width,
                                         uint32_t val) {
  const uintptr_t ad = reinterpret_cast<uintptr_t>(byte_addr);
  uint32_t *w = reinterpret_cast<uint32_t *>(ad & ~(uintptr_t)3);
  const int sh = (int)(ad & 3) * 8 + bit_in_byte;
  const uint32_t m = ((1u << width) - 1u) << sh;
  atomicAnd(w, ~m);
  atomicOr(w, (val << sh) & m);
}
__device__ __forceinline__ void put_code13(uint8_t *strip, int64_t n_cap, int64_t t, uint32_t code) {
  rmw_bits(strip + t, 0, 8, code & 0xffu);
  rmw_bits(strip + n_cap + t / 2, (int)(t & 1) * 4, 4, (code >> 8) & 15u);
  rmw_bits(strip + n_cap + n_cap / 2 + t / 8, (int)(t & 7), 1, (code >> 12) & 1u);
}
// raw = {lo bytes 0-3, lo bytes 4-7, 8 nibbles, 8 bits (low byte)} of 8 consecutive tokens ->
// the u16-layout uint4 (token 2q in the low half of word q)
__device__ __forceinline__ uint4 unpack13(const uint4 &raw) {
  uint32_t o[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t lo = __byte_perm(q < 2 ? raw.x : raw.y, 0u, (q & 1) ? 0x4342u : 0x4140u);
    const uint32_t n2 = (raw.z >> (8 * q)) & 0xffu;
    const uint32_t b2 = (raw.w >> (2 * q)) & 3u;
    o[q] = lo | ((n2 & 0xfu) << 8) | ((n2 & 0xf0u) << 20) | ((b2 & 1u) << 12) | ((b2 & 2u) << 27);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// mass_d() as two 32-bit words, branch-free (the P1 histogram's hot loop): every step is
// the same exact operation as in mass_d; delta <= 2^23 (|z̃| <= 2^22, g <= 128).
__device__ __forceinline__ void mass_parts(uint32_t delta, float kappa, uint32_t &lo, uint32_t &hi) {
  const float df = __fsub_rn(__int_as_float(0x4B000000 + (int)delta), 8388608.0f);
  const float x0 = -__fmul_rn(df, kappa);
  const float x = fmaxf(x0, -64.0f);  // keeps 2^(40+n) normal; x0 < -40 -> 0 below
  const float r = __fadd_rn(x, 12582912.0f);
  float nf = __fsub_rn(r, 12582912.0f);
  const bool adj = nf > x;
  nf = adj ? __fsub_rn(nf, 1.0f) : nf;
  const int ni = __float_as_int(r) - 0x4B400000 - (adj ? 1 : 0);
  const float v = __fmul_rn(exp2_poly(__fsub_rn(x, nf)), pow2f(40 + ni));
  const uint32_t b = __float_as_uint(v);
  const int sh = (int)(b >> 23) - 150;  // v = m * 2^sh, m in [2^23, 2^24)
  const uint32_t m = (b & 0x7FFFFFu) | 0x800000u;
  uint32_t l = sh >= 0 ? (m << sh) : (sh > -32 ? (m >> -sh) : 0u);
  uint32_t h = sh > 8 ? (m >> (32 - sh)) : 0u;
  const bool zero = x0 < -40.0f;
  lo = zero ? 0u : l;
  hi = zero ? 0u : h;
}
#endif

// R5: Θ = ceil(τ_q · S / 2^24)  (τ_q <= 2^24, S < 2^63)
HC_HD uint64_t threshold(uint32_t tau_q, uint64_t S) {
  uint64_t lo = (uint64_t)tau_q * S;
  uint64_t hi = __umul64hi((uint64_t)tau_q, S);
  uint64_t add = (1ull << 24) - 1;
  uint64_t lo2 = lo + add;
  hi += (lo2 < lo) ? 1ull : 0ull;
  return (hi << 40) | (lo2 >> 24);
}

// R4's mass W(Δ) = trunc(p(f) * 2^(40+n)), x = -(float)Δ*κ, n = floor(x), f = x - n, 0 for
// x < -40 -- the same IEEE steps as mass() / mass_d() (hc_device.cuh), bit for bit, with the
// floor, the int->float of n and the final truncation on the conversion pipe (F2I / I2F),
// which runs beside the FMA / ALU pipes this pass is otherwise bound by.
__device__ __forceinline__ uint64_t wmass(uint32_t dl, float kappa) {
  const float df = __fsub_rn(__int_as_float(0x4B000000 + (int)dl), 8388608.0f);  // exact, Δ <= 2^23
  const float x0 = -__fmul_rn(df, kappa);
  const float x = fmaxf(x0, -64.0f);          // keeps 2^(40+n) normal; x0 < -40 -> 0 below
  const int ni = __float2int_rd(x);            // floor (exact for |x| <= 64)
  const float f = __fsub_rn(x, __int2float_rn(ni));
  const float v = __fmul_rn(exp2_poly(f), pow2f(40 + ni));
  const uint64_t w = __float2ull_rz(v);        // truncation toward zero, v < 2^41
  return x0 < -40.0f ? 0ull : w;
}

// wmass for two tokens at once: the same IEEE steps with the adds / multiplies / polynomial on
// the packed fp32x2 pipe (FADD2 / FMUL2 / FFMA2: each lane rounds as the scalar op), so both
// results are bit-identical to wmass() (x - float(n) == x + (-float(n)); -(df κ) == df (-κ)).
__device__ __forceinline__ void wmass2(uint32_t d0, uint32_t d1, float kappa, uint64_t &w0, uint64_t &w1) {
  const float2 df = __fadd2_rn(make_float2(__int_as_float(0x4B000000 + (int)d0), __int_as_float(0x4B000000 + (int)d1)),
                               make_float2(-8388608.0f, -8388608.0f));
  const float2 x0 = __fmul2_rn(df, make_float2(-kappa, -kappa));
  const float xa = fmaxf(x0.x, -64.0f), xb = fmaxf(x0.y, -64.0f);
  const int na = __float2int_rd(xa), nb = __float2int_rd(xb);
  const float2 f = __fadd2_rn(make_float2(xa, xb), make_float2(-__int2float_rn(na), -__int2float_rn(nb)));
  float2 p = make_float2(0x1.c6e292p-13f, 0x1.c6e292p-13f);  // exp2_poly, Horner in pairs
  p = __ffma2_rn(p, f, make_float2(0x1.46301cp-10f, 0x1.46301cp-10f));
  p = __ffma2_rn(p, f, make_float2(0x1.3d24eap-7f, 0x1.3d24eap-7f));
  p = __ffma2_rn(p, f, make_float2(0x1.c68562p-5f, 0x1.c68562p-5f));
  p = __ffma2_rn(p, f, make_float2(0x1.ebfd9ap-3f, 0x1.ebfd9ap-3f));
  p = __ffma2_rn(p, f, make_float2(0x1.62e42ap-1f, 0x1.62e42ap-1f));
  p = __ffma2_rn(p, f, make_float2(0x1.000000p+0f, 0x1.000000p+0f));
  const float2 v = __fmul2_rn(p, make_float2(pow2f(40 + na), pow2f(40 + nb)));
  w0 = x0.x < -40.0f ? 0ull : __float2ull_rz(v.x);
  w1 = x0.y < -40.0f ? 0ull : __float2ull_rz(v.y);
}

// 16-B read-only load that bypasses L1 (value rows: read once per head group)
__device__ __forceinline__ uint4 ldg_nc16(const uint16_t *p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// ---- mbarrier + bulk-copy (TMA engine) helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// per-(b, query head) selection state, 128 B, in the workspace
struct alignas(16) HeadState {
  int32_t M;            // max z (atomicMax), init INT_MIN
  int32_t zmin;         // min z (atomicMin), init INT_MAX
  uint32_t amax;        // bits of max|t| (atomicMax on non-negative float bits), init 0
  int32_t e;            // table scale exponent
  float kappa;          // κ_h = κ0 · 2^-e
  int32_t shift;        // coarse bucket = Δ >> shift
  int32_t bstar;        // boundary coarse bucket, kNB = "all strict"
  uint32_t cnt_before;  // #tokens in buckets < bstar
  uint64_t mass_before; // mass in buckets < bstar
  uint64_t S;           // total mass
  uint64_t theta;       // Θ
  uint32_t delta_star;  // exact boundary Δ* (tokens with Δ < Δ* are kept)
  uint32_t r_ties;      // #ties at Δ* kept (lowest indices)
  int64_t ksel;         // k_sel
  int64_t kstar;        // k* if τ decided, else -1
  uint64_t sel_mass;    // mass of the kept set (renorm)
  uint32_t gather_done; // completion counter of the gather's last-block reduction
  uint32_t h1_done;     // completion counter of hist1 (last CTA runs bound1)
  uint32_t h2_done;     // completion counter of hist2 (last CTA runs bound2)
  // hc_select_pass.cu (K1 / K2 / K3 of the decode selection); zeroed by k_table / the prep
  uint32_t c1_done;     // K1 completion counter (the row's last CTA bounds the cut)
  uint32_t c2_done;     // K2 completion counter (the last CTA resolves the cut)
  uint32_t ticket;      // K3 chunk tickets (decoupled look-back order)
  uint32_t r_lo, r_hi;  // refine range of Δ (inclusive)
  int32_t fshift;       // refine bin width 2^fshift
  uint32_t state;       // 1 / 2: refine pass 1 / 2 pending, 3: resolved, 4: error
};
static_assert(sizeof(HeadState) == 128, "HeadState size");

// per-(b, KV head) state of the shared selection (R8, hc_group.cu), in the workspace
struct alignas(16) GroupState {
  uint64_t SA;          // Σ_j A_j
  uint64_t theta;       // Θ = ceil(τ_q·S_A / 2^24)
  uint64_t ntot;        // candidates
  uint64_t cb, mb;      // count / mass of the keys below the current prefix bucket
  uint64_t prefix;      // fixed high bits of the boundary key D*
  uint64_t dstar;       // exact boundary key (2^48 = keep all)
  uint64_t r_ties;      // ties at D* kept (lowest indices)
  int64_t ksel, kstar;
  uint64_t rho[4];      // ρ_h = floor((2^104 - 1) / S_h)
  int32_t done;         // boundary resolved
  int32_t pad[3];
};

}  // namespace hc
