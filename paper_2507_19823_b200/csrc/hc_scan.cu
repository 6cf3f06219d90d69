// hc_scan.cu -- row a2: approximate scores against the quantized key cache,
// Eq. 3:  z̃_j = Σ_{i=1..g} T_{i, P_{j,i}}.
//
// B200 design:
//  * one CTA per SM (persistent over token tiles), 512 threads;
//  * a tile = TPT*512 consecutive tokens of one (b, kv) unit; every thread owns
//    2 chunks of 8 consecutive tokens and keeps G int32 accumulators per token in
//    registers across the whole group loop (the sum is exact integer, R2/R3, so the
//    association is free);
//  * the group loop streams the unit's T slice i (cpow2 × G × int16 = 64 KiB at
//    c = 8192, G = 4) into shared memory with cp.async.bulk (TMA bulk copy engine)
//    on an mbarrier, double-buffered: slice i+2 is in flight while slice i is used;
//  * the P strip of group i (group-major layout, contiguous per group) is read
//    with 128-bit L1-bypassing loads, one group ahead of use;
//  * one 8-byte LDS per (token, group) returns the 4 GQA heads' table entries.
#include <stdlib.h>
#include <string.h>

#include "hc_internal.h"

namespace hc {

constexpr int kScanThreads = 512;
#ifndef HC_LOOKUP_BATCH
#define HC_LOOKUP_BATCH 1
#endif
constexpr bool kLookupBatch = HC_LOOKUP_BATCH;

__device__ __forceinline__ uint4 ld_stream(const uint16_t *p) {
  uint4 v;
  // streamed once: evict-first in L2, so the layer's tables T stay resident
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// packed 13-bit code planes (f3(ii)): 8 tokens = 8 B lo + 4 B nibbles + 1 B bits
__device__ __forceinline__ uint4 ld_raw13(const uint8_t *strip, int64_t n_cap, int64_t tok) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint32_t lo0, lo1, nib;
  uint16_t bit;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(lo0), "=r"(lo1) : "l"(strip + tok), "l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(nib) : "l"(strip + n_cap + tok / 2), "l"(pol));
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
               : "=h"(bit) : "l"(strip + n_cap + n_cap / 2 + tok / 8), "l"(pol));
  return make_uint4(lo0, lo1, nib, (uint32_t)bit);
}

template <int G>
struct Lut;
// Head pairs share a 32-bit word w = (odd head, signed) << 16 | (even head + 32768) (k_table).
// The even accumulator sums whole words (mod 2^32), the odd one w >> 16 (= the odd head,
// exactly, since the biased low field is in [1, 65535]); unbias() recovers
// Σ even = Σ w - 2^16·Σ odd - 32768·ng -- two integer adds per pair instead of three.
__device__ __forceinline__ int wadd(int acc, uint32_t w) { return (int)((uint32_t)acc + w); }
template <>
struct Lut<4> {  // 8-byte entries: 4 x int16
  static constexpr int kShift = 3;
  __device__ __forceinline__ static void add(const uint8_t *sb, uint32_t off, int (&acc)[4]) {
    const uint2 v = *reinterpret_cast<const uint2 *>(sb + off);
    acc[0] = wadd(acc[0], v.x);
    acc[1] += ((int)v.x) >> 16;
    acc[2] = wadd(acc[2], v.y);
    acc[3] += ((int)v.y) >> 16;
  }
};
template <>
struct Lut<2> {
  static constexpr int kShift = 2;
  __device__ __forceinline__ static void add(const uint8_t *sb, uint32_t off, int (&acc)[2]) {
    const uint32_t v = *reinterpret_cast<const uint32_t *>(sb + off);
    acc[0] = wadd(acc[0], v);
    acc[1] += ((int)v) >> 16;
  }
};
template <int G>
__device__ __forceinline__ void unbias(int (&acc)[8][G], int ng) {
  if constexpr (G >= 2) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int h = 0; h < G; h += 2)
        acc[t][h] = (int)((uint32_t)acc[t][h] - ((uint32_t)acc[t][h + 1] << 16) - 32768u * (uint32_t)ng);
  }
}
template <>
struct Lut<1> {
  static constexpr int kShift = 1;
  __device__ __forceinline__ static void add(const uint8_t *sb, uint32_t off, int (&acc)[1]) {
    acc[0] += (int)*reinterpret_cast<const int16_t *>(sb + off);
  }
};

// 8 codes (one uint4) -> 8 tokens' accumulators.  Codes are masked to cpow2-1, so
// any 16-bit pattern stays inside the slice (valid codes are < c <= cpow2).
// all 8 table words of a chunk loaded before any is consumed (8 LDS in flight per warp)
__device__ __forceinline__ void lookup8_g4(const uint4 &c, const uint8_t *sb, uint32_t mask,
                                           int (&acc)[8][4]) {
  const uint32_t w[4] = {c.x, c.y, c.z, c.w};
  uint2 v[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[2 * q] = *reinterpret_cast<const uint2 *>(sb + ((w[q] << 3) & mask));
    v[2 * q + 1] = *reinterpret_cast<const uint2 *>(sb + ((w[q] >> 13) & mask));
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    acc[t][0] = wadd(acc[t][0], v[t].x);
    acc[t][1] += ((int)v[t].x) >> 16;
    acc[t][2] = wadd(acc[t][2], v[t].y);
    acc[t][3] += ((int)v[t].y) >> 16;
  }
}

template <int G>
__device__ __forceinline__ void lookup8(const uint4 &c, const uint8_t *sb, uint32_t mask,
                                        int (&acc)[8][G]) {
  if constexpr (G == 4) {
    if (kLookupBatch) { lookup8_g4(c, sb, mask, acc); return; }
  }
  const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t o0 = (w[q] << Lut<G>::kShift) & mask;
    const uint32_t o1 = (w[q] >> (16 - Lut<G>::kShift)) & mask;
    Lut<G>::add(sb, o0, acc[2 * q]);
    Lut<G>::add(sb, o1, acc[2 * q + 1]);
  }
}

// group-split items add their exact integer partial sums into z (zeroed by k_table) with
// float atomics: every partial and every prefix is an integer below 2^23, so the fp32 sum
// is exact in any order and z is final after the scan (no partial planes, no reduce pass)
__device__ __forceinline__ void red_add4(float *p, float a0, float a1, float a2, float a3) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a0), "f"(a1), "f"(a2),
               "f"(a3)
               : "memory");
}

template <int G>
__device__ __forceinline__ void store_chunk_add(const LayerArgs &a, int b, int kv, int64_t tok,
                                                const int (&acc)[8][G]) {
  if (tok >= a.n_q) return;
  const int64_t rem_ = a.n_q - tok;
  const int nval = rem_ < 8 ? (int)rem_ : 8;
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float *zp = a.z + ((int64_t)b * a.Hq + kv * G + h) * a.z_stride + tok;
    if (nval == 8) {
      red_add4(zp, (float)acc[0][h], (float)acc[1][h], (float)acc[2][h], (float)acc[3][h]);
      red_add4(zp + 4, (float)acc[4][h], (float)acc[5][h], (float)acc[6][h], (float)acc[7][h]);
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < nval) atomicAdd(zp + u, (float)acc[u][h]);
    }
  }
}

template <int G>
__device__ __forceinline__ void store_chunk(const LayerArgs &a, float *zbase, int b, int kv,
                                            int64_t tok, const int (&acc)[8][G], int (&mx)[G],
                                            int (&mn)[G], bool add = false) {
  if (add) { store_chunk_add<G>(a, b, kv, tok, acc); return; }
  if (tok >= a.n_q) return;
  const int64_t rem_ = a.n_q - tok;
  const int nval = rem_ < 8 ? (int)rem_ : 8;
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float *zp = zbase + ((int64_t)b * a.Hq + kv * G + h) * a.z_stride + tok;
    if (nval == 8) {
      float4 v0 = make_float4((float)acc[0][h], (float)acc[1][h], (float)acc[2][h], (float)acc[3][h]);
      float4 v1 = make_float4((float)acc[4][h], (float)acc[5][h], (float)acc[6][h], (float)acc[7][h]);
      reinterpret_cast<float4 *>(zp)[0] = v0;
      reinterpret_cast<float4 *>(zp)[1] = v1;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        mx[h] = max(mx[h], acc[u][h]);
        mn[h] = min(mn[h], acc[u][h]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u < nval) {
          zp[u] = (float)acc[u][h];
          mx[h] = max(mx[h], acc[u][h]);
          mn[h] = min(mn[h], acc[u][h]);
        }
      }
    }
  }
}

// Work item = (unit, token tile, group split).  With nsplit > 1 each item sums only
// its groups [i0, i1) and adds the exact integer partial into z (store_chunk_add) -- so
// small-context configs can spread one unit's tokens AND groups over all SMs without
// re-streaming every slice.
// per-head max / min of the final scores (unsplit scan): warp reduce + one atomic per warp,
// so the select kernel needs no extra pass over z for them
template <int G>
__device__ __forceinline__ void fold_minmax(const LayerArgs &a, int b, int kv, const int (&mx)[G],
                                            const int (&mn)[G]) {
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const int vmx = __reduce_max_sync(0xffffffffu, mx[h]);
    const int vmn = __reduce_min_sync(0xffffffffu, mn[h]);
    if ((threadIdx.x & 31) == 0 && vmx != INT_MIN) {
      HeadState *hs = a.hs + (int64_t)b * a.Hq + kv * G + h;
      atomicMax(&hs->M, vmx);
      atomicMin(&hs->zmin, vmn);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Pipelined scan (used when the stream-K split does not apply: short rows, group splits,
// packed codes).  The CTA's work is one stream of (item, group) steps:
//  * table slices live in a 3-slot ring filled by bulk copies (TMA engine) on "full"
//    mbarriers; there is NO CTA-wide barrier per group: each warp, after its lookups in
//    slot s%3, bumps a shared counter, and the LAST warp to finish the slot refills it
//    with step s+3's slice -- warps drift up to two steps apart instead of draining at a
//    __syncthreads every group;
//  * each thread prefetches its code registers two steps ahead;
//  * both prefetchers run across item boundaries, so the next tile's slices and codes are
//    in flight while this tile's scores are stored.
// Same arithmetic, same z.
struct ScanCursor {
  int item, i, ng;
  const uint16_t *P;  // this thread's code pointer at group i0 of `item`
  const uint8_t *Pb;  // packed codes: the strip of group i0 of `item`
  const uint8_t *T;   // table slice of group i0 of `item`
  int64_t tile0;
};

template <int G, int TPT, bool P13>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan_pipe(LayerArgs a, int tiles_per_unit,
                                                                int total_tiles, int nsplit) {
  constexpr int kChunks = TPT / 8;
  constexpr int kTile = kScanThreads * TPT;
  constexpr int kSlots = 3;
  constexpr uint32_t kWarps = kScanThreads / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t slice_bytes = (uint32_t)a.cpow2 * G * 2;
  uint8_t *tbuf = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kSlots * slice_bytes);
  __shared__ uint32_t s_done[kSlots];
  if (threadIdx.x == 0) {
    for (int j = 0; j < kSlots; ++j) { mbar_init(&full[j], 1); s_done[j] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();
  if ((int)blockIdx.x >= total_tiles) return;
  const uint32_t mask = (uint32_t)(a.cpow2 - 1) << Lut<G>::kShift;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int woff = warp * (32 * TPT);  // this warp's first token inside a tile
  const int gper = (a.g + nsplit - 1) / nsplit;

  auto cset = [&](ScanCursor &c, int item) {
    c.item = item;
    c.i = 0;
    if (item < total_tiles) {
      const int sp = item % nsplit, tile = item / nsplit;
      const int u = tile / tiles_per_unit, tk = tile - u * tiles_per_unit;
      const int i0 = sp * gper;
      c.ng = min(a.g, i0 + gper) - i0;
      const int b = u / a.Hkv, kv = u - b * a.Hkv;
      c.tile0 = (int64_t)tk * kTile;
      c.P = a.codes + (int64_t)b * a.code_b_stride + ((int64_t)kv * a.g + i0) * a.n_cap + c.tile0 +
            woff + lane * 8;
      if (P13) c.Pb = a.pcodes + (int64_t)b * a.pc_b_stride + ((int64_t)kv * a.g + i0) * a.strip_bytes;
      c.T = reinterpret_cast<const uint8_t *>(a.T) + ((int64_t)u * a.g + i0) * slice_bytes;
    }
  };
  auto cadv = [&](ScanCursor &c) {
    if (++c.i >= c.ng) cset(c, c.item + gridDim.x);
  };
  auto ccodes = [&](const ScanCursor &c, uint4 (&r)[kChunks]) {
    const bool live = c.item < total_tiles;
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int64_t tok = c.tile0 + woff + k * 256 + lane * 8;
      const bool v = live && tok < a.n_q;
      if (P13)
        r[k] = v ? ld_raw13(c.Pb + (int64_t)c.i * a.strip_bytes, a.n_cap, tok) : make_uint4(0, 0, 0, 0);
      else
        r[k] = v ? ld_stream(c.P + (int64_t)c.i * a.n_cap + k * 256) : make_uint4(0, 0, 0, 0);
    }
  };
  // one thread: bulk-copy c's slice into `slot`.  Why no fence.proxy.async before this async-
  // proxy write into a slot the warps just read through the generic proxy (a WAR hazard across
  // proxies): every warp releases the slot only after ALL of its lookup results have been
  // consumed -- the empty asm statements below take every accumulator as an input, so each
  // LDS of the slot has returned its data into a register before the warp's counter
  // increment is even issued, and the refill is issued only by the warp that observes the
  // 16th increment.  No read of the slot is in flight when the bulk copy starts, so there is
  // nothing for the async write to overtake.  This is the ordering CUTLASS's TMA pipelines
  // rely on as well (the consumer's release is an mbarrier arrive after its reads; the
  // producer's refill carries no proxy fence).  A fence.proxy.async here would also wait for
  // this thread's own in-flight global loads (the code prefetch two steps ahead).  The
  // selection's z streams (hc_select_pass.cu), whose release is not data-dependent in the
  // same way, do issue the proxy fence.
  auto cslice = [&](const ScanCursor &c, int slot) {
    if (c.item < total_tiles) {
      mbar_expect_tx(&full[slot], slice_bytes);
      bulk_g2s(tbuf + slot * slice_bytes, c.T + (int64_t)c.i * slice_bytes, slice_bytes, &full[slot]);
    }
  };
  ScanCursor lc, lt;  // code cursor: step + 2; table cursor: step + 3
  cset(lc, blockIdx.x);
  cset(lt, blockIdx.x);
  uint4 rc0[kChunks], rc1[kChunks];
  ccodes(lc, rc0);
  cadv(lc);
  ccodes(lc, rc1);
  cadv(lc);
  for (int j = 0; j < kSlots; ++j) {
    if (threadIdx.x == 0) cslice(lt, j);
    cadv(lt);
  }

  uint32_t ph = 0;  // phase bit per slot
  int slot = 0;
  for (int item = blockIdx.x; item < total_tiles; item += gridDim.x) {
    const int sp = item % nsplit, tile = item / nsplit;
    const int u = tile / tiles_per_unit, tk = tile - u * tiles_per_unit;
    const int i0 = sp * gper;
    const int ng = min(a.g, i0 + gper) - i0;
    const int b = u / a.Hkv, kv = u - b * a.Hkv;
    const int64_t tile0 = (int64_t)tk * kTile;
    int acc[kChunks][8][G];
#pragma unroll
    for (int k = 0; k < kChunks; ++k)
#pragma unroll
      for (int u8 = 0; u8 < 8; ++u8)
#pragma unroll
        for (int h = 0; h < G; ++h) acc[k][u8][h] = 0;
    for (int i = 0; i < ng; ++i) {
      uint4 rc2[kChunks];
      ccodes(lc, rc2);  // step + 2 (possibly the next item's)
      cadv(lc);
      mbar_wait(&full[slot], (ph >> slot) & 1u);
      ph ^= 1u << slot;
      const uint8_t *sb = tbuf + slot * slice_bytes;
#pragma unroll
      for (int k = 0; k < kChunks; ++k) lookup8<G>(P13 ? unpack13(rc0[k]) : rc0[k], sb, mask, acc[k]);
      // Release the slot; the last warp out refills it with step + 3.  Every lookup result
      // has been consumed (the empty asm statements take all accumulators as inputs), so
      // this warp's reads of the slot are complete before its counter increment issues.
#pragma unroll
      for (int k = 0; k < kChunks; ++k)
#pragma unroll
        for (int u8 = 0; u8 < 8; u8 += 2) {
          if constexpr (G == 4)
            asm volatile("" ::"r"(acc[k][u8][0]), "r"(acc[k][u8][1]), "r"(acc[k][u8][2]), "r"(acc[k][u8][3]),
                         "r"(acc[k][u8 + 1][0]), "r"(acc[k][u8 + 1][1]), "r"(acc[k][u8 + 1][2]),
                         "r"(acc[k][u8 + 1][3]));
          else if constexpr (G == 2)
            asm volatile("" ::"r"(acc[k][u8][0]), "r"(acc[k][u8][1]), "r"(acc[k][u8 + 1][0]),
                         "r"(acc[k][u8 + 1][1]));
          else
            asm volatile("" ::"r"(acc[k][u8][0]), "r"(acc[k][u8 + 1][0]));
        }
      __syncwarp();
      if (lane == 0) {
        uint32_t old;
        asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old)
                     : "r"(smem_u32(&s_done[slot]))
                     : "memory");
        if (old == kWarps - 1) {
          asm volatile("st.relaxed.cta.shared::cta.u32 [%0], 0;" ::"r"(smem_u32(&s_done[slot])) : "memory");
          cslice(lt, slot);
        }
      }
      cadv(lt);
#pragma unroll
      for (int k = 0; k < kChunks; ++k) { rc0[k] = rc1[k]; rc1[k] = rc2[k]; }
      slot = slot == kSlots - 1 ? 0 : slot + 1;
    }
    int mx[G], mn[G];
#pragma unroll
    for (int h = 0; h < G; ++h) { mx[h] = INT_MIN; mn[h] = INT_MAX; }
    float *zbase = a.z;
    const bool zadd = nsplit > 1;
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      unbias<G>(acc[k], ng);
      store_chunk<G>(a, zbase, b, kv, tile0 + woff + k * 256 + lane * 8, acc[k], mx, mn, zadd);
    }
    if (nsplit == 1) fold_minmax<G>(a, b, kv, mx, mn);
  }
}

// ---------------------------------------------------------------------------------------
// Stream-K variant of k_scan_pipe: the (tile, group) steps of the launch are cut into
// `grid` EQUAL contiguous ranges, one per persistent CTA, so no SM idles in a last partial
// wave (config 3: 512 tiles on 148 SMs = 3.46 waves, 13 % of the scan lost to the tail).
// A tile whose groups straddle two CTAs is finished by the second to arrive: each writes
// its exact int32 partial (own groups, unbiased) to its slot, fences, bumps the tile's
// counter; the finisher adds the other's partial to its registers, stores z and folds
// max / min (the sums are exact integers, so the result equals the unsplit scan's).
// Needs steps per CTA >= 2 g (every tile straddles at most two CTAs; the launcher checks).
template <int G, int TPT>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan_sk(LayerArgs a, int tiles_per_unit,
                                                              int total_tiles, int *skpart,
                                                              uint32_t *skctr) {
  constexpr int kChunks = TPT / 8;
  constexpr int kTile = kScanThreads * TPT;
  constexpr int kSlots = 3;
  constexpr uint32_t kWarps = kScanThreads / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t slice_bytes = (uint32_t)a.cpow2 * G * 2;
  uint8_t *tbuf = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kSlots * slice_bytes);
  __shared__ uint32_t s_done[kSlots];
  if (threadIdx.x == 0) {
    for (int j = 0; j < kSlots; ++j) { mbar_init(&full[j], 1); s_done[j] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();
  const int g = a.g;
  const int64_t S = (int64_t)total_tiles * g;
  const int64_t s0 = S * blockIdx.x / gridDim.x, s1 = S * (blockIdx.x + 1) / gridDim.x;
  if (s0 >= s1) return;
  const uint32_t mask = (uint32_t)(a.cpow2 - 1) << Lut<G>::kShift;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int woff = warp * (32 * TPT);

  // step cursor: s = global step, i = its group, tok0 = its tile's first token (divisions
  // only when a tile starts)
  struct Cur { int64_t s; int i; int64_t tok0; const uint16_t *P; const uint8_t *T; };
  auto cpos = [&](Cur &c, int64_t st) {  // pointers of step st (tile st / g, group st % g)
    c.s = st;
    if (st >= s1) return;
    const int tile = (int)(st / g), i = (int)(st - (int64_t)tile * g);
    const int u = tile / tiles_per_unit, tk = tile - u * tiles_per_unit;
    const int b = u / a.Hkv, kv = u - b * a.Hkv;
    c.i = i;
    c.tok0 = (int64_t)tk * kTile;
    c.P = a.codes + (int64_t)b * a.code_b_stride + ((int64_t)kv * g + i) * a.n_cap + c.tok0 + woff + lane * 8;
    c.T = reinterpret_cast<const uint8_t *>(a.T) + ((int64_t)u * g + i) * slice_bytes;
  };
  auto cadv = [&](Cur &c) {
    if (c.s + 1 < s1 && c.i + 1 < g) {  // same tile: next group's strip and slice
      ++c.s;
      ++c.i;
      c.P += a.n_cap;
      c.T += slice_bytes;
    } else {
      cpos(c, c.s + 1);
    }
  };
  auto ccodes = [&](const Cur &c, uint4 (&r)[kChunks]) {
    const bool live = c.s < s1;
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      const int64_t tok = c.tok0 + woff + k * 256 + lane * 8;
      r[k] = (live && tok < a.n_q) ? ld_stream(c.P + k * 256) : make_uint4(0, 0, 0, 0);
    }
  };
  auto cslice = [&](const Cur &c, int slot) {
    if (c.s < s1) {
      mbar_expect_tx(&full[slot], slice_bytes);
      bulk_g2s(tbuf + slot * slice_bytes, c.T, slice_bytes, &full[slot]);
    }
  };
  Cur lc, lt;
  cpos(lc, s0);
  cpos(lt, s0);
  uint4 rc0[kChunks], rc1[kChunks];
  ccodes(lc, rc0);
  cadv(lc);
  ccodes(lc, rc1);
  cadv(lc);
  for (int j = 0; j < kSlots; ++j) {
    if (threadIdx.x == 0) cslice(lt, j);
    cadv(lt);
  }
  uint32_t ph = 0;
  int slot = 0;
  int64_t st = s0;
  while (st < s1) {
    const int tile = (int)(st / g);
    const int64_t t_lo = (int64_t)tile * g, t_hi = t_lo + g;
    const int64_t e = t_hi < s1 ? t_hi : s1;  // steps of this tile done by this CTA: [st, e)
    const int ng = (int)(e - st);
    const bool whole = st == t_lo && e == t_hi;
    const int u = tile / tiles_per_unit, tk = tile - u * tiles_per_unit;
    const int b = u / a.Hkv, kv = u - b * a.Hkv;
    const int64_t tile0 = (int64_t)tk * kTile;
    int acc[kChunks][8][G];
#pragma unroll
    for (int k = 0; k < kChunks; ++k)
#pragma unroll
      for (int u8 = 0; u8 < 8; ++u8)
#pragma unroll
        for (int h = 0; h < G; ++h) acc[k][u8][h] = 0;
    for (int i = 0; i < ng; ++i) {
      uint4 rc2[kChunks];
      ccodes(lc, rc2);
      cadv(lc);
      mbar_wait(&full[slot], (ph >> slot) & 1u);
      ph ^= 1u << slot;
      const uint8_t *sb = tbuf + slot * slice_bytes;
#pragma unroll
      for (int k = 0; k < kChunks; ++k) lookup8<G>(rc0[k], sb, mask, acc[k]);
#pragma unroll
      for (int k = 0; k < kChunks; ++k)
#pragma unroll
        for (int u8 = 0; u8 < 8; u8 += 2) {
          if constexpr (G == 4)
            asm volatile("" ::"r"(acc[k][u8][0]), "r"(acc[k][u8][1]), "r"(acc[k][u8][2]), "r"(acc[k][u8][3]),
                         "r"(acc[k][u8 + 1][0]), "r"(acc[k][u8 + 1][1]), "r"(acc[k][u8 + 1][2]),
                         "r"(acc[k][u8 + 1][3]));
          else if constexpr (G == 2)
            asm volatile("" ::"r"(acc[k][u8][0]), "r"(acc[k][u8][1]), "r"(acc[k][u8 + 1][0]),
                         "r"(acc[k][u8 + 1][1]));
          else
            asm volatile("" ::"r"(acc[k][u8][0]), "r"(acc[k][u8 + 1][0]));
        }
      __syncwarp();
      if (lane == 0) {
        uint32_t old;
        asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old)
                     : "r"(smem_u32(&s_done[slot]))
                     : "memory");
        if (old == kWarps - 1) {
          asm volatile("st.relaxed.cta.shared::cta.u32 [%0], 0;" ::"r"(smem_u32(&s_done[slot])) : "memory");
          cslice(lt, slot);
        }
      }
      cadv(lt);
#pragma unroll
      for (int k = 0; k < kChunks; ++k) { rc0[k] = rc1[k]; rc1[k] = rc2[k]; }
      slot = slot == kSlots - 1 ? 0 : slot + 1;
    }
#pragma unroll
    for (int k = 0; k < kChunks; ++k) unbias<G>(acc[k], ng);
    bool finish = whole;
    if (!whole) {
      // my partial -> my slot (0: this tile is my first, 1: my last).  Per WARP (each warp owns
      // a disjoint token range of the tile): the warp's second arrival (over the two CTAs)
      // adds the other CTA's partial for its tokens and finishes them -- no CTA barrier, one
      // fence per warp (release / acquire around the counter by lane 0, ordered for the
      // other lanes by __syncwarp)
      const int myslot = st == s0 ? 0 : 1;
      int *mine = skpart + ((int64_t)blockIdx.x * 2 + myslot) * (kTile * G);
#pragma unroll
      for (int k = 0; k < kChunks; ++k)
#pragma unroll
        for (int u8 = 0; u8 < 8; ++u8) {
          int *dst = mine + ((int64_t)(woff + k * 256 + lane * 8 + u8)) * G;
          if constexpr (G == 4)
            *reinterpret_cast<int4 *>(dst) = make_int4(acc[k][u8][0], acc[k][u8][1], acc[k][u8][2], acc[k][u8][3]);
          else
#pragma unroll
            for (int h = 0; h < G; ++h) dst[h] = acc[k][u8][h];
        }
      __syncwarp();
      uint32_t prev = 0;
      if (lane == 0) {
        __threadfence();
        prev = atomicAdd(&skctr[(int64_t)tile * kWarps + warp], 1u);
        if (prev == 1u) skctr[(int64_t)tile * kWarps + warp] = 0u;
        __threadfence();
      }
      finish = __shfl_sync(0xffffffffu, prev, 0) == 1u;
      __syncwarp();
      if (finish) {
        // the other contributor: the previous CTA (tile = its last) or the next (its first)
        const int oc = myslot == 0 ? (int)blockIdx.x - 1 : (int)blockIdx.x + 1;
        const int os = myslot == 0 ? 1 : 0;
        const int *other = skpart + ((int64_t)oc * 2 + os) * (kTile * G);
#pragma unroll
        for (int k = 0; k < kChunks; ++k)
#pragma unroll
          for (int u8 = 0; u8 < 8; ++u8) {
            const int *src = other + ((int64_t)(woff + k * 256 + lane * 8 + u8)) * G;
            if constexpr (G == 4) {
              const int4 v = __ldcg(reinterpret_cast<const int4 *>(src));
              acc[k][u8][0] += v.x; acc[k][u8][1] += v.y; acc[k][u8][2] += v.z; acc[k][u8][3] += v.w;
            } else {
#pragma unroll
              for (int h = 0; h < G; ++h) acc[k][u8][h] += __ldcg(src + h);
            }
          }
      }
    }
    if (finish) {
      int mx[G], mn[G];
#pragma unroll
      for (int h = 0; h < G; ++h) { mx[h] = INT_MIN; mn[h] = INT_MAX; }
#pragma unroll
      for (int k = 0; k < kChunks; ++k)
        store_chunk<G>(a, a.z, b, kv, tile0 + woff + k * 256 + lane * 8, acc[k], mx, mn, false);
      fold_minmax<G>(a, b, kv, mx, mn);
    }
    st = e;
  }
}

// ---------------------------------------------------------------------------------------
// 8-bit table variant (R2b): one 4-byte LDS per (token, group) -- 3.5 instead of
// 6.15 shared-memory wavefronts per warp lookup -- and SWAR accumulation: the entry holds
// the 4 heads as (int8 + 128) bytes; acc_e += w & 0x00FF00FF (heads 0, 2), acc_o +=
// (w >> 8) & 0x00FF00FF (heads 1, 3), 16-bit fields never overflow for g <= 257, and
// z_h = field - 128*ng exactly.  Two registers per token let a thread own 32 tokens
// (tile = 16384 tokens), which halves the table-slice ingress per token.
// Same pipeline as k_scan_pipe: a 3-slot ring of (table slice,
// code strip) pairs filled by bulk copies on one "full" mbarrier per slot, released by the
// last warp out, prefetch across item boundaries.
template <int TPT>
__global__ void __launch_bounds__(kScanThreads, 1) k_scan8_pipe(LayerArgs a, int tiles_per_unit,
                                                                 int total_tiles, int nsplit) {
  constexpr int G = 4;
  constexpr int kChunks = TPT / 8;
  constexpr int kTile = kScanThreads * TPT;
  constexpr uint32_t kCodeBytes = kTile * 2;
  constexpr int kSlots = 3;
  constexpr uint32_t kWarps = kScanThreads / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t slice_bytes = (uint32_t)a.cpow2 * 4;
  uint8_t *tbuf = smem;
  uint8_t *cbuf = smem + kSlots * slice_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(cbuf + kSlots * kCodeBytes);
  __shared__ uint32_t s_done[kSlots];
  if (threadIdx.x == 0) {
    for (int j = 0; j < kSlots; ++j) { mbar_init(&full[j], 1); s_done[j] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();
  if ((int)blockIdx.x >= total_tiles) return;
  const uint32_t mask = (uint32_t)(a.cpow2 - 1) << 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int woff = warp * (32 * TPT);
  const int gper = (a.g + nsplit - 1) / nsplit;
  int lt_item = blockIdx.x, lt_i = 0, lt_ng = 0;
  const uint16_t *lt_P = nullptr;
  const uint8_t *lt_T = nullptr;
  uint32_t lt_cbytes = 0;
  auto lset = [&](int item) {
    lt_item = item;
    lt_i = 0;
    if (item < total_tiles) {
      const int sp = item % nsplit, tile = item / nsplit;
      const int u = tile / tiles_per_unit, tk = tile - u * tiles_per_unit;
      const int i0 = sp * gper;
      lt_ng = min(a.g, i0 + gper) - i0;
      const int b = u / a.Hkv, kv = u - b * a.Hkv;
      const int64_t tile0 = (int64_t)tk * kTile;
      const int64_t avail = a.n_cap - tile0;
      lt_cbytes = (uint32_t)(avail < kTile ? avail : kTile) * 2;
      lt_P = a.codes + (int64_t)b * a.code_b_stride + ((int64_t)kv * a.g + i0) * a.n_cap + tile0;
      lt_T = reinterpret_cast<const uint8_t *>(a.T) + ((int64_t)u * a.g + i0) * slice_bytes;
    }
  };
  auto ladv = [&]() {
    if (++lt_i >= lt_ng) lset(lt_item + gridDim.x);
  };
  auto lfill = [&](int slot) {  // one thread: table slice + code strip of the lookahead step
    if (lt_item < total_tiles) {
      mbar_expect_tx(&full[slot], slice_bytes + lt_cbytes);
      bulk_g2s(tbuf + slot * slice_bytes, lt_T + (int64_t)lt_i * slice_bytes, slice_bytes, &full[slot]);
      bulk_g2s(cbuf + slot * kCodeBytes, lt_P + (int64_t)lt_i * a.n_cap, lt_cbytes, &full[slot]);
    }
  };
  lset(blockIdx.x);
  for (int j = 0; j < kSlots; ++j) {
    if (threadIdx.x == 0) lfill(j);
    ladv();
  }
  uint32_t ph = 0;
  int slot = 0;
  for (int item = blockIdx.x; item < total_tiles; item += gridDim.x) {
    const int sp = item % nsplit, tile = item / nsplit;
    const int u = tile / tiles_per_unit, tk = tile - u * tiles_per_unit;
    const int i0 = sp * gper;
    const int ng = min(a.g, i0 + gper) - i0;
    const int b = u / a.Hkv, kv = u - b * a.Hkv;
    const int64_t tile0 = (int64_t)tk * kTile;
    uint32_t ae[kChunks][8], ao[kChunks][8];
#pragma unroll
    for (int k = 0; k < kChunks; ++k)
#pragma unroll
      for (int t = 0; t < 8; ++t) { ae[k][t] = 0u; ao[k][t] = 0u; }
    for (int i = 0; i < ng; ++i) {
      mbar_wait(&full[slot], (ph >> slot) & 1u);
      ph ^= 1u << slot;
      const uint8_t *sb = tbuf + slot * slice_bytes;
      const uint8_t *cs = cbuf + slot * kCodeBytes + (size_t)woff * 2;
#pragma unroll
      for (int k = 0; k < kChunks; ++k) {
        const uint4 c = *reinterpret_cast<const uint4 *>(cs + (k * 256 + lane * 8) * 2);
        const uint32_t w4[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t e0 = *reinterpret_cast<const uint32_t *>(sb + ((w4[q] << 2) & mask));
          const uint32_t e1 = *reinterpret_cast<const uint32_t *>(sb + ((w4[q] >> 14) & mask));
          ae[k][2 * q] += e0 & 0x00FF00FFu;
          ao[k][2 * q] += (e0 >> 8) & 0x00FF00FFu;
          ae[k][2 * q + 1] += e1 & 0x00FF00FFu;
          ao[k][2 * q + 1] += (e1 >> 8) & 0x00FF00FFu;
        }
      }
      // every read of the slot (codes and table) has been consumed by the adds above
#pragma unroll
      for (int k = 0; k < kChunks; ++k)
        asm volatile("" ::"r"(ae[k][0]), "r"(ae[k][1]), "r"(ae[k][2]), "r"(ae[k][3]), "r"(ae[k][4]),
                     "r"(ae[k][5]), "r"(ae[k][6]), "r"(ae[k][7]), "r"(ao[k][0]), "r"(ao[k][1]),
                     "r"(ao[k][2]), "r"(ao[k][3]), "r"(ao[k][4]), "r"(ao[k][5]), "r"(ao[k][6]),
                     "r"(ao[k][7]));
      __syncwarp();
      if (lane == 0) {
        uint32_t old;
        asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old)
                     : "r"(smem_u32(&s_done[slot]))
                     : "memory");
        if (old == kWarps - 1) {
          asm volatile("st.relaxed.cta.shared::cta.u32 [%0], 0;" ::"r"(smem_u32(&s_done[slot])) : "memory");
          lfill(slot);
        }
      }
      ladv();
      slot = slot == kSlots - 1 ? 0 : slot + 1;
    }
    const int bias = 128 * ng;
    int mx[G], mn[G];
#pragma unroll
    for (int h = 0; h < G; ++h) { mx[h] = INT_MIN; mn[h] = INT_MAX; }
    float *zbase = a.z;
    const bool zadd = nsplit > 1;
#pragma unroll
    for (int k = 0; k < kChunks; ++k) {
      int acc[8][G];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        acc[t][0] = (int)(ae[k][t] & 0xffffu) - bias;
        acc[t][2] = (int)(ae[k][t] >> 16) - bias;
        acc[t][1] = (int)(ao[k][t] & 0xffffu) - bias;
        acc[t][3] = (int)(ao[k][t] >> 16) - bias;
      }
      store_chunk<G>(a, zbase, b, kv, tile0 + woff + k * 256 + lane * 8, acc, mx, mn, zadd);
    }
    if (nsplit == 1) fold_minmax<G>(a, b, kv, mx, mn);
  }
}

template <int G, int TPT, bool P13>
static cudaError_t scan_pipe_launch(const LayerArgs &a, cudaStream_t s) {
  constexpr int kTile = kScanThreads * TPT;
  const int tiles_per_unit = (int)((a.n_q + kTile - 1) / kTile);
  const int units = a.B * a.Hkv;
  const int nsplit = a.scan_split;
  const int total = tiles_per_unit * units * nsplit;
  if (total == 0) return cudaSuccess;
  const size_t smem = (size_t)3 * a.cpow2 * G * 2 + 3 * 8;
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_scan_pipe<G, TPT, P13>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    if (e != cudaSuccess) return e;
    configured[dev] = 1;
  }
  const int grid = total < a.num_sms ? total : a.num_sms;
  cudaEvent_t eb, ee;
  scan_events(&eb, &ee);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const unsigned evflag = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  if (eb) cudaEventRecordWithFlags(eb, s, evflag);
  launch_chain(k_scan_pipe<G, TPT, P13>, dim3(grid), dim3(kScanThreads), smem, s, a, tiles_per_unit, total, nsplit);
  note_launch();
  if (ee) cudaEventRecordWithFlags(ee, s, evflag);
  return cudaGetLastError();
}

static int scan_streamk() {
  static int v = -1;
  if (v < 0) {
    const char *ev = getenv("HC_SCAN_SK");
    v = (ev && !strcmp(ev, "0")) ? 0 : 1;
  }
  return v;
}

// stream-K launch when every CTA gets >= 2 tiles of steps (else false: use the pipe kernel)
template <int G, int TPT>
static bool scan_sk_launch(const LayerArgs &a, cudaStream_t s, cudaError_t *err) {
  constexpr int kTile = kScanThreads * TPT;
  const int tiles_per_unit = (int)((a.n_q + kTile - 1) / kTile);
  const int total = tiles_per_unit * a.B * a.Hkv;
  const int grid = a.num_sms < kSkMaxCtas ? a.num_sms : kSkMaxCtas;
  if (!a.skpart || !a.skctr || total < 2 * grid || (int64_t)total * (kScanThreads / 32) > a.skctr_n || total == 0)
    return false;
  const size_t smem = (size_t)3 * a.cpow2 * G * 2 + 3 * 8;
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_scan_sk<G, TPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         226 * 1024);
    if (e != cudaSuccess) { *err = e; return true; }
    configured[dev] = 1;
  }
  cudaEvent_t eb, ee;
  scan_events(&eb, &ee);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const unsigned evflag = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  if (eb) cudaEventRecordWithFlags(eb, s, evflag);
  launch_chain(k_scan_sk<G, TPT>, dim3(grid), dim3(kScanThreads), smem, s, a, tiles_per_unit, total, a.skpart,
               a.skctr);
  note_launch();
  if (ee) cudaEventRecordWithFlags(ee, s, evflag);
  *err = cudaGetLastError();
  return true;
}

template <int G>
static cudaError_t scan_g(const LayerArgs &a, cudaStream_t s) {
  if (!a.pcodes && scan_streamk() && a.scan_split == 1) {
    cudaError_t e = cudaSuccess;
    if (a.scan_tpt == 8 ? scan_sk_launch<G, 8>(a, s, &e) : scan_sk_launch<G, 16>(a, s, &e)) return e;
  }
  if (a.pcodes)  // packed 13-bit codes
    return a.scan_tpt == 8 ? scan_pipe_launch<G, 8, true>(a, s) : scan_pipe_launch<G, 16, true>(a, s);
  return a.scan_tpt == 8 ? scan_pipe_launch<G, 8, false>(a, s) : scan_pipe_launch<G, 16, false>(a, s);
}

static cudaError_t scan8_pipe_launch(const LayerArgs &a, cudaStream_t s) {
  constexpr int TPT = 32;
  constexpr int kTile = kScanThreads * TPT;
  const int tiles_per_unit = (int)((a.n_q + kTile - 1) / kTile);
  const int units = a.B * a.Hkv;
  const int nsplit = a.scan_split;
  const int total = tiles_per_unit * units * nsplit;
  if (total == 0) return cudaSuccess;
  const size_t smem = (size_t)3 * a.cpow2 * 4 + 3 * (size_t)kTile * 2 + 3 * 8;
  static int configured[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_scan8_pipe<TPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         226 * 1024);
    if (e != cudaSuccess) return e;
    configured[dev] = 1;
  }
  const int grid = total < a.num_sms ? total : a.num_sms;
  cudaEvent_t eb, ee;
  scan_events(&eb, &ee);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  const unsigned evflag = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  if (eb) cudaEventRecordWithFlags(eb, s, evflag);
  launch_chain(k_scan8_pipe<TPT>, dim3(grid), dim3(kScanThreads), smem, s, a, tiles_per_unit, total, nsplit);
  note_launch();
  if (ee) cudaEventRecordWithFlags(ee, s, evflag);
  return cudaGetLastError();
}

cudaError_t launch_scan(const LayerArgs &a, cudaStream_t s) {
  if (a.lut8) return scan8_pipe_launch(a, s);
  switch (a.G) {
    case 1: return scan_g<1>(a, s);
    case 2: return scan_g<2>(a, s);
    case 4: return scan_g<4>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hc
