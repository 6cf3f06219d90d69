// hc_internal.h -- launch interfaces between the C-ABI host layer (hc_api.cu)
// and the sm_100a kernels.  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hc_device.cuh"

namespace hc {

constexpr int kSkMaxCtas = 160;  // stream-K scan: max persistent CTAs (partial slots in the workspace)

// number of kernels this library has enqueued (or captured into a graph)
void note_launch(int n = 1);
// set the thread's hc_last_error() message; returns st
int set_error(int st, const char *msg);

// Programmatic dependent launch (PDL) along the decode chain (encode -> table -> [resident]
// -> scan -> select -> gather -> next layer's encode): each chain kernel triggers its
// dependents at entry and waits (griddepcontrol.wait) before touching memory written by
// its predecessors, so the next kernel's launch and prologue overlap this kernel's tail.
// Opt-in (HC_PDL=1): measured neutral in the graph-captured step and slower for eager
// calls, so plain stream order is the default; the kernels are PDL-safe either way.
bool pdl_enabled();
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
cudaError_t launch_chain(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                         Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
// profiling hook: events recorded around the next scan launch (may be null)
void scan_events(cudaEvent_t *begin, cudaEvent_t *end);

// row -> element offset:  (r / R1) * s1 + (r % R1) * s2 + s0
struct RowMap {
  int64_t R1, s1, s2, s0;
};

struct EncodeArgs {
  const uint16_t *keys;
  RowMap kmap;           // key row offset (elements)
  int64_t rows;
  const float *C;        // [cbg][c][dbar]
  int d, g, c, cbg;
  uint16_t *codes;
  RowMap omap;           // code offset of (r, group 0)
  int64_t gstride;       // elements between groups
  // optional fused value-row copy (append): vdst[vdmap(r)] = vsrc[vsmap(r)], d halves
  const uint16_t *vsrc;
  RowMap vsmap;
  uint16_t *vdst;
  RowMap vdmap;
  // bulk encode only: optional row gather (key row of r = kidx[r], valid if < n_keys)
  const int64_t *kidx;
  int64_t n_keys;
  // packed 13-bit codes (f3(ii)): if pcodes, row r's group-i code goes to token ptok of
  // strip psmap(r) + i (strip_bytes each, n_cap tokens) instead of codes/omap
  uint8_t *pcodes;
  RowMap psmap;
  int64_t strip_bytes, pn_cap, ptok;
};
cudaError_t launch_encode(const EncodeArgs &a, cudaStream_t s);
// many rows: codebook slice staged in shared memory, rows per thread (hc_kmeans.cu)
cudaError_t launch_encode_bulk(const EncodeArgs &a, cudaStream_t s);
// f4: one MiniBatchKMeans step; enc.codes = labels [g][b], enc.kidx = sample
cudaError_t launch_kmeans_step(const EncodeArgs &enc, const int64_t *sample, int64_t b, float *C,
                               int64_t *counts, unsigned long long *n, unsigned long long *S,
                               cudaStream_t st);

struct RowCopyArgs {
  const uint16_t *src;
  RowMap smap;
  uint16_t *dst;
  RowMap dmap;
  int64_t rows;
  int d;
};
cudaError_t launch_rowcopy(const RowCopyArgs &a, cudaStream_t s);

struct LayerArgs {
  // shape
  int B, Hkv, G, Hq, d, g, c, cbg, dbar, cpow2;
  int lut8;               // 1: 8-bit table variant (R2b), entries = 4 x (int8 + 128) in a u32
  int64_t n_q, n_res, n_cand, n_cap, res_cap;
  // inputs
  const uint16_t *q;      // [B][Hq][d]
  const float *C;         // layer codebook [cbg][c][dbar]
  const uint16_t *codes;  // layer 0 of batch 0 base + l*Hkv*g*n_cap ; batch stride below
  int64_t code_b_stride;  // elements between batches
  const uint8_t *pcodes;  // packed 13-bit codes (f3(ii)) at layer l, batch 0; null = u16 codes
  int64_t pc_b_stride;    // bytes between batches
  int64_t strip_bytes;    // bytes per (b, l, kv, group) strip = 13 n_cap / 8
  const uint16_t *res_k;  // [B][L][Hkv][W][d] at layer l (batch stride below)
  const uint16_t *res_v;
  int64_t res_b_stride;   // elements between batches
  int64_t res_slot0;      // slot of candidate n_q: (n_q) % W
  const uint16_t *V;      // value store at layer l, batch 0
  int v_placement;        // 0 = HBM (bulk-copy ring gather), 1 = host-mapped (zero-copy loads)
  int64_t v_b_stride;     // elements between batches
  int64_t v_kv_stride;    // elements between KV heads
  // budget
  uint32_t tau_q;
  int64_t k_max;
  int renorm;
  float kappa0;
  // workspace
  HeadState *hs;          // [B*Hq]
  int16_t *T;             // [units][g][cpow2][G]
  const float *cb_absmax; // layer [cbg][dbar]: max_m |C[ci][m][e]| (R2 bound)
  int tsplit;             // k_table parts: contiguous ranges of the g * cpow2 entries
  int tunits;             // k_table units per CTA (<= kTableU, tunits * d * G <= kTableQ)
  float *z;               // [B*Hq][z_stride]
  int64_t z_stride;
  // outputs
  int32_t *sel_idx;       // [B*Hq][k_max]
  float *sel_w;
  int64_t *sel_k;         // [B*Hq] (may be null)
  float *out;             // [B*Hq][d]
  int num_sms;
  int scan_tpt;           // tokens per thread in the scan (8 or 16)
  int scan_split;         // group splits per token tile (1 = write z directly)
  float *zpart;           // [scan_split][B*Hq][z_stride] partial sums when scan_split > 1
  // shared per-KV-head selection (R8, hc_group.cu)
  GroupState *grp;                 // [B*Hkv]
  unsigned long long *grp_hist;    // [B*Hkv][4 levels][kNB][count, mass]
  uint32_t *grp_chunk;             // [B*Hkv][chunks][strict, ties]
  unsigned long long *grp_key;     // [B*Hkv][z_stride] order key D of every candidate
  // completion counters of this layer's gather kernel, zeroed by k_table (no memset node
  // between the chain kernels)
  uint32_t *gdone;
  int gdone_n;
  // the selection's coarse count histograms [B*Hq][kNB], zeroed by k_table (or null)
  uint32_t *sel_ghist;
  // k_gather_rows on a sub-range of each row's list (sequence-sharded finish): entries
  // [g_off[row], g_off[row] + g_cnt[row]) with local token index = sel_idx - g_base
  const int64_t *g_off, *g_cnt;
  int64_t g_base;
  // k_gather_union: kept counts per row from this array instead of hs[row].ksel (standalone
  // hc_gather_values), and the token range [gtok_lo, gtok_hi) the GPU sums (heterogeneous
  // split: the host owns the rest; decode: [0, n_cand))
  const int64_t *k_in;
  int64_t gtok_lo, gtok_hi;
  // stream-K scan (k_scan_sk): per-CTA partial slots [sms][2][tile][G] int32 and per-tile
  // arrival counters (zeroed by k_table)
  int *skpart;
  uint32_t *skctr;
  int skctr_n;
};

cudaError_t launch_init(const LayerArgs &a, cudaStream_t s);
cudaError_t launch_table(const LayerArgs &a, cudaStream_t s);
cudaError_t launch_resident(const LayerArgs &a, cudaStream_t s);
cudaError_t launch_cbabs(const float *C, int64_t slices, int c, int dbar, float *out, cudaStream_t s);
cudaError_t launch_scan(const LayerArgs &a, cudaStream_t s);

// Eq. 4 selection over `rows` independent score rows (query heads):
// z [rows][z_stride] (exact integers stored as fp32), hs[row].{M,zmin,kappa} set.
struct SelArgs {
  HeadState *hs;
  const float *z;
  int64_t z_stride;
  int rows;
  int64_t n;              // candidates per row
  uint32_t tau_q;
  int64_t k_max;
  int renorm;
  int32_t *sel_idx;       // [rows][k_max]
  float *sel_w;           // [rows][k_max]
  int64_t *sel_k;         // [rows] (may be null)
  // hc_select_pass.cu state (workspace): coarse (count, mass) histograms (zeroed before K1 by
  // k_table / the float prep), refine histograms and chunk counters (zeroed by K1)
  uint32_t *ghist;             // [rows][kNB] coarse counts
  unsigned long long *gmass;   // [rows][kNB] coarse exact masses (directly after ghist)
  uint32_t *fcnt;              // [rows][kNB]
  uint32_t *cntlo;             // [rows][nch] per chunk: tokens above the refine range
  unsigned long long *pre;     // [rows][nch] per chunk: exclusive (strict << 32 | ties) prefix
  unsigned long long *list;    // [rows][cap] in-range tokens (index << 32 | Δ)
  int64_t nch, cap;            // chunks per row (kSelChunk tokens each), list capacity per row
};
// fused rows a3-a5 (one cluster of CTAs per row; round 1, HC_SELECT=fused); nsplit: scan
// partial planes in la.zpart
cudaError_t launch_select_fused(const SelArgs &s, const LayerArgs &la, int nsplit, int do_gather,
                                int num_sms, cudaStream_t st);
// rows a3-a4 (hc_select_pass.cu): rows of <= 64K candidates in one cluster kernel, longer rows
// in three passes (force = 1: the passes for any length); nsplit > 1: z carries no folded max/min
// wg: K3 fused with Eq. 5 over HBM values (k_sel_write_gather) when non-null: wg->out gets the
// output, wpart [rows][select_wg_maxc][128] / wdone [rows] (zeroed) are its partials / counters
struct SelGather { const LayerArgs *a; float *wpart; uint32_t *wdone; int used; };  // used: set when K3G ran
cudaError_t launch_select(SelArgs s, int nsplit, int num_sms, cudaStream_t st, int force = 0,
                          SelGather *wg = nullptr);
// K3G alone (the sharded finish: s.pre built by the shard's counts, idx_base = the shard's base)
cudaError_t launch_select_write_gather(const SelArgs &s, const LayerArgs &a, float *wpart, uint32_t *wdone,
                                       int num_sms, cudaStream_t st, int64_t idx_base);
// contributor slots per row of k_sel_write_gather (CTAs over contiguous ranges of `per` items)
inline int select_wg_maxc(int64_t nch, int64_t per) { return (int)((nch + per - 1) / per + 1); }
constexpr int kSelChunk = 4096;
// HeadState::state of the selection passes (hc_select_pass.cu; the sharded finish marks rows done)
constexpr uint32_t kStRefine1 = 1, kStRefine2 = 2, kStDone = 3, kStError = 4;
constexpr int kTableU = 8;     // k_table: units per CTA (max)
constexpr int kTableQ = 8192;  // k_table: staged query floats per CTA (32 KiB)  // tokens per chunk of the selection passes (16 KB of z)
inline int64_t select_chunks(int64_t n) { return (n + kSelChunk - 1) / kSelChunk; }
inline int64_t select_list_cap(int64_t n) { int64_t c = n / 16; return c < 4096 ? 4096 : c; }

// sequence-sharded phases (hc_shard.cu)
int shard_chunks(int64_t n);
cudaError_t launch_shard_stats(const LayerArgs &a, int nsplit, int32_t *stats, cudaStream_t st);
cudaError_t launch_shard_hist1(const LayerArgs &a, const int32_t *gstats, unsigned long long *h1,
                               cudaStream_t st);
cudaError_t launch_shard_hist2(const LayerArgs &a, const SelArgs &s, const int32_t *gstats,
                               const unsigned long long *h1, unsigned long long *h2, cudaStream_t st);
cudaError_t launch_shard_counts(const LayerArgs &a, const SelArgs &s, const unsigned long long *h2,
                                uint32_t *chunk, unsigned long long *cnt, cudaStream_t st);
cudaError_t launch_shard_finish(const LayerArgs &a, const SelArgs &s, const uint32_t *chunk,
                                const unsigned long long *allcnt, int rank, int64_t base,
                                float *part, float *out, cudaStream_t st, int64_t *grange = nullptr,
                                float *rpart = nullptr, uint32_t *rdone = nullptr,
                                float *upart = nullptr, uint32_t *udone = nullptr,
                                unsigned long long *pre = nullptr, float *wpart = nullptr);

// f4 (iii) App. B block-wise prefill attention (hc_prefill.cu), d = 128
cudaError_t launch_blockwise_attn(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t n,
                                  int Hq, int Hkv, int64_t bs, float *out, cudaStream_t s);

// f3(ii) packed codes (hc_encode.cu)
cudaError_t launch_pack13(const uint16_t *src, int64_t strips, int64_t n, int64_t src_stride,
                          uint8_t *dst, int64_t n_cap, cudaStream_t s);

// R8 shared per-KV-head selection (hc_group.cu): sel_idx / sel_w / hs.ksel of the G rows
int grp_chunks(int64_t n);
cudaError_t launch_group_select(const LayerArgs &a, int nsplit, cudaStream_t st);

// Eq. 5 with GQA union de-duplication (hc_gather.cu)
int gather_union_chunks(int64_t n_cand);
cudaError_t launch_gather_union(const LayerArgs &a, float *part, uint32_t *done, cudaStream_t s);
cudaError_t launch_add_partial(float *out, const float *part, int64_t n, cudaStream_t s);
int gather_rows_chunks(int64_t k_cap);
cudaError_t launch_gather_rows(const LayerArgs &a, int64_t k_cap, float *part, uint32_t *done,
                               cudaStream_t s);

// standalone select (R5b): float scores -> fixed-point z, hs init (M, zmin, e, kappa)
cudaError_t launch_select_float_prep(const float *scores, int64_t rows, int64_t n, float *z,
                                     int64_t z_stride, HeadState *hs, float kappa0,
                                     cudaStream_t s, uint32_t *ghist = nullptr,
                                     unsigned long long *gmass = nullptr);

}  // namespace hc
