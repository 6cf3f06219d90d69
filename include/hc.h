/*
 * hc.h -- C ABI of the B200 (sm_100a) HCAttention decode hot path (libhc.so).
 *
 * HCAttention (arXiv 2507.19823) §3.2 "Heterogeneous Attention Computation":
 * keys are grouped-vector quantized, scores are table
 * lookups z̃_j = Σ_i T[i][P_ji] with T = q̄·C (Eq. 3), ã =
 * softmax(z̃/√d), tokens are selected by cumulative mass τ (Eq. 4,
 * P:240-252) and the output is Σ_{i∈Π_k*} ã*_i V_i (Eq. 5).
 * Citations "P:n" are lines of PAPER.md; "R<k>" are DESIGN.md §2 readings.
 *
 * Conventions (all entry points):
 *  - Tensors are caller-owned.  Pointers are DEVICE pointers unless stated;
 *    fp16 tensors are passed as uint16_t* (IEEE binary16 bit patterns).
 *  - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default)
 *    and never allocate or synchronise; they are CUDA-graph capturable.
 *  - Argument validation is synchronous: a non-HC_OK status is returned and
 *    nothing is launched; hc_last_error() gives a one-line reason (thread-local).
 *    Asynchronous CUDA faults surface as HC_ERR_CUDA from a later call.
 *  - Layouts are row-major, innermost index last.
 */
#ifndef HC_H_
#define HC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HC_OK = 0,
    HC_ERR_ARG = 1,         /* bad scalar argument (tau outside (0,1], k_max < 1, NULL ptr) */
    HC_ERR_SHAPE = 2,       /* dimension mismatch (g does not divide d, ...) */
    HC_ERR_RANGE = 3,       /* index / layer / value out of range */
    HC_ERR_CAPACITY = 4,    /* append beyond n_cap */
    HC_ERR_EMPTY = 5,       /* no candidates (n_q + n_res == 0) */
    HC_ERR_CUDA = 6,        /* a CUDA runtime error (launch or earlier async fault) */
    HC_ERR_NCCL = 7,        /* an NCCL call of the sequence-sharded path failed */
    HC_ERR_UNSUPPORTED = 8, /* valid but not built for (e.g. c > 8192, G not in {1,2,4}) */
    HC_ERR_WORKSPACE = 9    /* workspace NULL or smaller than *_workspace_bytes() */
} hc_status;

typedef void *hc_stream_t; /* cudaStream_t */

/* Grouped vector quantizer (§3.1): d-dim keys split into g groups of
 * dbar = d/g dims; c centroids per codebook slice; cbg codebook slices
 * (cbg == g: one codebook per group as C ∈ R^{g×c×dbar}; cbg == 1: one
 * codebook shared by all groups, Table 4b).
 * lut_bits: precision of the query/codebook table T (R2): 0 or 16 = 16-bit fixed point
 * (default, >= fp16 precision); 8 = the 8-bit table variant (R2b: ~bf16
 * worst-case precision, half the shared-memory traffic; requires G == 4).
 * Supported by the kernels: d % g == 0, dbar in {1,2,4,8,16}, 1 <= c <= 8192. */
typedef struct {
    int32_t d, g, c, cbg;
    int32_t lut_bits;
    int32_t code_bits; /* 0 or 16: u16 codes; 13: packed codes (NEXT f3(ii), see below) */
} hc_vq;

/* Packed 13-bit code layout (code_bits = 13, requires c <= 8192 and lut_bits = 16): every
 * (b, l, kv, group) strip of n_cap tokens is HC_STRIP13_BYTES(n_cap) = 13*n_cap/8 bytes:
 *   [lo: n_cap bytes, code & 0xff][nib: n_cap/2 bytes, (code >> 8) & 15, token t in byte
 *   t/2, low nibble for even t][bit: n_cap/8 bytes, code >> 12, token t at bit t%8 of byte t/8]
 * and hc_kcache.codes points at B*L*Hkv*g such strips (same order as the u16 layout).
 * 19 % fewer code bytes than u16 at g = 32 (52 vs 64 B per token and KV head). */
#define HC_STRIP13_BYTES(n_cap) ((int64_t)(n_cap) * 13 / 8)

/* Budget (R5): tau ∈ (0,1] is Eq. 4's cumulative-mass threshold (τ = 0.9 in
 * §4.1); k_max >= 1 caps the kept set: k_sel = min(k*(τ), k_max);
 * renorm = 0 keeps Eq. 5's unrenormalised ã* (default), 1 divides by the kept mass;
 * select_only = 0: the GPU computes Eq. 5 (default); 1: stop after the selection (sel_idx /
 * sel_w / sel_k must be given, `out` is not written) so Eq. 5 can run on the host over the
 * offloaded values -- the paper's own split (hc_host_weighted_sum).
 * shared_kv = 0: one selection per query head (default, DESIGN R5/R7); 1: ONE selection
 * per KV head shared by its G query heads, on their head-averaged attention mass (DESIGN
 * R8); each head keeps its own weights W_h/S_h over the shared
 * rows, so a value row is read once for G heads.  Takes renorm = 0 (else
 * HC_ERR_UNSUPPORTED); the G rows of sel_idx / sel_k are identical. */
typedef struct {
    float tau;
    int64_t k_max;
    int32_t renorm;
    int32_t select_only;
    int32_t shared_kv;
} hc_budget;

#define HC_MAX_LAYERS 256

/* Quantized key cache of one model (all layers).  Host struct; device buffers.
 *  codes    [B][L][Hkv][g][n_cap] uint16, GROUP-MAJOR (the index matrix P of P:227,
 *           0-based, one contiguous strip per (b,l,kv,group)); n_cap % 64 == 0.
 *  codebook [L][cbg][c][dbar] fp32 (one codebook set per layer, shared by its KV heads);
 *  cb_absmax [L][cbg][dbar] its per-dimension max |C| (optional, see hc_codebook_absmax).
 *  Recent window (R7, optional, res_cap = W >= 0): the newest n_res[l] <= W tokens keep
 *  exact keys/values resident: res_k/res_v [B][L][Hkv][W][d] fp16, token at global
 *  position p lives in slot p % W.  Candidates of a layer are the quantized tokens
 *  0..n_q-1 followed by the resident tokens n_q..n_q+n_res-1.
 *  n_q[l], n_res[l] are host-side counts, advanced by hc_append_kv. */
typedef struct {
    int32_t B, L, Hkv, G; /* batch, layers, KV heads, GQA group size (Hq = G*Hkv) */
    hc_vq vq;
    int64_t n_cap;
    uint16_t *codes;
    const float *codebook;
    const float *cb_absmax; /* optional [L][cbg][dbar]: max_m |C[l][ci][m][e]| (R2's bound;
                               hc_codebook_absmax fills it once); NULL = recomputed per call */
    int32_t res_cap;
    uint16_t *res_k;
    uint16_t *res_v;
    int64_t n_q[HC_MAX_LAYERS];
    int32_t n_res[HC_MAX_LAYERS];
} hc_kcache;

/* Value store (A8, "fully offloading the value matrix V").
 *  base [B][L][Hkv][n_cap][d] fp16.  placement HC_V_DEVICE: HBM pointer.
 *  HC_V_HOST_MAPPED: pinned host memory mapped into the device address space
 *  (cudaHostAlloc Mapped/Portable or cudaHostRegister Mapped), passed as its
 *  device-accessible address; rows are read zero-copy over the host link by the
 *  gather kernel, only the selected ones. */
enum { HC_V_DEVICE = 0, HC_V_HOST_MAPPED = 1 };
typedef struct {
    int32_t placement;
    uint16_t *base;
    int64_t n_cap;
} hc_vstore;

/* Optional debug taps of hc_decode_attention (any member may be NULL).
 *  z     [B][Hq][n_q+n_res] int32  fixed-point scores z̃ (R3), scale 2^-e
 *  e     [B][Hq] int32             table scale exponents (R2)
 *  S     [B][Hq] uint64            total mass Σ W (R4)
 *  M     [B][Hq] int32             max score
 *  kstar [B][Hq] int64             k*(τ) when τ decides the cut, -1 when the cap does */
typedef struct {
    int32_t *z;
    int32_t *e;
    uint64_t *S;
    int32_t *M;
    int64_t *kstar;
} hc_decode_debug;

const char *hc_last_error(void);
const char *hc_version(void);

/* Number of kernels this library has enqueued on streams (or captured into CUDA graphs)
 * since load.  Used by bench.py to report gpu_launches. */
uint64_t hc_launch_count(void);

/* Profiling hook (bench.py's roofline): record the two cudaEvent_t's (passed as void*)
 * on the call's stream immediately before and after the NEXT quantized-key scan kernel
 * launched by hc_decode_attention from this thread (one-shot; NULLs disable).  Inside
 * stream capture they become external event-record nodes of the graph. */
hc_status hc_profile_scan_events(void *begin_event, void *end_event);
/* Same, around the whole Eq. 3 stage of the NEXT hc_decode_attention call from this thread:
 * the table build (row a1) + the resident-token scorer + the quantized-key scan (row a2). */
hc_status hc_profile_eq3_events(void *begin_event, void *end_event);

/* Host value-store memory (A8): page-lock caller-allocated host memory (e.g. an
 * anonymous mapping advised for 2 MiB transparent huge pages, so random row reads by host
 * threads and by the GPU do not miss the TLB on every row) and map it into the device
 * address space (cudaHostRegister Portable | Mapped).  *dev_ptr = the device-accessible
 * address to put in hc_vstore.base (HC_V_HOST_MAPPED).  Synchronous; not for the hot path. */
hc_status hc_host_register(void *host, size_t bytes, void **dev_ptr);
hc_status hc_host_unregister(void *host);

/* Codebook constant of R2: out[l][ci][e] = max_m |codebook[l][ci][m][e]| for all L layers.
 * codebook [L][cbg][c][dbar] fp32, out [L][cbg][dbar] fp32 (device).  Call once per codebook
 * and store the result in hc_kcache.cb_absmax. */
hc_status hc_codebook_absmax(const float *codebook, hc_vq vq, int32_t L, float *out,
                             hc_stream_t stream);

/* Key encoding, R1 ("represented as nearest neighbor of the centroids"):
 *   codes[i*code_stride + r] = argmin_m ||keys[r][i*dbar:(i+1)*dbar] - C[ci][m]||², ties -> lowest m.
 * keys [rows][d] fp16; codebook [cbg][c][dbar] fp32 (ONE layer's codebook);
 * codes uint16 group-major with code_stride >= rows.  rows == 0 is a no-op. */
hc_status hc_quantize_keys(const uint16_t *keys, int64_t rows, const float *codebook, hc_vq vq,
                           uint16_t *codes, int64_t code_stride, hc_stream_t stream);

/* NEXT f4 -- codebook training: ONE MiniBatchKMeans step ("MiniBatchKMeans ...
 * batch size of 10,000"; Sculley 2010 Alg. 1 in its batched scikit-learn form, DESIGN F4):
 *   labels[i*b + s] = R1 nearest centroid of keys[sample[s]]'s group-i sub-vector under the
 *   codebook as it is at the start of the step; then for every centroid m of slice ci with
 *   n_m > 0 assigned sub-vectors summing to s_m:
 *     C_m <- (C_m·v_m + s_m) / (v_m + n_m)   (double, then fp32 round-to-nearest),
 *     v_m <- v_m + n_m.
 * keys [n_keys][d] fp16 (device); sample [b] int64 key-row indices (device; rows outside
 * [0, n_keys) are skipped, label 0xFFFF); codebook [cbg][c][dbar] fp32 and counts [cbg][c]
 * int64 (device, updated in place; counts start at 0 for a fresh codebook); labels [g][b]
 * u16 (device, optional).  s_m is summed exactly (int64 units of 2^-24), so the result
 * is independent of thread order.  ws >= hc_kmeans_workspace_bytes(vq, b). */
size_t hc_kmeans_workspace_bytes(hc_vq vq, int64_t b);

/* NEXT f4 (iii) -- App. B block-wise prefill attention (DESIGN F5): query i of
 * block kb = i / bs attends to the anchor block (keys j < bs) and causally to its own block
 * (kb*bs <= j <= i); block 0 is causal.  out[i][h] = softmax over that key set of
 * q[i][h]·k[j][h/(Hq/Hkv)] / sqrt(d), applied to v.  q [n][Hq][d], k, v [n][Hkv][d] fp16,
 * out [n][Hq][d] fp32 (device).  d = 128, bs % 64 == 0, Hq % Hkv == 0. */
hc_status hc_blockwise_attention(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t n,
                                 int32_t Hq, int32_t Hkv, int32_t d, int64_t bs, float *out,
                                 hc_stream_t stream);

/* Prefill append: "when a block operation concludes, the quantization of the key cache"
 * -- encode n new keys per sequence (R1, bulk encoder) into codes positions
 * [n_q, n_q + n) of `layer` and copy their values into the value store; n_q += n.
 * k, v [B][n][Hkv][d] fp16 (device).  16-bit codes, no resident window in use
 * (n_res == 0), else HC_ERR_UNSUPPORTED; HC_ERR_CAPACITY if n_q + n > n_cap. */
hc_status hc_prefill_append(hc_kcache *kc, const hc_vstore *vs, int32_t layer, const uint16_t *k,
                            const uint16_t *v, int64_t n, hc_stream_t stream);

/* Pack u16 codes into the 13-bit strip layout (code_bits = 13, above): for s < strips,
 * t < n: strip s of dst (HC_STRIP13_BYTES(n_cap) bytes each) gets src[s*src_stride + t].
 * Codes must be < 8192 (HC_ERR_RANGE is not checked on the device: higher bits are
 * dropped).  n <= n_cap, n_cap % 64 == 0; tokens >= n of each strip are left unchanged.
 * Device pointers; asynchronous on `stream`. */
hc_status hc_pack_codes13(const uint16_t *src, int64_t strips, int64_t n, int64_t src_stride,
                          uint8_t *dst, int64_t n_cap, hc_stream_t stream);
hc_status hc_kmeans_step(const uint16_t *keys, int64_t n_keys, const int64_t *sample, int64_t b,
                         hc_vq vq, float *codebook, int64_t *counts, uint16_t *labels, void *ws,
                         size_t ws_bytes, hc_stream_t stream);

/* Append one decode token for layer `layer` (all B sequences, all Hkv heads).
 * k_new, v_new [B][Hkv][d] fp16.  With res_cap == 0 the key is encoded (R1) into
 * codes at position n_q[layer] and v is written to the value store there.  With a
 * window, the token enters the window; if it was full, the oldest resident token is
 * encoded into P and its value moved to the value store first.
 * Advances kc->n_q[layer] / kc->n_res[layer].  HC_ERR_CAPACITY if n_q would exceed n_cap. */
hc_status hc_append_kv(hc_kcache *kc, const hc_vstore *vs, int32_t layer, const uint16_t *k_new,
                       const uint16_t *v_new, hc_stream_t stream);

/* Bytes of device workspace hc_decode_attention needs for this cache shape
 * (independent of the current n; sized for n_cap + res_cap). */
size_t hc_decode_workspace_bytes(const hc_kcache *kc, hc_budget budget);

/* One decode step of one layer for all B×Hq query heads (rows a1-a5):
 *   q [B][Hq][d] fp16 (query head h uses KV head h / G)
 *   out [B][Hq][d] fp32 = Σ_{j∈sel} ã_j V_j  (Eq. 5)
 *   sel_idx [B][Hq][k_max] int32 (optional): kept global token indices, ascending
 *   sel_w   [B][Hq][k_max] fp32  (optional): their weights ã_j
 *   sel_k   [B][Hq] int64        (optional): k_sel
 * HC_ERR_EMPTY if the layer has no tokens.  ws: >= hc_decode_workspace_bytes. */
hc_status hc_decode_attention(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs,
                              int32_t layer, hc_budget budget, float *out, int32_t *sel_idx,
                              float *sel_w, int64_t *sel_k, const hc_decode_debug *dbg, void *ws,
                              size_t ws_bytes, hc_stream_t stream);

/* hc_append_kv + hc_decode_attention in one call (a decode step appends the new token, then
 * attends over the cache including it; PAPER.md P:227 then P:229-287): the append's encode /
 * value copy runs on a library-owned side stream forked from `stream` (event edges; one side
 * stream per device and host thread) concurrently with the table build, and the scan waits for
 * it -- the result equals the two calls in sequence.  Arguments as in the two calls (no debug
 * taps); kc->n_q / n_res advance as in hc_append_kv.  Graph-capturable. */
hc_status hc_append_decode_attention(const uint16_t *q, hc_kcache *kc, const hc_vstore *vs, int32_t layer,
                                     const uint16_t *k_new, const uint16_t *v_new, hc_budget budget, float *out,
                                     int32_t *sel_idx, float *sel_w, int64_t *sel_k, void *ws, size_t ws_bytes,
                                     hc_stream_t stream);

/* Standalone Eq. 4 selection on real-valued scores (R5b):
 *   scores [rows][n] fp32 (z̃ = q·Kᵀ, unscaled; softmax uses 1/√d)
 *   idx [rows][k_max] int32 ascending, w [rows][k_max] fp32, k [rows] int64. */
size_t hc_select_workspace_bytes(int64_t rows, int64_t n, hc_budget budget);
hc_status hc_select_topk(const float *scores, int64_t rows, int64_t n, int32_t d, hc_budget budget,
                         int32_t *idx, float *w, int64_t *k, void *ws, size_t ws_bytes,
                         hc_stream_t stream);

/* ---- Host-side Eq. 5 (the paper's "CPU part").
 * out[row][e] = Σ_{r<k[row]} w[row][r] · V_row(idx[row][r])[e], fp32 accumulation in index
 * order, on `threads` host threads (0 = all cores).  All pointers are HOST pointers:
 *   idx [rows][k_stride] int32, w [rows][k_stride] fp32, k [rows] int64 (e.g. the D2H copies
 *   of hc_decode_attention's selection with select_only = 1), row = b*Hq + hq;
 *   V: value store of ONE layer, fp16, row j of (b, kv = hq / G) at
 *      V + b*v_b_stride + kv*v_kv_stride + j*d  (elements);
 *   n_valid: rows 0..n_valid-1 of every (b, kv) hold values (the layer's n_q); only kept
 *      tokens j < n_valid are summed (resident-window tokens j >= n_q live in HBM: add them
 *      with hc_gather_values(tok_begin = n_q));
 *   out [rows][d] fp32.
 * hc_host_weighted_sum runs synchronously; hc_enqueue_host_weighted_sum enqueues the same
 * work as a host node on `stream` (cudaLaunchHostFunc; graph-capturable), executing after
 * prior work on the stream (e.g. the D2H copies of idx / w / k). */
hc_status hc_host_weighted_sum(const int32_t *idx, const float *w, const int64_t *k, int64_t rows,
                               int64_t k_stride, const uint16_t *V, int64_t v_b_stride,
                               int64_t v_kv_stride, int64_t n_valid, int32_t Hq, int32_t G, int32_t d,
                               float *out, int32_t threads);
hc_status hc_enqueue_host_weighted_sum(const int32_t *idx, const float *w, const int64_t *k,
                                       int64_t rows, int64_t k_stride, const uint16_t *V,
                                       int64_t v_b_stride, int64_t v_kv_stride, int64_t n_valid,
                                       int32_t Hq, int32_t G, int32_t d, float *out, int32_t threads,
                                       hc_stream_t stream);

/* ---- Heterogeneous Eq. 5 (§3.2 "Heterogeneous Attention Computation"): the
 * kept value rows are summed partly on the GPU (zero-copy pull over the host link) and
 * partly by host threads over host DRAM (the paper's CPU part), concurrently, split
 * by token index at t_split <= n_q (DESIGN §8b f1; paper_2507_19823_b200/hetero.py):
 *   out = Σ_{j∈sel, j<t_split} ã_j V_j   (hc_*host_weighted_sum_range, host; value store only)
 *       + Σ_{j∈sel, j>=t_split} ã_j V_j  (hc_gather_values, GPU; incl. the resident window)
 *   joined by hc_add_partial.
 *
 * hc_host_weighted_sum_range: as hc_host_weighted_sum restricted to kept tokens
 *   tok_begin <= j < tok_end (rows with no kept token in range get 0).  Work items are
 *   (KV unit, 4096-token chunk); the G heads of a unit run back to back over a chunk so
 *   shared rows come from the core's cache; chunk partials are added in chunk order (the
 *   result does not depend on `threads`).  F16C/AVX-512 or AVX2 when the CPU has them.
 *   HC_ERR_RANGE if tok_begin < 0, tok_end < tok_begin or tok_end > n_valid. */
hc_status hc_host_weighted_sum_range(const int32_t *idx, const float *w, const int64_t *k, int64_t rows,
                                     int64_t k_stride, const uint16_t *V, int64_t v_b_stride,
                                     int64_t v_kv_stride, int64_t n_valid, int32_t Hq, int32_t G, int32_t d,
                                     int64_t tok_begin, int64_t tok_end, float *out, int32_t threads);
hc_status hc_enqueue_host_weighted_sum_range(const int32_t *idx, const float *w, const int64_t *k,
                                             int64_t rows, int64_t k_stride, const uint16_t *V,
                                             int64_t v_b_stride, int64_t v_kv_stride, int64_t n_valid,
                                             int32_t Hq, int32_t G, int32_t d, int64_t tok_begin,
                                             int64_t tok_end, float *out, int32_t threads,
                                             hc_stream_t stream);

/* Doorbell host worker: the host share of the split without graph host nodes (a
 * cudaLaunchHostFunc node costs ~250 us round trip; this path ~10 us).  A persistent host
 * thread (with its own OpenMP team of `threads`) polls per-job mailboxes in pinned mapped
 * memory.  A job = one host share of Eq. 5 for `rows` = B*Hq query heads over a host value
 * store V (HOST pointer of layer 0, strides in elements as hc_host_weighted_sum) into out
 * [rows][d] fp32 (HOST memory, e.g. pinned); its staging for the selection is owned by the
 * worker.  On `stream` (kernels only, graph-capturable):
 *   hc_host_worker_submit: copies each row's kept entries with index < t_split from the
 *     DEVICE selection (sel_idx/sel_w [rows][k_stride] ascending, sel_k [rows]) into the
 *     job's staging, then rings the job's doorbell with {t_split, v_off}; the worker then
 *     computes out = Σ_{kept j < t_split} w_j V[v_off + ...]_j (v_off = element offset of
 *     the layer in V) exactly as hc_host_weighted_sum_range(tok 0..t_split); n_valid = the
 *     layer's n_q (HC_ERR_RANGE if t_split > n_valid: window tokens are not in the host store);
 *   hc_host_worker_wait: a kernel that returns once the job's last submission is done (so
 *     later work on the stream sees out), or after timeout_s seconds, when the job is marked
 *     failed (hc_host_worker_status then returns HC_ERR_CUDA) and `out` is filled with NaN
 *     (if it is mapped pinned memory) so no consumer can take a stale share for a result;
 *     a result the worker finishes after a newer submission arrived is discarded.
 * Submissions of one job must not overlap (wait before the next submit).  add_job returns
 * HC_ERR_CAPACITY beyond max_jobs; create / add_job / destroy are setup calls for one
 * thread (the worker itself only reads jobs that add_job has published).  destroy stops the
 * thread (no wait may be pending). */
typedef struct hc_host_worker hc_host_worker;
hc_status hc_host_worker_create(int32_t threads, int32_t max_jobs, double timeout_s, hc_host_worker **out);
hc_status hc_host_worker_destroy(hc_host_worker *w);
hc_status hc_host_worker_add_job(hc_host_worker *w, int64_t rows, int64_t k_stride, const uint16_t *V,
                                 int64_t v_b_stride, int64_t v_kv_stride, int32_t Hq, int32_t G, int32_t d,
                                 float *out, int32_t *job);
hc_status hc_host_worker_submit(hc_host_worker *w, int32_t job, const int32_t *sel_idx, const float *sel_w,
                                const int64_t *sel_k, int64_t t_split, int64_t n_valid, int64_t v_off,
                                hc_stream_t stream);
hc_status hc_host_worker_wait(hc_host_worker *w, int32_t job, hc_stream_t stream);
hc_status hc_host_worker_status(hc_host_worker *w);
/* Maintenance / test hook: paused != 0 stops serving doorbells (pending waits then time out). */
hc_status hc_host_worker_pause(hc_host_worker *w, int32_t paused);

/* GPU Eq. 5 over a GIVEN selection, restricted to kept tokens tok_begin <= j < tok_end:
 *   out[b][h] = Σ_{r<sel_k[row], tok_begin<=sel_idx[row][r]<tok_end} sel_w[row][r] · V_j
 * with row = b*Hq + h.  sel_idx/sel_w [B*Hq][k_stride] (ascending indices per row) and
 * sel_k [B*Hq] are DEVICE arrays as hc_decode_attention writes them; V is the layer's value
 * store (HBM or host-mapped: only kept rows in range are read; rows kept by several GQA
 * heads once).  ws: hc_decode_workspace_bytes(kc, budget with k_max = k_stride); its
 * gather region is used (the selection arrays are the caller's).  An empty range writes 0.
 * HC_ERR_RANGE for tok_begin < 0 or tok_end < tok_begin. */
hc_status hc_gather_values(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, const int32_t *sel_idx,
                           const float *sel_w, const int64_t *sel_k, int64_t k_stride, int64_t tok_begin,
                           int64_t tok_end, float *out, void *ws, size_t ws_bytes, hc_stream_t stream);

/* out[i] += part[i] for i < n (fp32).  part may be host-mapped pinned memory (the host
 * share of the heterogeneous split, read zero-copy after the host node finished). */
hc_status hc_add_partial(float *out, const float *part, int64_t n, hc_stream_t stream);

/* ---- Sequence-sharded decode, one layer, R ranks (one per GPU).
 * Rank `rank` holds the contiguous GLOBAL token range [shard_base, shard_base + n_q[layer])
 * of every (b, layer, kv) unit (its own codes and value rows; no resident window).  The
 * scores are exact integers (R2/R3) and the softmax mass is a function of Δ = M − z only
 * (R4), so the global Eq. 4 selection is assembled from integer collectives that the
 * CALLER performs between the phases (NCCL over NVLink on GPUs; any backend works):
 *   hc_shard_begin   table + scan;   stats [rows][2] int32 {max z, -min z}  -> all-reduce MAX
 *   hc_shard_hist1   (global stats)  h1 [rows][4096][2] uint64 (count, mass)  -> all-reduce SUM
 *   hc_shard_hist2   (global h1)     h2 [rows][4096] uint64 (fine counts)     -> all-reduce SUM
 *   hc_shard_counts  (global h2)     cnt [rows][2] uint64 (#Δ<Δ*, #Δ==Δ*)     -> all-gather
 *   hc_shard_finish  (allcnt [R][rows][2]) writes this rank's kept tokens (global indices) at
 *                    their GLOBAL positions of sel_idx/sel_w [rows][k_max] (other ranks'
 *                    positions untouched) and its Eq. 5 numerator share out [rows][d] fp32
 *                                                                               -> all-reduce SUM
 * rows = B*Hq.  Every rank evaluates the same bounds on the same reduced integers, so the
 * kept index set equals the unsharded one bit for bit (R-invariance).  The workspace
 * (hc_shard_workspace_bytes) carries state between the phases of one layer. */
size_t hc_shard_workspace_bytes(const hc_kcache *kc, hc_budget budget);

/* ---- The sequence-sharded decode in ONE call: the five phases below
 * with the four exchanges between them issued by the library as NCCL collectives on `stream`
 * (all-reduce MAX of the score range, all-reduce SUM of the two integer histograms,
 * all-gather of the per-rank (strict, tie) counts, all-reduce SUM of the Eq. 5 numerators):
 * one layer, this rank's shard [shard_base, shard_base + n_q[layer]) of every unit, the
 * global Eq. 4 selection and the full output out [B][Hq][d] fp32 on every rank.
 *   sel_idx / sel_w [B*Hq][k_max] (required): this rank's kept tokens (GLOBAL indices,
 *     ascending) at their GLOBAL positions of each row's list; other ranks' slots untouched;
 *   sel_k [B*Hq] (optional): the global k_sel.
 * comm: an NCCL communicator of the `world` ranks (hc_nccl_comm_init, or any ncclComm_t of
 * the process's libnccl.so.2); NULL only with world == 1.  ws >= hc_decode_sharded_workspace_
 * bytes(kc, budget, world) (phase state + exchange buffers).  Graph-capturable (NCCL
 * collectives are).  NCCL is loaded at run time (dlopen libnccl.so.2, HC_NCCL_LIB overrides);
 * NCCL failures return HC_ERR_NCCL. */
typedef struct ncclComm *ncclComm_t; /* NCCL's opaque communicator (nccl.h) */
#define HC_NCCL_UNIQUE_ID_BYTES 128
hc_status hc_nccl_get_unique_id(void *id /* HC_NCCL_UNIQUE_ID_BYTES bytes, host */);
hc_status hc_nccl_comm_init(ncclComm_t *comm, int32_t world, const void *id, int32_t rank);
hc_status hc_nccl_comm_destroy(ncclComm_t comm);
size_t hc_decode_sharded_workspace_bytes(const hc_kcache *kc, hc_budget budget, int32_t world);
hc_status hc_decode_attention_sharded(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs,
                                      int32_t layer, hc_budget budget, float *out, int32_t *sel_idx,
                                      float *sel_w, int64_t *sel_k, int32_t rank, int32_t world,
                                      int64_t shard_base, ncclComm_t comm, void *ws, size_t ws_bytes,
                                      hc_stream_t stream);
hc_status hc_shard_begin(const uint16_t *q, const hc_kcache *kc, const hc_vstore *vs, int32_t layer,
                         hc_budget budget, int32_t *stats, void *ws, size_t ws_bytes,
                         hc_stream_t stream);
hc_status hc_shard_hist1(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                         const int32_t *gstats, uint64_t *h1, void *ws, size_t ws_bytes,
                         hc_stream_t stream);
hc_status hc_shard_hist2(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                         const int32_t *gstats, const uint64_t *h1, uint64_t *h2, void *ws,
                         size_t ws_bytes, hc_stream_t stream);
hc_status hc_shard_counts(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                          const uint64_t *h2, uint64_t *cnt, void *ws, size_t ws_bytes,
                          hc_stream_t stream);
hc_status hc_shard_finish(const hc_kcache *kc, const hc_vstore *vs, int32_t layer, hc_budget budget,
                          const uint64_t *allcnt, int32_t rank, int32_t world, int64_t shard_base,
                          float *out, int32_t *sel_idx, float *sel_w, int64_t *sel_k, void *ws,
                          size_t ws_bytes, hc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* HC_H_ */
