// hc_host.cu -- the paper's "CPU part" of Eq. 2 (§3.2):
// Eq. 5's sparse weighted sum over the offloaded values, executed on host threads from
// the selection the GPU produced -- for the whole token range, or for the token range
// [tok_begin, tok_end) the host owns in the heterogeneous split (the GPU pulls the rest
// over the host link, hc_gather_values; DESIGN §8b f1).
//
// Work item = (KV unit u = (b, kv), token chunk of g_chunk tokens).  For each of the
// unit's G query heads the item cuts the head's ascending kept list to the chunk (binary
// search) and accumulates w_j·V_j in fp32; heads run back to back over the same chunk, so
// a row kept by several heads is read from DRAM once and from the core's L2 afterwards
// (the GQA union, as in k_gather_union).  Chunk partials are added in chunk order:
// results do not depend on the thread count or schedule.
// fp16 -> fp32 with F16C (AVX-512 or AVX2, runtime-dispatched), rows prefetched
// g_pf entries ahead; scalar table fallback on CPUs without F16C.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <thread>
#include <vector>

#include "../../include/hc.h"
#include "hc_internal.h"

namespace {

int64_t g_chunk = 4096;                // tokens per work item (HC_HOST_CHUNK)
std::atomic<uint64_t> g_ready_wait_ns{0};  // HC_WORKER_STATS: thread-time spent waiting on staging
int g_pf = 32;                        // kept rows prefetched ahead (HC_HOST_PF)
int g_hint = 0;                       // 0: T0, 1: T1, 2: T2 (HC_HOST_HINT)

float g_h2f[65536];
std::atomic<int> g_h2f_ready{0};

float half_bits_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h >> 15) << 31, exp = (h >> 10) & 0x1f, man = h & 0x3ff;
  uint32_t bits;
  if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else {
      float v = (float)man * 5.9604644775390625e-08f;  // man * 2^-24
      memcpy(&bits, &v, 4);
      bits |= sign;
    }
  } else if (exp == 31) {
    bits = sign | 0x7f800000u | (man << 13);
  } else {
    bits = sign | ((exp + 112u) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

void init_table() {
  if (g_h2f_ready.load(std::memory_order_acquire)) return;
  for (uint32_t h = 0; h < 65536; ++h) g_h2f[h] = half_bits_to_float((uint16_t)h);
  g_h2f_ready.store(1, std::memory_order_release);
}

enum Isa { kScalar = 0, kAvx2 = 1, kAvx512 = 2 };
Isa detect_isa() {
  static int isa = -1;
  if (const char *ev = getenv("HC_HOST_ISA")) {  // test override: scalar | avx2 | avx512
    if (!strcmp(ev, "scalar")) return kScalar;
    if (!strcmp(ev, "avx2") && __builtin_cpu_supports("avx2") && __builtin_cpu_supports("f16c") &&
        __builtin_cpu_supports("fma"))
      return kAvx2;
  }
  if (isa < 0) {
    __builtin_cpu_init();
    if (__builtin_cpu_supports("avx512f") && __builtin_cpu_supports("f16c") && __builtin_cpu_supports("fma"))
      isa = kAvx512;
    else if (__builtin_cpu_supports("avx2") && __builtin_cpu_supports("f16c") && __builtin_cpu_supports("fma"))
      isa = kAvx2;
    else
      isa = kScalar;
  }
  return (Isa)isa;
}

struct HostArgs {
  const int32_t *idx;
  const float *w;
  const int64_t *k;
  int64_t rows, k_stride;
  const uint16_t *V;
  int64_t v_b_stride, v_kv_stride;
  int32_t Hq, G, d;
  float *out;
  int32_t threads;
  int64_t tok_begin, tok_end;  // host-owned token range (global indices)
  bool owned_once;
  // streaming input (doorbell worker): unit u's rows are valid once ready[u] == epoch;
  // the range is then used as given (no clamp pass over the rows)
  const volatile uint32_t *ready = nullptr;
  uint32_t epoch = 0;
};

inline void prefetch_row(const uint16_t *p, int d) {
  const char *c = reinterpret_cast<const char *>(p);
  if (g_hint == 0) for (int o = 0; o < d * 2; o += 64) _mm_prefetch(c + o, _MM_HINT_T0);
  else if (g_hint == 1) for (int o = 0; o < d * 2; o += 64) _mm_prefetch(c + o, _MM_HINT_T1);
  else for (int o = 0; o < d * 2; o += 64) _mm_prefetch(c + o, _MM_HINT_T2);
}

// acc[0..d) += Σ_{r in [lo, hi)} w[r] · V[ix[r]]
__attribute__((target("avx512f,f16c,fma"))) void accum_avx512(const uint16_t *Vb, const int32_t *ix,
                                                              const float *wt, int64_t lo, int64_t hi,
                                                              int d, float *acc) {
  if (d == 128) {
    __m512 a[8];
    for (int q = 0; q < 8; ++q) a[q] = _mm512_loadu_ps(acc + 16 * q);
    for (int64_t r = lo; r < hi; ++r) {
      if (r + g_pf < hi) prefetch_row(Vb + (int64_t)ix[r + g_pf] * 128, 128);
      const uint16_t *v = Vb + (int64_t)ix[r] * 128;
      const __m512 w = _mm512_set1_ps(wt[r]);
      for (int q = 0; q < 8; ++q)
        a[q] = _mm512_fmadd_ps(w, _mm512_cvtph_ps(_mm256_loadu_si256((const __m256i *)(v + 16 * q))), a[q]);
    }
    for (int q = 0; q < 8; ++q) _mm512_storeu_ps(acc + 16 * q, a[q]);
    return;
  }
  for (int64_t r = lo; r < hi; ++r) {
    if (r + g_pf < hi) prefetch_row(Vb + (int64_t)ix[r + g_pf] * d, d);
    const uint16_t *v = Vb + (int64_t)ix[r] * d;
    const __m512 w = _mm512_set1_ps(wt[r]);
    for (int e = 0; e < d; e += 16)
      _mm512_storeu_ps(acc + e, _mm512_fmadd_ps(w, _mm512_cvtph_ps(_mm256_loadu_si256((const __m256i *)(v + e))),
                                                _mm512_loadu_ps(acc + e)));
  }
}

__attribute__((target("avx2,f16c,fma"))) void accum_avx2(const uint16_t *Vb, const int32_t *ix,
                                                         const float *wt, int64_t lo, int64_t hi, int d,
                                                         float *acc) {
  for (int64_t r = lo; r < hi; ++r) {
    if (r + g_pf < hi) prefetch_row(Vb + (int64_t)ix[r + g_pf] * d, d);
    const uint16_t *v = Vb + (int64_t)ix[r] * d;
    const __m256 w = _mm256_set1_ps(wt[r]);
    for (int e = 0; e < d; e += 8)
      _mm256_storeu_ps(acc + e, _mm256_fmadd_ps(w, _mm256_cvtph_ps(_mm_loadu_si128((const __m128i *)(v + e))),
                                                _mm256_loadu_ps(acc + e)));
  }
}

void accum_scalar(const uint16_t *Vb, const int32_t *ix, const float *wt, int64_t lo, int64_t hi, int d,
                  float *acc) {
  for (int64_t r = lo; r < hi; ++r) {
    if (r + g_pf < hi) __builtin_prefetch(Vb + (int64_t)ix[r + g_pf] * d, 0, 0);
    const uint16_t *v = Vb + (int64_t)ix[r] * d;
    const float wr = wt[r];
    for (int e = 0; e < d; ++e) acc[e] += wr * g_h2f[v[e]];
  }
}

int64_t lower_bound_i32(const int32_t *a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

void run(const HostArgs &a) {
  const Isa isa = detect_isa();
  // dev overrides, read once (thread-safe static init; run() is called from several threads)
  static const bool env_read = [] {
    if (const char *ev = getenv("HC_HOST_PF")) g_pf = atoi(ev);
    if (const char *ev = getenv("HC_HOST_HINT")) g_hint = atoi(ev);
    if (const char *ev = getenv("HC_HOST_CHUNK")) { const long v = atol(ev); if (v >= 256) g_chunk = v; }
    return true;
  }();
  (void)env_read;
  if (isa == kScalar) init_table();
  const int nt = a.threads > 0 ? a.threads : omp_get_max_threads();
  const int G = a.G, d = a.d;
  const int64_t units = a.rows / G;
  // clamp the range to the tokens actually kept (lists are ascending)
  int64_t last = a.tok_end - 1;
  if (!a.ready) {
    last = -1;
    for (int64_t row = 0; row < a.rows; ++row)
      if (a.k[row] > 0 && a.idx[row * a.k_stride + a.k[row] - 1] > last) last = a.idx[row * a.k_stride + a.k[row] - 1];
  }
  const int64_t t0 = a.tok_begin, t1 = a.tok_end < last + 1 ? a.tok_end : last + 1;
  const int64_t nch = t1 > t0 ? (t1 - t0 + g_chunk - 1) / g_chunk : 0;
  if (nch == 0) {
    memset(a.out, 0, sizeof(float) * (size_t)a.rows * d);
    return;
  }
  // chunk partials [units][nch][G][d], reused across calls by the calling thread
  thread_local std::vector<float> part;
  const size_t need = (size_t)units * nch * G * d;
  if (part.size() < need) part.resize(need);
  float *P = part.data();
  const int64_t items = units * nch;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1)
  for (int64_t it = 0; it < items; ++it) {
    const int64_t u = it / nch, c = it - u * nch;
    if (a.ready) {  // wait for this unit's staged lists (units arrive in order)
      if (a.ready[u] != a.epoch) {
        const auto w0 = std::chrono::steady_clock::now();
        while (a.ready[u] != a.epoch) _mm_pause();
        g_ready_wait_ns.fetch_add((uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                                      std::chrono::steady_clock::now() - w0).count(),
                                  std::memory_order_relaxed);
      }
      std::atomic_thread_fence(std::memory_order_acquire);
    }
    const int64_t j0 = t0 + c * g_chunk, j1 = j0 + g_chunk < t1 ? j0 + g_chunk : t1;
    const int64_t b = (u * G) / a.Hq, kv = ((u * G) % a.Hq) / G;
    const uint16_t *Vb = a.V + b * a.v_b_stride + kv * a.v_kv_stride;
    float *pp = P + (size_t)it * G * d;
    memset(pp, 0, sizeof(float) * (size_t)G * d);
    for (int h = 0; h < G; ++h) {
      const int64_t row = u * G + h;
      const int32_t *ix = a.idx + row * a.k_stride;
      const float *wt = a.w + row * a.k_stride;
      const int64_t kk = a.k[row];
      const int64_t lo = lower_bound_i32(ix, kk, j0), hi = lower_bound_i32(ix, kk, j1);
      if (lo >= hi) continue;
      float *acc = pp + (size_t)h * d;
      if (isa == kAvx512 && d % 16 == 0) accum_avx512(Vb, ix, wt, lo, hi, d, acc);
      else if (isa != kScalar && d % 8 == 0) accum_avx2(Vb, ix, wt, lo, hi, d, acc);
      else { init_table(); accum_scalar(Vb, ix, wt, lo, hi, d, acc); }
    }
  }
  // out[row] = Σ_c partial[u][c][h] in chunk order
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t row = 0; row < a.rows; ++row) {
    const int64_t u = row / G, h = row - u * G;
    float *o = a.out + row * d;
    for (int e = 0; e < d; ++e) o[e] = 0.0f;
    for (int64_t c = 0; c < nch; ++c) {
      const float *pp = P + ((size_t)(u * nch + c) * G + h) * d;
      for (int e = 0; e < d; ++e) o[e] += pp[e];
    }
  }
}

void CUDART_CB host_cb(void *p) {
  HostArgs *a = static_cast<HostArgs *>(p);
  run(*a);
  if (a->owned_once) delete a;
}

hc_status check(const int32_t *idx, const float *w, const int64_t *k, const uint16_t *V, float *out,
                int64_t rows, int32_t Hq, int32_t G, int32_t d, int64_t tok_begin, int64_t tok_end,
                int64_t n_valid) {
  if (!idx || !w || !k || !V || !out) return HC_ERR_ARG;
  if (rows < 0 || Hq <= 0 || G <= 0 || d <= 0 || d > 256 || Hq % G || rows % G) return HC_ERR_SHAPE;
  // only rows [0, n_valid) of each (b, kv) exist in the host store: a range past it would
  // read beyond the layer's values (or the resident window's tokens, which live in HBM)
  if (tok_begin < 0 || tok_end < tok_begin || n_valid < 0 || tok_end > n_valid) return HC_ERR_RANGE;
  return HC_OK;
}

hc_status enqueue(const HostArgs &proto, hc_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  // a captured host node may run many times: its argument block lives as long as the library
  HostArgs *a = new HostArgs(proto);
  a->owned_once = cap != cudaStreamCaptureStatusActive;
  if (cudaLaunchHostFunc(s, host_cb, a) != cudaSuccess) {
    delete a;
    return HC_ERR_CUDA;
  }
  return HC_OK;
}


// ---------------------------------------------------------------------------------------
// Doorbell host worker: the heterogeneous split without graph host nodes (a host node costs
// ~250 us round trip on the B200 box, tools/hostnode_latency.py).  A persistent host thread
// polls per-job mailboxes in pinned mapped memory:
//   GPU  k_submit: every row copies its kept entries with index < t_split (binary search in
//        the ascending list) into the job's host staging, writes k_host[row]; the last CTA
//        (device completion counter, system-scope fences) writes the descriptor
//        {t_split, V offset} and bumps req[job];
//   host worker: sees req != seen, runs the engine (OpenMP, its own team), writes out_host,
//        then done[job] = req (release);
//   GPU  k_wait: one thread spins (globaltimer-bounded, __nanosleep) until done == req, so
//        the consumer kernels (hc_add_partial) see out_host.
// Everything the GPU does is kernels: graph-capturable; replays re-ring the same mailbox.
struct Mailbox {      // pinned, mapped; one per job
  volatile uint32_t req, done;
  volatile int64_t t_split, v_off;
  volatile uint32_t err;
};

struct Job {
  int64_t rows, k_stride;
  const uint16_t *V;   // host pointer of the store's layer 0 (offset per submit)
  int64_t v_b_stride, v_kv_stride;
  int32_t Hq, G, d;
  float *out;          // host
  float *out_d;        // device alias of out (pinned mapped), or null: poisoned by k_wait on timeout
  int32_t *idx_h;      // staging (pinned mapped) [rows][k_stride]
  float *w_h;
  int64_t *k_h;        // [rows]
  int32_t *idx_d;      // device aliases of the staging
  float *w_d;
  int64_t *k_d;
  Mailbox *mb_h, *mb_d;
  uint32_t *ctr;       // device: [0] completion counter of k_submit, [1] epoch, [2..] per-unit rows staged
  uint32_t *ready_h, *ready_d;  // pinned mapped [units]: epoch of the unit's last staging
  uint32_t seen;
};

}  // namespace

namespace hc {  // the worker's kernels (named for launch lists)

__global__ void k_submit(const int32_t *sel_idx, const float *sel_w, const int64_t *sel_k, int64_t k_stride,
                         int64_t rows, int G, int64_t t_split, int64_t v_off, int32_t *idx_h, float *w_h,
                         int64_t *k_h, Mailbox *mb, uint32_t *ctr, volatile uint32_t *ready) {
  // the epoch of this submission: the device counter is only advanced by the last CTA to
  // finish, after every CTA has read it here
  __shared__ uint32_t s_epoch;
  __shared__ int64_t s_p;
  if (threadIdx.x == 0) s_epoch = *(volatile uint32_t *)&ctr[1] + 1u;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // ring first: the worker starts at once and
    mb->t_split = t_split;                    // consumes units as their ready flags flip
    mb->v_off = v_off;
    __threadfence_system();
    mb->req = epoch;
    __threadfence_system();
  }
  // rows in unit-major order, gridDim.x rows in flight: early units become ready early
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    if (threadIdx.x == 0) {
      const int32_t *li = sel_idx + row * k_stride;
      int64_t lo = 0, hi = sel_k[row];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)li[mid] < t_split) lo = mid + 1; else hi = mid;
      }
      s_p = lo;
      k_h[row] = lo;
    }
    __syncthreads();
    const int64_t p = s_p;
    const int32_t *si = sel_idx + row * k_stride;
    const float *sw = sel_w + row * k_stride;
    int32_t *di = idx_h + row * k_stride;
    float *dw = w_h + row * k_stride;
    if ((k_stride & 3) == 0) {
      const int64_t p4 = p & ~(int64_t)3;
      for (int64_t e = (int64_t)threadIdx.x * 4; e < p4; e += (int64_t)blockDim.x * 4) {
        *reinterpret_cast<int4 *>(di + e) = *reinterpret_cast<const int4 *>(si + e);
        *reinterpret_cast<float4 *>(dw + e) = *reinterpret_cast<const float4 *>(sw + e);
      }
      for (int64_t e = p4 + threadIdx.x; e < p; e += blockDim.x) { di[e] = si[e]; dw[e] = sw[e]; }
    } else {
      for (int64_t e = threadIdx.x; e < p; e += blockDim.x) { di[e] = si[e]; dw[e] = sw[e]; }
    }
    __threadfence_system();  // this thread's staging writes before the unit's count
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t u = row / G;
      const uint32_t prev = atomicAdd(&ctr[2 + u], 1u);
      if (prev == (uint32_t)G - 1u) {  // the unit's last row: publish it
        ctr[2 + u] = 0u;
        __threadfence_system();
        ready[u] = epoch;
        __threadfence_system();
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&ctr[0], 1u);
    if (prev == gridDim.x - 1) {  // every CTA has read the epoch: advance it
      ctr[0] = 0u;
      *(volatile uint32_t *)&ctr[1] = epoch;
    }
  }
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// On timeout the job is marked failed (hc_host_worker_status -> HC_ERR_CUDA) AND its output
// is poisoned with NaN, so a consumer that runs anyway (hc_add_partial) cannot pass a stale
// or half-written host share off as a result.
__global__ void k_wait(Mailbox *mb, uint64_t timeout_ns, float *out, int64_t n_out) {
  __shared__ int s_fail;
  if (threadIdx.x == 0) {
    const uint32_t want = mb->req;
    const uint64_t t0 = gtimer();
    s_fail = 0;
    while (mb->done != want) {
      __nanosleep(1000);
      if (gtimer() - t0 > timeout_ns) { mb->err = 1u; s_fail = 1; break; }
    }
    __threadfence_system();
  }
  __syncthreads();
  if (s_fail && out) {
    for (int64_t i = threadIdx.x; i < n_out; i += blockDim.x) out[i] = __int_as_float(0x7fc00000);
    __threadfence_system();
  }
}

}  // namespace hc

struct hc_host_worker {
  std::vector<Job> jobs;
  std::atomic<int> njobs{0};
  std::atomic<bool> stop{false};
  std::atomic<bool> paused{false};
  std::thread th;
  // HC_WORKER_STATS=1: time in the engine and idle time between jobs, printed by destroy
  bool stats = false;
  double busy_s = 0, idle_s = 0;
  long jobs_run = 0;
  int threads;
  uint64_t timeout_ns;
  int max_jobs;
};

namespace {

void worker_loop(hc_host_worker *w) {
  int idle = 0;
  auto last_done = std::chrono::steady_clock::now();
  while (!w->stop.load(std::memory_order_acquire)) {
    bool did = false;
    const int nj = w->paused.load(std::memory_order_acquire) ? 0 : w->njobs.load(std::memory_order_acquire);
    for (int j = 0; j < nj; ++j) {
      Job &jb = w->jobs[j];
      const uint32_t r = jb.mb_h->req;
      if (r == jb.seen) continue;
      std::atomic_thread_fence(std::memory_order_acquire);
      HostArgs a{jb.idx_h, jb.w_h, jb.k_h, jb.rows, jb.k_stride, jb.V + jb.mb_h->v_off, jb.v_b_stride,
                 jb.v_kv_stride, jb.Hq, jb.G, jb.d, jb.out, w->threads, 0, jb.mb_h->t_split, false};
      a.ready = jb.ready_h;
      a.epoch = r;
      const auto t0 = std::chrono::steady_clock::now();
      run(a);
      jb.seen = r;
      // a submission that arrived while this one ran can only follow a timed-out wait (the
      // stream waits for `done` before the next submit): its staging was overwritten under
      // the engine, so this result is stale -- do not publish it; the next poll serves the
      // new request (the timed-out wait already marked the job failed and poisoned `out`)
      std::atomic_thread_fence(std::memory_order_acquire);
      if (jb.mb_h->req != r) continue;
      std::atomic_thread_fence(std::memory_order_release);
      jb.mb_h->done = r;
      if (w->stats) {
        const auto t1 = std::chrono::steady_clock::now();
        w->busy_s += std::chrono::duration<double>(t1 - t0).count();
        w->idle_s += std::chrono::duration<double>(t0 - last_done).count();
        ++w->jobs_run;
        last_done = t1;
      }
      did = true;
    }
    if (did) { idle = 0; continue; }
    if (++idle < 200000) _mm_pause();
    else std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

}  // namespace

extern "C" {

hc_status hc_host_weighted_sum_range(const int32_t *idx, const float *w, const int64_t *k, int64_t rows,
                                     int64_t k_stride, const uint16_t *V, int64_t v_b_stride,
                                     int64_t v_kv_stride, int64_t n_valid, int32_t Hq, int32_t G, int32_t d,
                                     int64_t tok_begin, int64_t tok_end, float *out, int32_t threads) {
  hc_status st = check(idx, w, k, V, out, rows, Hq, G, d, tok_begin, tok_end, n_valid);
  if (st) return st;
  HostArgs a{idx, w, k, rows, k_stride, V, v_b_stride, v_kv_stride, Hq, G, d, out, threads,
             tok_begin, tok_end, false};
  run(a);
  return HC_OK;
}

hc_status hc_enqueue_host_weighted_sum_range(const int32_t *idx, const float *w, const int64_t *k,
                                             int64_t rows, int64_t k_stride, const uint16_t *V,
                                             int64_t v_b_stride, int64_t v_kv_stride, int64_t n_valid,
                                             int32_t Hq, int32_t G, int32_t d, int64_t tok_begin,
                                             int64_t tok_end, float *out, int32_t threads,
                                             hc_stream_t stream) {
  hc_status st = check(idx, w, k, V, out, rows, Hq, G, d, tok_begin, tok_end, n_valid);
  if (st) return st;
  return enqueue(HostArgs{idx, w, k, rows, k_stride, V, v_b_stride, v_kv_stride, Hq, G, d, out, threads,
                          tok_begin, tok_end, false},
                 stream);
}

hc_status hc_host_weighted_sum(const int32_t *idx, const float *w, const int64_t *k, int64_t rows,
                               int64_t k_stride, const uint16_t *V, int64_t v_b_stride,
                               int64_t v_kv_stride, int64_t n_valid, int32_t Hq, int32_t G, int32_t d,
                               float *out, int32_t threads) {
  return hc_host_weighted_sum_range(idx, w, k, rows, k_stride, V, v_b_stride, v_kv_stride, n_valid, Hq, G,
                                    d, 0, n_valid, out, threads);
}

hc_status hc_enqueue_host_weighted_sum(const int32_t *idx, const float *w, const int64_t *k,
                                       int64_t rows, int64_t k_stride, const uint16_t *V,
                                       int64_t v_b_stride, int64_t v_kv_stride, int64_t n_valid,
                                       int32_t Hq, int32_t G, int32_t d, float *out, int32_t threads,
                                       hc_stream_t stream) {
  return hc_enqueue_host_weighted_sum_range(idx, w, k, rows, k_stride, V, v_b_stride, v_kv_stride, n_valid,
                                            Hq, G, d, 0, n_valid, out, threads, stream);
}

hc_status hc_host_worker_create(int32_t threads, int32_t max_jobs, double timeout_s, hc_host_worker **out) {
  if (!out || max_jobs < 1 || timeout_s <= 0) return HC_ERR_ARG;
  hc_host_worker *w = new hc_host_worker();
  w->threads = threads > 0 ? threads : omp_get_max_threads();
  w->timeout_ns = (uint64_t)(timeout_s * 1e9);
  w->max_jobs = max_jobs;
  if (const char *ev = getenv("HC_WORKER_STATS")) w->stats = atoi(ev) != 0;
  g_ready_wait_ns.store(0);
  w->jobs.resize(max_jobs);  // fixed storage: the worker reads entries while jobs are added
  w->th = std::thread(worker_loop, w);
  *out = w;
  return HC_OK;
}

hc_status hc_host_worker_destroy(hc_host_worker *w) {
  if (!w) return HC_ERR_ARG;
  w->stop.store(true, std::memory_order_release);
  if (w->th.joinable()) w->th.join();
  if (w->stats && w->jobs_run > 1)
    fprintf(stderr,
            "[hc_host_worker] %ld jobs: engine %.1f us/job, idle between jobs %.1f us/job, "
            "staging waits %.1f thread-us/job\n",
            w->jobs_run, 1e6 * w->busy_s / w->jobs_run, 1e6 * w->idle_s / (w->jobs_run - 1),
            1e-3 * (double)g_ready_wait_ns.load() / w->jobs_run);
  for (int j = 0; j < w->njobs.load(); ++j) {
    Job &jb = w->jobs[j];
    cudaFreeHost(jb.idx_h);
    cudaFreeHost(jb.w_h);
    cudaFreeHost(jb.k_h);
    cudaFreeHost((void *)jb.mb_h);
    cudaFreeHost(jb.ready_h);
    cudaFree(jb.ctr);
  }
  delete w;
  return HC_OK;
}

hc_status hc_host_worker_add_job(hc_host_worker *w, int64_t rows, int64_t k_stride, const uint16_t *V,
                                 int64_t v_b_stride, int64_t v_kv_stride, int32_t Hq, int32_t G, int32_t d,
                                 float *out, int32_t *job) {
  if (!w || !V || !out || !job) return HC_ERR_ARG;
  if (rows <= 0 || k_stride < 1 || Hq <= 0 || G <= 0 || d <= 0 || d > 256 || Hq % G || rows % G)
    return HC_ERR_SHAPE;
  const int j = w->njobs.load();
  if (j >= w->max_jobs) return HC_ERR_CAPACITY;
  Job jb{};
  jb.rows = rows; jb.k_stride = k_stride; jb.V = V; jb.v_b_stride = v_b_stride; jb.v_kv_stride = v_kv_stride;
  jb.Hq = Hq; jb.G = G; jb.d = d; jb.out = out;
  const unsigned fl = cudaHostAllocMapped | cudaHostAllocPortable;
  bool ok = cudaHostAlloc((void **)&jb.idx_h, (size_t)rows * k_stride * 4, fl) == cudaSuccess &&
            cudaHostAlloc((void **)&jb.w_h, (size_t)rows * k_stride * 4, fl) == cudaSuccess &&
            cudaHostAlloc((void **)&jb.k_h, (size_t)rows * 8, fl) == cudaSuccess &&
            cudaHostAlloc((void **)&jb.mb_h, sizeof(Mailbox), fl) == cudaSuccess &&
            cudaHostAlloc((void **)&jb.ready_h, (size_t)(rows / G) * 4, fl) == cudaSuccess &&
            cudaMalloc((void **)&jb.ctr, (size_t)(2 + rows / G) * 4) == cudaSuccess &&
            cudaMemset(jb.ctr, 0, (size_t)(2 + rows / G) * 4) == cudaSuccess;
  if (ok) {
    memset((void *)jb.mb_h, 0, sizeof(Mailbox));
    memset(jb.ready_h, 0, (size_t)(rows / G) * 4);
    ok = cudaHostGetDevicePointer((void **)&jb.idx_d, jb.idx_h, 0) == cudaSuccess &&
         cudaHostGetDevicePointer((void **)&jb.w_d, jb.w_h, 0) == cudaSuccess &&
         cudaHostGetDevicePointer((void **)&jb.k_d, jb.k_h, 0) == cudaSuccess &&
         cudaHostGetDevicePointer((void **)&jb.mb_d, (void *)jb.mb_h, 0) == cudaSuccess &&
         cudaHostGetDevicePointer((void **)&jb.ready_d, jb.ready_h, 0) == cudaSuccess;
  }
  if (!ok) return HC_ERR_CUDA;
  if (cudaHostGetDevicePointer((void **)&jb.out_d, out, 0) != cudaSuccess) {
    jb.out_d = nullptr;  // out not mapped: the timeout still sets the error flag
    cudaGetLastError();
  }
  jb.seen = 0;
  w->jobs[j] = jb;
  w->njobs.store(j + 1, std::memory_order_release);
  *job = j;
  return HC_OK;
}

hc_status hc_host_worker_submit(hc_host_worker *w, int32_t job, const int32_t *sel_idx, const float *sel_w,
                                const int64_t *sel_k, int64_t t_split, int64_t n_valid, int64_t v_off,
                                hc_stream_t stream) {
  if (!w || !sel_idx || !sel_w || !sel_k) return HC_ERR_ARG;
  if (job < 0 || job >= w->njobs.load()) return HC_ERR_RANGE;
  if (t_split < 0 || v_off < 0 || n_valid < 0 || t_split > n_valid) return HC_ERR_RANGE;
  Job &jb = w->jobs[job];
  static int ctas = -1;  // rows in flight (unit-major order); HC_SUBMIT_CTAS dev override
  if (ctas < 0) { const char *ev = getenv("HC_SUBMIT_CTAS"); ctas = ev ? atoi(ev) : 64; if (ctas < 1) ctas = 64; }
  const unsigned grid = (unsigned)(jb.rows < ctas ? jb.rows : ctas);
  hc::k_submit<<<grid, 256, 0, (cudaStream_t)stream>>>(sel_idx, sel_w, sel_k, jb.k_stride, jb.rows, jb.G, t_split,
                                                   v_off, jb.idx_d, jb.w_d, jb.k_d, jb.mb_d, jb.ctr, jb.ready_d);
  hc::note_launch();
  return cudaGetLastError() == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

hc_status hc_host_worker_wait(hc_host_worker *w, int32_t job, hc_stream_t stream) {
  if (!w) return HC_ERR_ARG;
  if (job < 0 || job >= w->njobs.load()) return HC_ERR_RANGE;
  const Job &jb = w->jobs[job];
  hc::k_wait<<<1, 256, 0, (cudaStream_t)stream>>>(jb.mb_d, w->timeout_ns, jb.out_d, jb.rows * jb.d);
  hc::note_launch();
  return cudaGetLastError() == cudaSuccess ? HC_OK : HC_ERR_CUDA;
}

hc_status hc_host_worker_pause(hc_host_worker *w, int32_t paused) {
  if (!w) return HC_ERR_ARG;
  w->paused.store(paused != 0, std::memory_order_release);
  return HC_OK;
}

hc_status hc_host_worker_status(hc_host_worker *w) {
  if (!w) return HC_ERR_ARG;
  for (int j = 0; j < w->njobs.load(); ++j)
    if (w->jobs[j].mb_h->err) return HC_ERR_CUDA;
  return HC_OK;
}

}  // extern "C"
