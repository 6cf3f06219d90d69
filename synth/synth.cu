// synth/synth.cu -- device-side twin of synth/__init__.py (input generation only,
// none of the method's arithmetic).  Integer splitmix64 counter streams, so the
// device tensors are bit-identical to the numpy ones.
#include <cuda_fp16.h>
#include <stdint.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

__device__ __forceinline__ uint64_t fin(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// out[s * strip_stride + j] = code(keys[s], j, c) for j < n, s < nstrips
__global__ void k_codes(uint16_t *out, const uint64_t *keys, int64_t nstrips, int64_t strip_stride,
                        int64_t n, uint32_t c, int64_t start) {
  const int64_t s = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (s >= nstrips) return;
  const uint64_t key = keys[s];
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = fin(key + (uint64_t)(j + start + 1) * GOLDEN);
    out[s * strip_stride + j] = (uint16_t)(((u >> 32) * (uint64_t)c) >> 32);
  }
}

__device__ __forceinline__ uint16_t v16(uint64_t u) {
  const int64_t x = (int64_t)(u & 0xffff) + (int64_t)((u >> 16) & 0xffff) +
                    (int64_t)((u >> 32) & 0xffff) + (int64_t)(u >> 48) - 131070;
  const float f = (float)x * 0x1p-15f;  // exact
  return __half_as_ushort(__float2half_rn(f));
}

// out[s * strip_stride + j*d + e] = v16(u64(keys[s], j*d + e)), rows [0, n)
__global__ void k_values(uint16_t *out, const uint64_t *keys, int64_t nstrips, int64_t strip_stride,
                         int64_t n, int d, int64_t start) {
  const int64_t s = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (s >= nstrips) return;
  const uint64_t key = keys[s];
  const int64_t tot = n * d;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; t < tot;
       t += (int64_t)gridDim.x * blockDim.x * 8) {
    uint16_t h[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) h[q] = v16(fin(key + (uint64_t)(t + start * d + q + 1) * GOLDEN));
    uint4 v;
    v.x = h[0] | ((uint32_t)h[1] << 16);
    v.y = h[2] | ((uint32_t)h[3] << 16);
    v.z = h[4] | ((uint32_t)h[5] << 16);
    v.w = h[6] | ((uint32_t)h[7] << 16);
    *reinterpret_cast<uint4 *>(out + s * strip_stride + t) = v;
  }
}

extern "C" int synth_codes(uint16_t *out, const uint64_t *keys, int64_t nstrips,
                           int64_t strip_stride, int64_t n, uint32_t c, int64_t start, void *stream) {
  if (nstrips <= 0 || n <= 0) return 0;
  dim3 grid((unsigned)((n + 255) / 256 < 64 ? (n + 255) / 256 : 64), (unsigned)(nstrips < 65535 ? nstrips : 65535),
            (unsigned)((nstrips + 65534) / 65535));
  k_codes<<<grid, 256, 0, (cudaStream_t)stream>>>(out, keys, nstrips, strip_stride, n, c, start);
  return (int)cudaGetLastError();
}

extern "C" int synth_values(uint16_t *out, const uint64_t *keys, int64_t nstrips,
                            int64_t strip_stride, int64_t n, int d, int64_t start, void *stream) {
  if (nstrips <= 0 || n <= 0) return 0;
  const int64_t tot8 = n * d / 8;
  dim3 grid((unsigned)((tot8 + 255) / 256 < 256 ? (tot8 + 255) / 256 : 256), (unsigned)(nstrips < 65535 ? nstrips : 65535),
            (unsigned)((nstrips + 65534) / 65535));
  k_values<<<grid, 256, 0, (cudaStream_t)stream>>>(out, keys, nstrips, strip_stride, n, d, start);
  return (int)cudaGetLastError();
}
