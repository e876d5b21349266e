// dfr_overflow.cu — GPU Monte Carlo of the Fast Radix overflow model
// (§3.1).
//
// Fast Radix deals a pass into buckets of ESTIMATED capacity ceil(N/M)
// (Alg. 3 l.2) and sends a record whose bucket is full to
// overflow space (Alg. 3 l.8-9).  For uniform inputs the overflow of one pass
// is the balls-into-bins excess  sum_i max(0, X_i - ceil(N/M))  of N records
// over M buckets; the paper models its expected fraction with Eq. 1 / Eq. 2
// (P:296-301).  This kernel samples it: one CTA per trial throws the N records
// into M shared-memory counters and reduces the excess.
//
// Random numbers: SplitMix64 as a counter-based generator (the published
// definition): trial t uses the stream key k_t = mix(key + (t+1)*GAMMA) and
// record b goes to bucket  hi32(mix(k_t + (b+1)*GAMMA)) * M >> 32.
#include <cuda_runtime.h>

#include <cstdint>

#include "dfr.h"

namespace dfr {
namespace {

constexpr unsigned long long GAMMA = 0x9E3779B97F4A7C15ull;
constexpr int MC_THREADS = 512;
constexpr uint32_t MC_MAX_M = 16384;  // 64 KB of counters

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void __launch_bounds__(MC_THREADS) k_overflow_mc(unsigned long long n, uint32_t m,
                                                           uint32_t trials, unsigned long long key,
                                                           unsigned long long* out) {
  extern __shared__ uint32_t cnt[];
  __shared__ unsigned long long s_part[MC_THREADS / 32];
  const unsigned long long cap = (n + m - 1) / m;  // the estimated bucket capacity ceil(N/M)
  for (uint32_t t = blockIdx.x; t < trials; t += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const unsigned long long kt = mix64(key + (unsigned long long)(t + 1) * GAMMA);
    for (unsigned long long b = threadIdx.x; b < n; b += blockDim.x) {
      const unsigned long long r = mix64(kt + (b + 1) * GAMMA);
      const uint32_t bin = __umulhi((uint32_t)(r >> 32), m);  // hi32(r) * m >> 32
      atomicAdd(&cnt[bin], 1u);
    }
    __syncthreads();
    unsigned long long ex = 0;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
      ex += cnt[i] > cap ? cnt[i] - cap : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) ex += __shfl_xor_sync(0xffffffffu, ex, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = ex;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long s = 0;
      for (int w = 0; w < MC_THREADS / 32; ++w) s += s_part[w];
      out[t] = s;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace dfr

extern "C" int dfr_overflow_mc(uint64_t n, uint32_t m, uint32_t trials, uint64_t key,
                               uint64_t* d_overflow, dfr_stream_t stream) {
  if (trials == 0) return DFR_OK;
  if (!d_overflow || m < 1 || m > dfr::MC_MAX_M) return DFR_ERR_INVALID;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return DFR_ERR_CUDA;
  const size_t smem = (size_t)m * 4;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute((const void*)dfr::k_overflow_mc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return DFR_ERR_CUDA;
  const uint32_t grid = trials < (uint32_t)(4 * sms) ? trials : (uint32_t)(4 * sms);
  dfr::k_overflow_mc<<<grid, dfr::MC_THREADS, smem, (cudaStream_t)stream>>>(
      n, m, trials, key, reinterpret_cast<unsigned long long*>(d_overflow));
  return cudaGetLastError() == cudaSuccess ? DFR_OK : DFR_ERR_CUDA;
}
