// Memory-side ceiling of a deal pass on B200: read 2^28 u64 keys linearly and
// write them as runs of R keys into S output streams (tile t's run s lands at
// s * (n / S) + t * R), no ranking.  Compares with a plain copy.  The deal's
// write pattern at 2^28 uniform keys is S = 256 streams of ~16-key runs.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scatter_bw scatter_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void copy_k(const uint64_t* __restrict__ a, uint64_t* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// one CTA of 256 threads per 4096-key tile (grid-stride over tiles): key i of
// the tile goes to run s = i / R (mod S), position within run i % R
template <int R>
__global__ void scatter_k(const uint64_t* __restrict__ a, uint64_t* __restrict__ b, size_t n, int S) {
  const size_t tiles = n / 4096, stream_len = n / S;
  for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < 4096; i += 256) {
      const int run = i / R, s = run % S, k = run / S;  // 4096 / R runs over S streams
      const size_t o = (size_t)s * stream_len + t * (size_t)(4096 / S) + (size_t)k * R + i % R;
      b[o] = a[t * 4096 + i];
    }
  }
}

// the same streams, but lane-scattered: consecutive keys of a tile go to
// different streams (key i -> stream i % 256, position i / 256 in its run), so
// every warp store touches 32 runs (a deal writing straight from registers)
__global__ void scatter_lanes_k(const uint64_t* __restrict__ a, uint64_t* __restrict__ b, size_t n) {
  const size_t tiles = n / 4096, stream_len = n / 256;
  for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (int i = threadIdx.x; i < 4096; i += 256) {
      const size_t o = (size_t)(i % 256) * stream_len + t * 16 + i / 256;
      b[o] = a[t * 4096 + i];
    }
  }
}

int main() {
  const size_t n = (size_t)1 << 28;
  uint64_t *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 1, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    const int K = 10;
    for (int k = 0; k < K; ++k) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= K;
    printf("%-28s %.3f ms  %.2f TB/s (read+write)\n", name, ms, 2.0 * n * 8 / (ms * 1e-3) / 1e12);
  };
  timeit("copy", [&] { copy_k<<<sms * 8, 256>>>(a, b, n); });
  timeit("scatter S=256 R=16", [&] { scatter_k<16><<<sms * 8, 256>>>(a, b, n, 256); });
  timeit("scatter S=256 R=32", [&] { scatter_k<32><<<sms * 8, 256>>>(a, b, n, 128); });
  timeit("scatter S=64 R=64", [&] { scatter_k<64><<<sms * 8, 256>>>(a, b, n, 64); });
  timeit("lane-scattered S=256 R=16", [&] { scatter_lanes_k<<<sms * 8, 256>>>(a, b, n); });
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
