// Microbenchmark (tools only): counting "x < me" over a smem array, 32-bit
// integer compare vs packed fp16x2 HSET2+HADD2 on 14-bit integer patterns.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void k_int(const uint32_t* g, uint32_t* out, int iters) {
  __shared__ uint32_t s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = g[i];
  __syncthreads();
  const uint32_t me = s[(threadIdx.x * 37) & 1023];
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int b = ((it * 67 + threadIdx.x / 32 * 4) & 255) * 4;
#pragma unroll
    for (int x = 0; x < 16; x += 4) {
      uint4 v = *reinterpret_cast<const uint4*>(&s[(b + x) & 1023]);
      acc += (int)(v.x - me) < 0; acc += (int)(v.y - me) < 0;
      acc += (int)(v.z - me) < 0; acc += (int)(v.w - me) < 0;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_h2(const uint32_t* g, uint32_t* out, int iters) {
  __shared__ uint32_t s[1024];  // 2048 halves
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = g[i];
  __syncthreads();
  const unsigned short meb = reinterpret_cast<const unsigned short*>(s)[(threadIdx.x * 37) & 2047];
  const __half2 me2 = __halves2half2(__ushort_as_half(meb), __ushort_as_half(meb));
  __half2 acc = __float2half2_rn(0.f);
  for (int it = 0; it < iters; ++it) {
    const int b = ((it * 67 + threadIdx.x / 32 * 4) & 255) * 4;
#pragma unroll
    for (int x = 0; x < 8; x += 2) {  // 4 words = 8 halves per 2 LDS.64
      uint2 v = *reinterpret_cast<const uint2*>(&s[(b + x) & 1023]);
      acc = __hadd2(acc, __hlt2(*reinterpret_cast<__half2*>(&v.x), me2));
      acc = __hadd2(acc, __hlt2(*reinterpret_cast<__half2*>(&v.y), me2));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)__low2float(acc) + (uint32_t)__high2float(acc);
}
// correctness of fp16 ordering on patterns [0x0400, 0x43ff]
__global__ void k_check(uint32_t* bad) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;  // 0 .. 2^28
  const unsigned short x = 0x0400 + (a & 0x3fff), y = 0x0400 + ((a >> 14) & 0x3fff);
  __half2 hx = __halves2half2(__ushort_as_half(x), __ushort_as_half(y));
  __half2 hy = __halves2half2(__ushort_as_half(y), __ushort_as_half(x));
  __half2 r = __hlt2(hx, hy);
  const bool lo = __low2float(r) != 0.f, hi = __high2float(r) != 0.f;
  if (lo != (x < y) || hi != (y < x)) atomicAdd(bad, 1u);
}

int main() {
  const int n = 1024; uint32_t h[n];
  uint32_t s = 12345;
  for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; h[i] = s >> 1; }
  uint32_t *g, *out, *bad; cudaMalloc(&g, 4 * n); cudaMalloc(&out, 4 << 22); cudaMalloc(&bad, 4);
  cudaMemcpy(g, h, 4 * n, cudaMemcpyHostToDevice);
  cudaMemset(bad, 0, 4);
  k_check<<<(1 << 28) / 256, 256>>>(bad);
  uint32_t hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("fp16 order mismatches over 2^28 pairs: %u\n", hb);
  // make halves valid: patterns 0x0400..0x43ff
  for (int i = 0; i < n; ++i) h[i] = (0x0400 + (h[i] & 0x3fff)) | ((0x0400 + ((h[i] >> 14) & 0x3fff)) << 16);
  uint32_t* g2; cudaMalloc(&g2, 4 * n); cudaMemcpy(g2, h, 4 * n, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512, iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  k_int<<<blocks, threads>>>(g, out, iters);
  cudaEventRecord(a); k_int<<<blocks, threads>>>(g, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  double members = (double)blocks * threads * iters * 16;
  printf("int32 LEA: %.3f ms, %.3f SM-cycles per warp-member\n", ms, ms * 1e-3 * 1.965e9 / (members / 32 / sms));
  k_h2<<<blocks, threads>>>(g2, out, iters);
  cudaEventRecord(a); k_h2<<<blocks, threads>>>(g2, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("fp16x2   : %.3f ms, %.3f SM-cycles per warp-member  (%s)\n", ms, ms * 1e-3 * 1.965e9 / (members / 32 / sms), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
