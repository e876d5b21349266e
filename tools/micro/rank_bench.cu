// Microbenchmark (tools only, not product): throughput of warp peer-mask
// primitives on sm_100a: match.any.sync vs 8 ballots (two codegen forms).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; return x; }

__global__ void k_match(uint32_t* sink, int iters) {
  uint32_t s = hash(threadIdx.x + blockIdx.x * 977), acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t d = (s >> (i & 7)) & 255u;
    acc += __match_any_sync(0xffffffffu, d);
    s = s * 1664525u + 1013904223u;
  }
  if (acc == 0x12345) sink[0] = acc;
}
__global__ void k_ballot_c(uint32_t* sink, int iters) {
  uint32_t s = hash(threadIdx.x + blockIdx.x * 977), acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t d = (s >> (i & 7)) & 255u;
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const bool set = (d >> b) & 1u;
      const uint32_t v = __ballot_sync(0xffffffffu, set);
      peers &= set ? v : ~v;
    }
    acc += peers;
    s = s * 1664525u + 1013904223u;
  }
  if (acc == 0x12345) sink[0] = acc;
}
__device__ __forceinline__ uint32_t peers_ptx(uint32_t d) {
  uint32_t peers;
  asm("{\n .reg .pred p;\n .reg .b32 v, t;\n"
      " and.b32 t, %1, 1; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; mov.b32 %0, v;\n"
      " and.b32 t, %1, 2; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
      " and.b32 t, %1, 4; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
      " and.b32 t, %1, 8; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
      " and.b32 t, %1, 16; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
      " and.b32 t, %1, 32; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
      " and.b32 t, %1, 64; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
      " and.b32 t, %1, 128; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
      "}" : "=r"(peers) : "r"(d));
  return peers;
}
__global__ void k_ballot_ptx(uint32_t* sink, int iters) {
  uint32_t s = hash(threadIdx.x + blockIdx.x * 977), acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t d = (s >> (i & 7)) & 255u;
    acc += peers_ptx(d);
    s = s * 1664525u + 1013904223u;
  }
  if (acc == 0x12345) sink[0] = acc;
}
// xor-accumulate form: diff |= v ^ spread(bit)
__global__ void k_ballot_xor(uint32_t* sink, int iters) {
  uint32_t s = hash(threadIdx.x + blockIdx.x * 977), acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t d = (s >> (i & 7)) & 255u;
    uint32_t diff = 0;
    const int x = (int)(d << 24);
#pragma unroll
    for (int b = 7; b >= 0; --b) {
      const int xb = x << (7 - b);
      const uint32_t v = __ballot_sync(0xffffffffu, xb < 0);
      diff |= v ^ (uint32_t)(xb >> 31);
    }
    acc += ~diff;
    s = s * 1664525u + 1013904223u;
  }
  if (acc == 0x12345) sink[0] = acc;
}
__global__ void k_empty(uint32_t* sink, int iters) {
  uint32_t s = hash(threadIdx.x + blockIdx.x * 977), acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t d = (s >> (i & 7)) & 255u;
    acc += d;
    s = s * 1664525u + 1013904223u;
  }
  if (acc == 0x12345) sink[0] = acc;
}

int main() {
  uint32_t* sink; cudaMalloc(&sink, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, void (*k)(uint32_t*, int)) {
    k<<<blocks, threads>>>(sink, iters);
    cudaEventRecord(a);
    k<<<blocks, threads>>>(sink, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double warp_ops = (double)blocks * threads / 32 * iters;
    double per_sm_cycles = ms * 1e-3 * 1.965e9 / (warp_ops / sms);
    printf("%-14s %8.3f ms  %.2f SM-cycles per warp-op  (%s)\n", name, ms, per_sm_cycles, cudaGetErrorString(cudaGetLastError()));
  };
  run("empty", k_empty);
  run("match_any", k_match);
  run("ballot_c", k_ballot_c);
  run("ballot_ptx", k_ballot_ptx);
  run("ballot_xor", k_ballot_xor);
  return 0;
}
