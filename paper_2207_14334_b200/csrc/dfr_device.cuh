// dfr_device.cuh — device building blocks of the B200 DFR sort (sm_100a).
//
// Citations: P:L = PAPER.md line L (arXiv 2207.14334), S:L = SPEC.md line L.
// Shares nothing with oracle/ (test infrastructure).
//
// Vocabulary (§2): a *pass* processes every record of a
// range on one digit; a *count* builds per-digit histograms; the *deal*
// places records into *buckets*.  A *segment* here is one DFR invocation
// (Alg. 4) on a contiguous bucket: the whole input at level 0,
// a large bucket (Alg. 4 l.11 "recurse on the large bucket") at level >= 1.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace dfr {

constexpr int THREADS = 256;             // one CTA = 8 warps
constexpr int WARPS = THREADS / 32;
// tuning knobs (tools/variants.sh builds alternatives side by side)
#ifndef DFR_LB_SLEEP
#define DFR_LB_SLEEP 64  // ns of back-off when a look-back round makes no progress
#endif
#ifndef DFR_RANK_G
#define DFR_RANK_G 2  // keys whose peer masks are computed together in warp_rank
#endif
#ifndef DFR_COLD
#define DFR_COLD __noinline__  // rare paths called from the diversion's window loop
#endif
#ifndef DFR_HIST_MINB
#define DFR_HIST_MINB 4  // histogram: minimum resident CTAs per SM (register cap)
#endif
#ifndef DFR_CLAIM_AFTER_BARRIER
#define DFR_CLAIM_AFTER_BARRIER 1  // deal: claim the next ticket after the look-back barrier
#endif
// streaming TMA loads: keys are read once per pass, so they may leave L2 first
// (DFR_TMA_EVICT_FIRST=1: L2::evict_first cache hint)
#if DFR_TMA_EVICT_FIRST
#define DFR_TMA_LOAD                                                                              \
  "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"                 \
  " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
#else
#define DFR_TMA_LOAD "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
#endif
#ifndef DFR_LEVEL1_CHAIN
#define DFR_LEVEL1_CHAIN 1  // recursion level 1 through the stand-alone kernels (else in k_levels)
#endif
#ifndef DFR_HIST_TILES
#define DFR_HIST_TILES 8  // histogram: deal tiles counted per step of its tile loop
#endif
#ifndef DFR_DEAL_PF
#define DFR_DEAL_PF 1  // deal: L2 prefetch of the next tile when its ticket is claimed
#endif
#ifndef DFR_FUSED_SB
#define DFR_FUSED_SB 3  // fused pass: sub-bucket bits below the group (4 or 8 sub-buckets per digit)
#endif
#ifndef DFR_LB_EARLY
#define DFR_LB_EARLY 0  // deal: the look-back's first round trip issued before the reorder
#endif
#ifndef DFR_FUSED_NT
#define DFR_FUSED_NT 256  // fused pass: threads per CTA (3 CTAs/SM)
#endif
#ifndef DFR_RUN_ATOMS
#define DFR_RUN_ATOMS 0  // atomic deal ranks: one atomic per run of equal digits in consecutive lanes
#endif
#ifndef DFR_HIST_COPIES
#define DFR_HIST_COPIES 1  // histogram: shared-memory counter sets per CTA (warp w uses w % copies)
#endif
#ifndef DFR_HIST_U
#define DFR_HIST_U 8  // histogram: 16-byte loads in flight per thread
#endif
#ifndef DFR_LB
#define DFR_LB 8  // look-back predecessors loaded per round trip
#endif
#ifndef DFR_WO_UNROLL
#define DFR_WO_UNROLL 6  // deal write-out unroll
#endif
#ifndef DFR_DV_CU
#define DFR_DV_CU 1  // diversion rank-count loop unroll
#endif
#ifndef DFR_FRANK8
#define DFR_FRANK8 1  // fused pass: sub-bucket words 4..7 compared in one round trip
#endif
#ifndef DFR_FRANK_SB
#define DFR_FRANK_SB 1  // fused pass: ranks by one thread per sub-bucket (<= DFR_FRANK_MA keys branch-free; longer ones via a work list; 0: one thread per key, r02c)
#endif
#ifndef DFR_FRANK_NB
#define DFR_FRANK_NB 4  // fused ranks: sub-buckets per batch of loads
#endif
#ifndef DFR_FRANK_MA
#define DFR_FRANK_MA 4  // fused ranks: sub-buckets of up to this many keys are ranked branch-free by their own thread
#endif
#ifndef DFR_FRANK_BL
#define DFR_FRANK_BL 2  // fused ranks: threads per long sub-bucket (each ranks 8 / BL keys of a group of 8)
#endif
#ifndef DFR_FWO_UNROLL
#define DFR_FWO_UNROLL 2  // fused pass: write-out unroll
#endif
#ifndef DFR_FLB_EARLY
#define DFR_FLB_EARLY 0  // fused pass: the look-back's first round trip issued before the ranks
#endif
#ifndef DFR_FLOAD_EARLY
#define DFR_FLOAD_EARLY 1  // fused pass (with DFR_FRANK_SB): the next tile's keys load during the ranks
#endif
#ifndef DFR_FLB
#define DFR_FLB 4  // fused pass: look-back predecessors loaded per round trip
#endif
constexpr int LB_PAD = 32;  // status rows in front of pass 0's table (>= DFR_LB, DFR_FLB)
static_assert(DFR_LB <= LB_PAD && DFR_FLB <= LB_PAD, "look-back pad");
constexpr int WO_UNROLL = DFR_WO_UNROLL, DV_CU = DFR_DV_CU, FWO_UNROLL = DFR_FWO_UNROLL;
constexpr int HCOPIES = DFR_HIST_COPIES;
static_assert(WARPS % HCOPIES == 0, "histogram copies");
constexpr int KPT = 16;                  // keys per thread per tile
constexpr int TILE = THREADS * KPT;      // 4096 keys per tile (hist / deal)
#ifndef DFR_WIN
#define DFR_WIN 1280
#endif
constexpr int WIN = DFR_WIN;             // diversion window (keys) per CTA
constexpr int MID_CAP = 4096;            // C: buckets N_d < s <= C finish on-chip
#ifndef DFR_SMALL_N
#define DFR_SMALL_N (1 << 21)
#endif
constexpr int SMALL_N = DFR_SMALL_N;     // inputs up to this size: all levels in k_levels
constexpr int MID_CAP_S = 1024;          // buckets up to this size: the 4-CTA/SM mid kernel
constexpr int MAX_ND = 256;              // composite index uses 8 bits
constexpr int MAX_PASSES = 4;            // top passes per group (p <= 3 for n < 2^30)
constexpr uint32_t FLAG_AGG = 1u << 30;  // look-back: tile aggregate available
constexpr uint32_t FLAG_INC = 2u << 30;  // look-back: inclusive prefix available
constexpr uint32_t VAL_MASK = (1u << 30) - 1;

// Seg::flags
constexpr uint32_t SEG_SKIP_DIVERT = 1u << 8;  // no diversion scan this level
constexpr uint32_t SEG_COPY = 1u << 9;         // finished, data in B: copy to A
constexpr uint32_t SEG_DONE = 1u << 10;        // finished in A
constexpr uint32_t SEG_SORTED = 1u << 11;      // passes reach digit 0: sorted after them

struct Seg {                    // one DFR invocation on a contiguous bucket
  uint32_t start, len;          // element range in the arrays
  int32_t hi;                   // top remaining digit; digits above are constant
  uint32_t buf;                 // buffer id holding the data: 0 = A (caller), 1 = B, 2 = C (scratch)
  uint32_t p;                   // top passes of this invocation (Alg. 4 l.4)
  int32_t low;                  // lowest digit of the group = hi - p + 1
  uint32_t tile0;               // first tile id (exclusive prefix over segments)
  uint32_t chunk0;              // first diversion chunk id
  uint32_t hist_off;            // first histogram row (one row of 256 per pass)
  uint32_t flags;               // bits 0..3: pass j skipped; SEG_* above
  uint32_t final_buf;           // buffer id holding the data after the passes
  uint32_t ntiles;              // tiles of this segment
  unsigned long long diff;      // OR over the segment of (key ^ key[start])
  uint32_t route;               // pass j: source id bits 4j..4j+1, destination id bits 4j+2..4j+3
  uint32_t pad;
};
static_assert(sizeof(Seg) == 64, "Seg layout");

struct MidE {                   // a bucket N_d < len <= C finished on-chip
  uint32_t start;
  uint16_t len;
  int8_t hi;
  uint8_t buf;
};

struct Ctl {
  uint32_t cur;                 // index of the current segment queue (0/1)
  uint32_t nseg;                // segments in the current level
  uint32_t total_tiles;
  uint32_t total_chunks;
  uint32_t ticket[MAX_PASSES];  // dynamic tile tickets per pass (forward progress)
  uint32_t next_count;          // segments queued for the next level
  uint32_t mid_count;           // mid buckets queued (all levels)
  uint32_t level;               // current level (0 = top call)
  uint32_t overflow;            // queue overflow guard (should stay 0)
  unsigned long long level0_large;
  unsigned long long mid_buckets;
  unsigned long long global_segments;
  uint32_t level0_p, level0_run;
  uint32_t levels_run, max_p;
  uint32_t fused_ok;            // level 0 ran the fused last pass (plan kernel's verdict)
  uint32_t fused_tiles;         // run-aligned tiles of the fused pass
  uint32_t fticket;             // dynamic tile ticket of the fused pass
  uint32_t fused_regular;       // fused pass: tickets below this have chain predecessor ticket - chains
  uint32_t fused_chains;        // fused pass: look-back chains (16, or 1 without the chain histogram)
  uint32_t fr_next_chunk;       // Fast Radix: overflow chunks handed out so far
  uint32_t fr_tiles;            // Fast Radix: tiles of the pass that reads the estimated layout
  uint32_t fr_overflow;         // Fast Radix: records the estimated pass dealt to overflow
  uint32_t mround[12];          // keys-only mid rounds: [r + 1] buckets queued for round r + 1
};

template <class K>
struct Params {
  K* A;                 // caller keys
  K* B;                 // scratch keys ("buffer the same size as the input")
  uint32_t* Av;         // caller values (pairs) or null
  uint32_t* Bv;         // scratch values or null
  K* C;                 // second scratch buffer (fused level 0 only, else null)
  uint32_t* Cv;
  Ctl* ctl;
  Seg* segq[2];
  MidE* midq;
  MidE* midq2;          // keys-only mid rounds: the queue of the odd rounds (capacity mid_cap)
  uint32_t* hist;       // histogram / bucket-offset rows, 256 u32 each
  uint32_t* status;     // look-back status words [MAX_PASSES][tiles_max][256]
  size_t status_stride; // words per pass
  uint32_t max_segs;
  uint32_t mid_cap;     // capacity of midq
  uint32_t hist_rows;   // capacity of hist (rows)
  uint32_t n_d;         // diversion threshold N_d
  uint32_t chunk;       // diversion chunk = WIN - 16/sizeof(K) - n_d
  uint32_t n;           // elements of the whole array
  uint32_t fuse;        // level 0 may fuse its last deal with the diversion (host decision; C != null)
  uint32_t* H;          // joint histogram of the group's two low digits [d_mid][d_low] (fuse)
  uint4* ftiles;        // run-aligned tiles of the fused pass in ticket order:
                        // (offset in the segment, length, ticket of the previous tile of its
                        // chain or ~0u, chain)
  uint32_t* J;          // fused level 0: [256][16] counts of (top digit, top 4 bits of the
                        // middle digit), then [16][256] chain bases (exclusive over chains)
  uint32_t skip_trivial;
  // keys only (dfr_config.stable_deals == 0): a deal whose tile is constant in
  // the group digits below its own ranks keys of equal digit in any order
  // (shared-memory atomics instead of the ballot multi-split).  Output-
  // invariant: equal keys are indistinguishable, every later pass of the group
  // is stable, and the buckets are then sorted on all lower digits (DESIGN R5)
  uint32_t unstable;
  uint32_t full_lsd;    // ablation: the top call sorts all D digits LSD (dfr_config.full_lsd)
  // Fast Radix estimation (dfr_config.fast_radix; Alg. 3): the
  // level-0 pass on the lowest group digit deals into ESTIMATED buckets of
  // fr_cap = ceil(n/256) keys at d * fr_cap of its destination buffer; a key
  // ranked past its bucket's capacity goes to the overflow chunk of
  // FR_CHUNK keys its bucket's rank falls in (chunks handed out on first
  // touch, after the 256 main regions: "virtually extending overflown
  // buckets"); the next pass reads bucket by bucket, main region then chunks.
  uint32_t fr;          // 1: level 0 runs Fast Radix estimation
  uint32_t fr_cap;
  uint32_t fr_kmax;     // chunk-table columns per bucket
  uint32_t* fr_ct;      // [256][fr_kmax] chunk id + 1 (0: not handed out; ~0u: being handed out)
  uint2* fr_tab;        // tiles of the pass that reads the estimated layout: (offset, length)
  uint32_t* fr_cnt;     // [2][256]: next-digit counts (exact offsets of the next pass), top-digit counts
  int D;                // digits per key
  __device__ __forceinline__ K* kbuf(uint32_t id) const { return id == 0 ? A : (id == 1 ? B : C); }
  __device__ __forceinline__ uint32_t* vbuf(uint32_t id) const {
    return id == 0 ? Av : (id == 1 ? Bv : Cv);
  }
};

// ------------------------------------------------------------------ helpers
template <class K>
__device__ __forceinline__ uint32_t digit_of(K k, int d) {
  return (uint32_t)(k >> (8 * d)) & 255u;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// ld_relaxed at p + OFF bytes (immediate offset: no address arithmetic)
template <int OFF>
__device__ __forceinline__ uint32_t ld_relaxed_off(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1+%2];" : "=r"(v) : "l"(p), "n"(OFF) : "memory");
  return v;
}
template <int LB, int K = 0>
__device__ __forceinline__ void ld_lookback(const uint32_t* p, uint32_t (&v)[LB]) {
  if constexpr (K < LB) {
    v[K] = ld_relaxed_off<-1024 * K>(p);
    ld_lookback<LB, K + 1>(p, v);
  }
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- TMA bulk copies (cp.async.bulk) + mbarrier ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// an mbarrier's memory is reused for other data after this (PTX: invalidate first)
__device__ __forceinline__ void mbar_inval(unsigned long long* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one thread: expect `bytes` and launch a 1-D bulk copy global -> shared
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// explicit shared-space accesses on 32-bit shared addresses (the compiler
// otherwise falls back to generic LD/ST when smem pointers travel in structs)
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// predicated shared load: ~0u when !pred (no access)
__device__ __forceinline__ uint32_t lds32_if(uint32_t a, bool pred) {
  uint32_t v = ~0u;
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.u32 %0, [%1];\n}"
               : "+r"(v)
               : "r"(a), "r"((uint32_t)pred));
  return v;
}
// predicated on x <= lim / x < lim (the compare inside the asm: no bool materialized)
__device__ __forceinline__ uint32_t lds32_if_le(uint32_t a, uint32_t x, uint32_t lim) {
  uint32_t v = ~0u;
  asm volatile("{\n .reg .pred p;\n setp.le.u32 p, %2, %3;\n @p ld.shared.u32 %0, [%1];\n}"
               : "+r"(v)
               : "r"(a), "r"(x), "r"(lim));
  return v;
}
__device__ __forceinline__ uint32_t lds32_if_lt(uint32_t a, uint32_t x, uint32_t lim) {
  uint32_t v = ~0u;
  asm volatile("{\n .reg .pred p;\n setp.lt.u32 p, %2, %3;\n @p ld.shared.u32 %0, [%1];\n}"
               : "+r"(v)
               : "r"(a), "r"(x), "r"(lim));
  return v;
}
__device__ __forceinline__ void sts16_if_le(uint32_t a, uint32_t v, uint32_t x, uint32_t lim) {
  asm volatile("{\n .reg .pred p;\n setp.le.u32 p, %2, %3;\n @p st.shared.u16 [%0], %1;\n}" ::"r"(a),
               "h"((unsigned short)v), "r"(x), "r"(lim)
               : "memory");
}
__device__ __forceinline__ uint2 lds64v(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
template <class T>
__device__ __forceinline__ T ldsk(uint32_t a);
template <>
__device__ __forceinline__ uint32_t ldsk<uint32_t>(uint32_t a) { return lds32(a); }
template <>
__device__ __forceinline__ unsigned long long ldsk<unsigned long long>(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
// predicated 16-bit shared store (no access when !pred)
__device__ __forceinline__ void sts16_if(uint32_t a, uint32_t v, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.u16 [%0], %1;\n}" ::"r"(a),
               "h"((unsigned short)v), "r"((uint32_t)pred)
               : "memory");
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, unsigned long long v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__device__ __forceinline__ __half2 __ushort_as_half2_pair(uint32_t h) {
  const __half x = __ushort_as_half((unsigned short)h);
  return __halves2half2(x, x);
}
__device__ __forceinline__ __half2 u2h2(uint32_t v) { return *reinterpret_cast<const __half2*>(&v); }
__device__ __forceinline__ void red_add_shared(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
// shared-memory add returning the old value (ATOMS.ADD)
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t saddr, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(saddr), "r"(v) : "memory");
  return r;
}

// least p >= 0 with len <= n_d * 256^p  (Alg. 4 l.4; reading S:284)
__host__ __device__ __forceinline__ int est_top_passes(uint64_t len, uint32_t n_d) {
  int p = 0;
  uint64_t cap = n_d;
  while (len > cap && p < 8) {
    cap = (cap > (~0ull >> 8)) ? ~0ull : (cap << 8);
    ++p;
  }
  return p;
}

// highest digit index <= hi whose byte of `diff` is non-zero, or -1
__device__ __forceinline__ int highest_nonconst(unsigned long long diff, int hi) {
  for (int d = hi; d >= 0; --d)
    if ((diff >> (8 * d)) & 255ull) return d;
  return -1;
}

// exclusive block scan of one value per thread (NT threads); returns the
// exclusive prefix, writes the block total to *total (all threads).
// s_warp needs NT/32 words.
template <int NT = THREADS>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp,
                                                    uint32_t* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = lane < NW ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < NW) s_warp[lane] = t;  // inclusive per warp
  }
  __syncthreads();
  uint32_t wpre = w ? s_warp[w - 1] : 0;
  *total = s_warp[NW - 1];
  __syncthreads();
  return wpre + x - v;
}

// Warp-level multi-split rank (stable): items are (j, lane) in j-major order;
// the rank of an item = number of earlier items of this warp with the same
// digit.  The peers of a lane (lanes holding the same digit in this step) are
// found with 8 ballots, one per digit bit — vote/ALU work only: MATCH.ANY costs
// ~64 SM cycles per instruction on sm_100a, and a shared-memory match spends
// the shared-memory pipe, which is this kernel's bottleneck.  The lowest peer
// advances the warp's running count of the digit with one atomicAdd and
// broadcasts the old value.  whist (256 u32) must be zero on entry.
// io[j]: in = digit (256 marks an invalid item, only when !FULL);
// out = digit | rank << 16.
template <bool FULL>
__device__ __forceinline__ uint32_t warp_peers(uint32_t d) {
  // lanes whose digit equals this lane's: AND over the digit bits of the
  // bit's ballot, complemented where this lane's bit is 0
#ifndef DFR_PEERS_C
  // per bit: lop3 -> predicate, vote, predicated not, and (4 SASS instructions)
  uint32_t peers;
  if (FULL)
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
  else  // digit 256 marks an empty slot: a ninth bit
    asm("{\n .reg .pred p;\n .reg .b32 v, t;\n"
        " and.b32 t, %1, 1; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; mov.b32 %0, v;\n"
        " and.b32 t, %1, 2; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        " and.b32 t, %1, 4; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        " and.b32 t, %1, 8; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        " and.b32 t, %1, 16; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        " and.b32 t, %1, 32; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        " and.b32 t, %1, 64; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        " and.b32 t, %1, 128; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        " and.b32 t, %1, 256; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 v, p, 0xffffffff; @!p not.b32 v, v; and.b32 %0, %0, v;\n"
        "}" : "=r"(peers) : "r"(d));
  return peers;
#endif
  // C form (-DDFR_PEERS_C; 5 instructions per bit): the bit moved to the sign
  // position, its ballot xor the spread of the lane's own bit marks the lanes
  // that differ in that bit
  constexpr int NB = FULL ? 8 : 9;
  const int x = (int)(d << (32 - NB));
  uint32_t diff = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int xb = x << b;
    const uint32_t v = __ballot_sync(0xffffffffu, xb < 0);
    diff |= v ^ (uint32_t)(xb >> 31);
  }
  return ~diff;
}

template <int N, bool FULL, bool LDS = false>
__device__ __forceinline__ void warp_rank(uint32_t (&io)[N], uint32_t* whist) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  // peer masks of G items first (independent ballot chains), then their
  // counter updates in item order
  constexpr int G = DFR_RANK_G;
  static_assert(N % G == 0, "items per group");
#pragma unroll
  for (int j0 = 0; j0 < N; j0 += G) {
    uint32_t peers[G];
#pragma unroll
    for (int g = 0; g < G; ++g) peers[g] = warp_peers<FULL>(io[j0 + g]);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t d = io[j0 + g];
      uint32_t old = 0;
      if (LDS) {
        // every lane reads the counter, the last peer lane writes it back (a
        // warp's shared-memory accesses are performed in instruction order)
        const bool ok = FULL || d < 256;
        old = ok ? whist[d] : 0u;
        if (ok && lane == 31 - __clz(peers[g])) whist[d] = old + __popc(peers[g]);
      } else {
        const uint32_t leader = __ffs(peers[g]) - 1;
        if (lane == leader && (FULL || d < 256)) old = atomicAdd(&whist[d], __popc(peers[g]));
        old = __shfl_sync(0xffffffffu, old, leader);
      }
      io[j0 + g] = d | ((old + __popc(peers[g] & lt)) << 16);
    }
  }
}

// cooperative copy of n elements by nt threads (this one: tid): 16-byte
// vectors when dst and src share their alignment, four accesses in flight
template <class T>
__device__ __forceinline__ void coop_copy(T* dst, const T* src, uint32_t n, uint32_t tid,
                                          uint32_t nt) {
  if ((((uintptr_t)dst ^ (uintptr_t)src) & 15) == 0) {
    constexpr uint32_t E = 16 / sizeof(T);
    uint32_t head = (uint32_t)(((16 - ((uintptr_t)src & 15)) & 15) / sizeof(T));
    if (head > n) head = n;
    const uint32_t nv = (n - head) / E;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    uint32_t v = tid;
    for (; v + 3 * nt < nv; v += 4 * nt) {
      const uint4 x0 = s4[v], x1 = s4[v + nt], x2 = s4[v + 2 * nt], x3 = s4[v + 3 * nt];
      d4[v] = x0;
      d4[v + nt] = x1;
      d4[v + 2 * nt] = x2;
      d4[v + 3 * nt] = x3;
    }
    for (; v < nv; v += nt) d4[v] = s4[v];
    for (uint32_t i = tid; i < head; i += nt) dst[i] = src[i];
    for (uint32_t i = head + nv * E + tid; i < n; i += nt) dst[i] = src[i];
  } else {
    uint32_t i = tid;
    for (; i + 3 * nt < n; i += 4 * nt) {
      const T x0 = src[i], x1 = src[i + nt], x2 = src[i + 2 * nt], x3 = src[i + 3 * nt];
      dst[i] = x0;
      dst[i + nt] = x1;
      dst[i + 2 * nt] = x2;
      dst[i + 3 * nt] = x3;
    }
    for (; i < n; i += nt) dst[i] = src[i];
  }
}

// programmatic dependent launch: wait for the previous grid in the stream
// (all its memory operations visible), then let the next grid be scheduled
// (its CTAs block in their own wait) -- hides kernel-boundary latency
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// binary search: largest i in [0, n) with key(i) <= t (key non-decreasing, key(0) = 0)
template <class F>
__device__ __forceinline__ uint32_t upper_index(uint32_t n, uint32_t t, F key) {
  uint32_t lo = 0, hi = n;  // answer in [lo, hi)
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (key(mid) <= t)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// ---- bucket-start bitmask search (diversion) -------------------------------
// last set bit at position <= i and >= lim, or -1
__device__ __forceinline__ int prev_set(const uint32_t* bm, int i, int lim) {
  int w = i >> 5;
  uint32_t m = bm[w] & (0xffffffffu >> (31 - (i & 31)));
  while (true) {
    if (m) {
      int s = w * 32 + 31 - __clz(m);
      return s >= lim ? s : -1;
    }
    if (--w < 0 || w * 32 + 31 < lim) return -1;
    m = bm[w];
  }
}
// first set bit at position > i and <= lim (lim < nbits), or -1
__device__ __forceinline__ int next_set(const uint32_t* bm, int i, int lim) {
  int p = i + 1;
  if (p > lim) return -1;
  int w = p >> 5;
  uint32_t m = bm[w] & (0xffffffffu << (p & 31));
  while (true) {
    if (m) {
      int e = w * 32 + __ffs(m) - 1;
      return e <= lim ? e : -1;
    }
    ++w;
    if (w * 32 > lim) return -1;
    m = bm[w];
  }
}

template <class K>
struct Comp {  // composite (remaining bits, index-in-bucket) for the small sort
  using T = unsigned long long;
};
template <>
struct Comp<uint32_t> {
  using T = uint32_t;
};

}  // namespace dfr
