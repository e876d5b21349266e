// dfr_phases.cuh — the steps of one DFR level as device functions.
//
// A level processes every queued segment (bucket) of the recursion at once:
//   plan    Alg. 4 l.4: p = est(len) capped at the remaining digits
//           (reading S:284), tile/chunk/histogram-row layout
//   hist    Alg. 1 l.2-3 / P:118-120: one read of the segment counts all p
//           group digits at once (one histogram row per pass) + the
//           per-segment diff mask OR(k ^ k0) used to skip constant digits
//   plan2   P:120 "convert counts into indices": exclusive scan per digit;
//           single-bin digits are identity passes and are skipped
//   scatter Alg. 4 l.6: one stable deal per group digit, LSD order,
//           A<->B; per-tile offsets by single-pass decoupled look-back
//   divert  Alg. 4 l.7-14: scan for bucket boundaries of the
//           top-p prefix; buckets <= N_d are sorted on-chip (stable, the
//           insertion-sort result) into the caller's buffer; larger
//           buckets recurse (l.11): <= C on-chip (mid queue), > C through the
//           global segment queue (next level)
//   mid     Alg. 4 applied recursively inside shared memory for N_d < s <= C
//
// Every phase is written for a grid of THREADS-thread CTAs and is called both
// from stand-alone kernels (level 0) and from the cooperative level kernel.
#pragma once
#include "dfr_device.cuh"

namespace dfr {

#ifdef DFR_FPROF
// fused-pass phase profile (timing experiments only): SM cycles per phase
// summed over CTAs (thread 0's view), [8] tiles, [9] tiles with ties
__device__ unsigned long long g_fprof[16];
#define FPROF_MARK(k)                          \
  do {                                         \
    if (threadIdx.x == 0) {                    \
      const long long now_ = clock64();        \
      fp_[k] += (unsigned long long)(now_ - fp_last_); \
      fp_last_ = now_;                         \
    }                                          \
  } while (0)
#else
#define FPROF_MARK(k) \
  do {                \
  } while (0)
#endif
#ifdef DFR_LB_STATS
// look-back statistics of the fused pass (timing experiments only):
// [0] extra rounds (not resolved in the first), [1] rounds that slept, [2] tiles
__device__ unsigned long long g_lb_stats[4];
#endif

// A device queue/stack capacity was exceeded.  The capacities are sized so
// that this cannot happen; the flag is reported in dfr_stats and
// a DFR_DEBUG build traps at once.
__device__ __forceinline__ void flag_overflow(Ctl* c, uint32_t bit) {
  atomicOr(&c->overflow, bit);
#ifdef DFR_DEBUG
  printf("dfr: device queue overflow (flag %u)\n", bit);
  __trap();
#endif
}

template <class K, bool PAIRS>
struct Phases {
  using V = uint32_t;
  using CT = typename Comp<K>::T;
  static constexpr int VEC = 16 / sizeof(K);
  static constexpr int CT_BITS = 8 * sizeof(CT);

  // ------------------------------------------------------------ smem sizes
  // warp-private digit counters + the fused level's chain histogram (256 x 16)
  static constexpr size_t SMEM_HIST = HCOPIES * MAX_PASSES * 256 * 4 + 4096 * 4 + 64;
  static constexpr int F_CHAINS = 16;  // fused pass: chains = top 4 bits of the middle digit
  // The deal kernel runs SC_NT threads per CTA over tiles of TILE keys
  // (4 CTAs/SM with the permutation deal: 32 warps hide the look-back and load latencies)
  static constexpr int SC_NT = 256;
  static constexpr int SCATTER_HDR_WORDS = (SC_NT / 32 + 1) * 256 + 256 + 32 + 256;
  static constexpr size_t SMEM_SCATTER =
      SCATTER_HDR_WORDS * 4 + 2 * TILE * sizeof(K) + (PAIRS ? 2 * TILE * 4 : 0);
  // PERM deal: header | permutation | one tile
  // (the tile buffers hold the 16-byte aligned superset of a tile: SUP_K / SUP_V)
  static constexpr int SUP_K = TILE + 2 * (16 / (int)sizeof(K)), SUP_V = TILE + 8;
  static constexpr size_t SMEM_SCATTER_P =
      SCATTER_HDR_WORDS * 4 + TILE * 2 + SUP_K * sizeof(K) + (PAIRS ? SUP_V * 4 : 0);
  // 2 windows (+ values) | fp16 composites | order | bitmask, misc, mbarriers
  static constexpr size_t SMEM_DIVERT = 1 * (WIN * sizeof(K) + (PAIRS ? WIN * 4 : 0)) +
                                        (4 * WIN + 64) * 2 + WIN * 2 + (WIN / 32 + 12) * 4 + 16 + 16;
  template <int CAP>
  static constexpr size_t smem_mid() {
    return 2 * CAP * sizeof(K) + (PAIRS ? 2 * CAP * 4 : 0) + (CAP + 8) * sizeof(CT) +
           3 * WARPS * 256 * 4 + 256 * 4 + (CAP / 32 + 8) * 4 + 512 * 8 + 128;
  }
  static constexpr size_t SMEM_MID = smem_mid<MID_CAP>();
  static constexpr size_t SMEM_MID_S = smem_mid<MID_CAP_S>();
  static constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
  // k_levels: hist, the permutation deal and the diversion (mid buckets run
  // in k_mid / k_mid_s)
  static constexpr size_t SMEM_LEVEL = cmax(cmax(SMEM_HIST, SMEM_SCATTER_P), SMEM_DIVERT);

  // ---------------------------------------------------------------- plan
  // ONE block: take the queued segments of the next level, compute p, low,
  // tiles, chunks and histogram rows (exclusive prefixes), zero the rows.
  static __device__ void plan(const Params<K>& P, uint32_t* sm) {
    Ctl* c = P.ctl;
    uint32_t* s_warp = sm;  // 8
    __shared__ uint32_t s_tot[4];
    const uint32_t cur = 1u - c->cur;
    uint32_t nseg = c->next_count;
    if (nseg > P.max_segs) {
      if (threadIdx.x == 0) flag_overflow(c, 1u);
      nseg = P.max_segs;
    }
    Seg* q = P.segq[cur];
    uint32_t tile_run = 0, chunk_run = 0, row_run = 0, maxp = 0;
    for (uint32_t b = 0; b < nseg; b += THREADS) {
      const uint32_t i = b + threadIdx.x;
      uint32_t tiles = 0, chunks = 0, rows = 0, p = 0;
      Seg s;
      if (i < nseg) {
        s = q[i];
        s.diff = 0;
        s.final_buf = s.buf;
        s.route = 0;
        chunks = (s.len + P.chunk - 1) / P.chunk;
        if (s.hi < 0) {  // digits exhausted: all keys equal (Alg. 2 l.17-18)
          s.p = 0;
          s.low = 0;
          s.flags = s.buf ? SEG_COPY : SEG_DONE;
          if (!s.buf) chunks = 0;
        } else {
          int pp = est_top_passes(s.len, P.n_d);
          if (pp > s.hi + 1 || (P.full_lsd && c->level + 1u == 0u)) pp = s.hi + 1;  // (ablation: all digits)
          p = (uint32_t)pp;
          s.p = p;
          s.low = s.hi - pp + 1;
          s.flags = 0;
          tiles = (s.len + TILE - 1) / TILE;
          rows = p;
        }
        s.ntiles = tiles;
      }
      uint32_t tt, tc, tr;
      uint32_t et = block_excl_scan(tiles, s_warp, &tt);
      uint32_t ec = block_excl_scan(chunks, s_warp, &tc);
      uint32_t er = block_excl_scan(rows, s_warp, &tr);
      if (i < nseg) {
        s.tile0 = tile_run + et;
        s.chunk0 = chunk_run + ec;
        s.hist_off = row_run + er;
        q[i] = s;
        if (p > maxp) maxp = p;
      }
      tile_run += tt;
      chunk_run += tc;
      row_run += tr;
    }
    // max p over the block
    maxp = __reduce_max_sync(0xffffffffu, maxp);
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = maxp;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t m = 0;
      for (int w = 0; w < WARPS; ++w) m = max(m, s_warp[w]);
      s_tot[0] = m;
    }
    __syncthreads();
    if (row_run > P.hist_rows) {
      if (threadIdx.x == 0) flag_overflow(c, 2u);
      row_run = P.hist_rows;
    }
    for (uint32_t r = 0; r < row_run; ++r) P.hist[(size_t)r * 256 + threadIdx.x] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      c->cur = cur;
      c->nseg = nseg;
      c->total_tiles = tile_run;
      c->total_chunks = chunk_run;
      for (int j = 0; j < MAX_PASSES; ++j) c->ticket[j] = 0;
      c->next_count = 0;
      c->max_p = s_tot[0];
      c->level += 1;  // k_init starts it at ~0u, so the top call is level 0
      c->levels_run = c->level;
    }
    __syncthreads();
  }

  // ---------------------------------------------------------------- hist
  static __device__ void hist_flush(const Params<K>& P, Seg* q, uint32_t si, const Seg& s,
                                    uint32_t* sh, unsigned long long diff, uint32_t* jh) {
    __syncthreads();
    if (jh) {  // the fused level's (top digit, chain) histogram; its marginal is the top digit's
      uint32_t m = 0;
      for (uint32_t x = 0; x < (uint32_t)F_CHAINS; ++x) {
        const uint32_t i = threadIdx.x * F_CHAINS + ((x + threadIdx.x) & (F_CHAINS - 1));
        const uint32_t v = jh[i];
        jh[i] = 0;
        m += v;
        if (v) atomicAdd(&P.J[i], v);
      }
      sh[2 * 256 + threadIdx.x] += m;  // warp 0's row of the top group digit (pass 2)
    }
    for (uint32_t j = 0; j < s.p; ++j) {
      uint32_t v = 0;
#pragma unroll
      for (int w = 0; w < HCOPIES; ++w) {
        v += sh[(w * MAX_PASSES + j) * 256 + threadIdx.x];
        sh[(w * MAX_PASSES + j) * 256 + threadIdx.x] = 0;
      }
      if (v) atomicAdd(&P.hist[(size_t)(s.hist_off + j) * 256 + threadIdx.x], v);
    }
    // diff: warp OR then one atomic per warp
    unsigned long long d = diff;
#pragma unroll
    for (int o = 16; o; o >>= 1) d |= __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0 && d) atomicOr(&q[si].diff, d);
    __syncthreads();
  }

  // warp-private sub-histograms (no cross-warp contention).  A warp whose 32
  // keys share the whole group prefix (sorted, skewed, constant inputs) adds
  // 32 once per digit; otherwise each lane adds 1 to its digit's counter.
  // bin of (top group digit, top 4 bits of the middle one): the fused pass's chains
  static __device__ __forceinline__ uint32_t chain_bin(K k, int low) {
    return digit_of(k, low + 2) * F_CHAINS + (digit_of(k, low + 1) >> 4);
  }
  template <int NP, bool JT>
  static __device__ __forceinline__ void count_key(uint32_t shw, uint32_t jsh, K k, bool valid, int low) {
    const uint32_t lane = threadIdx.x & 31;
    const K pre = k >> (8 * low);
    const K pre0 = __shfl_sync(0xffffffffu, pre, 0);
    if (__all_sync(0xffffffffu, valid && pre == pre0)) {
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < (JT ? NP - 1 : NP); ++j) red_add_shared(shw + 4 * (j * 256 + digit_of(k, low + j)), 32u);
        if (JT) red_add_shared(jsh + 4 * chain_bin(k, low), 32u);
      }
    } else if (valid) {
#pragma unroll
      for (int j = 0; j < (JT ? NP - 1 : NP); ++j) red_add_shared(shw + 4 * (j * 256 + digit_of(k, low + j)), 1u);
      if (JT) red_add_shared(jsh + 4 * chain_bin(k, low), 1u);
    }
  }

  // one tile: diff mask + counts of the NP group digits
  template <int NP, bool JT = false>
  static __device__ __forceinline__ void hist_tile(const K* tp, uint32_t cnt, K kref, int low,
                                                   uint32_t shw, unsigned long long& diff,
                                                   uint32_t jsh = 0) {
    // a tile at any offset (recursion levels): warp 0 counts the < VEC head
    // keys before the 16-byte boundary, the rest takes the vector path
    const uintptr_t mis = reinterpret_cast<uintptr_t>(tp) & 15;
    if (mis && (mis % sizeof(K)) == 0) {
      const uint32_t h = min(cnt, (uint32_t)((16 - mis) / sizeof(K)));
      if (threadIdx.x < 32) {
        const bool ok = threadIdx.x < h;
        const K k = ok ? tp[threadIdx.x] : K(0);
        if (ok) diff |= (unsigned long long)(k ^ kref);
        count_key<NP, JT>(shw, jsh, k, ok, low);
      }
      tp += h;
      cnt -= h;
    }
    if ((reinterpret_cast<uintptr_t>(tp) & 15) == 0) {
      const uint32_t nv = cnt / VEC;
      const uint4* vp = reinterpret_cast<const uint4*>(tp);
      // independent 16-byte loads in flight per thread; a full block is at
      // most one tile (u32 keys: 4)
      constexpr int U_TILE = TILE * (int)sizeof(K) / 16 / THREADS;
      constexpr int U = DFR_HIST_U < U_TILE ? DFR_HIST_U : U_TILE;
      uint32_t vb = 0;
      for (; vb + U * THREADS <= nv; vb += U * THREADS) {  // full blocks: no bounds checks
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldg(vp + vb + u * THREADS + threadIdx.x);
        // one warp vote per block: do all U*VEC*32 keys share lane 0's group
        // prefix?  OR of (k ^ k0) | (k0 ^ kref) over the segment equals the
        // OR of (k ^ kref), so the diff mask comes from the same accumulator
        const K k0 = __shfl_sync(0xffffffffu, reinterpret_cast<const K*>(&x[0])[0], 0);
        K acc = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const K* kk = reinterpret_cast<const K*>(&x[u]);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc |= kk[e] ^ k0;
        }
        diff |= (unsigned long long)(acc | (k0 ^ kref));
        if (__all_sync(0xffffffffu, (acc >> (8 * low)) == K(0))) {
          if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (int j = 0; j < (JT ? NP - 1 : NP); ++j)
              red_add_shared(shw + 4 * (j * 256 + digit_of(k0, low + j)), 32u * U * VEC);
            if (JT) red_add_shared(jsh + 4 * chain_bin(k0, low), 32u * U * VEC);
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const K* kk = reinterpret_cast<const K*>(&x[u]);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
#pragma unroll
              for (int j = 0; j < (JT ? NP - 1 : NP); ++j) red_add_shared(shw + 4 * (j * 256 + digit_of(kk[e], low + j)), 1u);
              if (JT) red_add_shared(jsh + 4 * chain_bin(kk[e], low), 1u);
            }
          }
        }
      }
      for (; vb < nv; vb += THREADS) {
        const uint32_t v = vb + threadIdx.x;
        const bool ok = v < nv;
        uint4 x = ok ? __ldg(vp + v) : make_uint4(0, 0, 0, 0);
        const K* kk = reinterpret_cast<const K*>(&x);
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          if (ok) diff |= (unsigned long long)(kk[e] ^ kref);
          count_key<NP, JT>(shw, jsh, kk[e], ok, low);
        }
      }
      if (nv * VEC < cnt && threadIdx.x < 32) {  // < VEC leftover keys, warp 0
        const uint32_t ii = nv * VEC + threadIdx.x;
        const bool ok = ii < cnt;
        K k = ok ? tp[ii] : K(0);
        if (ok) diff |= (unsigned long long)(k ^ kref);
        count_key<NP, JT>(shw, jsh, k, ok, low);
      }
    } else {
      for (uint32_t ib = 0; ib < cnt; ib += THREADS) {
        const uint32_t i = ib + threadIdx.x;
        const bool ok = i < cnt;
        K k = ok ? tp[i] : K(0);
        if (ok) diff |= (unsigned long long)(k ^ kref);
        count_key<NP, JT>(shw, jsh, k, ok, low);
      }
    }
  }

  // contiguous tile ranges per block; counts the p group digits of every
  // tile of its segment with warp-aggregated shared-memory counting over
  // 128-bit loads, flushes once per segment with global atomics; zeroes the
  // tile's look-back status words for the coming passes.
  static __device__ void hist(const Params<K>& P, uint32_t* sm) {
    Ctl* c = P.ctl;
    const uint32_t total = c->total_tiles, nseg = c->nseg;
    if (total == 0) return;
    Seg* q = P.segq[c->cur];
    if (P.fuse && c->level == 0) {
      // fused level 0: clear the joint histogram and the fused pass's status
      // rows beyond the deal tiles (it may have up to 65536 run-aligned tiles)
      const uint32_t gid = blockIdx.x * THREADS + threadIdx.x, gsz = gridDim.x * THREADS;
      for (uint32_t x = gid; x < 65536u; x += gsz) P.H[x] = 0;
      uint32_t* st2 = P.status + 2 * P.status_stride;
      for (size_t x = (size_t)total * 256 + gid; x < (size_t)65536 * 256; x += gsz) st2[x] = 0;
    }
    const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
    const uint32_t t0 = blockIdx.x * per;
    const uint32_t t1 = min(total, t0 + per);
    if (t0 >= t1) return;
    uint32_t* sh = sm;  // [HCOPIES][MAX_PASSES][256]; warp w counts into copy w % HCOPIES
    const uint32_t shw = smem_u32(sh + ((threadIdx.x >> 5) % HCOPIES) * MAX_PASSES * 256);
    for (int j = 0; j < HCOPIES * MAX_PASSES; ++j) sh[j * 256 + threadIdx.x] = 0;
    // the fused level: also the (top digit, chain) histogram of the group
    uint32_t* jh = (P.fuse && c->level == 0) ? sm + HCOPIES * MAX_PASSES * 256 : nullptr;
    const uint32_t jsh = jh ? smem_u32(jh) : 0u;
    if (jh)
      for (uint32_t x = threadIdx.x; x < 4096u; x += THREADS) jh[x] = 0;
    uint32_t si = upper_index(nseg, t0, [&](uint32_t i) { return q[i].tile0; });
    Seg s = q[si];
    unsigned long long diff = 0;
    __syncthreads();
    for (uint32_t t = t0; t < t1; ++t) {
      while (t >= s.tile0 + s.ntiles) {  // next segment with tiles
        hist_flush(P, q, si, s, sh, diff, s.p == 3 ? jh : nullptr);
        diff = 0;
        ++si;
        s = q[si];
      }
      const uint32_t lt = t - s.tile0;
      const uint32_t base = s.start + lt * TILE;
      // up to HT deal tiles of the segment per step (fewer per-step overheads)
      const uint32_t nt = min(min((uint32_t)DFR_HIST_TILES, t1 - t), s.tile0 + s.ntiles - t);
      const uint32_t cnt = min(nt * TILE, s.len - lt * TILE);
      for (uint32_t j = 0; j < s.p; ++j)
        for (uint32_t u = 0; u < nt; ++u)
          P.status[j * P.status_stride + (size_t)(t + u) * 256 + threadIdx.x] = 0;
      t += nt - 1;
      const K* src = P.kbuf(s.buf);
      const K kref = src[s.start];
      const K* tp = src + base;
      switch (s.p) {
        case 1: hist_tile<1>(tp, cnt, kref, s.low, shw, diff); break;
        case 2: hist_tile<2>(tp, cnt, kref, s.low, shw, diff); break;
        case 3:
          if (jh)
            hist_tile<3, true>(tp, cnt, kref, s.low, shw, diff, jsh);
          else
            hist_tile<3>(tp, cnt, kref, s.low, shw, diff);
          break;
        default: hist_tile<4>(tp, cnt, kref, s.low, shw, diff); break;
      }
    }
    hist_flush(P, q, si, s, sh, diff, s.p == 3 ? jh : nullptr);
  }

  // --------------------------------------------------------------- plan2
  // One block per segment: counts -> exclusive bucket offsets (in place),
  // pass skipping, final buffer; a segment whose group digits are all
  // constant is re-queued at once with its highest non-constant digit.
  static __device__ void plan2(const Params<K>& P, uint32_t* sm) {
    Ctl* c = P.ctl;
    const uint32_t nseg = c->nseg;
    Seg* q = P.segq[c->cur];
    Seg* nq = P.segq[1u - c->cur];
    uint32_t* s_warp = sm;
    for (uint32_t si = blockIdx.x; si < nseg; si += gridDim.x) {
      const Seg s = q[si];
      if (s.flags & (SEG_COPY | SEG_DONE)) continue;
      uint32_t skip = 0;
      for (uint32_t j = 0; j < s.p; ++j) {
        uint32_t* row = P.hist + (size_t)(s.hist_off + j) * 256;
        const uint32_t cnt = row[threadIdx.x];
        const int single = __syncthreads_or(cnt == s.len);
        if (single && P.skip_trivial) skip |= 1u << j;
        uint32_t tot;
        const uint32_t ex = block_excl_scan(cnt, s_warp, &tot);
        row[threadIdx.x] = ex;
      }
      const uint32_t executed = s.p - __popc(skip);
      uint32_t flags = skip;
      if (executed == 0) {
        const int hn = highest_nonconst(s.diff, s.low - 1);
        if (hn < 0) {
          flags |= s.buf ? SEG_COPY : SEG_DONE;
        } else {
          flags |= SEG_SKIP_DIVERT;
          if (threadIdx.x == 0) {
            const uint32_t idx = atomicAdd(&c->next_count, 1u);
            if (idx < P.max_segs) {
              Seg ns = {};
              ns.start = s.start;
              ns.len = s.len;
              ns.hi = hn;
              ns.buf = s.buf;
              nq[idx] = ns;
            } else {
              flag_overflow(c, 4u);
            }
          }
        }
      }
      // recursion levels: when the passes end on digit 0 every bucket of the
      // scan (Alg. 4 l.8) is a constant key -- insertion sort and recursion
      // leave it as it is -- so the diversion only moves the segment to A
      if (executed > 0 && s.low == 0 && (c->level > 0 || P.full_lsd)) flags |= SEG_SORTED;
      // buffer route of the executed passes: ping-pong between the data's
      // buffer and another one; a level 0 with the second scratch buffer runs
      // A -> C -> B -> C, so that its third pass (the fused pass, B -> A)
      // lands in the caller's buffer without a copy
      const bool three = P.C != nullptr && c->level == 0;
      uint32_t route = 0, cur = s.buf;
      for (uint32_t j = 0; j < s.p; ++j) {
        if ((skip >> j) & 1u) continue;
        const uint32_t nb = three ? (cur == 2u ? 1u : 2u) : (cur == 0u ? 1u : 0u);
        route |= (cur | nb << 2) << (4 * j);
        cur = nb;
      }
      if (threadIdx.x == 0) {
        q[si].flags = flags;
        q[si].route = route;
        q[si].final_buf = cur;
        if (c->level == 0) {
          c->level0_p = s.p;
          c->level0_run = executed;
        }
      }
      __syncthreads();
    }
  }

  // ------------------------------------------------------------- scatter
  // One stable deal on group digit low+j for every active segment.  A
  // persistent CTA claims a tile of TILE keys by dynamic ticket (forward
  // progress for the look-back), pulls it into shared memory with one TMA bulk
  // copy, ranks it with the warp-level multi-split, publishes its per-digit
  // aggregate, resolves its exclusive per-digit prefix by decoupled look-back
  // over the segment's earlier tiles, reorders the tile by digit in shared
  // memory and writes every digit run contiguously.
  static __device__ __forceinline__ bool pass_active(const Seg& s, int j) {
    return (uint32_t)j < s.p && !((s.flags >> j) & 1u) &&
           !(s.flags & (SEG_SKIP_DIVERT | SEG_COPY | SEG_DONE));
  }
  static __device__ __forceinline__ uint32_t route_src(const Seg& s, int j) {
    return (s.route >> (4 * j)) & 3u;
  }
  static __device__ __forceinline__ uint32_t route_dst(const Seg& s, int j) {
    return (s.route >> (4 * j + 2)) & 3u;
  }


  // rank, publish, reorder, look back, write out — one staged tile
  // PERM: the keys are not held in registers through the rank; the tile is
  // reordered as a permutation of positions (u16, `perm`) and the write-out
  // gathers keys through it — 32 fewer registers per thread (u64), which lets
  // 4 CTAs share an SM.
  // Fast Radix: the overflow chunk of bucket d holding its overflow ranks
  // [k * FR_CHUNK, (k+1) * FR_CHUNK): handed out on first touch (a lock word
  // while the id is drawn)
  static constexpr uint32_t FR_CHUNK = 4096, FR_LOCK = ~0u;
  static __device__ __forceinline__ uint32_t fr_chunk(const Params<K>& P, uint32_t d, uint32_t k) {
    uint32_t* e = P.fr_ct + (size_t)d * P.fr_kmax + k;
    uint32_t v = *(volatile uint32_t*)e;
    if (v == 0u) {
      v = atomicCAS(e, 0u, FR_LOCK);
      if (v == 0u) {
        v = atomicAdd(&P.ctl->fr_next_chunk, 1u) + 1u;
        atomicExch(e, v);
        return v - 1u;
      }
    }
    while (v == FR_LOCK) v = *(volatile uint32_t*)e;
    return v - 1u;
  }

  // FRM (Fast Radix mode): 0 counted deal; 1 deal into estimated buckets (with
  // overflow chunks), counting the next digit; 2 deal reading the estimated
  // layout through the tile table, counting the next (top) digit
  template <int SC_NT, bool FULL, bool FUSEH, bool PERM, int FRM = 0, class Hook>
  static __device__ __forceinline__ void deal_tile(const Hook& after_lookback, const Params<K>& P,
                                                   const Seg& s, int j,
                                                   uint32_t t, uint32_t lt, uint32_t cnt, int dg,
                                                   uint32_t* status, K* sk, V* sv, uint32_t* whist,
                                                   int* s_dst, uint32_t* s_warp, K* dst, V* dstv,
                                                   uint32_t bstart, uint16_t* perm, uint32_t sup,
                                                   uint32_t nh_s, bool uns) {
    constexpr int SC_W = SC_NT / 32;
    constexpr int SC_KPT = TILE / SC_NT;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* mywh = whist + w * 256;
    uint32_t* tcount = whist + SC_W * 256;  // 256 tile counts (zeroed with whist)
    // warp-striped items: (jj, lane) -> w*32*SC_KPT + jj*32 + lane
    K key[SC_KPT];
    V val[SC_KPT];
    uint32_t dr[SC_KPT];
    const uint32_t tc_s = smem_u32(tcount);
    uns = (!PAIRS && uns) || FRM == 2;  // FRM 2: every tile lies in one bucket of the lower digit
    if (uns) {  // (R5) rank = the tile counter's old value: keys of equal digit in any order
#pragma unroll
      for (int jj = 0; jj < SC_KPT; ++jj) {
        const uint32_t idx = w * 32 * SC_KPT + jj * 32 + lane;
        key[jj] = sk[(PERM ? (sup & 0xffu) : 0u) + idx];
        dr[jj] = (FULL || idx < cnt) ? digit_of(key[jj], dg) : 256u;
#if DFR_RUN_ATOMS
        // runs of equal digits in consecutive lanes (locally sorted input)
        // reserve their ranks with one atomic per run instead of serializing
        // on the counter
        const uint32_t dprev = __shfl_up_sync(0xffffffffu, dr[jj], 1);
        const uint32_t bsame = __ballot_sync(0xffffffffu, lane > 0 && dr[jj] == dprev);
        if (bsame) {
          const uint32_t starts = ~bsame, le = 0xffffffffu >> (31 - lane);
          const uint32_t st0 = 31 - __clz(starts & le), nxt = starts & ~le;
          const uint32_t rlen = (nxt ? (uint32_t)__ffs(nxt) - 1u : 32u) - st0;
          uint32_t old = 0;
          if (lane == st0 && (FULL || idx < cnt)) old = atom_add_shared(tc_s + 4 * dr[jj], rlen);
          old = __shfl_sync(0xffffffffu, old, st0);
          if (FULL || idx < cnt) dr[jj] |= (old + lane - st0) << 16;
          if (FRM == 1 && (FULL || idx < cnt)) red_add_shared(nh_s + 4 * digit_of(key[jj], dg + 1), 1u);
          if (FRM == 2 && (FULL || idx < cnt))
            red_add_shared(fr_joint_addr(smem_u32(whist), nh_s,
                                         digit_of(key[jj], dg + 1) * FR_CHAINS + (dr[jj] & 0xffu) / (256 / FR_CHAINS)),
                           1u);
          continue;
        }
#endif
        if (FULL || idx < cnt) {
          dr[jj] |= atom_add_shared(tc_s + 4 * dr[jj], 1u) << 16;
          if (FRM == 1) red_add_shared(nh_s + 4 * digit_of(key[jj], dg + 1), 1u);
          if (FRM == 2)  // (top digit, top 3 bits of this one), see fr_joint_addr
            red_add_shared(fr_joint_addr(smem_u32(whist), nh_s,
                                         digit_of(key[jj], dg + 1) * FR_CHAINS + (dr[jj] & 0xffu) / (256 / FR_CHAINS)),
                           1u);
        }
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < SC_KPT; ++jj) {
        const uint32_t idx = w * 32 * SC_KPT + jj * 32 + lane;
        key[jj] = sk[(PERM ? (sup & 0xffu) : 0u) + idx];  // PERM: the tile starts koff into sk
        if (PAIRS && !PERM) val[jj] = sv[idx];
        dr[jj] = (FULL || idx < cnt) ? digit_of(key[jj], dg) : 256u;
        if (FULL || idx < cnt) {
          red_add_shared(tc_s + 4 * dr[jj], 1u);  // tile histogram
          if (FRM == 1) red_add_shared(nh_s + 4 * digit_of(key[jj], dg + 1), 1u);  // the next digit (Alg. 3 l.5-6)
        }
      }
    }
    __syncthreads();
    if (FUSEH) {  // joint histogram [this digit][digit below] for the fused last pass
      const K* tk = sk + (PERM ? (sup & 0xffu) : 0u);
      const uint32_t lo0 = digit_of(tk[0], s.low), lo1 = digit_of(tk[cnt - 1], s.low);
      if (lo0 == lo1) {  // input sorted by the digit below: the whole tile shares it
        // (counted path: fplan takes these counts from the look-back's
        // inclusive prefixes instead; Fast Radix tiles follow a table)
        if (FRM == 2 && threadIdx.x < 256 && tcount[threadIdx.x])
          atomicAdd(&P.H[threadIdx.x * 256 + lo0], tcount[threadIdx.x]);
      } else {  // a tile across a boundary of the digit below (one per run of it)
        for (uint32_t i = threadIdx.x; i < cnt; i += SC_NT) {
          const K k = tk[i];
          atomicAdd(&P.H[digit_of(k, dg) * 256 + digit_of(k, s.low)], 1u);
        }
      }
    }
    // publish the tile aggregate as early as possible: successors' look-backs
    // then rarely wait for this tile
    const uint32_t dd = threadIdx.x;
    const bool dig_thread = dd < 256;
    uint32_t run = 0;
    constexpr int LB = DFR_LB;  // predecessors per look-back round trip
    uint32_t lbv[LB];
    if (dig_thread) {
      run = tcount[dd];
      st_relaxed(status + (size_t)t * 256 + dd, (lt == 0 ? FLAG_INC : FLAG_AGG) | run);
#if DFR_LB_EARLY
      // the look-back's first round trip, in flight during the reorder
      if (lt > 0) ld_lookback<LB>(status + (size_t)(t - 1) * 256 + dd, lbv);
#endif
    }
    if (w == 0) {  // tile offsets of the 256 digits (8 per lane) into s_dst, free until the look-back
      const uint4 c0 = *reinterpret_cast<const uint4*>(tcount + 8 * lane);
      const uint4 c1 = *reinterpret_cast<const uint4*>(tcount + 8 * lane + 4);
      const uint32_t c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      uint32_t sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) sum += c[k];
      uint32_t x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      uint32_t e0 = x - sum;
      uint32_t ex[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ex[k] = e0;
        e0 += c[k];
      }
      *reinterpret_cast<uint4*>(s_dst + 8 * lane) = make_uint4(ex[0], ex[1], ex[2], ex[3]);
      *reinterpret_cast<uint4*>(s_dst + 8 * lane + 4) = make_uint4(ex[4], ex[5], ex[6], ex[7]);
      if (uns) {  // the reorder's bases (s_dst is rewritten by the look-back meanwhile)
        *reinterpret_cast<uint4*>(whist + 8 * lane) = make_uint4(ex[0], ex[1], ex[2], ex[3]);
        *reinterpret_cast<uint4*>(whist + 8 * lane + 4) = make_uint4(ex[4], ex[5], ex[6], ex[7]);
      }
    }
    if (!uns) warp_rank<SC_KPT, FULL, PERM>(dr, mywh);
    __syncthreads();  // ranks and tile offsets done
    // per digit: warp bases in the tile = tile offset of the digit + counts of
    // the digit in earlier warps
    uint32_t lstart = 0;
    if (dig_thread) lstart = (uint32_t)s_dst[dd];
    if (!uns) {
      if (dig_thread) {
        uint32_t acc = lstart;
#pragma unroll
        for (int e = 0; e < SC_W; ++e) {
          const uint32_t x = whist[e * 256 + dd];
          whist[e * 256 + dd] = acc;
          acc += x;
        }
      }
      __syncthreads();
    }
    // reorder the tile by digit in shared memory (stable unless uns)
    const uint32_t* const rb = uns ? whist : mywh;
#pragma unroll
    for (int jj = 0; jj < SC_KPT; ++jj) {
      const uint32_t dgt = dr[jj] & 0xffffu;
      if (FULL || dgt < 256) {
        const uint32_t pos = rb[dgt] + (dr[jj] >> 16);
        if (PERM) {
          perm[pos] = (uint16_t)((sup & 0xffu) + w * 32 * SC_KPT + jj * 32 + lane);
        } else {
          sk[pos] = key[jj];
          if (PAIRS) sv[pos] = val[jj];
        }
      }
    }
    if (dig_thread) {
      uint32_t excl = 0;
#ifdef DFR_D_NOLB  // timing experiment only: wrong output
      if (false) {
#else
      if (lt > 0) {  // decoupled look-back, up to LB predecessors per round trip
#endif
        int tt = (int)t - 1;
        bool first = true;
        while (true) {
          // LB predecessors tt, tt-1, ... in one round trip; rows before the
          // segment's first tile t0 may be read (status has LB pad rows in
          // front) but are never used: t0 publishes FLAG_INC, and the walk
          // stops at the first FLAG_INC or unpublished entry
          uint32_t v[LB];
          if (DFR_LB_EARLY && first) {
#pragma unroll
            for (int i = 0; i < LB; ++i) v[i] = lbv[i];
          } else {
            ld_lookback<LB>(status + (size_t)tt * 256 + dd, v);
          }
          first = false;
          int k = 0;
          bool done = false;
#pragma unroll
          for (; k < LB; ++k) {
            if ((v[k] >> 30) == 0) break;  // not published yet: retry from here
            excl += v[k] & VAL_MASK;
            if (v[k] & FLAG_INC) {
              done = true;
              break;
            }
          }
          if (done) break;
          if (k == 0) __nanosleep(DFR_LB_SLEEP);  // predecessor not published: yield the issue slots
          tt -= k;
        }
        st_relaxed(status + (size_t)t * 256 + dd, FLAG_INC | ((excl + run) & VAL_MASK));
      }
      // counts are mod 2^30 (n <= 2^30): a non-empty run's prefix is < 2^30
      excl &= VAL_MASK;
      // run offset of the digit relative to the tile's local offsets, mod 2^32
      // (Fast Radix estimated pass: the rank inside the digit's bucket)
      s_dst[dd] = FRM == 1 ? (int)(excl - lstart) : (int)(s.start + bstart + excl - lstart);
    }
#if DFR_CLAIM_AFTER_BARRIER
    __syncthreads();
    after_lookback();  // thread 0: claim the next tile (its atomic overlaps the write-out)
#else
    after_lookback();  // thread 0: claim the next tile, start its TMA load
    __syncthreads();
#endif
    // coalesced write of each digit run
#pragma unroll WO_UNROLL
    for (uint32_t i = threadIdx.x; i < (FULL ? (uint32_t)TILE : cnt); i += SC_NT) {
      const uint32_t src = PERM ? (uint32_t)perm[i] : i;
      const K k = sk[src];
      const uint32_t dk = digit_of(k, dg);
      uint32_t o = (uint32_t)s_dst[dk] + i;  // < 2^30: unsigned math
      if (FRM == 1) {  // estimated bucket dk: main region, or the overflow chunk of rank o
        if (o < P.fr_cap) {
          o += dk * P.fr_cap;
        } else {
          const uint32_t ov = o - P.fr_cap;
          o = 256u * P.fr_cap + fr_chunk(P, dk, ov / FR_CHUNK) * FR_CHUNK + ov % FR_CHUNK;
        }
      }
#ifdef DFR_DEBUG
      if (FRM != 1 && (o < s.start || o >= s.start + s.len)) {
        printf("scatter OOB: t=%u i=%u o=%u seg=[%u,%u)\n", t, i, o, s.start, s.start + s.len);
        __trap();
      }
#endif
      dst[o] = k;
      if (PAIRS) dstv[o] = sv[PERM ? src - (sup & 0xffu) + (sup >> 8) : src];
    }
  }

  // One stable deal on group digit low+j for every active segment.  A
  // persistent CTA claims a tile of TILE keys by dynamic ticket (forward
  // progress for the look-back), pulls it into shared memory with one TMA bulk
  // copy, ranks it with the warp-level multi-split, publishes its per-digit
  // aggregate, reorders the tile by digit in shared memory, resolves its
  // exclusive per-digit prefix by decoupled look-back over the segment's
  // earlier tiles and writes every digit run contiguously.
  // thread 0: claim a ticket into ti[0..2] (ticket, segment, tma) and, for a
  // full aligned tile of an active segment, start its TMA bulk load
  // (DEFER: ticket, segment and eligibility only; issue_tile starts the copy
  // later — ti is then final before the caller's next barrier)
  // SUP: the copy covers the 16-byte aligned superset of the tile (the tile
  // starts koff keys / voff values into the buffer, ti[3] = koff | voff << 8),
  // so that tiles of segments at any offset (recursion levels) still use TMA
  // element offset and length of tile t (local index lt) of segment s in
  // pass j: consecutive TILE-key pieces of the segment, or (FRM == 2) the
  // Fast Radix tile table over the estimated layout
  template <int FRM = 0>
  static __device__ __forceinline__ void tile_loc(const Params<K>& P, const Seg& s, uint32_t t,
                                                  uint32_t lt, uint32_t& off, uint32_t& cnt) {
    if (FRM == 2) {
      const uint2 e = P.fr_tab[t];
      off = e.x;
      cnt = e.y;
    } else {
      off = s.start + lt * TILE;
      cnt = min((uint32_t)TILE, s.len - lt * TILE);
    }
  }

  template <bool DEFER = false, bool SUP = false, int FRM = 0>
  static __device__ __forceinline__ void claim_tile(const Params<K>& P, int j, const Seg* q,
                                                    uint32_t nseg, uint32_t total, uint32_t* ti,
                                                    K* kb, V* vb, unsigned long long* bar) {
    const uint32_t t = atomicAdd(&P.ctl->ticket[j], 1u);
    ti[0] = t;
    ti[2] = 0;
    if (t >= total) return;
    const uint32_t si = FRM == 2 ? 0u : upper_index(nseg, t, [&](uint32_t i) { return q[i].tile0; });
    ti[1] = si;
    const Seg& s = q[si];
    const uint32_t lt = t - s.tile0;
    uint32_t off, tcnt;
    tile_loc<FRM>(P, s, t, lt, off, tcnt);
    if (!pass_active(s, j) || tcnt < (uint32_t)TILE) return;
    const uint32_t sb = route_src(s, j);
    const K* src = P.kbuf(sb) + off;
    const V* srcv = PAIRS ? P.vbuf(sb) + off : nullptr;
    const bool aligned = !(reinterpret_cast<uintptr_t>(src) & 15) &&
                         !(PAIRS && (reinterpret_cast<uintptr_t>(srcv) & 15));
    if (SUP) ti[3] = 0;
    if (aligned) {
    } else if (SUP) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(src), a0 = a & ~(uintptr_t)15;
      const uintptr_t k0 = reinterpret_cast<uintptr_t>(P.kbuf(sb));
      if (a0 < k0 || a0 + sup_bytes(a - a0, TILE * sizeof(K)) > k0 + (uintptr_t)P.n * sizeof(K)) return;
      uint32_t off = (uint32_t)((a - a0) / sizeof(K));
      if (PAIRS) {
        const uintptr_t b = reinterpret_cast<uintptr_t>(srcv), b0 = b & ~(uintptr_t)15;
        const uintptr_t v0 = reinterpret_cast<uintptr_t>(P.vbuf(sb));
        if (b0 < v0 || b0 + sup_bytes(b - b0, TILE * 4) > v0 + (uintptr_t)P.n * 4) return;
        off |= (uint32_t)((b - b0) / 4) << 8;
      }
      ti[3] = off;
    } else {
      return;
    }
    ti[2] = 1;
#if DFR_DEAL_PF
    // the copy starts only after the current tile's write-out: pull the
    // tile into L2 meanwhile
    if (DEFER) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(TILE * sizeof(K)))
                   : "memory");
      if (PAIRS) {
        const uintptr_t b = reinterpret_cast<uintptr_t>(srcv) & ~(uintptr_t)15;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"((uint32_t)(TILE * 4)) : "memory");
      }
    }
#endif
    if (!DEFER) issue_tile<SUP, FRM>(P, j, q, ti, kb, vb, bar);
  }
  static __device__ __forceinline__ uint32_t sup_bytes(uintptr_t head, uint32_t bytes) {
    return (uint32_t)((head + bytes + 15) & ~(uintptr_t)15);
  }
  // thread 0: start the TMA bulk copy of the claimed tile in ti (ti[2] = 1)
  template <bool SUP = false, int FRM = 0>
  static __device__ __forceinline__ void issue_tile(const Params<K>& P, int j, const Seg* q,
                                                    const uint32_t* ti, K* kb, V* vb,
                                                    unsigned long long* bar) {
    if (!ti[2]) return;
    const Seg& s = q[ti[1]];
    const uint32_t lt = ti[0] - s.tile0;
    const uint32_t sb = route_src(s, j);
    uint32_t off, tcnt;
    tile_loc<FRM>(P, s, ti[0], lt, off, tcnt);
    const K* src = P.kbuf(sb) + off;
    const V* srcv = PAIRS ? P.vbuf(sb) + off : nullptr;
    uint32_t kbytes = TILE * sizeof(K), vbytes = TILE * 4;
    if (SUP && ti[3]) {
      const uint32_t koff = ti[3] & 0xffu, voff = ti[3] >> 8;
      kbytes = sup_bytes(koff * sizeof(K), TILE * sizeof(K));
      src -= koff;
      if (PAIRS) {
        vbytes = sup_bytes(voff * 4, TILE * 4);
        srcv -= voff;
      }
    }
    fence_proxy_async();
    const uint32_t bytes = kbytes + (PAIRS ? vbytes : 0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        DFR_TMA_LOAD ::"r"(
            smem_u32(kb)),
        "l"(src), "r"(kbytes), "r"(smem_u32(bar))
        : "memory");
    if (PAIRS)
      asm volatile(
          DFR_TMA_LOAD ::"r"(
              smem_u32(vb)),
          "l"(srcv), "r"(vbytes), "r"(smem_u32(bar))
          : "memory");
  }

  // Persistent CTA with two tile buffers (!PERM) or one tile buffer and a
  // position permutation (PERM, the default deal).  The next tile's ticket is claimed,
  // and its TMA load started, as soon as the current tile has published its
  // inclusive prefix: the load and the ticket round trip overlap the current
  // tile's write-out, and tickets are still claimed in (nearly) completion
  // order, which keeps the look-back of later tiles short.
  // FUSEH: the middle pass of a fused level 0 also counts the joint histogram
  // PERM (deal_tile): one tile buffer, refilled once the write-out is done
  template <int SC_NT, bool FUSEH = false, bool PERM = false, int FRM = 0>
  static __device__ void scatter(const Params<K>& P, int j, uint32_t* sm) {
    constexpr int SC_W = SC_NT / 32;
    Ctl* c = P.ctl;
    const uint32_t total = FRM == 2 ? c->fr_tiles : c->total_tiles, nseg = c->nseg;
    if ((uint32_t)j >= c->max_p) return;  // no segment of this level has pass j
    if (P.fuse && j == 2 && c->level == 0 && *(volatile uint32_t*)&c->fused_ok) return;  // fused pass did it
    const Seg* q = P.segq[c->cur];
    uint32_t* whist = sm;                                         // SC_W*256
    int* s_dst = reinterpret_cast<int*>(whist + (SC_W + 1) * 256);  // 256 (after tcount)
    uint32_t* s_warp = reinterpret_cast<uint32_t*>(s_dst + 256);  // 16
    uint32_t* ti = s_warp + 16;                                   // 2 x 4 words
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(ti + 8);  // 2, 8-aligned
    uint32_t* nh = sm + SCATTER_HDR_WORDS - 256;  // Fast Radix: next-digit counters of this CTA
    if (FRM) {
      nh[threadIdx.x] = 0;
      __syncthreads();
    }
    uint16_t* const perm = reinterpret_cast<uint16_t*>(sm + SCATTER_HDR_WORDS);  // PERM: TILE
    K* const kb0 = PERM ? reinterpret_cast<K*>(perm + TILE)
                        : reinterpret_cast<K*>(sm + SCATTER_HDR_WORDS);  // (1 or 2) x TILE keys
    V* const vb0 = reinterpret_cast<V*>(kb0 + (PERM ? SUP_K : 2 * TILE));  // (1 or 2) x TILE values
    uint32_t* status = P.status + (size_t)j * P.status_stride;
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
      claim_tile<false, PERM, FRM>(P, j, q, nseg, total, ti, kb0, vb0, &bar[0]);
    }
    uint32_t phases = 0;  // mbarrier parity per buffer
    // the segment record and its bucket-offset row are re-read only when a
    // tile of another segment comes up (level 0: once per CTA)
    uint32_t cur_si = ~0u, bstart = 0;
    bool skewed = false;  // the segment's digit of this pass is skewed: stable ranks
    Seg s;

    if (PERM) {
      for (int e = threadIdx.x; e < (SC_W + 1) * 256; e += SC_NT) whist[e] = 0;
    }
    for (int it = 0;; ++it) {
      const int cb = PERM ? 0 : (it & 1);
      if (!PERM) {
        for (int e = threadIdx.x; e < (SC_W + 1) * 256; e += SC_NT) whist[e] = 0;
      }
      // PERM: the previous tile's closing barrier already made ti visible and
      // the zeroed counters; the first tile needs this one
      if (!PERM || it == 0) __syncthreads();  // ti[cb] visible; whist zeroed; other buffer free
      const uint32_t t = ti[cb * 4 + 0];
      if (t >= total) break;
      const uint32_t si = ti[cb * 4 + 1];
      if (si != cur_si) {
        cur_si = si;
        s = q[si];
        uint32_t cntd = 0;
        if (threadIdx.x < 256 && pass_active(s, j) && FRM != 1) {
          bstart = P.hist[(size_t)(s.hist_off + j) * 256 + threadIdx.x];
          const uint32_t nx = threadIdx.x == 255 ? s.len : P.hist[(size_t)(s.hist_off + j) * 256 + threadIdx.x + 1];
          cntd = nx - bstart;
        }
        // a skewed digit (> 1/16 of the segment) puts many lanes of a warp on
        // one tile counter: the atomic ranks (R5) would serialize on it, the
        // ballot multi-split does not
        skewed = __syncthreads_or(cntd > s.len / 16) != 0;
      }
      const bool tma = ti[cb * 4 + 2] != 0;
      const uint32_t sup = (PERM && tma) ? ti[3] : 0u;  // the tile's offsets in the aligned copy
      K* sk = kb0 + cb * TILE;
      V* sv = vb0 + cb * TILE;
      auto claim_next = [&]() {
        if (threadIdx.x == 0) {
          const int nb = PERM ? 0 : (cb ^ 1);
          claim_tile<false, PERM, FRM>(P, j, q, nseg, total, ti + nb * 4, kb0 + nb * TILE,
                                       vb0 + nb * TILE, &bar[nb]);
        }
      };
      // claim the next tile once this one's prefix is known (tickets in
      // completion order); PERM: its copy starts after the write-out
      auto hook = [&]() {
        if (!PERM)
          claim_next();
        else if (threadIdx.x == 0)
          claim_tile<true, true, FRM>(P, j, q, nseg, total, ti, kb0, vb0, &bar[0]);
      };
      if (!pass_active(s, j)) {
        claim_next();
        if (PERM) __syncthreads();
        continue;
      }
      const uint32_t lt = t - s.tile0;
      uint32_t base, cnt;
      tile_loc<FRM>(P, s, t, lt, base, cnt);
      const uint32_t sb = route_src(s, j), db = route_dst(s, j);
      const K* src = P.kbuf(sb);
      K* dst = P.kbuf(db);
      const V* srcv = P.vbuf(sb);
      V* dstv = P.vbuf(db);
      const int dg = s.low + j;
      if (tma) {
        mbar_wait(&bar[cb], (phases >> cb) & 1u);
        phases ^= 1u << cb;
      } else {  // ragged tail / unaligned tile: plain coalesced loads
        for (uint32_t i = threadIdx.x; i < cnt; i += SC_NT) sk[i] = src[base + i];
        if (PAIRS)
          for (uint32_t i = threadIdx.x; i < cnt; i += SC_NT) sv[i] = srcv[base + i];
        __syncthreads();
      }
      // (R5) keys only: ranks in any order when the tile is constant in the
      // group digits below dg (the input of pass j is sorted by them)
      bool uns = false;
      if (!PAIRS && P.unstable && !skewed) {
        if (j == 0) {
          uns = true;
        } else {
          const K* tk = sk + (PERM ? (sup & 0xffu) : 0u);
          const K x = (tk[0] ^ tk[cnt - 1]) >> (8 * s.low);
          uns = (x & ((K(1) << (8 * j)) - 1)) == 0;
        }
      }
      if (cnt == (uint32_t)TILE)
        deal_tile<SC_NT, true, FUSEH, PERM, FRM>(hook, P, s, j, t, lt, cnt, dg, status, sk, sv, whist,
                                                 s_dst, s_warp, dst, dstv, bstart, perm, sup,
                                                 smem_u32(nh), uns);
      else
        deal_tile<SC_NT, false, FUSEH, PERM, FRM>(hook, P, s, j, t, lt, cnt, dg, status, sk, sv, whist,
                                                  s_dst, s_warp, dst, dstv, bstart, perm, sup,
                                                  smem_u32(nh), uns);
      if (PERM) {  // single buffer: refill it once every thread is done with the write-out
        if (FRM == 2) {  // rows 1..SC_W-1 hold the joint counters: only row 0 and the tile counts
          whist[threadIdx.x] = 0;
          whist[SC_W * 256 + threadIdx.x] = 0;
        } else {
          for (int e = threadIdx.x; e < (SC_W + 1) * 256; e += SC_NT) whist[e] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          fence_proxy_async();
          issue_tile<PERM, FRM>(P, j, q, ti, kb0, vb0, &bar[0]);
        }
      }
      fence_proxy_async();  // generic smem accesses before a later TMA into this buffer
    }
    // every claimed ticket < total was processed, so no bulk copy is in flight
    // here, and every thread passed its last wait before the loop's final barrier
    if (threadIdx.x == 0) {
      mbar_inval(&bar[0]);
      mbar_inval(&bar[1]);
    }
    if (FRM == 1) {  // this CTA's next-digit counts (Fast Radix)
      __syncthreads();
      const uint32_t v = nh[threadIdx.x];
      if (v) atomicAdd(&P.fr_cnt[threadIdx.x], v);
    }
    if (FRM == 2) {
      __syncthreads();
      fr_joint_flush(P, whist, nh);
    }
  }
  // Fast Radix, pass mid (FRM 2): the (top digit, top 3 bits of the middle
  // digit) counts of the fused pass's FR_CHAINS chains (what the histogram
  // kernel counts on the counted path; their marginal gives the top digit's
  // bucket offsets, Alg. 3 l.5-6): 2048 counters in the deal's unused warp
  // rows 1..7 (1792) and the next-digit row (256), flushed once per CTA into
  // P.J[top digit][chain] (the first FR_CHAINS of the F_CHAINS slots)
  static constexpr int FR_CHAINS = 8;
  static __device__ __forceinline__ uint32_t fr_joint_addr(uint32_t whist_a, uint32_t nh_a, uint32_t b) {
    return b < 1792u ? whist_a + 4 * (256u + b) : nh_a + 4 * (b - 1792u);
  }
  static __device__ __forceinline__ void fr_joint_flush(const Params<K>& P, uint32_t* whist, uint32_t* nh) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t b = threadIdx.x * 8 + e;
      const uint32_t v = b < 1792u ? whist[256 + b] : nh[b - 1792u];
      if (v) atomicAdd(&P.J[(b / FR_CHAINS) * F_CHAINS + b % FR_CHAINS], v);
    }
  }

  // ------------------------------------------------------- Fast Radix
  // Fast Radix estimation at level 0 (dfr_config.fast_radix; Alg. 3,
  // P:211-246, applied to the top call's group of p = 3 digits lo, mid, hi):
  //   pass lo   deals A into ESTIMATED buckets (capacity ceil(n/256)) in
  //             C, overflow into chunks after the main regions (FRM = 1), and
  //             counts digit mid -- no histogram read of the input
  //   pass mid  reads C bucket by bucket (main region, then its chunks: the
  //             stable bucket order) through a tile table and deals
  //             into exact buckets of B (FRM = 2), counting digit hi (Alg. 3
  //             l.5-6: the top digit counted in the penultimate pass) and the
  //             joint histogram of the fused pass
  //   pass hi   the fused last pass (one chain: no chain histogram) B -> A
  // No pass is skipped (no histogram tells which digits are constant).

  // grid: the level-0 segment's route and flags, zeroed status rows, chunk
  // table, counters and the fused pass's joint histogram
  static __device__ __forceinline__ void zero_words(uint32_t* p, size_t n, uint32_t gid, uint32_t gsz) {
    const size_t head = min(n, (size_t)(((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15) / 4));
    for (size_t x = gid; x < head; x += gsz) p[x] = 0;
    uint4* q = reinterpret_cast<uint4*>(p + head);
    const size_t nv = (n - head) / 4;
    for (size_t x = gid; x < nv; x += gsz) q[x] = make_uint4(0, 0, 0, 0);
    for (size_t x = head + 4 * nv + gid; x < n; x += gsz) p[x] = 0;
  }
  static __device__ void fr_prep(const Params<K>& P) {
    Ctl* c = P.ctl;
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
    if (gid == 0) {
      Seg* q = P.segq[c->cur];
      Seg s = q[0];
      s.flags = 0;
      s.route = (0u | 2u << 2) | (2u | 1u << 2) << 4 | (1u | 2u << 2) << 8;  // A->C, C->B, B->C
      s.final_buf = 2;
      s.diff = ~0ull;  // unknown: every lower digit may vary
      q[0] = s;
      c->level0_p = s.p;
      c->level0_run = s.p;
      c->fr_next_chunk = 0;
      c->fr_tiles = 0;
      c->fr_overflow = 0;
    }
    // (16-byte stores: the status rows and the chunk table are ~0.26 GB at 2^28)
    zero_words(P.status, 3 * P.status_stride, gid, gsz);
    zero_words(P.fr_ct, (size_t)256 * P.fr_kmax, gid, gsz);
    for (uint32_t x = gid; x < 512u; x += gsz) P.fr_cnt[x] = 0;
    for (uint32_t x = gid; x < 65536u; x += gsz) P.H[x] = 0;
  }

  // one CTA of 256 threads after pass lo: bucket d's count is pass lo's
  // inclusive prefix of its last tile; the table of pass mid's tiles (each
  // bucket's main region in TILE pieces, then its overflow chunks) and pass
  // mid's exact bucket offsets (from the mid-digit counts pass lo took)
  static __device__ void fr_plan(const Params<K>& P) {
    Ctl* c = P.ctl;
    __shared__ uint32_t s_warp[WARPS];
    const Seg s = P.segq[c->cur][0];
    const uint32_t d = threadIdx.x;
    const uint32_t total = P.status[(size_t)(s.ntiles - 1) * 256 + d] & VAL_MASK;
    const uint32_t cap = P.fr_cap;
    const uint32_t main = min(total, cap), ovf = total - main;
    const uint32_t nmain = (main + TILE - 1) / TILE, novf = (ovf + FR_CHUNK - 1) / FR_CHUNK;
    uint32_t tt;
    uint32_t t0 = block_excl_scan(nmain + novf, s_warp, &tt);
    for (uint32_t k = 0; k < nmain; ++k)
      P.fr_tab[t0++] = make_uint2(d * cap + k * TILE, min((uint32_t)TILE, main - k * TILE));
    for (uint32_t k = 0; k < novf; ++k)
      P.fr_tab[t0++] = make_uint2(256u * cap + (P.fr_ct[(size_t)d * P.fr_kmax + k] - 1u) * FR_CHUNK,
                                  min(FR_CHUNK, ovf - k * FR_CHUNK));
    uint32_t tot2;
    const uint32_t ex = block_excl_scan(P.fr_cnt[d], s_warp, &tot2);
    P.hist[(size_t)(s.hist_off + 1) * 256 + d] = ex;
    uint32_t tov;
    block_excl_scan(ovf, s_warp, &tov);
    if (d == 0) {
      c->fr_tiles = tt;
      c->fr_overflow = tov;
    }
  }

  // ------------------------------------------------------- small sort core
  // rank of item i inside its bucket [bs, be) of the smem composite array
  static __device__ __forceinline__ uint32_t bucket_rank(const CT* cmp, int bs, int be, CT me) {
    uint32_t r = 0;
    int x = bs;
    for (; x + 4 <= be; x += 4) {
      const CT a = cmp[x], b = cmp[x + 1], c = cmp[x + 2], d = cmp[x + 3];
      r += (uint32_t)(a < me) + (uint32_t)(b < me) + (uint32_t)(c < me) + (uint32_t)(d < me);
    }
    for (; x < be; ++x) r += cmp[x] < me;
    return r;
  }
  static __device__ __forceinline__ uint32_t bucket_rank_wide(const K* keys, int bs, int be,
                                                              int i, K me) {
    uint32_t r = 0;
    for (int x = bs; x < be; ++x) {
      const K o = keys[x];
      r += (o < me) || (o == me && x < i);
    }
    return r;
  }

  // ---------------------------------------------------------------- divert
  // bucket of blen keys at gstart, held in buffer `buf`, larger than N_d:
  // recurse on the remaining digits (Alg. 4 l.11)
  static __device__ void push_bucket(const Params<K>& P, const Seg& s, uint32_t buf,
                                     uint32_t gstart, uint32_t blen) {
    Ctl* c = P.ctl;
    const int hn = highest_nonconst(s.diff, s.low - 1);
    if (c->level == 0) atomicAdd(&c->level0_large, 1ull);
    if (hn < 0 && buf == 0) return;  // constant keys, already in place
    if (blen <= (uint32_t)MID_CAP) {
      const uint32_t idx = atomicAdd(&c->mid_count, 1u);
      atomicAdd(&c->mid_buckets, 1ull);
      if (idx < P.mid_cap) {
        MidE m;
        m.start = gstart;
        m.len = (uint16_t)blen;
        m.hi = (int8_t)hn;
        m.buf = (uint8_t)buf;
        P.midq[idx] = m;
      } else {
        flag_overflow(c, 8u);
      }
    } else {
      const uint32_t idx = atomicAdd(&c->next_count, 1u);
      atomicAdd(&c->global_segments, 1ull);
      if (idx < P.max_segs) {
        Seg ns = {};
        ns.start = gstart;
        ns.len = blen;
        ns.hi = hn;
        ns.buf = buf;
        P.segq[1u - c->cur][idx] = ns;
      } else {
        flag_overflow(c, 16u);
      }
    }
  }

  static __device__ __forceinline__ void bucket_bounds_fast(const uint32_t* bm, int i, int& bs,
                                                            int& be) {
    // bits at or before i within 3 words, bits after i within 3 words (N_d <= 64)
    const int w = i >> 5;
    const uint32_t le = 0xffffffffu >> (31 - (i & 31));
    const uint32_t m0 = bm[w] & le, m1 = bm[w - 1], m2 = bm[w - 2];
    bs = m0 ? (w * 32 + 31 - __clz(m0))
            : (m1 ? ((w - 1) * 32 + 31 - __clz(m1)) : (m2 ? ((w - 2) * 32 + 31 - __clz(m2)) : -(1 << 20)));
    const uint32_t n0 = bm[w] & ~le, n1 = bm[w + 1], n2 = bm[w + 2];
    be = n0 ? (w * 32 + __ffs(n0) - 1)
            : (n1 ? ((w + 1) * 32 + __ffs(n1) - 1) : (n2 ? ((w + 2) * 32 + __ffs(n2) - 1) : (1 << 20)));
  }

  // Diversion scan of one level (Alg. 4 l.7-14).  A CTA owns the buckets that
  // START in its chunk of CH = WIN - VEC - N_d keys; it holds one window of
  // WIN keys (16-byte aligned start <= chunk start - 1; one TMA bulk copy into
  // a single window buffer, refilled after each window) so that every owned bucket of <= N_d
  // keys lies inside the window.  Those are sorted on-chip into the caller's
  // buffer in the stable (insertion-sort) order; larger buckets are
  // queued (Alg. 4 l.11).
  //
  // Per window (DV_NT threads, DKPT positions each, position i = tid + DV_NT*m):
  //   A  keys -> registers; bucket-start bitmask by ballot; composites := +inf
  //   B  bucket bounds from the bitmask; the 16-bit composite of each owned
  //      small-bucket key at cmp[4*bs + idx] (4-aligned groups per bucket)
  //   C  rank = number of bucket keys with a smaller composite, counted four
  //      at a time with packed fp16x2 compares (HSET2 + HADD2; composites are
  //      positive normal fp16 bit patterns, so integer order = fp16 order);
  //      order[bs + rank] = i
  //   D  (lossy composites) read-back: a slot claimed by another key means a
  //      tie -> that bucket is re-ranked exactly on the full keys by a warp
  //   E  coalesced write of every owned slot: out[j] = window[order[j]]
  // The composite is exact — (remaining bits, index in bucket) — when the R
  // remaining bits fit 14 - idx bits; otherwise it is the top 16 remaining bits
  // (scaled onto the signed normal fp16 values, Compo::get<true>).
  static constexpr uint16_t H_INF = 0x7c00;   // +inf: never below a composite
  static constexpr uint16_t H_BASE = 0x0400;  // smallest positive normal fp16
  static constexpr uint32_t DV_NONE = 0xffffffffu;
  static constexpr uint32_t DV_HOLE = 0xffffu;  // order slot not filled (window positions < WIN)
#ifndef DFR_DV_NT
#define DFR_DV_NT 128
#define DFR_DV_MINB 8
#endif
  static constexpr int DV_NT = DFR_DV_NT;     // threads of the stand-alone divert kernel
  static constexpr size_t DV_WIN_BYTES = WIN * sizeof(K) + (PAIRS ? WIN * 4 : 0);
  static constexpr int DV_CMP = 4 * WIN + 64;  // halves

  struct DivertSmem {
    char* win[2];       // window buffers (keys, then values for pairs); both point at one
                        // buffer: 8 CTAs/SM hide its refill (divert())
    uint16_t* cmp;      // fp16 composites
    uint16_t* order;    // slot -> window position of the key ranked there
    uint32_t* bm;       // bucket-start bitmask (4 zero words on each side)
    uint32_t* misc;     // [2*b]: segment of the window in buffer b, [2*b+1]: tma flag
    unsigned long long* bar;  // one mbarrier per buffer
  };

  // composite of a key with R remaining bits at index idx of its bucket
  struct Compo {
    K mask;        // remaining bits
    int sh, sl;    // (rem >> sh) << sl
    int sh16;      // diversion, lossy: the top 16 remaining bits are rem >> sh16
    uint32_t im;   // index mask (exact mode)
    bool exact;
    __device__ __forceinline__ void init(int R, int nd) {
      const int idxb = nd <= 64 ? 6 : 8;
      mask = R ? (K)(~K(0) >> (8 * sizeof(K) - R)) : K(0);
      exact = R + idxb <= 14;
      sh = exact ? 0 : R - 14;
      // lossy: the top 16 remaining bits; with R = 8 (possible when n_d > 64 makes the
      // index 8 bits wide) the 16 bits reach into the bucket's shared prefix,
      // which is constant inside a bucket, so they still order it
      sh16 = (exact || R < 16) ? 0 : R - 16;
      sl = exact ? idxb : 0;
      im = exact ? 0xffu : 0u;
    }
    __device__ __forceinline__ uint16_t operator()(K k, uint32_t idx) const {
      return (uint16_t)(H_BASE + (((uint32_t)((k & mask) >> sh) << sl) | (idx & im)));
    }
    // LOSSY: the top 16 of the R remaining bits scaled onto the 61440 normal
    // fp16 values of both signs, in order (negatives for the lower half:
    // -0x7BFF .. -0x0400, then +0x0400 .. +0x7BFF): ties 3.7x rarer than with
    // 14 bits; exact: (rem << idxb) | idx
    template <bool LOSSY>
    __device__ __forceinline__ uint16_t get(K k, uint32_t idx) const {
      if (LOSSY) {
        const uint32_t v = (((uint32_t)(k >> sh16) & 0xffffu) * 61440u) >> 16;
        return (uint16_t)(v < 30720u ? (0x8000u | (0x0400u + 30719u - v)) : (0x0400u + v - 30720u));
      }
      return (uint16_t)(H_BASE + (((uint32_t)(k & mask) << sl) | idx));
    }
  };

  // window geometry of chunk ch of segment s: r0 = segment index of window
  // position 0 (16-byte aligned in memory), off = first owned position
  static __device__ __forceinline__ void window_of(const Params<K>& P, const Seg& s, uint32_t ch,
                                                   int& c0, int& r0, int& off) {
    constexpr int VEC = 16 / sizeof(K);
    c0 = (int)(ch - s.chunk0) * (int)P.chunk;
    const long long a = (long long)s.start + c0 - 1;  // absolute index of the key before the chunk
    const long long a0 = a >= 0 ? (a & ~(long long)(VEC - 1)) : -(long long)VEC;
    r0 = (int)(a0 - (long long)s.start);
    off = c0 - r0;
  }

  // thread 0: chunk ch goes to buffer b; start its TMA when the window lies
  // inside the array and the segment diverts this level
  static __device__ __forceinline__ void divert_prefetch(const Params<K>& P, const Seg* q,
                                                         uint32_t nseg, uint32_t total,
                                                         uint32_t ch, const DivertSmem& S, int b) {
    S.misc[2 * b] = 0;
    S.misc[2 * b + 1] = 0;
    if (ch >= total) return;
    const uint32_t si = upper_index(nseg, ch, [&](uint32_t i) { return q[i].chunk0; });
    S.misc[2 * b] = si;
    const Seg& s = q[si];
    if (s.flags & (SEG_DONE | SEG_SKIP_DIVERT | SEG_COPY | SEG_SORTED)) return;
    int c0, r0, off;
    window_of(P, s, ch, c0, r0, off);
    const long long abs0 = (long long)s.start + r0;
    if (abs0 < 0 || abs0 + WIN > (long long)P.n) return;
    const K* xs = P.kbuf(s.final_buf) + abs0;
    const V* xv = PAIRS ? P.vbuf(s.final_buf) + abs0 : nullptr;
    if ((reinterpret_cast<uintptr_t>(xs) & 15) || (PAIRS && (reinterpret_cast<uintptr_t>(xv) & 15)))
      return;
    fence_proxy_async();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(S.bar + b)),
                 "r"((uint32_t)DV_WIN_BYTES)
                 : "memory");
    asm volatile(
        DFR_TMA_LOAD ::"r"(
            smem_u32(S.win[b])),
        "l"(xs), "r"((uint32_t)(WIN * sizeof(K))), "r"(smem_u32(S.bar + b))
        : "memory");
    if (PAIRS)
      asm volatile(
          DFR_TMA_LOAD ::"r"(
              smem_u32(S.win[b] + WIN * sizeof(K))),
          "l"(xv), "r"((uint32_t)(WIN * 4)), "r"(smem_u32(S.bar + b))
          : "memory");
    S.misc[2 * b + 1] = 1;
  }

  // a bucket > N_d starting at segment index rb: find its end (gallop over
  // the segment), queue it (Alg. 4 l.9-11)
  static __device__ DFR_COLD void divert_large(const Params<K>& P, const Seg& s, int rb,
                                                   int known, int shift) {
    const K* xs = P.kbuf(s.final_buf) + s.start;
    const K pre = xs[rb] >> shift;
    const uint32_t len = s.len;
    uint32_t lo = (uint32_t)max(known - 1, rb);  // index known to share the prefix
    uint32_t hi = len;
    uint32_t step = 64;
    while (true) {  // gallop
      const uint32_t probe = lo + step;
      if (probe >= hi) break;
      if ((xs[probe] >> shift) != pre) {
        hi = probe;
        break;
      }
      lo = probe;
      step <<= 1;
    }
    while (hi - lo > 1) {  // first index in (lo, hi] with a different prefix
      const uint32_t mid = (lo + hi) >> 1;
      if ((xs[mid] >> shift) != pre)
        hi = mid;
      else
        lo = mid;
    }
    push_bucket(P, s, s.final_buf, s.start + (uint32_t)rb, hi - (uint32_t)rb);
  }

  // exact stable ranks of the bucket [bs, be) of the window, by one warp
  static __device__ DFR_COLD void rerank_exact(uint32_t sk_a, uint32_t order_a, int bs, int be) {
    const int lane = threadIdx.x & 31;
    for (int y = bs + lane; y < be; y += 32) {
      const K ky = ldsk<K>(sk_a + sizeof(K) * y);
      uint32_t r = 0;
      for (int z = bs; z < be; ++z) {
        const K kz = ldsk<K>(sk_a + sizeof(K) * z);
        r += (kz < ky) || (kz == ky && z < y);
      }
      sts16(order_a + 2 * (bs + r), (uint32_t)y);
    }
  }

  // highest set bit of the 96-bit word (hi:mid:lo), counted from bit 0 of lo,
  // or -1 (branch-free selects)
  static __device__ __forceinline__ int top_bit96(uint32_t hi, uint32_t mid, uint32_t lo) {
    const int th = 95 - __clz(hi), tm = 63 - __clz(mid), tl = 31 - __clz(lo);
    return hi ? th : (mid ? tm : tl);
  }
  // lowest set bit of the 96-bit word (hi:mid:lo), or 96
  static __device__ __forceinline__ int low_bit96(uint32_t lo, uint32_t mid, uint32_t hi) {
    const int bl = __ffs(lo) - 1, bmid = 31 + __ffs(mid), bh = 63 + __ffs(hi);
    return lo ? bl : (mid ? bmid : (hi ? bh : 96));
  }

  // warp-wide exact re-rank of every bucket flagged in bmk (lanes' info),
  // then its slots written out again (a bucket that straddles two warps is
  // done by both, with identical results)
  static __device__ DFR_COLD void fixup_flagged(uint32_t sk_a, uint32_t sv_a, uint32_t order_a,
                                                    uint32_t bmk, uint32_t info, bool b, K* outk,
                                                    V* outv) {
    const int lane = threadIdx.x & 31;
    while (bmk) {
      const uint32_t inf = __shfl_sync(0xffffffffu, info, __ffs(bmk) - 1);
      bmk &= ~__ballot_sync(0xffffffffu, b && (info & 0xfffu) == (inf & 0xfffu));
      const int bs = inf & 0xfff, be = bs + ((inf >> 12) & 0x1ff);
      rerank_exact(sk_a, order_a, bs, be);
      __syncwarp();
      for (int j = bs + lane; j < be; j += 32) {
        const uint32_t src = lds16(order_a + 2 * j);
        outk[j] = ldsk<K>(sk_a + sizeof(K) * src);
        if (PAIRS) outv[j] = lds32(sv_a + 4 * src);
      }
      __syncwarp();
    }
  }



  // Positions: warp w holds the contiguous range [w*WPW, (w+1)*WPW) of the
  // window, 32 consecutive positions per step m.  The bucket-start ballot
  // words of its own steps stay in registers; bucket bounds come from the
  // lane's own word plus warp-uniform carries (last start before the step,
  // first start after it), seeded by the two edge words of each neighbouring
  // warp (shared memory).
  template <int NT, bool LOSSY, bool EDGE>
  static __device__ __forceinline__ void divert_window(const Params<K>& P, const Seg& s,
                                                       const DivertSmem& S, uint32_t sk_a,
                                                       uint32_t sv_a, int r0, int off,
                                                       const Compo& comp) {
    constexpr int NW = NT / 32, WPW = WIN / NW, DKPT = WPW / 32;
    constexpr uint32_t KB = sizeof(K);
    constexpr int NONE_LO = -(1 << 20), NONE_HI = 1 << 20;
    static_assert(DKPT >= 2, "two edge words per warp");
    static_assert(WIN % NW == 0 && WPW % 32 == 0, "each warp holds whole 32-position steps");
    const int CH = (int)P.chunk;
    const int nd = (int)P.n_d;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int len = (int)s.len;
    const int shift = 8 * s.low;
    const int wbase = w * WPW;
    const uint32_t cmp_a = smem_u32(S.cmp), order_a = smem_u32(S.order);
    const uint32_t bm_a = smem_u32(S.bm);  // word index = position / 32 (zero words beyond both ends)
    const K pmask = (K)(~K(0) << shift);  // the group prefix bits of a key
    // ---- A: keys, bucket-start words
    uint32_t bw[DKPT];  // (keys are re-read in B: registers buy occupancy here)
#pragma unroll
    for (int m = 0; m < DKPT; ++m) {
      const int i = wbase + 32 * m + lane;
      const K km = ldsk<K>(sk_a + KB * i);
      const K kp = ldsk<K>(sk_a + KB * (i > 0 ? i - 1 : 0));
      bool st = ((km ^ kp) & pmask) != K(0);
      if (m == 0) st |= i == 0;
      if (EDGE) {
        const int r = r0 + i;
        st |= (unsigned)(r - 1) >= (unsigned)(len - 1);  // r <= 0 or r >= len
      }
      bw[m] = __ballot_sync(0xffffffffu, st);
    }
    if (lane < 2) sts32(bm_a + 4 * (w * DKPT + lane), lane ? bw[1] : bw[0]);
    if (lane == 2) sts32(bm_a + 4 * (w * DKPT + DKPT - 2), bw[DKPT - 2]);
    if (lane == 3) sts32(bm_a + 4 * (w * DKPT + DKPT - 1), bw[DKPT - 1]);
    if (nd > 64)  // generic N_d: every word through shared memory
#pragma unroll
      for (int m = 2; m < DKPT - 2; ++m)
        if (lane == 0) sts32(bm_a + 4 * (w * DKPT + m), bw[m]);
    {  // composites := +inf (the pad of every bucket's last group of four)
      const uint4 inf4 = make_uint4(0x7c007c00u, 0x7c007c00u, 0x7c007c00u, 0x7c007c00u);
      for (int x = threadIdx.x; x < DV_CMP / 8; x += NT) sts128(cmp_a + 16 * x, inf4);
    }
    __syncthreads();
    // ---- B: bounds, composites of owned small-bucket keys, large starts
    const uint32_t le = 0xffffffffu >> (31 - lane);
    uint32_t info[DKPT];      // bs | size << 12 | rank << 24, or DV_NONE
    uint32_t mev[(DKPT + 1) / 2];  // the composites of the lane's positions, two per word
#pragma unroll
    for (int m = 0; m < (DKPT + 1) / 2; ++m) mev[m] = 0;
    uint32_t lg = 0;
    if (nd <= 64) {
      // first start after each step (backward carry), seeded by the next warp
      int nxt[DKPT];
      {
        const uint32_t e0 = lds32(bm_a + 4 * (w * DKPT + DKPT)),
                       e1 = lds32(bm_a + 4 * (w * DKPT + DKPT + 1));
        int c = e0 ? wbase + WPW + __ffs(e0) - 1 : (e1 ? wbase + WPW + 31 + __ffs(e1) : NONE_HI);
#pragma unroll
        for (int m = DKPT - 1; m >= 0; --m) {
          nxt[m] = c;
          if (bw[m]) c = wbase + 32 * m + __ffs(bw[m]) - 1;
        }
      }
      // last start before each step (forward carry), seeded by the previous warp
      const uint32_t f1 = lds32(bm_a + 4 * (w * DKPT - 1)), f2 = lds32(bm_a + 4 * (w * DKPT - 2));
      int prv = f1 ? wbase - 1 - __clz(f1) : (f2 ? wbase - 33 - __clz(f2) : NONE_LO);
#pragma unroll
      for (int m = 0; m < DKPT; ++m) {
        const int i = wbase + 32 * m + lane;
        const int base = wbase + 32 * m;
        const uint32_t lo = bw[m] & le, hi = bw[m] & ~le;
        const int bs = lo ? base + 31 - __clz(lo) : prv;
        const int be = hi ? base + __ffs(hi) - 1 : nxt[m];
        if (bw[m]) prv = base + 31 - __clz(bw[m]);
        bool own = bs >= off && bs < off + CH;
        if (EDGE) own &= r0 + bs < len;
        const bool small = be - bs <= nd;
        info[m] = DV_NONE;
        if (own && small) {
          info[m] = (uint32_t)bs | ((uint32_t)(be - bs) << 12);
          const uint32_t c16 = comp.template get<LOSSY>(ldsk<K>(sk_a + KB * i), (uint32_t)(i - bs));
          mev[m >> 1] |= c16 << (16 * (m & 1));
          sts16(cmp_a + 2 * (3 * bs + i), c16);
          if (LOSSY) sts16(order_a + 2 * i, DV_HOLE);  // slot i: filled in C unless a tie
        }
        lg |= (uint32_t)(own && !small && i == bs) << m;
      }
    } else {  // generic N_d (up to 256): word-wise search in shared memory
      __syncthreads();
      const uint32_t* bmp = S.bm;
#pragma unroll
      for (int m = 0; m < DKPT; ++m) {
        const int i = wbase + 32 * m + lane;
        int bs = prev_set(bmp, i, max(1, i - nd));
        int be = bs >= 1 ? next_set(bmp, i, min(WIN - 1, bs + nd)) : -1;
        if (be < 0) be = NONE_HI;
        if (bs < 0) bs = NONE_LO;
        bool own = bs >= off && bs < off + CH;
        if (EDGE) own &= r0 + bs < len;
        const bool small = be - bs <= nd;
        info[m] = DV_NONE;
        if (own && small) {
          info[m] = (uint32_t)bs | ((uint32_t)(be - bs) << 12);
          const uint32_t c16 = comp.template get<LOSSY>(ldsk<K>(sk_a + KB * i), (uint32_t)(i - bs));
          mev[m >> 1] |= c16 << (16 * (m & 1));
          sts16(cmp_a + 2 * (3 * bs + i), c16);
          if (LOSSY) sts16(order_a + 2 * i, DV_HOLE);  // slot i: filled in C unless a tie
        }
        lg |= (uint32_t)(own && !small && i == bs) << m;
      }
    }
    if (lg)  // rare: queue the large buckets that start here
      for (int m = 0; m < DKPT; ++m)
        if ((lg >> m) & 1u) {
          const int rb = r0 + wbase + 32 * m + lane;
          divert_large(P, s, rb, rb + 1, shift);
        }
    __syncthreads();
    // ---- C: ranks
#pragma unroll
    for (int m = 0; m < DKPT; ++m) {
      const int i = wbase + 32 * m + lane;
      const bool ok = info[m] != DV_NONE;
      const int bs = ok ? (int)(info[m] & 0xfff) : 0;
      const int ng = ok ? (int)(((info[m] >> 12) & 0x1ff) + 3) >> 2 : 0;
      const uint32_t me = (mev[m >> 1] >> (16 * (m & 1))) & 0xffffu;
      const __half2 me2 = __halves2half2(__ushort_as_half((unsigned short)me),
                                         __ushort_as_half((unsigned short)me));
      uint32_t pa = cmp_a + 8 * bs;
      const uint32_t pe = pa + 8 * ng;
      __half2 acc = __float2half2_rn(0.f);
#pragma unroll DV_CU
      for (; pa < pe; pa += 8) {
        const uint2 v = lds64v(pa);
        acc = __hadd2(acc, __hlt2(*reinterpret_cast<const __half2*>(&v.x), me2));
        acc = __hadd2(acc, __hlt2(*reinterpret_cast<const __half2*>(&v.y), me2));
      }
      const uint32_t rk = (uint32_t)__half2ushort_rz(__hadd(__low2half(acc), __high2half(acc)));
      if (ok) {
        sts16(order_a + 2 * (bs + rk), (uint32_t)i);
        info[m] |= rk << 24;
      }
    }
    __syncthreads();
    // ---- E: coalesced write of every owned slot.  (lossy) Two keys with
    // equal composites take the same rank, which leaves a slot of their
    // bucket unfilled: the lane that finds the hole flags the bucket
    K* outk = P.A + s.start + r0;
    V* outv = P.Av + s.start + r0;
    uint32_t hole = 0;
#pragma unroll
    for (int m = 0; m < DKPT; ++m) {
      if (info[m] != DV_NONE) {
        const int j = wbase + 32 * m + lane;
        const uint32_t src = lds16(order_a + 2 * j);
        if (LOSSY && src == DV_HOLE) {
          hole |= 1u << m;
        } else {
          outk[j] = ldsk<K>(sk_a + KB * src);
          if (PAIRS) outv[j] = lds32(sv_a + 4 * src);
        }
      }
    }
    // ---- D: (rare) flagged buckets re-ranked exactly on the full keys and
    // written again; the barrier also frees the window, composites and order
    if (LOSSY && __syncthreads_or(hole != 0)) {
#pragma unroll
      for (int m = 0; m < DKPT; ++m) {
        const bool b = (hole >> m) & 1u;
        const uint32_t bmk = __ballot_sync(0xffffffffu, b);
        if (bmk) fixup_flagged(sk_a, sv_a, order_a, bmk, info[m], b, outk, outv);
      }
      __syncthreads();
    } else if (!LOSSY) {
      __syncthreads();
    }
  }

  template <int NT>
  static __device__ __forceinline__ void divert(const Params<K>& P, uint32_t* sm) {
    Ctl* c = P.ctl;
    if (P.fuse && c->level == 0 && *(volatile uint32_t*)&c->fused_ok) return;  // done by the fused pass
    const uint32_t total = c->total_chunks, nseg = c->nseg;
    const Seg* q = P.segq[c->cur];
    DivertSmem S;
    char* base = reinterpret_cast<char*>(sm);
    S.win[0] = base;
    S.win[1] = base;  // one window buffer: 8 CTAs/SM (DFR_DV_MINB) hide its refill
    S.cmp = reinterpret_cast<uint16_t*>(base + DV_WIN_BYTES);
    S.order = S.cmp + DV_CMP;
    uint32_t* bm0 = reinterpret_cast<uint32_t*>(S.order + WIN);
    S.bm = bm0 + 4;
    S.misc = S.bm + WIN / 32 + 4;
    S.bar = reinterpret_cast<unsigned long long*>(S.misc + 4);
    if (threadIdx.x < 4) {
      bm0[threadIdx.x] = 0;
      S.bm[WIN / 32 + threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) {
      mbar_init(S.bar, 1);
      mbar_init(S.bar + 1, 1);
      fence_mbar_init();
      divert_prefetch(P, q, nseg, total, blockIdx.x, S, 0);
    }
    __syncthreads();
    uint32_t parity = 0;
    int b = 0;
    uint32_t cur_si = ~0u;  // the segment record and composite plan change rarely
    Seg s;
    Compo comp;
    for (uint32_t ch = blockIdx.x; ch < total; ch += gridDim.x) {
      const uint32_t si = S.misc[2 * b];
      if (si != cur_si) {
        cur_si = si;
        s = q[si];
        comp.init(8 * s.low, (int)P.n_d);
      }
      const bool tma = S.misc[2 * b + 1] != 0;
      int c0, r0, off;
      window_of(P, s, ch, c0, r0, off);
      if (s.flags & (SEG_DONE | SEG_SKIP_DIVERT | SEG_COPY | SEG_SORTED)) {
        // finished bucket left in B: copy out
        if ((s.flags & SEG_COPY) || ((s.flags & SEG_SORTED) && s.final_buf)) {
          const int c1 = min((int)s.len, c0 + (int)P.chunk);
          const int nt = blockDim.x;
          int r = c0 + threadIdx.x;
          K* dA = P.A + s.start;
          const K* sB = P.kbuf(s.final_buf) + s.start;
          for (; r + 3 * nt < c1; r += 4 * nt) {  // four loads in flight
            const K x0 = sB[r], x1 = sB[r + nt], x2 = sB[r + 2 * nt], x3 = sB[r + 3 * nt];
            dA[r] = x0;
            dA[r + nt] = x1;
            dA[r + 2 * nt] = x2;
            dA[r + 3 * nt] = x3;
          }
          for (; r < c1; r += nt) dA[r] = sB[r];
          if (PAIRS)
            for (int rv = c0 + threadIdx.x; rv < c1; rv += nt)
              P.Av[s.start + rv] = P.vbuf(s.final_buf)[s.start + rv];
        }
        __syncthreads();
        if (threadIdx.x == 0) divert_prefetch(P, q, nseg, total, ch + gridDim.x, S, 0);
        __syncthreads();
        continue;
      }
      const uint32_t sk_a = smem_u32(S.win[b]);
      const uint32_t sv_a = sk_a + WIN * sizeof(K);
      if (tma) {
        mbar_wait(S.bar + b, (parity >> b) & 1u);
        parity ^= 1u << b;
      } else {  // window at an array edge / unaligned: plain loads
        K* wk = reinterpret_cast<K*>(S.win[b]);
        V* wv = reinterpret_cast<V*>(S.win[b] + WIN * sizeof(K));
        const K* xs = P.kbuf(s.final_buf);
        const V* xv = PAIRS ? P.vbuf(s.final_buf) : nullptr;
        for (int i = threadIdx.x; i < WIN; i += blockDim.x) {
          const long long a = (long long)s.start + r0 + i;
          const bool ok = a >= 0 && a < (long long)P.n;
          wk[i] = ok ? xs[a] : K(0);
          if (PAIRS) wv[i] = ok ? xv[a] : 0u;
        }
        __syncthreads();
      }
      const bool edge = r0 < 0 || r0 + WIN > (int)s.len;
      if (comp.exact) {
        if (edge) divert_window<NT, false, true>(P, s, S, sk_a, sv_a, r0, off, comp);
        else      divert_window<NT, false, false>(P, s, S, sk_a, sv_a, r0, off, comp);
      } else {
        if (edge) divert_window<NT, true, true>(P, s, S, sk_a, sv_a, r0, off, comp);
        else      divert_window<NT, true, false>(P, s, S, sk_a, sv_a, r0, off, comp);
      }
      // divert_window ends on a barrier: window buffer, composites and order free
      if (threadIdx.x == 0) divert_prefetch(P, q, nseg, total, ch + gridDim.x, S, 0);
      __syncthreads();  // the next window's segment / tma flag visible
    }
    // no copy in flight (the last prefetch found ch >= total); the shared
    // memory is reused by the next phase of k_levels
    if (threadIdx.x == 0) {
      mbar_inval(S.bar);
      mbar_inval(S.bar + 1);
    }
  }

  // ============================================================ fused last pass
  // Level 0 with p = 3 group digits (lo, mid, hi) on large keys-only inputs:
  // after the passes on lo and mid the data is sorted by (mid, lo), so every
  // run of equal (mid, lo) -- an "s-run" -- is contiguous, and the buckets of
  // the level (Alg. 4 l.8: equal top-3-digit prefix) are exactly the keys of
  // one s-run that share digit hi.  A tile made of one whole s-run therefore
  // holds its buckets complete, and the last deal (Alg. 4 l.6, digit hi) and
  // the diversion of its small buckets (l.10-14: sorted) run on the
  // tile in one kernel: the keys are read once and written once, in their
  // final place (the separate deal + diversion move them twice).  The s-runs
  // come from the joint histogram H[mid][lo] counted by the deal on mid
  // (FUSEH); the plan kernel falls back (fused_ok = 0) to the plain deal +
  // diversion when an s-run exceeds a tile or a pass was skipped.
  //
  // Inside a tile the keys are split by (hi, the top FSB remaining bits): a
  // bucket's keys fall into 2^FSB sub-buckets that are already in order, so
  // the small sort only ranks inside a sub-bucket (mean 4 keys at 2^28 instead
  // of 16: a quarter of the compares, and of the warp divergence).
  // Per tile (FNT threads, up to FT_MAX keys):
  //   1 keys -> registers (coalesced loads; the tile was prefetched into L2);
  //     a slot in its sub-bucket by shared atomic
  //   2 one thread per digit value: bucket start, sub-bucket starts and
  //     composite-area bases (one packed block scan); tile aggregate published
  //   3 keys stored grouped by sub-bucket; the 16-bit composite (the next 16
  //     key bits) of each key of a small bucket stored in its sub-bucket's
  //     4-aligned composite area (padded with +inf); then, one thread per
  //     digit value, the decoupled look-back over the earlier tiles (their
  //     aggregates were published long before) and buckets > N_d queued for
  //     recursion (l.11)
  //   4 slot-major: rank = number of sub-bucket keys with a smaller composite
  //     (packed fp16x2 compares, as in the diversion); each key is written
  //     straight to its final place (a warp's 32 keys land in a permutation
  //     of a few consecutive sub-buckets).  The ranks of a sub-bucket of c
  //     keys sum to c(c-1)/2 unless two composites tie (tied keys share the
  //     lower rank); such a sub-bucket is re-ranked exactly on the full keys
  //     by a warp and written again.
  // Keys only: a bucket > N_d is written in slot order, which the recursion
  // sorts; equal keys are indistinguishable.
  static constexpr int FNT = 256, FKPT = 18, FNW = FNT / 32;
  // the longest s-run a tile holds (FKPT keys per thread would take 4608; the
  // shared memory of 3 CTAs/SM takes 4576 -- an s-run of 2^28 uniform keys
  // exceeds it with probability ~1e-9, and then the plain path runs)
  static constexpr int FT_MAX = 4576;
  static constexpr int FSB = 2;              // sub-bucket bits below the group
  static constexpr int FNS = 256 << FSB;     // sub-buckets per tile
  static constexpr int F_CMP = FT_MAX + 3 * FNS + 8;  // composite halves (areas padded to 4)
  struct FS {                                         // shared-memory layout, byte offsets
    static constexpr int KEYS = 0;                                      // K[FT_MAX], grouped
    static constexpr int CMP = KEYS + FT_MAX * (int)sizeof(K);          // u16[F_CMP]
    static constexpr int POS = CMP + F_CMP * 2;                         // u16[FT_MAX]: tile position
    static constexpr int CNT = POS + FT_MAX * 2;                         // u32[2][FNS] (two tiles)
    static constexpr int BDESC = CNT + 2 * FNS * 4;                     // u32[FNS]
    static constexpr int SDST = BDESC + FNS * 4;                        // int[256]
    static constexpr int FLAG = SDST + 1024;                            // u32[FNS/32] tie flags
    static constexpr int WARP = FLAG + FNS / 8;                         // u32[16]
    static constexpr int MISC = WARP + 64;                              // u32[16]
    static constexpr int BYTES = MISC + 64;
  };
  static_assert(FS::CMP % 16 == 0 && FS::CNT % 16 == 0 && FS::BDESC % 16 == 0,
                "fused smem alignment");
  static_assert(FS::BYTES + 1024 <= 233472 / 3, "three fused CTAs per SM");
  static_assert(FT_MAX <= FNT * FKPT && FT_MAX % 8 == 0, "fused tile");
  static_assert(FT_MAX < (1 << 13) && F_CMP / 4 < (1 << 11), "fused bucket descriptor fields");
  static constexpr size_t SMEM_FUSED = FS::BYTES;

  // One CTA of 1024 threads: the s-run tiles from H and their ticket order.
  // The look-back of the fused pass runs along F_CHAINS independent chains
  // (chain = top 4 bits of the middle digit): a tile's exclusive prefix per top
  // digit is the sum over the earlier tiles of ITS chain plus the chain's base,
  // the count of keys with that top digit in all earlier chains (from the
  // (top digit, chain) histogram the histogram kernel counted).  Tickets take
  // the chains round robin, so consecutive tickets belong to different chains
  // and a tile's predecessor in its chain was claimed F_CHAINS tickets
  // earlier: its inclusive prefix is nearly always published by then, and
  // the look-back rarely waits (one chain through all 65536 tiles cannot keep
  // up with the rate at which tiles arrive).
  // Grid of 256 CTAs (lo value l) x 256 threads (mid value d), before fplan
  // on the counted path: the middle pass added to H[mid][lo] only the tiles
  // that straddle a run of lo; the whole tiles [a, b) inside the run of lo = l
  // added nothing, and their digit counts are differences of the inclusive
  // prefixes the look-back left in the status rows: H[d][l] += I(b-1, d) - I(a-1, d)
  static __device__ void hfix(const Params<K>& P) {
    Ctl* c = P.ctl;
    const Seg s = P.segq[c->cur][0];
    if (!(P.fuse && c->level == 0 && c->nseg == 1 && s.p == 3 && (s.flags & 0xfu) == 0)) return;
    const uint32_t l = blockIdx.x, d = threadIdx.x;
    const uint32_t* st1 = P.status + P.status_stride;
    const uint32_t* lofs = P.hist + (size_t)s.hist_off * 256;  // lo bucket offsets (plan2)
    const uint32_t r0 = lofs[l], r1 = l == 255u ? s.len : lofs[l + 1];
    // tiles [a, b) lie inside [r0, r1) (the segment's last tile may be partial)
    const uint32_t a = (r0 + TILE - 1) / TILE, b = r1 == s.len ? (r1 + TILE - 1) / TILE : r1 / TILE;
    if (b > a) {
      const uint32_t ib = st1[(size_t)(b - 1) * 256 + d] & VAL_MASK;
      const uint32_t ia = a ? st1[(size_t)(a - 1) * 256 + d] & VAL_MASK : 0u;
      const uint32_t dif = (ib - ia) & VAL_MASK;  // mod 2^30 (n <= 2^30)
      if (dif) atomicAdd(&P.H[d * 256 + l], dif);
    }
  }

  static __device__ void fplan(const Params<K>& P) {
    Ctl* c = P.ctl;
    __shared__ uint32_t s_w[32], s_w2[32], s_m[32];
    const Seg s = P.segq[c->cur][0];
    const bool eligible = P.fuse && P.C != nullptr && c->level == 0 && c->nseg == 1 && s.p == 3 &&
                          (s.flags & (0xfu | SEG_SKIP_DIVERT | SEG_COPY | SEG_DONE | SEG_SORTED)) == 0 &&
                          route_src(s, 2) != 0;
    if (!eligible) {
      if (threadIdx.x == 0) c->fused_ok = 0;
      return;
    }
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // this thread: s-runs (middle digit, low digit) = ids [64t, 64t + 64); chain = t >> 6
    uint32_t h[64];
    const uint4* h4 = reinterpret_cast<const uint4*>(P.H + 64 * t);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint4 x = h4[k];
      h[4 * k] = x.x;
      h[4 * k + 1] = x.y;
      h[4 * k + 2] = x.z;
      h[4 * k + 3] = x.w;
    }
    uint32_t sum = 0, mx = 0, nz = 0;
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      sum += h[k];
      mx = max(mx, h[k]);
      nz += h[k] != 0;
    }
    uint32_t a = sum, b = nz;  // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
      if (lane >= o) {
        a += ya;
        b += yb;
      }
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 31) {
      s_w[w] = a;
      s_w2[w] = b;
    }
    if (lane == 0) s_m[w] = mx;
    // chains: 16 (top 4 bits of the middle digit) from the histogram kernel's
    // joint counts; Fast Radix: 8 (top 3 bits) from the middle pass's
    const uint32_t chains = P.fr ? (uint32_t)FR_CHAINS : (uint32_t)F_CHAINS;
    // chain bases per top digit: exclusive over the chains
    if (t < 256) {
      uint32_t acc = 0;
#pragma unroll
      for (int ch = 0; ch < F_CHAINS; ++ch) {
        const uint32_t x = (uint32_t)ch < chains ? P.J[t * F_CHAINS + ch] : 0u;
        P.J[4096 + ch * 256 + t] = acc;
        acc += x;
      }
    }
    __syncthreads();
    uint32_t pa = 0, tot = 0, ntl = 0, gmx = 0;
    for (int e = 0; e < 32; ++e) {
      if (e < w) pa += s_w[e];
      tot += s_w[e];
      ntl += s_w2[e];
      gmx = max(gmx, s_m[e]);
    }
    // tiles per chain (32 / chains warps per chain) and this thread's first index in its chain
    const uint32_t wpc = 32 / chains;
    uint32_t nch[F_CHAINS];
#pragma unroll
    for (int ch = 0; ch < F_CHAINS; ++ch) {
      nch[ch] = 0;
      if ((uint32_t)ch < chains)
        for (uint32_t e = 0; e < wpc; ++e) nch[ch] += s_w2[ch * wpc + e];
    }
    const int ch = (int)(w / wpc);
    uint32_t jb = b - nz;  // non-empty s-runs before mine in my chain
    for (uint32_t e = ch * wpc; e < (uint32_t)w; ++e) jb += s_w2[e];
    uint32_t nmin = nch[0];
#pragma unroll
    for (int e = 1; e < F_CHAINS; ++e)
      if ((uint32_t)e < chains) nmin = min(nmin, nch[e]);
    // ticket of the j-th tile of chain ch: round robin over the chains that
    // still have tiles (while every chain has: chains * j + ch)
    auto ticket = [&](uint32_t j) {
      if (j < nmin) return chains * j + (uint32_t)ch;
      uint32_t p = 0;
#pragma unroll
      for (int e = 0; e < F_CHAINS; ++e) p += min(nch[e], j) + ((e < ch && nch[e] > j) ? 1u : 0u);
      return p;  // (chains beyond `chains` have nch = 0)
    };
    if (P.fr) {  // the top digit's bucket offsets from the joint counts taken in the middle pass
      __shared__ uint32_t s_c[256];
      if (t < 256) {
        uint32_t m = 0;
#pragma unroll
        for (int ch = 0; ch < FR_CHAINS; ++ch) m += P.J[t * F_CHAINS + ch];
        s_c[t] = m;
      }
      __syncthreads();
      if (t < 256) {
        uint32_t e = 0;
        for (int x = 0; x < t; ++x) e += s_c[x];
        P.hist[(size_t)(s.hist_off + 2) * 256 + t] = e;
      }
    }
    const bool ok = gmx <= (uint32_t)FT_MAX && tot == s.len;
    if (ok) {
      uint32_t pos = pa + a - sum;
      uint32_t prev = jb ? ticket(jb - 1) : ~0u;
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const uint32_t x = h[k];
        if (x) {
          const uint32_t tk = ticket(jb);
          P.ftiles[tk] = make_uint4(pos, x, prev, (uint32_t)ch);
          prev = tk;
          ++jb;
        }
        pos += x;
      }
    }
    if (t == 0) {
      c->fused_ok = ok ? 1u : 0u;
      c->fused_tiles = ntl;
      c->fticket = 0;
      c->fused_regular = chains * nmin;  // tickets below this: chain predecessor = ticket - chains
      c->fused_chains = chains;
    }
  }

  // L2 prefetch of the 16-byte aligned superset of n keys at p (bulk async)
  static __device__ __forceinline__ void prefetch_keys_l2(const K* p, uint32_t n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p), a0 = a & ~(uintptr_t)15;
    const uint32_t bytes = (uint32_t)(((a + (uintptr_t)n * sizeof(K) + 15) & ~(uintptr_t)15) - a0);
    if (bytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(bytes) : "memory");
  }

  // exact stable re-rank of the sub-bucket [lst, lst+cb) of the grouped keys
  // by one warp (full keys, slot as tie-break), written to out[lst + rank]
  static __device__ DFR_COLD void fused_fix(uint32_t keys_a, uint32_t lst, uint32_t cb, K* out) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t y = lst + lane; y < lst + cb; y += 32) {
      const K ky = ldsk<K>(keys_a + sizeof(K) * y);
      uint32_t r = 0;
      for (uint32_t z = lst; z < lst + cb; ++z) {
        const K kz = ldsk<K>(keys_a + sizeof(K) * z);
        r += (kz < ky) || (kz == ky && z < y);
      }
      out[lst + r] = ky;
    }
  }

  // exclusive scan of one value per thread over NW warps with one barrier;
  // s_warp must not be reused before the caller's next barrier
  template <int NW = FNW>
  static __device__ __forceinline__ uint32_t fused_scan(uint32_t v, uint32_t* s_warp) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    uint32_t pre = 0;
#pragma unroll
    for (int q = 0; q < NW / 4; ++q) {
      const uint4 a = reinterpret_cast<const uint4*>(s_warp)[q];
      const uint32_t t[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) pre += (uint32_t)(4 * q + e) < w ? t[e] : 0u;
    }
    return pre + x - v;
  }

  // Compile-time geometry of the fused pass: a level-0 group of p = 3 digits
  // ends on the top digit, so its lowest digit is D - 3.
  static constexpr int F_LOW = (int)sizeof(K) - 3, F_DG = (int)sizeof(K) - 1;
  static constexpr int F_SBS = 8 * F_LOW - FSB;  // sub-bucket bits (key >> F_SBS) & 3
  static __device__ __forceinline__ uint32_t f_sub(K k) {
    return (uint32_t)(k >> (8 * F_DG)) << FSB | ((uint32_t)(k >> F_SBS) & ((1u << FSB) - 1));
  }
  // 16-bit composite of the bits below the sub-bucket bits.  u64: the next 16
  // bits scaled onto the normal fp16 values (lossy: ties are fixed up); u32:
  // all 6 remaining bits and the slot (< 256) -- exact and unique.
  static __device__ __forceinline__ uint32_t f_comp(K k, uint32_t slot) {
    if constexpr (sizeof(K) == 8) {
      // the 16 bits scaled onto the 61440 normal fp16 values of both signs, in
      // order (negatives first: -0x7bff .. -0x0400, then 0x0400 .. 0x7bff)
      const uint32_t v = (((uint32_t)(k >> (F_SBS - 16)) & 0xffffu) * 61440u) >> 16;
      return v < 30720u ? (0x8000u | (0x0400u + 30719u - v)) : (0x0400u + v - 30720u);
    } else {
      return 0x0400u + (((uint32_t)k & 63u) << 8 | slot);
    }
  }

  // ---- the fused pass with exact composites.  Inside a tile (one s-run) the
  // keys are split by (hi, the top GSB remaining bits) into sub-buckets, which
  // are already in order; inside a sub-bucket every key's remaining bits sit
  // at the top of a composite c = (k << G_CSH) | sb << 13 | slot (the slot, the
  // key's arrival rank in its sub-bucket, breaks ties between equal keys), so
  // the composites of a sub-bucket are distinct and ordered exactly as the
  // (key, slot) pairs: a key's rank is the number of sub-bucket composites
  // below its own -- no lossy compare, no tie fix-up.  The composite also
  // carries everything the write-out needs to rebuild the key (sb gives hi and
  // the sub-bucket bits; the tile's (mid, lo) bits are common), so one array
  // holds the tile: composites at their slot positions while ranking, then at
  // their final positions for the write-out.
  static constexpr int GSB = DFR_FUSED_SB;                  // sub-bucket bits below the group
  static constexpr int GNS = 256 << GSB;                    // sub-buckets per tile
  static constexpr int G_SBS = 8 * F_LOW - GSB;             // lowest sub-bucket bit
  static constexpr int G_CSH = 8 * (int)sizeof(K) - G_SBS;  // remaining bits -> top of c
  static_assert(G_CSH >= 13 + 8 + GSB, "composite fields: slot (13 bits) and sub-bucket");
  static_assert(GNS / 256 == 16 || GNS / 256 == 8 || GNS / 256 == 4, "4, 8 or 16 sub-buckets per digit value");
  static constexpr int GNT = DFR_FUSED_NT;                // threads per fused CTA (256 or 512)
  static constexpr int GKPT = (FT_MAX + GNT - 1) / GNT;   // keys per thread
  static constexpr int GMINB = GNT >= 512 ? 2 : 3;        // fused CTAs per SM
  static_assert(GNT % 128 == 0 && GNT / 32 <= 16, "fused CTA size");
  struct FX {                                              // shared-memory layout, byte offsets
    static constexpr int KEYS = 0;                         // K[FT_MAX + 4] composites (4 pad: rank loads)
    static constexpr int POS = KEYS + (FT_MAX + 4) * (int)sizeof(K);  // u16[FT_MAX]: final tile position
    static constexpr int CNT = POS + FT_MAX * 2;           // u32[2][GNS] (two tiles)
    static constexpr int BDESC = CNT + 2 * GNS * 4;        // u32[GNS]: start | compare count << 13
    static constexpr int SDST = BDESC + GNS * 4;           // int[256]
    static constexpr int WARP = SDST + 1024;               // u32[16]
    static constexpr int MISC = WARP + 64;                 // u32[16]: tickets; [8..11] the two tiles' prefixes
#if DFR_FRANK_SB
    static constexpr int WL = MISC + 64;                   // u32[FT_MAX / 5 + 5]: sub-buckets of > DFR_FRANK_MA keys (start | count << 13)
    static constexpr int BYTES = WL + (FT_MAX / 5 + 5) * 4;
#else
    static constexpr int BYTES = MISC + 64;
#endif
  };
  static_assert(FX::CNT % 16 == 0 && FX::BDESC % 16 == 0 && FX::MISC % 16 == 0, "fused smem alignment");
  static_assert(FX::BYTES + 1024 <= 233472 / 3, "three exact-composite fused CTAs per SM");
  static_assert(DFR_FRANK_MA >= 4 && DFR_FRANK_MA <= 8, "work list capacity FT_MAX / 5; ranks branch-free up to 8 keys");
  static constexpr size_t SMEM_FUSED_X = FX::BYTES;
  static constexpr K G_PRE = (K(1) << (8 * F_DG)) - (K(1) << (8 * F_LOW));  // the (mid, lo) bits
  static __device__ __forceinline__ uint32_t g_sub(K k) {
    return (uint32_t)(k >> (8 * F_DG)) << GSB | ((uint32_t)(k >> G_SBS) & ((1u << GSB) - 1));
  }
  // u64: the composite is the key rotated left by G_CSH: the remaining bits
  // on top, the (hi, mid, lo, sub-bucket) bits -- constant in a sub-bucket --
  // below; equal keys tie (checked).  u32: the 5 remaining bits on top, then
  // the sub-bucket and the slot: unique, exact.
  static constexpr bool LOSSY = sizeof(K) == 8;
  static __device__ __forceinline__ K g_comp(K k, uint32_t sb, uint32_t slot) {
    if constexpr (LOSSY)
      return k << G_CSH | k >> (8 * sizeof(K) - G_CSH);
    else
      return k << G_CSH | (K)(sb << 13 | slot);
  }
  static __device__ __forceinline__ uint32_t g_hi(K cpt) {  // the top digit of the key
    if constexpr (LOSSY)
      return (uint32_t)(cpt >> (8 * F_DG - G_SBS)) & 255u;
    else
      return (uint32_t)(cpt >> (13 + GSB)) & 255u;
  }
  static __device__ __forceinline__ K g_key(K cpt, K pre) {
    if constexpr (LOSSY) {
      return cpt >> G_CSH | cpt << (8 * sizeof(K) - G_CSH);
    } else {
      const uint32_t sb = (uint32_t)(cpt >> 13) & (GNS - 1);
      return (K)(sb >> GSB) << (8 * F_DG) | pre | (K)(sb & ((1u << GSB) - 1)) << G_SBS | cpt >> G_CSH;
    }
  }
  // composites in shared memory as two word arrays (u64: top words, then
  // low words; u32: one array), so that the rank loads of top words spread
  // over all 32 banks
  static constexpr int G_WORDS = FT_MAX + 4;  // 4 pad entries: the rank's 4-wide loads
  static __device__ __forceinline__ void st_comp(uint32_t a, uint32_t x, K c) {
    sts32(a + 4 * x, (uint32_t)(c >> (8 * sizeof(K) - 32)));
    if constexpr (sizeof(K) == 8) sts32(a + 4 * (G_WORDS + x), (uint32_t)c);
  }
  static __device__ __forceinline__ K ld_comp(uint32_t a, uint32_t x) {
    if constexpr (sizeof(K) == 8)
      return (K)lds32(a + 4 * x) << 32 | lds32(a + 4 * (G_WORDS + x));
    else
      return (K)lds32(a + 4 * x);
  }
  // exact ranks of every key of the tile in a small sub-bucket: full
  // composites, the slot breaking ties (the tile had tied top words)
  // (inlined: the register arrays must not be passed by address)
  static __device__ __forceinline__ void fused_exact(const uint32_t (&ds)[GKPT], uint32_t keys_a, uint32_t pos_a) {
#pragma unroll
    for (int m = 0; m < GKPT; ++m) {
      if (ds[m] == ~0u) continue;
      const uint32_t cb = (ds[m] >> 13) & 511u;
      if (!cb) continue;
      const uint32_t x = ds[m] & 8191u, slot = ds[m] >> 22, bl = x - slot;
      const K me = ld_comp(keys_a, x);  // this key's composite, still at its slot position
      uint32_t r = 0;
      for (uint32_t z = 0; z < cb; ++z) {
        const K cz = ld_comp(keys_a, bl + z);
        r += cz < me || (cz == me && z < slot);
      }
      sts16(pos_a + 2 * x, bl + r);
    }
  }

  // the same from the sub-bucket descriptors (start | count << 13; count 0: a
  // large bucket, kept in slot order), 8 threads per sub-bucket
  static __device__ DFR_COLD void fused_exact_sb(const uint32_t* bdesc, uint32_t keys_a, uint32_t pos_a) {
    for (uint32_t e = threadIdx.x; e < (uint32_t)GNS * 8; e += GNT) {
      const uint32_t bd = bdesc[e >> 3], cb = bd >> 13, bl = bd & 8191u;
      for (uint32_t s = e & 7u; s < cb; s += 8) {
        const K me = ld_comp(keys_a, bl + s);
        uint32_t r = 0;
        for (uint32_t z = 0; z < cb; ++z) {
          const K cz = ld_comp(keys_a, bl + z);
          r += cz < me || (cz == me && z < s);
        }
        sts16(pos_a + 2 * (bl + s), bl + r);
      }
    }
  }

  static __device__ void fused(const Params<K>& P, uint32_t* sm) {
    constexpr int SBW = 8 + GSB;  // ds: sub-bucket | slot << SBW
    Ctl* c = P.ctl;
    if (!*(volatile uint32_t*)&c->fused_ok) return;
    const Seg sv = P.segq[c->cur][0];
    const uint32_t ntiles = c->fused_tiles;
    constexpr int j = 2;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t nd = P.n_d;
    char* base = reinterpret_cast<char*>(sm);
    uint32_t* bdesc = reinterpret_cast<uint32_t*>(base + FX::BDESC);
    int* s_dst = reinterpret_cast<int*>(base + FX::SDST);
    uint32_t* s_warp = reinterpret_cast<uint32_t*>(base + FX::WARP);
    uint32_t* misc = reinterpret_cast<uint32_t*>(base + FX::MISC);
    const uint32_t keys_a = smem_u32(base + FX::KEYS), cnt0_a = smem_u32(base + FX::CNT),
                   pos_a = smem_u32(base + FX::POS);
    uint32_t* status = P.status + (size_t)j * P.status_stride;
    const K* src = P.kbuf(route_src(sv, j)) + sv.start;
    K* const out = P.A;
#if DFR_FRANK_SB
    const uint32_t wl_a = smem_u32(base + FX::WL);
#endif
    const uint32_t d = threadIdx.x;  // layout, look-back: one thread per digit value (d < 256)
    const bool dig = d < 256;
    const uint32_t brow = dig ? P.hist[(size_t)(sv.hist_off + j) * 256 + d] : 0u;  // bucket offsets of the top digit
    const uint32_t kofs = w * 32 * GKPT + lane;  // this thread's first key of a tile
    auto cnt_of = [&](uint32_t cb) { return reinterpret_cast<uint32_t*>(base + FX::CNT + cb * GNS * 4); };
    K key[GKPT];
    uint32_t ds[GKPT];  // sub-bucket | slot << SBW; then slot position | compare count << 13 | slot << 22;
                        // then final position; ~0u: no key
    // keys of tile tt -> registers, with the tile's chain link and chain
    auto load_keys = [&](uint32_t tt, uint32_t& prev, uint32_t& chn) -> uint32_t {
      uint32_t ln = 0;
      if (tt < ntiles) {
        const uint4 td = P.ftiles[tt];
        ln = td.y;
        prev = td.z;
        chn = td.w;
        const K* p = src + td.x + kofs;
        const int lim = (int)ln - (int)kofs;
#pragma unroll
        for (int m = 0; m < GKPT; ++m) key[m] = m * 32 < lim ? p[m * 32] : K(0);
      }
      return ln;
    };
    // sub-bucket and slot of every key (counter set cb); the tile's (mid, lo) bits
    auto count_keys = [&](uint32_t ln, uint32_t cb) {
      const int lim = (int)ln - (int)kofs;
      const uint32_t ca = cnt0_a + cb * GNS * 4;
#pragma unroll
      for (int m = 0; m < GKPT; ++m) {
        ds[m] = ~0u;
        if (m * 32 < lim) {
          const uint32_t sb = g_sub(key[m]);
          ds[m] = sb | atom_add_shared(ca + 4 * sb, 1u) << SBW;
        }
      }
      if (threadIdx.x == 0 && ln) *reinterpret_cast<K*>(misc + 8 + 2 * cb) = key[0] & G_PRE;
    };
    auto digit_counts = [&](uint32_t cb, uint32_t (&cs)[GNS / 256]) {
      const uint4* p = reinterpret_cast<const uint4*>(cnt_of(cb)) + (GNS / 1024) * d;
#pragma unroll
      for (int r = 0; r < GNS / 1024; ++r) {
        const uint4 v = dig ? p[r] : make_uint4(0, 0, 0, 0);
        cs[4 * r] = v.x;
        cs[4 * r + 1] = v.y;
        cs[4 * r + 2] = v.z;
        cs[4 * r + 3] = v.w;
      }
    };
    // the tile aggregate of digit d, published as soon as the counts are
    // complete; the first tile of a chain publishes its inclusive prefix
    // (the chain's base + its count) at once
    const uint32_t* jbase = P.J + 4096;
    const uint32_t regular = c->fused_regular, chains = c->fused_chains;
    auto publish = [&](uint32_t tt, uint32_t cb, uint32_t prev, uint32_t chn) {
      if (tt < ntiles && dig) {
        uint32_t cs[GNS / 256];
        digit_counts(cb, cs);
        uint32_t cdd = 0;
#pragma unroll
        for (int r = 0; r < GNS / 256; ++r) cdd += cs[r];
        st_relaxed(status + (size_t)tt * 256 + d,
                   prev == ~0u ? (FLAG_INC | ((jbase[chn * 256 + d] + cdd) & VAL_MASK)) : (FLAG_AGG | cdd));
      }
    };
    auto zero_counts = [&](uint32_t cb) {
      if (!dig) return;
      uint4* p = reinterpret_cast<uint4*>(cnt_of(cb)) + (GNS / 1024) * d;
#pragma unroll
      for (int r = 0; r < GNS / 1024; ++r) p[r] = make_uint4(0, 0, 0, 0);
    };
    zero_counts(0);
    zero_counts(1);
    // tickets are claimed one tile ahead, so that a tile's keys are in L2
    // (bulk prefetch at its claim) by the time they are loaded
    if (d == 0) {
      misc[0] = atomicAdd(&c->fticket, 1u);
      misc[1] = atomicAdd(&c->fticket, 1u);
      if (misc[1] < ntiles) {
        const uint4 tn = P.ftiles[misc[1]];
        prefetch_keys_l2(src + tn.x, tn.y);
      }
    }
    __syncthreads();
    uint32_t t = misc[0], tq = misc[1], cur = 0, tprev = ~0u, tch = 0;
#ifdef DFR_FPROF
    unsigned long long fp_[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long fp_last_ = clock64();
#endif
    uint32_t len = load_keys(t, tprev, tch);
    count_keys(len, 0);
    __syncthreads();
    publish(t, 0, tprev, tch);
    while (t < ntiles) {
      FPROF_MARK(0);  // (the previous tile's tail)
      // ---- layout (thread d: digit value d and its sub-buckets)
      uint32_t cs[GNS / 256];
      digit_counts(cur, cs);
      uint32_t cd = 0;
#pragma unroll
      for (int r = 0; r < GNS / 256; ++r) cd += cs[r];
      const bool small = cd <= nd;
      if (d == 0) misc[3] = 0;  // the tile's tie check (the last tile's was read before this barrier)
#if DFR_FRANK_SB
      // sub-buckets of > DFR_FRANK_MA (4) keys are ranked from a work list: their count rides
      // in the scan's upper half (both totals < 2^16)
      uint32_t nl = 0;
#pragma unroll
      for (int r = 0; r < GNS / 256; ++r) nl += small && cs[r] > (uint32_t)DFR_FRANK_MA;
      const uint32_t ex = fused_scan<GNT / 32>(cd | nl << 16, s_warp);
      const uint32_t lst = ex & 0xffffu;  // the bucket's first tile position
      if (d == 255) misc[4] = (ex >> 16) + nl;
      {
        uint32_t so = lst, wo = wl_a + 4 * (ex >> 16), bd[GNS / 256];
#pragma unroll
        for (int r = 0; r < GNS / 256; ++r) {
          bd[r] = so | (small ? cs[r] : 0u) << 13;  // a large bucket stays in slot order
          if (small && cs[r] > (uint32_t)DFR_FRANK_MA) {
            sts32(wo, bd[r]);
            wo += 4;
          }
          so += cs[r];
        }
        if (!small)  // (rare) written in slot order
          for (uint32_t x = lst; x < lst + cd; ++x) sts16(pos_a + 2 * x, x);
#else
      const uint32_t lst = fused_scan<GNT / 32>(cd, s_warp);  // the bucket's first tile position
      {
        uint32_t so = lst, bd[GNS / 256];
#pragma unroll
        for (int r = 0; r < GNS / 256; ++r) {
          bd[r] = so | ((small && cs[r] >= 2) ? cs[r] : 0u) << 13;
          so += cs[r];
        }
#endif
        uint4* bp = reinterpret_cast<uint4*>(bdesc) + (GNS / 1024) * d;
#pragma unroll
        for (int r = 0; r < GNS / 1024; ++r)
          if (dig) bp[r] = make_uint4(bd[4 * r], bd[4 * r + 1], bd[4 * r + 2], bd[4 * r + 3]);
      }
      __syncthreads();
      FPROF_MARK(1);
      // the ticket after the next one (consumed after the ranks: the atomic is
      // in flight meanwhile)
      uint32_t tw = 0;
      if (d == 0) tw = atomicAdd(&c->fticket, 1u);
      // ---- composites at their slot positions
#pragma unroll
      for (int m = 0; m < GKPT; ++m) {
        if (ds[m] != ~0u) {
          const uint32_t sb = ds[m] & (GNS - 1), slot = ds[m] >> SBW;
          const uint32_t bd = bdesc[sb];
          const uint32_t x = (bd & 8191u) + slot, cb = bd >> 13;
          key[m] = g_comp(key[m], sb, slot);
          st_comp(keys_a, x, key[m]);
#if !DFR_FRANK_SB
          ds[m] = x | cb << 13 | (cb ? slot << 22 : 0u);
#endif
        }
      }
      __syncthreads();
      FPROF_MARK(2);
#if DFR_FRANK_SB
      // ---- ranks, one thread per sub-bucket: the composites' top words (u32:
      // the composites) of a sub-bucket of 2..MA (4) keys are ranked against one
      // another branch-free (words past its end predicated off, read as ~0u:
      // never below a key's): every pair is compared once, the loser of a
      // compare moving up and the other down from the slot order, so equal
      // words keep slot order; equal words raise the tie flag (u64: equal
      // keys, or keys that differ only below the top word: the tile is then
      // re-ranked on the full composites).  Longer sub-buckets come from the
      // work list, DFR_FRANK_BL (2) threads each, every thread ranking 4 keys
      // of a group of 8 against the same 8 loaded words; a tie there makes the
      // sum of (rank - slot) over the sub-bucket non-zero
#if DFR_FLB_EARLY
      // the look-back's first round trip, in flight during the ranks (an
      // aggregate read early is still this predecessor's aggregate)
      uint32_t lbe[DFR_FLB];
      if (dig && tprev != ~0u && t < regular) {
#pragma unroll
        for (int i = 0; i < DFR_FLB; ++i) {
          const int r = (int)tprev - (int)chains * i;
          lbe[i] = r >= 0 ? ld_relaxed(status + (size_t)r * 256 + d) : FLAG_INC;
        }
      }
#endif
#if DFR_FLOAD_EARLY
      // the composites are in shared memory: the registers take the next tile's keys
      const uint32_t tn = tq;
      uint32_t nprev = ~0u, nchn = 0;
      const uint32_t lenn = load_keys(tn, nprev, nchn);
#endif
      {
        bool tie = false;
        constexpr int NB = GNS / GNT >= DFR_FRANK_NB ? DFR_FRANK_NB : GNS / GNT;  // sub-buckets per batch of loads
#pragma unroll
        for (int i0 = 0; i0 < GNS / GNT; i0 += NB) {
          constexpr int MA = DFR_FRANK_MA;  // longest sub-bucket ranked here
          uint32_t bd[NB], h[NB][MA];
#pragma unroll
          for (int q = 0; q < NB; ++q) bd[q] = bdesc[(i0 + q) * GNT + threadIdx.x];
#pragma unroll
          for (int q = 0; q < NB; ++q) {
            const uint32_t cb = bd[q] >> 13, a0 = keys_a + 4 * (bd[q] & 8191u);
#pragma unroll
            for (int i = 0; i < MA; ++i) {  // word i: 2 <= cb <= MA and i < cb
              const uint32_t lo = i < 1 ? 2u : (uint32_t)i + 1u;
              h[q][i] = lds32_if_le(a0 + 4 * i, cb - lo, (uint32_t)MA - lo);
            }
          }
#pragma unroll
          for (int q = 0; q < NB; ++q) {
            const uint32_t cb = bd[q] >> 13, bl = bd[q] & 8191u, p0 = pos_a + 2 * bl;
            uint32_t r[MA];
#pragma unroll
            for (int i = 0; i < MA; ++i) r[i] = bl + i;
#pragma unroll
            for (int i = 0; i < MA; ++i)
#pragma unroll
              for (int k = i + 1; k < MA; ++k) {  // equal words keep slot order
                const uint32_t l = h[q][k] < h[q][i];
                r[i] += l;
                r[k] -= l;
              }
#pragma unroll
            for (int i = 0; i < MA; ++i) sts16_if_le(p0 + 2 * i, r[i], cb - (i + 1), (uint32_t)(MA - (i + 1)));
            if (LOSSY) {  // equal words among the sub-bucket's own (the pads are equal to one another)
#pragma unroll
              for (int k = 1; k < MA; ++k) {
                bool e = false;
#pragma unroll
                for (int i = 0; i < k; ++i) e |= h[q][i] == h[q][k];
                tie |= e && cb - (k + 1) <= (uint32_t)(MA - (k + 1));
              }
            }
          }
        }
        const uint32_t nwl = misc[4];
        int dev = 0;  // sum of (rank - slot): 0 over a sub-bucket without equal words
        // BL threads per long sub-bucket, each ranking keys s, s + BL, ... of a
        // group of 8 against the same 8 loaded words
        constexpr uint32_t BL = DFR_FRANK_BL, KPL = 8 / BL;
        static_assert(BL == 1 || BL == 2 || BL == 4 || BL == 8, "threads per long sub-bucket");
#pragma unroll 1
        for (uint32_t e = threadIdx.x; e < nwl * BL; e += GNT) {
          const uint32_t bd = lds32(wl_a + 4 * (e / BL));
          const uint32_t cb = bd >> 13, bl = bd & 8191u, a0 = keys_a + 4 * bl;
#pragma unroll 1
          for (uint32_t s = e % BL; s < cb; s += 8) {
            uint32_t me[KPL], r[KPL];
#pragma unroll
            for (uint32_t k = 0; k < KPL; ++k) {
              me[k] = lds32_if_lt(a0 + 4 * (s + k * BL), s + k * BL, cb);
              r[k] = 0;
            }
#pragma unroll 1
            for (uint32_t z = 0; z < cb; z += 8) {  // 8 words per round trip, the ones past the end read as ~0u
              uint32_t hz[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) hz[q] = lds32_if_lt(a0 + 4 * (z + q), z + q, cb);
#pragma unroll
              for (int q = 0; q < 8; ++q)
#pragma unroll
                for (uint32_t k = 0; k < KPL; ++k) r[k] += hz[q] < me[k];
            }
#pragma unroll
            for (uint32_t k = 0; k < KPL; ++k)
              if (s + k * BL < cb) {
                sts16(pos_a + 2 * (bl + s + k * BL), bl + r[k]);
                dev += (int)r[k] - (int)(s + k * BL);
              }
          }
        }
        if (LOSSY) {  // the threads of a sub-bucket are adjacent lanes
          if (BL >= 2) dev += __shfl_xor_sync(0xffffffffu, dev, 1);
          if (BL >= 4) dev += __shfl_xor_sync(0xffffffffu, dev, 2);
          if (BL >= 8) dev += __shfl_xor_sync(0xffffffffu, dev, 4);
          tie |= dev != 0;
        }
        if (LOSSY && tie) misc[3] = 1u;
      }
      if (d == 0) {  // the claimed ticket: prefetch its keys into L2
        misc[1] = tw;
        if (tw < ntiles) {
          const uint4 tnw = P.ftiles[tw];
          prefetch_keys_l2(src + tnw.x, tnw.y);
        }
      }
#else
      // ---- ranks: the number of smaller composites in the sub-bucket.  u64:
      // the top words of equal keys (or, with odds 2^-32 per pair, of keys
      // that differ only in their low bits) tie and share the lower rank; the
      // sum over the tile of (rank - slot) is then negative, and the tile is
      // re-ranked exactly on the full composites (slot as the tie-break)
      int dev = 0;
#pragma unroll
      for (int m = 0; m < GKPT; ++m) {
        if (ds[m] != ~0u) {
          const uint32_t cb = (ds[m] >> 13) & 511u;
          uint32_t pos = ds[m] & 8191u;
          if (cb) {  // cb >= 2: the number of smaller top words among the
            // sub-bucket's composites (u32: the whole composite), four loads
            // at once masked by the sub-bucket size
            const uint32_t slot = ds[m] >> 22, bl = pos - slot;
            const uint32_t a0 = keys_a + 4 * bl;  // the top words (u32: the composites)
            const uint32_t me = (uint32_t)(key[m] >> (8 * sizeof(K) - 32));
            // (words past the sub-bucket: predicated off, read as ~0u)
            const uint32_t h0 = lds32(a0), h1 = lds32(a0 + 4), h2 = lds32_if(a0 + 8, cb > 2),
                           h3 = lds32_if(a0 + 12, cb > 3);
            const uint32_t r = (h0 < me) + (h1 < me) + (h2 < me) + (h3 < me);
            uint32_t rr = r;
#if DFR_FRANK8
            if (cb > 4) {  // words 4..7 in one round trip; a longer sub-bucket loops (rare)
              const uint32_t h4 = lds32(a0 + 16), h5 = lds32_if(a0 + 20, cb > 5),
                             h6 = lds32_if(a0 + 24, cb > 6), h7 = lds32_if(a0 + 28, cb > 7);
              rr += (h4 < me) + (h5 < me) + (h6 < me) + (h7 < me);
#pragma unroll 1
              for (uint32_t z = 8; z < cb; ++z) rr += lds32(a0 + 4 * z) < me;
            }
#else
#pragma unroll 1
            for (uint32_t z = 4; z < cb; ++z) rr += lds32(a0 + 4 * z) < me;
#endif
            pos = bl + rr;
            if (LOSSY) dev += (int)rr - (int)slot;  // sums to 0 over a sub-bucket without ties
          }
          sts16(pos_a + 2 * (ds[m] & 8191u), pos);
        }
      }
      if (LOSSY) {
#pragma unroll
        for (int o = 16; o; o >>= 1) dev += __shfl_xor_sync(0xffffffffu, dev, o);
        if (lane == 0 && dev) atomicAdd(reinterpret_cast<int*>(misc + 3), dev);
      }
      if (d == 0) {  // the claimed ticket: prefetch its keys into L2
        misc[1] = tw;
        if (tw < ntiles) {
          const uint4 tnw = P.ftiles[tw];
          prefetch_keys_l2(src + tnw.x, tnw.y);
        }
      }
#endif
      __syncthreads();  // positions and the tie check complete
      FPROF_MARK(3);
      if (LOSSY && misc[3] != 0) {  // (rare) tied top words
#if DFR_FRANK_SB
        fused_exact_sb(bdesc, keys_a, pos_a);
#else
        fused_exact(ds, keys_a, pos_a);
#endif
        __syncthreads();
      }
      // ---- the next tile's keys load while the look-back runs
#if DFR_FRANK_SB && DFR_FLOAD_EARLY
      tq = misc[1];
#else
      const uint32_t tn = tq;
      tq = misc[1];
      uint32_t nprev = ~0u, nchn = 0;
      const uint32_t lenn = load_keys(tn, nprev, nchn);
#endif
      // ---- decoupled look-back along this tile's chain (thread d, digit d)
      if (dig) {
        uint32_t excl;
        if (tprev == ~0u) {
          excl = jbase[tch * 256 + d];  // first tile of its chain: published with the counts
        } else {
          excl = 0;
          if (t < regular) {
            // the regular part of the ticket order: the chain predecessors are
            // t - chains, t - 2 chains, ...: DFR_FLB of them per round trip (the
            // chain's first tile is inclusive, so the walk stops there)
            constexpr int LB = DFR_FLB;
            int tt = (int)tprev;
            uint32_t lbv[LB];
#if DFR_FLB_EARLY
            bool first = true;
#endif
            while (true) {
#if DFR_FLB_EARLY
              if (first) {
#pragma unroll
                for (int i = 0; i < LB; ++i) lbv[i] = lbe[i];
                first = false;
              } else
#endif
#pragma unroll
              for (int i = 0; i < LB; ++i) {
                const int r = tt - (int)chains * i;
                lbv[i] = r >= 0 ? ld_relaxed(status + (size_t)r * 256 + d) : FLAG_INC;
              }
              int q = 0;
              bool done = false;
#pragma unroll
              for (; q < LB; ++q) {
                if ((lbv[q] >> 30) == 0) break;
                excl += lbv[q] & VAL_MASK;
                if (lbv[q] & FLAG_INC) {
                  done = true;
                  break;
                }
              }
              if (done) break;
#ifdef DFR_LB_STATS
              atomicAdd(&g_lb_stats[q == 0 ? 1 : 0], 1ull);
#endif
              if (q == 0) __nanosleep(DFR_LB_SLEEP);
              tt -= (int)chains * q;
            }
          } else {  // the tail of the order: follow the chain links
            uint32_t pt = tprev;
            while (true) {
              const uint32_t v = ld_relaxed(status + (size_t)pt * 256 + d);
              if ((v >> 30) == 0) {  // not published yet
                __nanosleep(DFR_LB_SLEEP);
                continue;
              }
              excl += v & VAL_MASK;
              if (v & FLAG_INC) break;
              pt = P.ftiles[pt].z;
            }
          }
#ifdef DFR_LB_STATS
          if (d == 0) atomicAdd(&g_lb_stats[2], 1ull);
#endif
          st_relaxed(status + (size_t)t * 256 + d, FLAG_INC | ((excl + cd) & VAL_MASK));
        }
        excl &= VAL_MASK;  // mod 2^30 (n <= 2^30): exact for a non-empty bucket
        const uint32_t gstart = sv.start + brow + excl;  // global index of bucket (d, this s-run)
        s_dst[d] = (int)(gstart - lst);
        if (!small) push_bucket(P, sv, 0u, gstart, cd);  // written to A below (Alg. 4 l.11)
      }
      __syncthreads();  // s_dst complete
      FPROF_MARK(4);
      // ---- this tile in final order: one linear pass, the keys rebuilt from
      // their composites
      {
        const K pre = *reinterpret_cast<const K*>(misc + 8 + 2 * cur);
#pragma unroll FWO_UNROLL
        for (uint32_t x = threadIdx.x; x < len; x += GNT) {
          const K cpt = ld_comp(keys_a, x);
          out[(uint32_t)s_dst[g_hi(cpt)] + lds16(pos_a + 2 * x)] = g_key(cpt, pre);
        }
      }
      // the next tile's keys have arrived meanwhile: count them, publish its aggregate
      count_keys(lenn, cur ^ 1u);
      __syncthreads();
      publish(tn, cur ^ 1u, nprev, nchn);
      FPROF_MARK(5);
#ifdef DFR_FPROF
      if (threadIdx.x == 0) fp_[8]++;
#endif
      // this tile's counters are read by no one any more
      zero_counts(cur);
      t = tn;
      len = lenn;
      tprev = nprev;
      tch = nchn;
      cur ^= 1u;
      FPROF_MARK(6);
    }
#ifdef DFR_FPROF
    if (threadIdx.x == 0)
      for (int k = 0; k < 10; ++k) atomicAdd(&g_fprof[k], fp_[k]);
#endif
  }

  // --------------------------------------------------------- mid (fast)
  // Keys-only buckets N_d < len <= C (Alg. 4 l.11 "recurse on the large
  // bucket"), one bucket per CTA iteration, in rounds.  Round r takes the
  // buckets queued for it and runs Alg. 4 on each with p' = 1 (est(len) = 1
  // for len <= N_d * 256): a deal on its highest non-constant digit hi, split
  // by 2 more bits into sub-buckets as in the fused pass, and every digit
  // bucket of <= N_d keys sorted on the spot (ranks by 16-bit composites,
  // ties re-ranked exactly), the keys written straight to their final place
  // in A.  A digit bucket > N_d is written in slot order and queued for round
  // r + 1 with the next digit (its keys are all in A by then); digits exhausted
  // (hi < 0, or a digit-0 bucket) means equal keys: nothing to sort.
  // (Pairs keep the shared-memory recursion of mid(): stability needs the
  // input order inside a bucket.)
  static __device__ void midf(const Params<K>& P, uint32_t* sm, int round) {
    constexpr bool WIDE = sizeof(K) == 8;
    Ctl* c = P.ctl;
    const MidE* q = (round & 1) ? P.midq2 : P.midq;
    MidE* nq = (round & 1) ? P.midq : P.midq2;
    const uint32_t total = min(round == 0 ? c->mid_count : c->mround[round], P.mid_cap);
    if (total == 0) return;
    uint32_t* nqc = &c->mround[round + 1];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t nd = P.n_d;
    char* base = reinterpret_cast<char*>(sm);
    uint32_t* bdesc = reinterpret_cast<uint32_t*>(base + FS::BDESC);
    uint32_t* flag = reinterpret_cast<uint32_t*>(base + FS::FLAG);
    uint32_t* s_warp = reinterpret_cast<uint32_t*>(base + FS::WARP);
    uint32_t* misc = reinterpret_cast<uint32_t*>(base + FS::MISC);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(base + FS::CNT);
    const uint32_t keys_a = smem_u32(base + FS::KEYS), cmp_a = smem_u32(base + FS::CMP),
                   cnt_a = smem_u32(cnt);
    const uint32_t d = threadIdx.x;
    const uint32_t kofs = w * 32 * FKPT + lane;
    reinterpret_cast<uint4*>(cnt)[d] = make_uint4(0, 0, 0, 0);
    if (d < FNS / 32) flag[d] = 0;
    if (d == 0) {
      misc[5] = 0;
      *reinterpret_cast<unsigned long long*>(misc + 6) = 0ull;
    }
    __syncthreads();
    // the keys of the next bucket are loaded while this one is ranked
    K key[FKPT];
    auto load = [&](const MidE& m) {
      if (m.hi < 0) return;  // (copied, not loaded)
      const K* p = P.kbuf(m.buf) + m.start + kofs;
      const int lim = (int)m.len - (int)kofs;
#pragma unroll
      for (int i = 0; i < FKPT; ++i) key[i] = i * 32 < lim ? p[i * 32] : K(0);
    };
    uint32_t e = blockIdx.x;
    MidE me = {0, 0, -1, 0};
    if (e < total) {
      me = q[e];
      load(me);
    }
    for (; e < total;) {
      const uint32_t en = e + gridDim.x;
      MidE mn = {0, 0, -1, 0};
      if (en < total) mn = q[en];
      const uint32_t len = me.len;
      const K* X = P.kbuf(me.buf) + me.start;
      K* const out = P.A + me.start;
      auto advance = [&]() {
        e = en;
        me = mn;
        load(me);
      };
      if (me.hi < 0) {  // digits exhausted: equal keys, sorted (Alg. 2 l.17-18)
        if (me.buf) coop_copy(out, X, len, threadIdx.x, THREADS);
        advance();
        continue;
      }
      // the bucket's highest non-constant digit (OR of k ^ k0)
      {
        const int lim = (int)len - (int)kofs;
        const K k0 = X[0];
#pragma unroll
        for (int m = 0; m < FKPT; ++m)
          if (!(m * 32 < lim)) key[m] = k0;
        K acc = 0;
#pragma unroll
        for (int m = 0; m < FKPT; ++m) acc |= key[m] ^ k0;
        unsigned long long a = (unsigned long long)acc;
#pragma unroll
        for (int o = 16; o; o >>= 1) a |= __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0 && a) atomicOr(reinterpret_cast<unsigned long long*>(misc + 6), a);
      }
      __syncthreads();
      const unsigned long long bdiff = *reinterpret_cast<volatile unsigned long long*>(misc + 6);
      const int dg = highest_nonconst(bdiff, me.hi);
      __syncthreads();  // every thread has read it
      if (d == 0) *reinterpret_cast<unsigned long long*>(misc + 6) = 0ull;
      if (dg < 0) {  // all keys equal: sorted (Alg. 2 l.17-18)
        if (me.buf) coop_copy(out, X, len, threadIdx.x, THREADS);
        advance();
        continue;
      }
      const int sbs = 8 * dg - FSB;  // sub-bucket bits (dg >= 1); below them R = sbs bits
      auto sub_of = [&](K k) -> uint32_t {
        return digit_of(k, dg) << FSB | (dg ? ((uint32_t)(k >> sbs) & ((1u << FSB) - 1)) : 0u);
      };
      // 16-bit composite of the bits below the sub-bucket bits: exact (the R
      // bits and the slot) when they fit 14 bits, else the top 16 of them
      // scaled onto the normal fp16 values (ties re-ranked exactly)
      const bool exact = sbs + 8 <= 14;
      auto comp_of = [&](K k, uint32_t slot) -> uint32_t {
        if (exact) return 0x0400u + (((uint32_t)k & ((1u << sbs) - 1)) << 8 | slot);
        const uint32_t v16 = sbs >= 16 ? (uint32_t)(k >> (sbs - 16)) & 0xffffu
                                       : ((uint32_t)k << (16 - sbs)) & 0xffffu;
        const uint32_t v = (v16 * 61440u) >> 16;
        return v < 30720u ? (0x8000u | (0x0400u + 30719u - v)) : (0x0400u + v - 30720u);
      };
      (void)WIDE;
      // ---- sub-bucket and slot of every key
      uint32_t ds[FKPT];
      {
        const int lim = (int)len - (int)kofs;
#pragma unroll
        for (int m = 0; m < FKPT; ++m) {
          ds[m] = ~0u;
          if (m * 32 < lim) {
            const uint32_t sb = sub_of(key[m]);
            uint32_t slot;
            asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(slot) : "r"(cnt_a + 4 * sb) : "memory");
            ds[m] = sb | slot << 10;
          }
        }
      }
      __syncthreads();
      // ---- layout (thread d: digit value d and its sub-buckets)
      const uint4 c4 = reinterpret_cast<const uint4*>(cnt)[d];
      const uint32_t cs[4] = {c4.x, c4.y, c4.z, c4.w};
      const uint32_t cd = c4.x + c4.y + c4.z + c4.w;
      const bool small = cd <= nd && dg > 0;  // a digit-0 bucket holds equal keys
      uint32_t padc = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) padc += (small && cs[r] >= 2) ? (cs[r] + 3) & ~3u : 0u;
      const uint32_t ex = fused_scan(cd | padc << 16, s_warp);
      const uint32_t lst = ex & 0xffffu;
      {
        uint32_t so = lst, co = ex >> 16;
        uint32_t bd[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const uint32_t ng = (small && cs[r] >= 2) ? (cs[r] + 3) >> 2 : 0u;
          bd[r] = (co >> 2) | ng << 11 | so << 18;
          if (ng) sts64(cmp_a + 2 * (co + 4 * ng - 4), 0x7c007c007c007c00ull);
          so += cs[r];
          co += 4 * ng;
        }
        reinterpret_cast<uint4*>(bdesc)[d] = make_uint4(bd[0], bd[1], bd[2], bd[3]);
      }
      if (cd > nd && dg > 0) {  // a large digit bucket: the next round, next digit (Alg. 4 l.11)
        const uint32_t idx = atomicAdd(nqc, 1u);
        if (idx < P.mid_cap) {
          MidE m;
          m.start = me.start + lst;
          m.len = (uint16_t)cd;
          m.hi = (int8_t)(dg - 1);
          m.buf = 0;
          nq[idx] = m;
        } else {
          flag_overflow(c, 64u);
        }
      }
      __syncthreads();
      // ---- keys grouped by sub-bucket, composites of the small ones
#pragma unroll
      for (int m = 0; m < FKPT; ++m) {
        if (ds[m] != ~0u) {
          const uint32_t slot = ds[m] >> 10;
          const uint32_t bd = bdesc[ds[m] & (FNS - 1)];
          const uint32_t x = (bd >> 18) + slot;
          if constexpr (sizeof(K) == 8)
            sts64(keys_a + 8 * x, (unsigned long long)key[m]);
          else
            sts32(keys_a + 4 * x, (uint32_t)key[m]);
          if ((bd >> 11) & 127u) sts16(cmp_a + 2 * (4 * (bd & 2047u) + slot), comp_of(key[m], slot));
        }
      }
      const uint32_t e_cur = e;
      (void)e_cur;
      advance();  // the next bucket's keys in flight during the ranks
      __syncthreads();
      // ---- slot-major ranks; every key to its final place
      int dev = 0;
      for (uint32_t x = threadIdx.x; x < len; x += FNT) {
        const K k = ldsk<K>(keys_a + sizeof(K) * x);
        const uint32_t bd = bdesc[sub_of(k)];
        const uint32_t ng = (bd >> 11) & 127u;
        uint32_t pos = x;
        if (ng) {
          const uint32_t bl = bd >> 18;
          const uint32_t pa = cmp_a + 8 * (bd & 2047u);
          const __half2 me2 = __ushort_as_half2_pair(lds16(pa + 2 * (x - bl)));
          __half2 acc = __float2half2_rn(0.f);
          for (uint32_t g = 0; g < ng; ++g) {
            const uint2 v = lds64v(pa + 8 * g);
            acc = __hadd2(acc, __hlt2(u2h2(v.x), me2));
            acc = __hadd2(acc, __hlt2(u2h2(v.y), me2));
          }
          pos = bl + (uint32_t)__half2ushort_rz(__hadd(__low2half(acc), __high2half(acc)));
          dev += (int)pos - (int)x;
        }
        out[pos] = k;
      }
      if (!exact) {
#pragma unroll
        for (int o = 16; o; o >>= 1) dev += __shfl_xor_sync(0xffffffffu, dev, o);
        if (lane == 0 && dev) atomicAdd(reinterpret_cast<int*>(misc + 5), dev);
      }
      __syncthreads();
      const int tie_sum = *reinterpret_cast<volatile int*>(misc + 5);
      __syncthreads();  // every thread has read it
      if (d == 0) misc[5] = 0;
      if (!exact && tie_sum != 0) {  // (rare) tied composites: re-rank those sub-buckets exactly
        uint32_t bad = 0;
        {
          const uint4 b4 = reinterpret_cast<const uint4*>(bdesc)[d];
          const uint32_t bds[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (small && cs[r] >= 2) {
              const uint32_t ca = cmp_a + 8 * (bds[r] & 2047u);
              bool eq = false;
              for (uint32_t y = 0; y + 1 < cs[r]; ++y) {
                const uint32_t a = lds16(ca + 2 * y);
                for (uint32_t z = y + 1; z < cs[r]; ++z) eq |= lds16(ca + 2 * z) == a;
              }
              bad |= (uint32_t)eq << r;
            }
        }
        if (bad) atomicOr(&flag[d >> 3], bad << (4 * (d & 7)));
        __syncthreads();
        for (uint32_t fw = w; fw < FNS / 32; fw += FNW) {
          uint32_t bits = flag[fw];
          while (bits) {
            const uint32_t sb = fw * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            fused_fix(keys_a, bdesc[sb] >> 18, cnt[sb], out);
          }
        }
        __syncthreads();
        if (d < FNS / 32) flag[d] = 0;
      }
      reinterpret_cast<uint4*>(cnt)[d] = make_uint4(0, 0, 0, 0);
      __syncthreads();
    }
  }

  // ------------------------------------------------------------------ mid
  // stable counting pass over smem range [lo, lo+L) on digit g: a -> b
  template <int MK>  // keys per thread: L <= THREADS * MK
  static __device__ void smem_pass(const K* a, K* b, const V* av, V* bv, int lo, int L, int g,
                                   uint32_t* whist, uint32_t* wmask, uint32_t* s_lstart,
                                   uint32_t* s_warp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < WARPS; ++e) whist[e * 256 + threadIdx.x] = 0;
    __syncthreads();
    K key[MK];
    V val[MK];
    uint32_t dr[MK];
#pragma unroll
    for (int jj = 0; jj < MK; ++jj) {
      const int rel = w * 32 * MK + jj * 32 + lane;
      const bool ok = rel < L;
      key[jj] = ok ? a[lo + rel] : K(0);
      if (PAIRS) val[jj] = ok ? av[lo + rel] : 0u;
      dr[jj] = ok ? digit_of(key[jj], g) : 256u;
    }
    if (w * 32 * MK < L) warp_rank<MK, false>(dr, whist + w * 256);  // warps past the range idle
    __syncthreads();
    uint32_t run = 0;
#pragma unroll
    for (int e = 0; e < WARPS; ++e) {
      const uint32_t x = whist[e * 256 + threadIdx.x];
      whist[e * 256 + threadIdx.x] = run;
      run += x;
    }
    uint32_t tot;
    s_lstart[threadIdx.x] = block_excl_scan(run, s_warp, &tot);
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < MK; ++jj) {
      const uint32_t dgt = dr[jj] & 0xffffu;
      if (dgt < 256) {
        const int pos = lo + s_lstart[dgt] + whist[w * 256 + dgt] + (dr[jj] >> 16);
        b[pos] = key[jj];
        if (PAIRS) bv[pos] = val[jj];
      }
    }
    __syncthreads();
  }

  // Alg. 4 inside shared memory for one bucket of N_d < len <= C (or the
  // whole input when n <= C): a stack of ranges; each range takes its top
  // passes over the non-constant digits, small sub-buckets are sorted at
  // once, larger ones are pushed back on the stack (recursion).
  // CAP: the largest bucket this instantiation holds; it takes the queued
  // buckets with len_lo < len <= CAP (k_mid_s: up to MID_CAP_S at 4 CTAs/SM,
  // k_mid: the rest at 2 CTAs/SM)
  template <int CAP>
  static __device__ void mid(const Params<K>& P, uint32_t* sm, int len_lo) {
    constexpr int MK = CAP / THREADS;
    Ctl* c = P.ctl;
    const uint32_t total = min(c->mid_count, P.mid_cap);
    K* S0 = reinterpret_cast<K*>(sm);
    K* S1 = S0 + CAP;
    V* V0 = reinterpret_cast<V*>(S1 + CAP);
    V* V1 = PAIRS ? V0 + CAP : V0;
    CT* cmp = reinterpret_cast<CT*>(PAIRS ? (void*)(V1 + CAP) : (void*)V0);
    uint32_t* whist = reinterpret_cast<uint32_t*>(cmp + CAP + 8);
    uint32_t* wmask = whist + WARPS * 256;  // 2*WARPS*256, kept zero between uses
    uint32_t* s_lstart = wmask + 2 * WARPS * 256;
    uint32_t* bm = s_lstart + 256;                   // CAP/32 + 8 words
    uint2* stack = reinterpret_cast<uint2*>(bm + CAP / 32 + 8);  // 512 entries
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(stack + 512);     // 32 words
    unsigned long long* s_diff = reinterpret_cast<unsigned long long*>(s_misc + 16);
    const int nd = (int)P.n_d;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int e = 0; e < 2 * WARPS; ++e) wmask[e * 256 + threadIdx.x] = 0;
    __syncthreads();

    for (uint32_t e = blockIdx.x; e < total; e += gridDim.x) {
      const MidE me = P.midq[e];
      const int len = me.len;
      if (len <= len_lo || len > CAP) continue;  // the other instantiation's bucket
      const K* X = P.kbuf(me.buf);
      const V* Xv = P.vbuf(me.buf);
      if (me.hi < 0) {  // digits exhausted: a constant bucket, sorted (Alg. 2 l.17-18)
        if (me.buf)  // left in the scratch buffer: copy out
          {
            coop_copy(P.A + me.start, X + me.start, (uint32_t)len, threadIdx.x, THREADS);
            if (PAIRS) coop_copy(P.Av + me.start, Xv + me.start, (uint32_t)len, threadIdx.x, THREADS);
          }
        continue;
      }
      {  // all MK loads of a thread in flight before its shared-memory stores
        K pk[MK];
        V pv[MK];
#pragma unroll
        for (int m = 0; m < MK; ++m) {
          const int i = threadIdx.x + THREADS * m;
          if (i < len) {
            pk[m] = X[me.start + i];
            if (PAIRS) pv[m] = Xv[me.start + i];
          }
        }
#pragma unroll
        for (int m = 0; m < MK; ++m) {
          const int i = threadIdx.x + THREADS * m;
          if (i < len) {
            S0[i] = pk[m];
            if (PAIRS) V0[i] = pv[m];
          }
        }
      }
      if (threadIdx.x == 0) {
        stack[0] = make_uint2((uint32_t)len << 16, (uint32_t)(me.hi + 1));
        s_misc[0] = 1;  // stack size
      }
      __syncthreads();
      while (true) {
        if (threadIdx.x == 0) {
          const uint32_t sz = s_misc[0];
          if (sz) {
            const uint2 top = stack[sz - 1];
            s_misc[0] = sz - 1;
            s_misc[1] = top.x;
            s_misc[2] = top.y;
            s_misc[3] = 1;
          } else {
            s_misc[3] = 0;
          }
          *s_diff = 0;
        }
        __syncthreads();
        if (!s_misc[3]) break;
        const int lo = s_misc[1] & 0xffff, L = s_misc[1] >> 16;
        const int h = (int)s_misc[2] - 1;
        // diff mask of the range
        const K kref = S0[lo];
        unsigned long long d = 0;
        for (int i = threadIdx.x; i < L; i += THREADS) d |= (unsigned long long)(S0[lo + i] ^ kref);
#pragma unroll
        for (int o = 16; o; o >>= 1) d |= __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0 && d) atomicOr(s_diff, d);
        __syncthreads();
        const unsigned long long diff = *s_diff;
        const int hn = highest_nonconst(diff, h);
        __syncthreads();
        if (hn < 0) continue;  // all keys equal: sorted
        int low;
        if (L <= nd) {
          low = hn + 1;  // the whole range is one small bucket
        } else {
          // top passes over the non-constant digits <= hn (Alg. 4 l.4-6)
          int pmax = est_top_passes((uint64_t)L, P.n_d);
          int gd[8], ng = 0;
          for (int dd = hn; dd >= 0 && ng < pmax; --dd)
            if ((diff >> (8 * dd)) & 255ull) gd[ng++] = dd;
          for (int x = ng - 1; x >= 0; --x) {  // least significant of the group first
            smem_pass<MK>(S0, S1, V0, V1, lo, L, gd[x], whist, wmask, s_lstart, s_misc + 8);
            for (int i = threadIdx.x; i < L; i += THREADS) {
              S0[lo + i] = S1[lo + i];
              if (PAIRS) V0[lo + i] = V1[lo + i];
            }
            __syncthreads();
          }
          low = gd[ng - 1];
        }
        // bucket starts over the range (bit at range end = sentinel)
        const int shift = 8 * low;
        const bool wide = (shift + 8 > CT_BITS);
        const int nbits = lo + L + 1;
        for (int b0 = 0; b0 < nbits; b0 += THREADS) {
          const int i = b0 + threadIdx.x;
          bool st = false;
          if (i >= lo && i <= lo + L) {
            if (i == lo || i == lo + L)
              st = true;
            else
              st = wide ? false : ((S0[i] >> shift) != (S0[i - 1] >> shift));
          }
          const uint32_t bb = __ballot_sync(0xffffffffu, st);
          if (lane == 0) bm[i >> 5] = bb;
        }
        __syncthreads();
        const CT remmask = (shift >= CT_BITS) ? ~CT(0) : ((CT(1) << shift) - 1);
        // small buckets: composite; large: push (Alg. 4 l.11)
        for (int b0 = 0; b0 < L; b0 += THREADS) {
          const int i = lo + b0 + threadIdx.x;
          if (b0 + (int)threadIdx.x < L) {
            const int bs = prev_set(bm, i, lo);
            const int bend = next_set(bm, i, lo + L);
            if (bend - bs <= nd) {
              if (!wide) cmp[i] = ((CT)(S0[i] & (K)remmask) << 8) | (CT)(i - bs);
            } else if (i == bs && low > 0) {
              const uint32_t sz = atomicAdd(&s_misc[0], 1u);
              if (sz < 512)
                stack[sz] = make_uint2((uint32_t)bs | ((uint32_t)(bend - bs) << 16), (uint32_t)low);
              else
                flag_overflow(c, 32u);
            }
          }
        }
        __syncthreads();
        // ranks (keys kept in registers, <= MK per thread)
        K key[MK];
        V val[MK];
        int dst[MK];
#pragma unroll
        for (int m = 0; m < MK; ++m) {
          const int i = lo + threadIdx.x + THREADS * m;
          dst[m] = -1;
          if (threadIdx.x + THREADS * m < L) {
            const int bs = prev_set(bm, i, lo);
            const int bend = next_set(bm, i, lo + L);
            if (bend - bs <= nd) {
              key[m] = S0[i];
              if (PAIRS) val[m] = V0[i];
              dst[m] = bs + (wide ? bucket_rank_wide(S0, bs, bend, i, key[m])
                                  : bucket_rank(cmp, bs, bend, cmp[i]));
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < MK; ++m) {
          if (dst[m] >= 0) {
            S0[dst[m]] = key[m];
            if (PAIRS) V0[dst[m]] = val[m];
          }
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < len; i += THREADS) {
        P.A[me.start + i] = S0[i];
        if (PAIRS) P.Av[me.start + i] = V0[i];
      }
      __syncthreads();
    }
  }
};

}  // namespace dfr
