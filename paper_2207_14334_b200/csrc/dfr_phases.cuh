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

template <class K, bool PAIRS>
struct Phases {
  using V = uint32_t;
  using CT = typename Comp<K>::T;
  static constexpr int VEC = 16 / sizeof(K);
  static constexpr int CT_BITS = 8 * sizeof(CT);

  // ------------------------------------------------------------ smem sizes
  static constexpr size_t SMEM_HIST = MAX_PASSES * 256 * 4 + 64;
  static constexpr size_t SMEM_SCATTER =
      WARPS * 256 * 4 + 256 * 4 * 2 + 64 + TILE * sizeof(K) + (PAIRS ? TILE * 4 : 0);
  static constexpr size_t SMEM_DIVERT =
      WIN * sizeof(K) + WIN * sizeof(CT) + (PAIRS ? WIN * 4 : 0) + (WIN / 32 + 8) * 4 + 64;
  static constexpr size_t SMEM_MID = 2 * MID_CAP * sizeof(K) + (PAIRS ? 2 * MID_CAP * 4 : 0) +
                                     MID_CAP * sizeof(CT) + WARPS * 256 * 4 + 256 * 4 +
                                     (MID_CAP / 32 + 8) * 4 + 512 * 8 + 128;
  static constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
  static constexpr size_t SMEM_LEVEL =
      cmax(cmax(SMEM_HIST, SMEM_SCATTER), cmax(SMEM_DIVERT, SMEM_MID));

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
      if (threadIdx.x == 0) c->overflow |= 1;
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
        chunks = (s.len + P.chunk - 1) / P.chunk;
        if (s.hi < 0) {  // digits exhausted: all keys equal (Alg. 2 l.17-18)
          s.p = 0;
          s.low = 0;
          s.flags = s.buf ? SEG_COPY : SEG_DONE;
          if (!s.buf) chunks = 0;
        } else {
          int pp = est_top_passes(s.len, P.n_d);
          if (pp > s.hi + 1) pp = s.hi + 1;
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
      if (threadIdx.x == 0) c->overflow |= 2;
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
                                    uint32_t* sh, unsigned long long diff) {
    __syncthreads();
    for (uint32_t j = 0; j < s.p; ++j) {
      uint32_t v = sh[j * 256 + threadIdx.x];
      if (v) atomicAdd(&P.hist[(size_t)(s.hist_off + j) * 256 + threadIdx.x], v);
      sh[j * 256 + threadIdx.x] = 0;
    }
    // diff: warp OR then one atomic per warp
    unsigned long long d = diff;
#pragma unroll
    for (int o = 16; o; o >>= 1) d |= __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0 && d) atomicOr(&q[si].diff, d);
    __syncthreads();
  }

  static __device__ __forceinline__ void count_key(uint32_t* sh, K k, bool valid, int low,
                                                   uint32_t p) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < MAX_PASSES; ++j) {
      if ((uint32_t)j < p) {  // warp-uniform
        const uint32_t d = valid ? digit_of(k, low + j) : 256u + j;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (valid && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&sh[j * 256 + d], __popc(peers));
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
    const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
    const uint32_t t0 = blockIdx.x * per;
    const uint32_t t1 = min(total, t0 + per);
    if (t0 >= t1) return;
    uint32_t* sh = sm;
    for (int j = 0; j < MAX_PASSES; ++j) sh[j * 256 + threadIdx.x] = 0;
    uint32_t si = upper_index(nseg, t0, [&](uint32_t i) { return q[i].tile0; });
    Seg s = q[si];
    unsigned long long diff = 0;
    __syncthreads();
    for (uint32_t t = t0; t < t1; ++t) {
      while (t >= s.tile0 + s.ntiles) {  // next segment with tiles
        hist_flush(P, q, si, s, sh, diff);
        diff = 0;
        ++si;
        s = q[si];
      }
      const uint32_t lt = t - s.tile0;
      const uint32_t base = s.start + lt * TILE;
      const uint32_t cnt = min((uint32_t)TILE, s.len - lt * TILE);
      for (uint32_t j = 0; j < s.p; ++j)
        P.status[j * P.status_stride + (size_t)t * 256 + threadIdx.x] = 0;
      const K* src = s.buf ? P.B : P.A;
      const K kref = src[s.start];
      const K* tp = src + base;
      if ((reinterpret_cast<uintptr_t>(tp) & 15) == 0) {
        const uint32_t nv = cnt / VEC;
        const uint4* vp = reinterpret_cast<const uint4*>(tp);
        for (uint32_t vb = 0; vb < nv; vb += THREADS) {
          const uint32_t v = vb + threadIdx.x;
          const bool ok = v < nv;
          uint4 x = ok ? __ldg(vp + v) : make_uint4(0, 0, 0, 0);
          const K* kk = reinterpret_cast<const K*>(&x);
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            if (ok) diff |= (unsigned long long)(kk[e] ^ kref);
            count_key(sh, kk[e], ok, s.low, s.p);
          }
        }
        for (uint32_t i = nv * VEC; i < cnt; i += THREADS) {  // < VEC keys, warp 0
          const uint32_t ii = i + threadIdx.x;
          const bool ok = ii < cnt;
          K k = ok ? tp[ii] : K(0);
          if (ok) diff |= (unsigned long long)(k ^ kref);
          if (threadIdx.x < 32) count_key(sh, k, ok, s.low, s.p);
        }
      } else {
        for (uint32_t ib = 0; ib < cnt; ib += THREADS) {
          const uint32_t i = ib + threadIdx.x;
          const bool ok = i < cnt;
          K k = ok ? tp[i] : K(0);
          if (ok) diff |= (unsigned long long)(k ^ kref);
          count_key(sh, k, ok, s.low, s.p);
        }
      }
    }
    hist_flush(P, q, si, s, sh, diff);
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
              atomicOr(&c->overflow, 4u);
            }
          }
        }
      }
      if (threadIdx.x == 0) {
        q[si].flags = flags;
        q[si].final_buf = s.buf ^ (executed & 1u);
        if (c->level == 0) {
          c->level0_p = s.p;
          c->level0_run = executed;
        }
      }
      __syncthreads();
    }
  }

  // ------------------------------------------------------------- scatter
  // One stable deal on group digit low+j for every active segment.  Tiles of
  // TILE keys are claimed by dynamic tickets; each tile ranks its keys with a
  // warp-level multi-split (match_any), publishes its per-digit aggregate,
  // resolves its exclusive per-digit prefix by decoupled look-back over the
  // preceding tiles of the same segment, reorders the tile through shared
  // memory by digit and writes each digit run contiguously.
  static __device__ void scatter(const Params<K>& P, int j, uint32_t* sm) {
    Ctl* c = P.ctl;
    const uint32_t total = c->total_tiles, nseg = c->nseg;
    if ((uint32_t)j >= c->max_p) return;  // no segment of this level has pass j
    Seg* q = P.segq[c->cur];
    uint32_t* whist = sm;                                   // WARPS*256
    int* s_dst = reinterpret_cast<int*>(whist + WARPS * 256);  // 256
    uint32_t* s_lstart = reinterpret_cast<uint32_t*>(s_dst + 256);  // 256
    uint32_t* s_misc = s_lstart + 256;                      // 16
    K* sk = reinterpret_cast<K*>(s_misc + 16);
    V* sv = reinterpret_cast<V*>(sk + TILE);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t* mywh = whist + w * 256;
    uint32_t* status = P.status + (size_t)j * P.status_stride;

    while (true) {
      if (threadIdx.x == 0) {
        const uint32_t t = atomicAdd(&c->ticket[j], 1u);
        s_misc[0] = t;
        s_misc[1] = t < total ? upper_index(nseg, t, [&](uint32_t i) { return q[i].tile0; }) : 0;
      }
      __syncthreads();
      const uint32_t t = s_misc[0];
      if (t >= total) break;
      const Seg s = q[s_misc[1]];
      if ((uint32_t)j >= s.p || ((s.flags >> j) & 1u) ||
          (s.flags & (SEG_SKIP_DIVERT | SEG_COPY | SEG_DONE))) {
        __syncthreads();
        continue;
      }
      const uint32_t lt = t - s.tile0;
      const uint32_t base = s.start + lt * TILE;
      const uint32_t cnt = min((uint32_t)TILE, s.len - lt * TILE);
      const uint32_t before = (uint32_t)j - __popc(s.flags & ((1u << j) - 1u));
      const uint32_t sb = s.buf ^ (before & 1u);
      const K* src = sb ? P.B : P.A;
      K* dst = sb ? P.A : P.B;
      const V* srcv = sb ? P.Bv : P.Av;
      V* dstv = sb ? P.Av : P.Bv;
      const int dg = s.low + j;

      // stage the tile in shared memory (16-byte vector loads when aligned)
      const K* tp = src + base;
      if ((reinterpret_cast<uintptr_t>(tp) & 15) == 0 && cnt == (uint32_t)TILE) {
        const uint4* vp = reinterpret_cast<const uint4*>(tp);
        uint4* sp = reinterpret_cast<uint4*>(sk);
#pragma unroll 4
        for (int v = threadIdx.x; v < TILE / VEC; v += THREADS) sp[v] = __ldg(vp + v);
      } else {
        for (uint32_t i = threadIdx.x; i < cnt; i += THREADS) sk[i] = tp[i];
      }
      if (PAIRS) {
        const V* vp = srcv + base;
        if ((reinterpret_cast<uintptr_t>(vp) & 15) == 0 && cnt == (uint32_t)TILE) {
          const uint4* v4 = reinterpret_cast<const uint4*>(vp);
          uint4* s4 = reinterpret_cast<uint4*>(sv);
#pragma unroll 4
          for (int v = threadIdx.x; v < TILE / 4; v += THREADS) s4[v] = __ldg(v4 + v);
        } else {
          for (uint32_t i = threadIdx.x; i < cnt; i += THREADS) sv[i] = vp[i];
        }
      }
#pragma unroll
      for (int e = 0; e < WARPS; ++e) whist[e * 256 + threadIdx.x] = 0;
      __syncthreads();

      // warp-striped items: (jj, lane) -> w*32*KPT + jj*32 + lane
      K key[KPT];
      V val[KPT];
      uint32_t dig[KPT], rank[KPT];
#pragma unroll
      for (int jj = 0; jj < KPT; ++jj) {
        const uint32_t idx = w * 32 * KPT + jj * 32 + lane;
        const bool ok = idx < cnt;
        key[jj] = sk[idx];
        if (PAIRS) val[jj] = sv[idx];
        dig[jj] = ok ? digit_of(key[jj], dg) : 256u;
      }
      warp_rank(dig, rank, mywh);
      __syncthreads();

      // per digit: exclusive offsets of each warp, tile aggregate
      const uint32_t dd = threadIdx.x;
      uint32_t run = 0;
#pragma unroll
      for (int e = 0; e < WARPS; ++e) {
        const uint32_t x = whist[e * 256 + dd];
        whist[e * 256 + dd] = run;
        run += x;
      }
      uint32_t* my_status = status + (size_t)t * 256 + dd;
      st_relaxed(my_status, (lt == 0 ? FLAG_INC : FLAG_AGG) | run);
      uint32_t tot;
      const uint32_t lstart = block_excl_scan(run, s_misc + 4, &tot);
      uint32_t excl = 0;
      if (lt > 0) {  // decoupled look-back over the segment's earlier tiles
        uint32_t tt = t - 1;
        while (true) {
          const uint32_t v = ld_relaxed(status + (size_t)tt * 256 + dd);
          if ((v >> 30) == 0) continue;  // predecessor not published yet
          excl += v & VAL_MASK;
          if (v & FLAG_INC) break;
          --tt;
        }
        st_relaxed(my_status, FLAG_INC | (excl + run));
      }
      const uint32_t bstart = P.hist[(size_t)(s.hist_off + j) * 256 + dd];
      s_dst[dd] = (int)(s.start + bstart + excl) - (int)lstart;
      s_lstart[dd] = lstart;
      __syncthreads();

      // reorder the tile by digit in shared memory (stable)
#pragma unroll
      for (int jj = 0; jj < KPT; ++jj) {
        if (dig[jj] < 256) {
          const uint32_t pos = s_lstart[dig[jj]] + mywh[dig[jj]] + rank[jj];
          sk[pos] = key[jj];
          if (PAIRS) sv[pos] = val[jj];
        }
      }
      __syncthreads();
      // coalesced write of each digit run
#pragma unroll 4
      for (uint32_t i = threadIdx.x; i < cnt; i += THREADS) {
        const K k = sk[i];
        const int o = s_dst[digit_of(k, dg)] + (int)i;
        dst[o] = k;
        if (PAIRS) dstv[o] = sv[i];
      }
      __syncthreads();
    }
  }

  // ------------------------------------------------------- small sort core
  // rank of item i inside its bucket [bs, be) of the smem composite array
  static __device__ __forceinline__ uint32_t bucket_rank(const CT* cmp, int bs, int be, CT me) {
    uint32_t r = 0;
    for (int x = bs; x < be; ++x) r += cmp[x] < me;
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
  static __device__ void push_bucket(const Params<K>& P, const Seg& s, uint32_t gstart,
                                     uint32_t blen) {
    Ctl* c = P.ctl;
    const int hn = highest_nonconst(s.diff, s.low - 1);
    if (c->level == 0) atomicAdd(&c->level0_large, 1ull);
    if (hn < 0 && s.final_buf == 0) return;  // constant keys, already in place
    if (blen <= (uint32_t)MID_CAP) {
      const uint32_t idx = atomicAdd(&c->mid_count, 1u);
      atomicAdd(&c->mid_buckets, 1ull);
      if (idx < P.mid_cap) {
        MidE m;
        m.start = gstart;
        m.len = (uint16_t)blen;
        m.hi = (int8_t)hn;
        m.buf = (uint8_t)s.final_buf;
        P.midq[idx] = m;
      } else {
        atomicOr(&c->overflow, 8u);
      }
    } else {
      const uint32_t idx = atomicAdd(&c->next_count, 1u);
      atomicAdd(&c->global_segments, 1ull);
      if (idx < P.max_segs) {
        Seg ns = {};
        ns.start = gstart;
        ns.len = blen;
        ns.hi = hn;
        ns.buf = s.final_buf;
        P.segq[1u - c->cur][idx] = ns;
      } else {
        atomicOr(&c->overflow, 16u);
      }
    }
  }

  static __device__ void divert(const Params<K>& P, uint32_t* sm) {
    Ctl* c = P.ctl;
    const uint32_t total = c->total_chunks, nseg = c->nseg;
    Seg* q = P.segq[c->cur];
    K* sk = reinterpret_cast<K*>(sm);
    CT* cmp = reinterpret_cast<CT*>(sk + WIN);
    V* sv = reinterpret_cast<V*>(cmp + WIN);
    uint32_t* bm = reinterpret_cast<uint32_t*>(PAIRS ? (void*)(sv + WIN) : (void*)sv);
    uint32_t* s_misc = bm + WIN / 32 + 8;
    const int CH = (int)P.chunk;
    const int nd = (int)P.n_d;
    const int W = 1 + CH + nd;  // window: lead key, chunk, halo of N_d
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

    for (uint32_t ch = blockIdx.x; ch < total; ch += gridDim.x) {
      if (threadIdx.x == 0) s_misc[0] = upper_index(nseg, ch, [&](uint32_t i) { return q[i].chunk0; });
      __syncthreads();
      const Seg s = q[s_misc[0]];
      __syncthreads();
      if (s.flags & (SEG_DONE | SEG_SKIP_DIVERT)) continue;
      const int c0 = (int)(ch - s.chunk0) * CH;  // segment-relative chunk start
      const int len = (int)s.len;
      if (s.flags & SEG_COPY) {  // finished bucket left in B: copy out (Alg. 4 comment)
        const int c1 = min(len, c0 + CH);
        for (int r = c0 + threadIdx.x; r < c1; r += THREADS) {
          P.A[s.start + r] = P.B[s.start + r];
          if (PAIRS) P.Av[s.start + r] = P.Bv[s.start + r];
        }
        continue;
      }
      const K* X = s.final_buf ? P.B : P.A;
      const V* Xv = s.final_buf ? P.Bv : P.Av;
      const int shift = 8 * s.low;
      const K* xs = X + s.start;

      K key[KPT];
      V val[KPT];
#pragma unroll
      for (int m = 0; m < KPT; ++m) {
        const int i = threadIdx.x + THREADS * m;
        const int r = c0 - 1 + i;
        const bool ok = i < W && r >= 0 && r < len;
        key[m] = ok ? xs[r] : K(0);
        if (PAIRS) val[m] = ok ? Xv[s.start + r] : 0u;
        sk[i] = key[m];
      }
      __syncthreads();
      // bucket-start bitmask: bit i <=> a bucket (equal top-p prefix) starts at i
#pragma unroll
      for (int m = 0; m < KPT; ++m) {
        const int i = threadIdx.x + THREADS * m;
        const int r = c0 - 1 + i;
        bool st = false;
        if (i < W) {
          if (r <= 0 || r >= len)
            st = true;
          else
            st = (sk[i] >> shift) != (sk[i - 1] >> shift);
        }
        const uint32_t b = __ballot_sync(0xffffffffu, st);
        if (lane == 0) bm[8 * m + w] = b;
      }
      if (threadIdx.x < 8) bm[WIN / 32 + threadIdx.x] = 0;
      __syncthreads();
      // classify; composite keys of owned small buckets
      const CT remmask = (shift >= CT_BITS) ? ~CT(0) : ((CT(1) << shift) - 1);
      uint32_t be_[KPT];  // packed (bucket start, bucket end) or 0xffffffff
#pragma unroll
      for (int m = 0; m < KPT; ++m) {
        const int i = threadIdx.x + THREADS * m;
        const int r = c0 - 1 + i;
        be_[m] = 0xffffffffu;
        if (i < 1 || i >= W || r >= len) continue;
        const int bs = prev_set(bm, i, max(1, i - nd));
        if (bs < 1 || bs > CH) continue;  // not owned, or a bucket > N_d
        const int bend = next_set(bm, i, min(W - 1, bs + nd));
        if (bend >= 0) {
          be_[m] = (uint32_t)bs | ((uint32_t)bend << 16);
          cmp[i] = ((CT)(key[m] & (K)remmask) << 8) | (CT)(i - bs);
        } else if (i == bs) {
          // an owned bucket > N_d: find its end, then queue it (Alg. 4 l.9-11)
          int e = next_set(bm, i, W - 1);
          uint32_t blen;
          if (e >= 0) {
            blen = (uint32_t)(e - i);
          } else {
            const K pre = key[m] >> shift;
            uint32_t lo = (uint32_t)(c0 - 1 + (W - 1));  // last in-window index (same prefix)
            uint32_t hi = (uint32_t)len;
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
            blen = hi - (uint32_t)r;
          }
          push_bucket(P, s, s.start + (uint32_t)r, blen);
        }
      }
      __syncthreads();
      uint32_t dst_[KPT];
#pragma unroll
      for (int m = 0; m < KPT; ++m) {
        const int i = threadIdx.x + THREADS * m;
        dst_[m] = 0;
        if (be_[m] != 0xffffffffu) {
          const int bs = be_[m] & 0xffff, bend = be_[m] >> 16;
          dst_[m] = bs + bucket_rank(cmp, bs, bend, cmp[i]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < KPT; ++m) {
        if (be_[m] != 0xffffffffu) {
          sk[dst_[m]] = key[m];
          if (PAIRS) sv[dst_[m]] = val[m];
        }
      }
      __syncthreads();
      K* outk = P.A + s.start;
      V* outv = P.Av + s.start;
#pragma unroll
      for (int m = 0; m < KPT; ++m) {
        if (be_[m] != 0xffffffffu) {
          const int i = threadIdx.x + THREADS * m;
          const int r = c0 - 1 + i;
          outk[r] = sk[i];
          if (PAIRS) outv[r] = sv[i];
        }
      }
      __syncthreads();
    }
  }

  // ------------------------------------------------------------------ mid
  // stable counting pass over smem range [lo, lo+L) on digit g: a -> b
  static __device__ void smem_pass(const K* a, K* b, const V* av, V* bv, int lo, int L, int g,
                                   uint32_t* whist, uint32_t* s_lstart, uint32_t* s_warp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < WARPS; ++e) whist[e * 256 + threadIdx.x] = 0;
    __syncthreads();
    K key[KPT];
    V val[KPT];
    uint32_t dig[KPT], rank[KPT];
#pragma unroll
    for (int jj = 0; jj < KPT; ++jj) {
      const int rel = w * 32 * KPT + jj * 32 + lane;
      const bool ok = rel < L;
      key[jj] = ok ? a[lo + rel] : K(0);
      if (PAIRS) val[jj] = ok ? av[lo + rel] : 0u;
      dig[jj] = ok ? digit_of(key[jj], g) : 256u;
    }
    warp_rank(dig, rank, whist + w * 256);
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
    for (int jj = 0; jj < KPT; ++jj) {
      if (dig[jj] < 256) {
        const int pos = lo + s_lstart[dig[jj]] + whist[w * 256 + dig[jj]] + rank[jj];
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
  static __device__ void mid(const Params<K>& P, uint32_t* sm) {
    Ctl* c = P.ctl;
    const uint32_t total = min(c->mid_count, P.mid_cap);
    K* S0 = reinterpret_cast<K*>(sm);
    K* S1 = S0 + MID_CAP;
    V* V0 = reinterpret_cast<V*>(S1 + MID_CAP);
    V* V1 = PAIRS ? V0 + MID_CAP : V0;
    CT* cmp = reinterpret_cast<CT*>(PAIRS ? (void*)(V1 + MID_CAP) : (void*)V0);
    uint32_t* whist = reinterpret_cast<uint32_t*>(cmp + MID_CAP);
    uint32_t* s_lstart = whist + WARPS * 256;
    uint32_t* bm = s_lstart + 256;                   // MID_CAP/32 + 8 words
    uint2* stack = reinterpret_cast<uint2*>(bm + MID_CAP / 32 + 8);  // 512 entries
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(stack + 512);     // 32 words
    unsigned long long* s_diff = reinterpret_cast<unsigned long long*>(s_misc + 16);
    const int nd = (int)P.n_d;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;

    for (uint32_t e = blockIdx.x; e < total; e += gridDim.x) {
      const MidE me = P.midq[e];
      const int len = me.len;
      const K* X = me.buf ? P.B : P.A;
      const V* Xv = me.buf ? P.Bv : P.Av;
      for (int i = threadIdx.x; i < len; i += THREADS) {
        S0[i] = X[me.start + i];
        if (PAIRS) V0[i] = Xv[me.start + i];
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
            smem_pass(S0, S1, V0, V1, lo, L, gd[x], whist, s_lstart, s_misc + 8);
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
                atomicOr(&c->overflow, 32u);
            }
          }
        }
        __syncthreads();
        // ranks (keys kept in registers, <= KPT per thread)
        K key[KPT];
        V val[KPT];
        int dst[KPT];
#pragma unroll
        for (int m = 0; m < KPT; ++m) {
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
        for (int m = 0; m < KPT; ++m) {
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
