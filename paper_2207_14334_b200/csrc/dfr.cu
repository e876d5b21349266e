// dfr.cu — kernels, host planner and C ABI of the B200 DFR sort.
//
// Launch sequence of one call (all on the caller's stream, no host sync):
//   cudaMallocAsync(workspace)
//   k_init     seed the level-0 segment (the whole input) and plan it
//   k_hist     one read: the p group-digit histograms + diff mask (Alg. 4 l.4-5)
//   k_plan2    counts -> bucket offsets; identity passes skipped
//   k_scatter  x p (host knows p for level 0): stable deals, LSD order (l.6)
//   k_divert   scan for large buckets; small ones sorted on-chip (l.7-14)
//   k_levels   cooperative kernel: recursion levels 1.. on the global
//              segment queue (l.11), looping on the device while it is non-empty
//   k_mid      buckets N_d < s <= C finished in shared memory
//   cudaFreeAsync(workspace)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>

#include "dfr.h"
#include "dfr_phases.cuh"

namespace cg = cooperative_groups;

namespace dfr {

// ------------------------------------------------------------------ kernels
template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS) k_init(const __grid_constant__ Params<K> P, uint32_t n,
                                                  int plan_now = 1) {
  extern __shared__ __align__(16) uint32_t sm[];
  Ctl* c = P.ctl;
  if (threadIdx.x == 0) {
    memset(c, 0, sizeof(Ctl));
    c->level = ~0u;
    c->cur = 0;
    c->next_count = 1;
    Seg s = {};
    s.start = 0;
    s.len = n;
    s.hi = P.D - 1;
    s.buf = 0;
    P.segq[1][0] = s;
  }
  if (P.J)  // the fused level's (top digit, chain) histogram, counted by k_hist
    for (uint32_t x = threadIdx.x; x < 4096u; x += blockDim.x) P.J[x] = 0;
  if (!plan_now) return;  // small inputs: k_levels plans level 0 itself
  __syncthreads();
  Phases<K, PAIRS>::plan(P, sm);
}

// stage API: a single segment with a forced group (digit_lo .. digit_lo+p-1)
template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS) k_init_stage(Params<K> P, uint32_t n, int digit_lo,
                                                        int p) {
  Ctl* c = P.ctl;
  if (threadIdx.x == 0) {
    memset(c, 0, sizeof(Ctl));
    c->cur = 0;
    c->nseg = 1;
    c->total_tiles = (n + TILE - 1) / TILE;
    c->total_chunks = 0;
    c->max_p = p;
    Seg s = {};
    s.start = 0;
    s.len = n;
    s.hi = digit_lo + p - 1;
    s.p = p;
    s.low = digit_lo;
    s.ntiles = c->total_tiles;
    s.final_buf = 0;
    P.segq[0][0] = s;
  }
  for (int r = 0; r < p; ++r) P.hist[r * 256 + threadIdx.x] = 0;
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS, DFR_HIST_MINB) k_hist(const __grid_constant__ Params<K> P) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, PAIRS>::hist(P, sm);
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS) k_plan2(const __grid_constant__ Params<K> P) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, PAIRS>::plan2(P, sm);
}

// Plan of recursion level 1 (the queue the level-0 diversion filled), run by
// the stand-alone kernels at full occupancy; an empty queue leaves an empty
// level, on which they return at once.
template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS) k_lplan(const __grid_constant__ Params<K> P) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Ctl* c = P.ctl;
  if (*(volatile uint32_t*)&c->next_count == 0) {
    if (threadIdx.x == 0) {
      c->nseg = 0;
      c->total_tiles = 0;
      c->total_chunks = 0;
      c->max_p = 0;
    }
    return;
  }
  Phases<K, PAIRS>::plan(P, sm);
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(Phases<K, PAIRS>::SC_NT, 4) k_scatter(const __grid_constant__ Params<K> P, int j) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, PAIRS>::template scatter<Phases<K, PAIRS>::SC_NT, false, true>(P, j, sm);
}

// the middle pass of a fused level 0: the deal plus the joint histogram
template <class K>
__global__ void __launch_bounds__(Phases<K, false>::SC_NT, 4) k_scatter_fh(const __grid_constant__ Params<K> P, int j) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, false>::template scatter<Phases<K, false>::SC_NT, true, true>(P, j, sm);
}

// Fast Radix (dfr_config.fast_radix, keys only): the estimated pass on the
// lowest group digit, its plan, and the middle pass reading the estimated layout
template <class K>
__global__ void __launch_bounds__(THREADS) k_fr_prep(const __grid_constant__ Params<K> P) {
  pdl_enter();
  Phases<K, false>::fr_prep(P);
}
template <class K>
__global__ void __launch_bounds__(Phases<K, false>::SC_NT, 4) k_scatter_fr(const __grid_constant__ Params<K> P, int j) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, false>::template scatter<Phases<K, false>::SC_NT, false, true, 1>(P, j, sm);
}
template <class K>
__global__ void __launch_bounds__(THREADS) k_fr_plan(const __grid_constant__ Params<K> P) {
  pdl_enter();
  Phases<K, false>::fr_plan(P);
}
template <class K>
__global__ void __launch_bounds__(Phases<K, false>::SC_NT, 4) k_scatter_frfh(const __grid_constant__ Params<K> P, int j) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, false>::template scatter<Phases<K, false>::SC_NT, true, true, 2>(P, j, sm);
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(Phases<K, PAIRS>::DV_NT, DFR_DV_MINB) k_divert(const __grid_constant__ Params<K> P) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, PAIRS>::template divert<Phases<K, PAIRS>::DV_NT>(P, sm);
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(256) k_hfix(const __grid_constant__ Params<K> P) {
  pdl_enter();
  Phases<K, PAIRS>::hfix(P);
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(1024) k_fplan(const __grid_constant__ Params<K> P) {
  pdl_enter();
  Phases<K, PAIRS>::fplan(P);
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(Phases<K, PAIRS>::GNT, Phases<K, PAIRS>::GMINB) k_fused(const __grid_constant__ Params<K> P) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, PAIRS>::fused(P, sm);
}

template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS, 2) k_mid(const __grid_constant__ Params<K> P, int len_lo) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, PAIRS>::template mid<MID_CAP>(P, sm, len_lo);
}
// keys only: the mid buckets, one round per digit (Phases::midf)
template <class K>
__global__ void __launch_bounds__(Phases<K, false>::FNT, 3) k_midf(const __grid_constant__ Params<K> P, int round) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, false>::midf(P, sm, round);
}

// the mid buckets of at most MID_CAP_S keys, at 4 CTAs/SM
template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS, 4) k_mid_s(const __grid_constant__ Params<K> P) {
  extern __shared__ __align__(16) uint32_t sm[];
  pdl_enter();
  Phases<K, PAIRS>::template mid<MID_CAP_S>(P, sm, 0);
}

// Recursion levels 1.. (Alg. 4 l.11 applied to every queued large bucket at
// once).  Cooperative launch: every CTA is resident, levels are separated by
// grid-wide barriers, and the loop ends on the device when the queue is empty.
template <class K, bool PAIRS>
__global__ void __launch_bounds__(THREADS, 4) k_levels(const __grid_constant__ Params<K> P) {
  extern __shared__ __align__(16) uint32_t sm[];
  cg::grid_group grid = cg::this_grid();
  using Ph = Phases<K, PAIRS>;
  for (int level = 0; level < 2 * P.D; ++level) {  // an iteration bound (depth <= D)
    if (*(volatile uint32_t*)&P.ctl->next_count == 0) break;
    grid.sync();
    if (blockIdx.x == 0) Ph::plan(P, sm);
    grid.sync();
    Ph::hist(P, sm);
    grid.sync();
    Ph::plan2(P, sm);
    grid.sync();
    for (int j = 0; j < MAX_PASSES; ++j) {
      if ((uint32_t)j >= *(volatile uint32_t*)&P.ctl->max_p) break;
      Ph::template scatter<THREADS, false, true>(P, j, sm);
      grid.sync();
    }
    Ph::template divert<THREADS>(P, sm);
    grid.sync();
  }
}

template <class K, bool PAIRS>
__global__ void k_seed_mid(Params<K> P, uint32_t n) {
  Ctl* c = P.ctl;
  memset(c, 0, sizeof(Ctl));
  MidE m;
  m.start = 0;
  m.len = (uint16_t)n;
  m.hi = (int8_t)(P.D - 1);
  m.buf = 0;
  P.midq[0] = m;
  c->mid_count = 1;
}

// ------------------------------------------------------------------ host
// launch with programmatic stream serialization (see pdl_enter)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
#ifdef DFR_NO_PDL
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

static std::atomic<unsigned long long> g_launches{0};

#ifdef DFR_DEBUG
#define DFR_CHECK_LAUNCH(name)                                                          \
  do {                                                                                  \
    cudaError_t e_ = cudaStreamSynchronize(st);                                          \
    if (e_ == cudaSuccess) e_ = cudaGetLastError();                                      \
    fprintf(stderr, "[dfr debug] %s: %s\n", name, cudaGetErrorString(e_));               \
  } while (0)
#else
#define DFR_CHECK_LAUNCH(name) \
  do {                         \
  } while (0)
#endif

struct PhaseEv {  // optional caller-provided events around each phase
  void* const* ev;
  cudaStream_t st;
  void begin(int i) const {
    if (ev && ev[2 * i]) cudaEventRecord((cudaEvent_t)ev[2 * i], st);
  }
  void end(int i) const {
    if (ev && ev[2 * i + 1]) cudaEventRecord((cudaEvent_t)ev[2 * i + 1], st);
  }
  void skip(int i) const {
    begin(i);
    end(i);
  }
};

struct Dev {
  int sms = 0;
  int occ_hist = 0, occ_scatter = 0, occ_divert = 0, occ_mid = 0, occ_mid_s = 0, occ_levels = 0,
      occ_fused = 0, occ_midf = 0;
};

template <class K, bool PAIRS>
static cudaError_t get_dev(Dev& out) {
  using Ph = Phases<K, PAIRS>;
  static std::once_flag once[16];
  static Dev devs[16];
  static cudaError_t errs[16];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [&]() {
    Dev d;
    cudaError_t err = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    // keep freed scratch cached in the stream-ordered pool: every call allocates
    // and frees its workspace (the paper times allocation), which must
    // then cost microseconds, not a re-map of gigabytes
    cudaMemPool_t pool;
    if (err == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      unsigned long long thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    auto setup = [&](const void* f, size_t smem, int* occ) {
      if (err != cudaSuccess) return;
      err = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, f, THREADS, smem);
    };
    setup((const void*)k_init<K, PAIRS>, 64, &d.occ_hist);
    setup((const void*)k_hist<K, PAIRS>, Ph::SMEM_HIST, &d.occ_hist);
    setup((const void*)k_plan2<K, PAIRS>, 64, &d.occ_mid);
    if (err == cudaSuccess && !PAIRS)
      err = cudaFuncSetAttribute((const void*)k_scatter_fh<K>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ph::SMEM_SCATTER_P);
    if (err == cudaSuccess && !PAIRS)
      err = cudaFuncSetAttribute((const void*)k_scatter_fr<K>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ph::SMEM_SCATTER_P);
    if (err == cudaSuccess && !PAIRS)
      err = cudaFuncSetAttribute((const void*)k_scatter_frfh<K>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ph::SMEM_SCATTER_P);
    if (err == cudaSuccess) {  // the deal (one tile buffer + permutation)
      err = cudaFuncSetAttribute((const void*)k_scatter<K, PAIRS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ph::SMEM_SCATTER_P);
      if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &d.occ_scatter, (const void*)k_scatter<K, PAIRS>, Ph::SC_NT, Ph::SMEM_SCATTER_P);
    }
    if (err == cudaSuccess) {  // the diversion runs DV_NT-thread CTAs
      err = cudaFuncSetAttribute((const void*)k_divert<K, PAIRS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ph::SMEM_DIVERT);
      if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &d.occ_divert, (const void*)k_divert<K, PAIRS>, Ph::DV_NT, Ph::SMEM_DIVERT);
    }
    setup((const void*)k_mid<K, PAIRS>, Ph::SMEM_MID, &d.occ_mid);
    setup((const void*)k_mid_s<K, PAIRS>, Ph::SMEM_MID_S, &d.occ_mid_s);
    if (err == cudaSuccess) {  // fused last pass: FNT-thread CTAs
      err = cudaFuncSetAttribute((const void*)k_fused<K, PAIRS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ph::SMEM_FUSED_X);
      if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ_fused, (const void*)k_fused<K, PAIRS>,
                                                            Ph::GNT, Ph::SMEM_FUSED_X);
    }
    setup((const void*)k_levels<K, PAIRS>, Ph::SMEM_LEVEL, &d.occ_levels);
    if (err == cudaSuccess && !PAIRS) {  // keys-only mid rounds: FNT-thread CTAs
      err = cudaFuncSetAttribute((const void*)k_midf<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Ph::SMEM_FUSED);
      if (err == cudaSuccess)
        err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ_midf, (const void*)k_midf<K>, Ph::FNT,
                                                            Ph::SMEM_FUSED);
    }
    devs[dev] = d;
    errs[dev] = err;
  });
  out = devs[dev];
  return errs[dev];
}

static inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// the buckets N_d < s <= C: keys only, D rounds of k_midf (one digit each);
// pairs, the shared-memory recursion of k_mid_s / k_mid
template <class K, bool PAIRS>
static void launch_mid(const Dev& dv, cudaStream_t st, const Params<K>& P) {
  using Ph = Phases<K, PAIRS>;
  if constexpr (!PAIRS) {
    for (int r = 0; r < (int)sizeof(K); ++r)
      launch_pdl(k_midf<K>, dv.sms * std::max(1, dv.occ_midf), Ph::FNT, Ph::SMEM_FUSED, st, P, r);
    g_launches += sizeof(K);
  } else {
    launch_pdl(k_mid_s<K, PAIRS>, dv.sms * std::max(1, dv.occ_mid_s), THREADS, Ph::SMEM_MID_S, st, P);
    launch_pdl(k_mid<K, PAIRS>, dv.sms * std::max(1, dv.occ_mid), THREADS, Ph::SMEM_MID, st, P, MID_CAP_S);
    g_launches += 2;
  }
}

struct Layout {
  size_t b_keys, b_vals, c_keys, ctl, segq0, segq1, midq, midq2, hist, status, fh, ftiles, fj, total;
  size_t fr_ct, fr_tab, fr_cnt, fr_cap, fr_kmax;
  size_t max_segs, mid_cap, hist_rows, tiles_max;
};

static Layout make_layout(size_t n, int kb, int vb, uint32_t n_d, int min_passes = 1,
                          bool fuse = false, bool fr = false) {
  Layout L{};
  L.max_segs = n / (MID_CAP + 1) + 2;
  L.mid_cap = n / (n_d + 1) + 2;
  // rows: sum of p over the segments of one level (p = 1 + [len > n_d*2^8] + ...)
  L.hist_rows = MAX_PASSES + L.max_segs;
  for (uint64_t cap = (uint64_t)n_d << 8; cap < n; cap <<= 8) L.hist_rows += n / (cap + 1) + 1;
  L.tiles_max = 2 * (n / TILE) + L.max_segs + 2;
  if (fuse && L.tiles_max < 65536) L.tiles_max = 65536;  // the fused pass: one tile per s-run
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  L.b_keys = take(n * kb);
  L.b_vals = vb ? take(n * vb) : 0;
  // fused level 0: A -> C -> B, fused pass B -> A.  Fast Radix: C holds the
  // 256 estimated buckets of ceil(n/256) keys, then overflow chunks (at most
  // n keys in all, plus one partly used chunk per bucket)
  using PhK = Phases<unsigned long long, false>;
  L.fr_cap = (n + 255) / 256;
  L.fr_kmax = n / PhK::FR_CHUNK + 2;
  const size_t c_elems = fr ? 256 * L.fr_cap + n + 256 * (size_t)PhK::FR_CHUNK : n;
  L.c_keys = fuse ? take(c_elems * kb) : 0;
  L.ctl = take(sizeof(Ctl));
  L.segq0 = take(L.max_segs * sizeof(Seg));
  L.segq1 = take(L.max_segs * sizeof(Seg));
  L.midq = take(L.mid_cap * sizeof(MidE));
  L.midq2 = take(L.mid_cap * sizeof(MidE));
  L.hist = take(L.hist_rows * 256 * 4);
  int passes = est_top_passes(n, n_d);  // no group of any level has more passes
  passes = passes < min_passes ? min_passes : (passes > MAX_PASSES ? MAX_PASSES : passes);
  // LB_PAD rows in front: the look-back loads up to DFR_LB rows below tile 0
  L.status = take(((size_t)passes * L.tiles_max + LB_PAD) * 256 * 4);
  L.fh = fuse ? take(65536 * 4) : 0;      // joint histogram of the two low group digits
  L.ftiles = fuse ? take(65536 * 16) : 0;  // run-aligned tiles of the fused pass
  L.fj = fuse ? take(2 * 4096 * 4) : 0;     // chain histogram and bases of the fused pass
  L.fr_ct = fr ? take(256 * L.fr_kmax * 4) : 0;                 // Fast Radix chunk table
  L.fr_tab = fr ? take((2 * (n / TILE) + 2 * 256 + 8) * 8) : 0;  // tiles of the middle pass
  L.fr_cnt = fr ? take(512 * 4) : 0;
  L.total = off;
  return L;
}

template <class K>
static Params<K> make_params(char* ws, const Layout& L, K* keys, uint32_t* vals, bool pairs,
                             uint32_t n_d, uint32_t skip, size_t n) {
  Params<K> P{};
  P.n = (uint32_t)n;
  P.A = keys;
  P.B = reinterpret_cast<K*>(ws + L.b_keys);
  P.Av = vals;
  P.Bv = pairs ? reinterpret_cast<uint32_t*>(ws + L.b_vals) : nullptr;
  P.C = L.c_keys ? reinterpret_cast<K*>(ws + L.c_keys) : nullptr;
  P.Cv = nullptr;
  P.ctl = reinterpret_cast<Ctl*>(ws + L.ctl);
  P.segq[0] = reinterpret_cast<Seg*>(ws + L.segq0);
  P.segq[1] = reinterpret_cast<Seg*>(ws + L.segq1);
  P.midq = reinterpret_cast<MidE*>(ws + L.midq);
  P.midq2 = reinterpret_cast<MidE*>(ws + L.midq2);
  P.hist = reinterpret_cast<uint32_t*>(ws + L.hist);
  P.status = reinterpret_cast<uint32_t*>(ws + L.status) + LB_PAD * 256;
  P.status_stride = L.tiles_max * 256;
  P.H = L.fh ? reinterpret_cast<uint32_t*>(ws + L.fh) : nullptr;
  P.ftiles = L.ftiles ? reinterpret_cast<uint4*>(ws + L.ftiles) : nullptr;
  P.J = L.fj ? reinterpret_cast<uint32_t*>(ws + L.fj) : nullptr;
  P.fr = L.fr_ct ? 1u : 0u;
  P.fr_cap = (uint32_t)L.fr_cap;
  P.fr_kmax = (uint32_t)L.fr_kmax;
  P.fr_ct = L.fr_ct ? reinterpret_cast<uint32_t*>(ws + L.fr_ct) : nullptr;
  P.fr_tab = L.fr_tab ? reinterpret_cast<uint2*>(ws + L.fr_tab) : nullptr;
  P.fr_cnt = L.fr_cnt ? reinterpret_cast<uint32_t*>(ws + L.fr_cnt) : nullptr;
  P.max_segs = (uint32_t)L.max_segs;
  P.mid_cap = (uint32_t)L.mid_cap;
  P.hist_rows = (uint32_t)L.hist_rows;
  P.n_d = n_d;
  P.chunk = WIN - (uint32_t)(16 / sizeof(K)) - n_d;
  P.skip_trivial = skip;
  P.D = (int)sizeof(K);
  return P;
}

static int cfg_nd(const dfr_config* cfg, uint32_t* n_d, uint32_t* skip, uint32_t* nofuse,
                  uint32_t* full_lsd, uint32_t* fast_radix, uint32_t* stable) {
  *stable = 0;
  *n_d = DFR_DEFAULT_ND;
  *skip = 1;
  *nofuse = 0;
  *full_lsd = 0;
  *fast_radix = 0;
  if (cfg) {
    if (cfg->fast_radix > 1 || cfg->stable_deals > 1) return DFR_ERR_INVALID;
    *stable = cfg->stable_deals;
    *fast_radix = cfg->fast_radix;
    if (cfg->full_lsd > 1) return DFR_ERR_INVALID;
    *full_lsd = cfg->full_lsd;
    *n_d = cfg->n_d ? cfg->n_d : DFR_DEFAULT_ND;
    *skip = cfg->skip_trivial_passes ? 1 : 0;
    if (cfg->fused_last_pass > 2) return DFR_ERR_INVALID;
    *nofuse = cfg->fused_last_pass == 2 ? 1 : 0;
  }
  if (*n_d < 8 || *n_d > (uint32_t)MAX_ND) return DFR_ERR_INVALID;
  return DFR_OK;
}

template <class K, bool PAIRS>
static int sort_impl(K* keys, uint32_t* vals, size_t n, cudaStream_t st, const dfr_config* cfg,
                     dfr_stats* stats) {
  using Ph = Phases<K, PAIRS>;
  uint32_t n_d, skip, nofuse, full_lsd, fast_radix, stable;
  if (cfg_nd(cfg, &n_d, &skip, &nofuse, &full_lsd, &fast_radix, &stable) != DFR_OK)
    return DFR_ERR_INVALID;
  if (full_lsd && sizeof(K) > (size_t)MAX_PASSES) return DFR_ERR_INVALID;  // D = 8 > passes a group holds
  if (stats) memset(stats, 0, sizeof(*stats));
  if (n <= 1) return DFR_OK;
  if (!keys || (PAIRS && !vals)) return DFR_ERR_INVALID;
  if (reinterpret_cast<uintptr_t>(keys) % sizeof(K)) return DFR_ERR_INVALID;
  if (PAIRS) {
    if (reinterpret_cast<uintptr_t>(vals) % 4) return DFR_ERR_INVALID;
    const char* ka = reinterpret_cast<const char*>(keys);
    const char* va = reinterpret_cast<const char*>(vals);
    if (ka < va + n * 4 && va < ka + n * sizeof(K)) return DFR_ERR_INVALID;
  }
  if (n > DFR_MAX_N) return DFR_ERR_TOO_LARGE;
  Dev dv;
  if (get_dev<K, PAIRS>(dv) != cudaSuccess) return DFR_ERR_CUDA;
  cudaGetLastError();

  int p0 = est_top_passes(n, n_d);
  if (p0 > (int)sizeof(K) || full_lsd) p0 = (int)sizeof(K);
  // fused last pass (Phases::fused): large keys-only top calls with 3 group
  // digits (s-runs of about n / 2^16 >= 2048 keys fill a tile)
  const bool fuse = !PAIRS && !nofuse && p0 == 3 && n >= ((size_t)1 << 27);
  // Fast Radix estimation (Alg. 3): on the fused level-0 path
  // (a bucket total of exactly 2^30 would read back as 0 from the 30-bit status)
  const bool fr = fuse && fast_radix && !full_lsd && n < DFR_MAX_N;
  const Layout L = make_layout(n, sizeof(K), PAIRS ? 4 : 0, n_d, full_lsd ? (int)sizeof(K) : 1, fuse, fr);
  char* ws = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&ws), L.total, st) != cudaSuccess) {
    cudaGetLastError();
    return DFR_ERR_ALLOC;
  }
  Params<K> P = make_params<K>(ws, L, keys, vals, PAIRS, n_d, skip, n);
  P.fuse = fuse ? 1u : 0u;
  P.full_lsd = full_lsd;
  P.unstable = (!PAIRS && !stable) ? 1u : 0u;
  const uint32_t nn = (uint32_t)n;
  const int sms = dv.sms;
  const PhaseEv pe{cfg ? cfg->phase_events : nullptr, st};

  if (n > (size_t)MID_CAP && n <= (size_t)SMALL_N) {
    // small inputs: every level, level 0 included, in the cooperative
    // k_levels (one launch instead of one per phase)
    for (int i = 0; i < DFR_PHASE_LEVELS; ++i) pe.skip(i);
    pe.begin(DFR_PHASE_LEVELS);
    k_init<K, PAIRS><<<1, THREADS, 64, st>>>(P, nn, 0);
    void* args[] = {&P};
    const uint32_t tiles = (nn + TILE - 1) / TILE;
    const int g_lv = (int)std::min<uint32_t>((uint32_t)(sms * std::max(1, dv.occ_levels)),
                                             std::max<uint32_t>(16u, 2u * tiles));
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_levels<K, PAIRS>, g_lv, THREADS,
                                                args, Ph::SMEM_LEVEL, st);
    pe.end(DFR_PHASE_LEVELS);
    if (e != cudaSuccess) {
      cudaFreeAsync(ws, st);
      return DFR_ERR_CUDA;
    }
    pe.begin(DFR_PHASE_MID);
    launch_mid<K, PAIRS>(dv, st, P);
    pe.end(DFR_PHASE_MID);
    g_launches += 2;
  } else if (n <= (size_t)MID_CAP) {  // the whole input fits one on-chip DFR
    for (int i = 0; i < DFR_PHASE_MID; ++i) pe.skip(i);
    pe.begin(DFR_PHASE_MID);
    k_seed_mid<K, PAIRS><<<1, 1, 0, st>>>(P, nn);
    launch_pdl(k_mid<K, PAIRS>, 1, THREADS, Ph::SMEM_MID, st, P, 0);
    pe.end(DFR_PHASE_MID);
    g_launches += 2;
  } else {
    const uint32_t tiles = (nn + TILE - 1) / TILE;
    const int g_hist = (int)std::min<uint32_t>(tiles, (uint32_t)(sms * std::max(1, dv.occ_hist)));
    const int g_sc = (int)std::min<uint32_t>(tiles, (uint32_t)(sms * std::max(1, dv.occ_scatter)));
    pe.begin(DFR_PHASE_HIST);
    k_init<K, PAIRS><<<1, THREADS, 64, st>>>(P, nn);
    if (fr) {  // Fast Radix: no histogram read of the input
      launch_pdl(k_fr_prep<K>, 4 * sms, THREADS, 0, st, P);
    } else {
      launch_pdl(k_hist<K, PAIRS>, g_hist, THREADS, Ph::SMEM_HIST, st, P);
    }
    pe.end(DFR_PHASE_HIST);
    pe.begin(DFR_PHASE_PLAN);
    if (!fr) launch_pdl(k_plan2<K, PAIRS>, 1, THREADS, 64, st, P);
    pe.end(DFR_PHASE_PLAN);
    for (int j = 0; j < MAX_PASSES; ++j) {
      if (j >= p0) {
        pe.skip(DFR_PHASE_SCATTER0 + j);
        continue;
      }
      pe.begin(DFR_PHASE_SCATTER0 + j);
      if (fr && j < 2) {  // the estimated pass, its plan, the pass reading the estimated layout
        if (j == 0) {
          launch_pdl(k_scatter_fr<K>, g_sc, Ph::SC_NT, Ph::SMEM_SCATTER_P, st, P, 0);
          launch_pdl(k_fr_plan<K>, 1, THREADS, 0, st, P);
        } else {
          const int g_fr = sms * std::max(1, dv.occ_scatter);
          launch_pdl(k_scatter_frfh<K>, g_fr, Ph::SC_NT, Ph::SMEM_SCATTER_P, st, P, 1);
        }
        g_launches += j == 0 ? 2 : 1;
        pe.end(DFR_PHASE_SCATTER0 + j);
        continue;
      }
      if (fuse && j == 2) {  // run-aligned tiles, then the fused last deal + diversion
        if (!fr) launch_pdl(k_hfix<K, PAIRS>, 256, 256, 0, st, P);
        launch_pdl(k_fplan<K, PAIRS>, 1, 1024, 0, st, P);
        const int g_f = sms * std::max(1, dv.occ_fused);
        launch_pdl(k_fused<K, PAIRS>, g_f, Ph::GNT, Ph::SMEM_FUSED_X, st, P);
        g_launches += fr ? 2 : 3;
      }
      if (fuse && j == 1 && !PAIRS)
        launch_pdl(k_scatter_fh<K>, g_sc, Ph::SC_NT, Ph::SMEM_SCATTER_P, st, P, j);
      else
        launch_pdl(k_scatter<K, PAIRS>, g_sc, Ph::SC_NT, Ph::SMEM_SCATTER_P, st, P, j);  // no-op when fused
      pe.end(DFR_PHASE_SCATTER0 + j);
    }
    const uint32_t chunks = (nn + P.chunk - 1) / P.chunk;
    const int g_dv = (int)std::min<uint32_t>(chunks, (uint32_t)(sms * std::max(1, dv.occ_divert)));
    pe.begin(DFR_PHASE_DIVERT);
    launch_pdl(k_divert<K, PAIRS>, g_dv, Ph::DV_NT, Ph::SMEM_DIVERT, st, P);
    pe.end(DFR_PHASE_DIVERT);
    pe.begin(DFR_PHASE_LEVELS);
    // level 1 through the stand-alone kernels (large recursions: c3, c4,
    // c5-low20 put most of their keys there), levels 2.. in k_levels
#if DFR_LEVEL1_CHAIN
    launch_pdl(k_lplan<K, PAIRS>, 1, THREADS, 64, st, P);
    launch_pdl(k_hist<K, PAIRS>, g_hist, THREADS, Ph::SMEM_HIST, st, P);
    launch_pdl(k_plan2<K, PAIRS>, 4 * sms, THREADS, 64, st, P);  // one block per segment
    for (int j = 0; j < MAX_PASSES; ++j)
      launch_pdl(k_scatter<K, PAIRS>, g_sc, Ph::SC_NT, Ph::SMEM_SCATTER_P, st, P, j);
    launch_pdl(k_divert<K, PAIRS>, g_dv, Ph::DV_NT, Ph::SMEM_DIVERT, st, P);
    g_launches += 4 + MAX_PASSES;
#endif
    void* args[] = {&P};
    const int g_lv = sms * std::max(1, dv.occ_levels);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_levels<K, PAIRS>, g_lv, THREADS,
                                                args, Ph::SMEM_LEVEL, st);
    pe.end(DFR_PHASE_LEVELS);
    if (e != cudaSuccess) {
      cudaFreeAsync(ws, st);
      return DFR_ERR_CUDA;
    }
    pe.begin(DFR_PHASE_MID);
    launch_mid<K, PAIRS>(dv, st, P);
    pe.end(DFR_PHASE_MID);
    g_launches += 5 + p0;
  }
  cudaError_t e = cudaGetLastError();
  int rc = (e == cudaSuccess) ? DFR_OK : DFR_ERR_CUDA;
  if (stats && rc == DFR_OK) {
    Ctl h;
    if (cudaMemcpyAsync(&h, P.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = DFR_ERR_CUDA;
    } else {
      stats->level0_p = h.level0_p;
      stats->level0_passes_run = h.level0_run;
      stats->level0_large = h.level0_large;
      stats->mid_buckets = h.mid_buckets;
      stats->global_segments = h.global_segments;
      stats->levels = h.levels_run;
      stats->overflow = h.overflow;
      stats->fused = h.fused_ok;
      stats->fr_overflow = h.fr_overflow;
    }
  }
  if (cudaFreeAsync(ws, st) != cudaSuccess && rc == DFR_OK) rc = DFR_ERR_CUDA;
  return rc;
}

// stage API helpers
template <class K, bool PAIRS>
static int stage_impl(const K* in, const uint32_t* vin, K* out, uint32_t* vout, size_t n,
                      int digit_lo, int p, uint32_t* d_counts, cudaStream_t st) {
  using Ph = Phases<K, PAIRS>;
  if (n == 0) return DFR_OK;
  if (n > DFR_MAX_N) return DFR_ERR_TOO_LARGE;
  if (!in || p < 1 || p > MAX_PASSES || digit_lo < 0 || digit_lo + p > (int)sizeof(K))
    return DFR_ERR_INVALID;
  Dev dv;
  if (get_dev<K, PAIRS>(dv) != cudaSuccess) return DFR_ERR_CUDA;
  cudaGetLastError();
  const Layout L = make_layout(n, 0, 0, 64, MAX_PASSES);
  char* ws = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&ws), L.total, st) != cudaSuccess) {
    cudaGetLastError();
    return DFR_ERR_ALLOC;
  }
  Params<K> P = make_params<K>(ws, L, const_cast<K*>(in), const_cast<uint32_t*>(vin), PAIRS, 64, 0, n);
  P.B = out;  // pass 0 deals A=in -> B=out
  P.Bv = vout;
  const uint32_t nn = (uint32_t)n;
  const uint32_t tiles = (nn + TILE - 1) / TILE;
  k_init_stage<K, PAIRS><<<1, THREADS, 0, st>>>(P, nn, digit_lo, p);
  DFR_CHECK_LAUNCH("k_init_stage");
  g_launches += d_counts ? 2 : 4;
  const int g_hist = (int)std::min<uint32_t>(tiles, (uint32_t)(dv.sms * std::max(1, dv.occ_hist)));
  k_hist<K, PAIRS><<<g_hist, THREADS, Ph::SMEM_HIST, st>>>(P);
  DFR_CHECK_LAUNCH("k_hist(stage)");
  if (d_counts) {
    cudaMemcpyAsync(d_counts, P.hist, (size_t)p * 256 * 4, cudaMemcpyDeviceToDevice, st);
  } else {
    k_plan2<K, PAIRS><<<1, THREADS, 64, st>>>(P);
    DFR_CHECK_LAUNCH("k_plan2(stage)");
    const int g_sc = (int)std::min<uint32_t>(tiles, (uint32_t)(dv.sms * std::max(1, dv.occ_scatter)));
    k_scatter<K, PAIRS><<<g_sc, Ph::SC_NT, Ph::SMEM_SCATTER_P, st>>>(P, 0);
    DFR_CHECK_LAUNCH("k_scatter(stage)");
  }
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(ws, st);
  return e == cudaSuccess ? DFR_OK : DFR_ERR_CUDA;
}

// (u64 key, u64 value) records (SPEC's 16-byte Record): the keys are
// sorted stably with their u32 input positions as the payload (the pairs
// path), then the values follow through that permutation.
__global__ void k_iota(uint32_t* v, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}
__global__ void k_gather_u64(const unsigned long long* src, const uint32_t* idx, unsigned long long* dst,
                             uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

static int sort_pairs_u64(unsigned long long* keys, unsigned long long* vals, size_t n, cudaStream_t st,
                          const dfr_config* cfg, dfr_stats* stats) {
  if (stats) memset(stats, 0, sizeof(*stats));
  if (n <= 1) return DFR_OK;
  if (!keys || !vals) return DFR_ERR_INVALID;
  if ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(vals)) % 8) return DFR_ERR_INVALID;
  {
    const char* ka = reinterpret_cast<const char*>(keys);
    const char* va = reinterpret_cast<const char*>(vals);
    if (ka < va + n * 8 && va < ka + n * 8) return DFR_ERR_INVALID;
  }
  if (n > DFR_MAX_N) return DFR_ERR_TOO_LARGE;
  Dev dv;
  if (get_dev<unsigned long long, true>(dv) != cudaSuccess) return DFR_ERR_CUDA;
  char* ws = nullptr;
  const size_t idx_bytes = align_up(n * 4);
  if (cudaMallocAsync(reinterpret_cast<void**>(&ws), idx_bytes + n * 8, st) != cudaSuccess) {
    cudaGetLastError();
    return DFR_ERR_ALLOC;
  }
  uint32_t* idx = reinterpret_cast<uint32_t*>(ws);
  unsigned long long* tmp = reinterpret_cast<unsigned long long*>(ws + idx_bytes);
  const int grid = 4 * dv.sms;
  k_iota<<<grid, 256, 0, st>>>(idx, (uint32_t)n);
  int rc = sort_impl<unsigned long long, true>(keys, idx, n, st, cfg, stats);
  if (rc == DFR_OK) {
    k_gather_u64<<<grid, 256, 0, st>>>(vals, idx, tmp, (uint32_t)n);
    if (cudaMemcpyAsync(vals, tmp, n * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess) rc = DFR_ERR_CUDA;
    g_launches += 2;
    if (rc == DFR_OK && cudaGetLastError() != cudaSuccess) rc = DFR_ERR_CUDA;
  }
  if (cudaFreeAsync(ws, st) != cudaSuccess && rc == DFR_OK) rc = DFR_ERR_CUDA;
  return rc;
}

}  // namespace dfr

// -------------------------------------------------------------------- C ABI
extern "C" {

int dfr_sort_u32_ex(uint32_t* d_keys, size_t n, dfr_stream_t stream, const dfr_config* cfg,
                    dfr_stats* stats) {
  return dfr::sort_impl<uint32_t, false>(d_keys, nullptr, n, (cudaStream_t)stream, cfg, stats);
}
int dfr_sort_u64_ex(uint64_t* d_keys, size_t n, dfr_stream_t stream, const dfr_config* cfg,
                    dfr_stats* stats) {
  return dfr::sort_impl<unsigned long long, false>(reinterpret_cast<unsigned long long*>(d_keys),
                                                   nullptr, n, (cudaStream_t)stream, cfg, stats);
}
int dfr_sort_pairs_u32_ex(uint32_t* d_keys, uint32_t* d_vals, size_t n, dfr_stream_t stream,
                          const dfr_config* cfg, dfr_stats* stats) {
  return dfr::sort_impl<uint32_t, true>(d_keys, d_vals, n, (cudaStream_t)stream, cfg, stats);
}
int dfr_sort_u32(uint32_t* d_keys, size_t n, dfr_stream_t stream) {
  return dfr_sort_u32_ex(d_keys, n, stream, nullptr, nullptr);
}
int dfr_sort_u64(uint64_t* d_keys, size_t n, dfr_stream_t stream) {
  return dfr_sort_u64_ex(d_keys, n, stream, nullptr, nullptr);
}
int dfr_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_vals, size_t n, dfr_stream_t stream) {
  return dfr_sort_pairs_u32_ex(d_keys, d_vals, n, stream, nullptr, nullptr);
}
int dfr_sort_pairs_u64_ex(uint64_t* d_keys, uint64_t* d_vals, size_t n, dfr_stream_t stream,
                          const dfr_config* cfg, dfr_stats* stats) {
  return dfr::sort_pairs_u64(reinterpret_cast<unsigned long long*>(d_keys),
                             reinterpret_cast<unsigned long long*>(d_vals), n, (cudaStream_t)stream, cfg,
                             stats);
}
int dfr_sort_pairs_u64(uint64_t* d_keys, uint64_t* d_vals, size_t n, dfr_stream_t stream) {
  return dfr_sort_pairs_u64_ex(d_keys, d_vals, n, stream, nullptr, nullptr);
}

int dfr_histogram_u32(const uint32_t* d_keys, size_t n, int digit_lo, int p, uint32_t* d_counts,
                      dfr_stream_t stream) {
  if (!d_counts) return DFR_ERR_INVALID;
  return dfr::stage_impl<uint32_t, false>(d_keys, nullptr, nullptr, nullptr, n, digit_lo, p,
                                          d_counts, (cudaStream_t)stream);
}
int dfr_histogram_u64(const uint64_t* d_keys, size_t n, int digit_lo, int p, uint32_t* d_counts,
                      dfr_stream_t stream) {
  if (!d_counts) return DFR_ERR_INVALID;
  return dfr::stage_impl<unsigned long long, false>(
      reinterpret_cast<const unsigned long long*>(d_keys), nullptr, nullptr, nullptr, n, digit_lo,
      p, d_counts, (cudaStream_t)stream);
}
int dfr_partition_pass_u64(const uint64_t* d_in, uint64_t* d_out, size_t n, int d,
                           dfr_stream_t stream) {
  if (n && (!d_in || !d_out || d_in == d_out)) return DFR_ERR_INVALID;
  return dfr::stage_impl<unsigned long long, false>(
      reinterpret_cast<const unsigned long long*>(d_in), nullptr,
      reinterpret_cast<unsigned long long*>(d_out), nullptr, n, d, 1, nullptr,
      (cudaStream_t)stream);
}
int dfr_partition_pass_pairs_u32(const uint32_t* d_keys_in, const uint32_t* d_vals_in,
                                 uint32_t* d_keys_out, uint32_t* d_vals_out, size_t n, int d,
                                 dfr_stream_t stream) {
  if (n && (!d_keys_in || !d_keys_out || d_keys_in == d_keys_out)) return DFR_ERR_INVALID;
  if ((d_vals_in == nullptr) != (d_vals_out == nullptr)) return DFR_ERR_INVALID;
  if (d_vals_in)
    return dfr::stage_impl<uint32_t, true>(d_keys_in, d_vals_in, d_keys_out, d_vals_out, n, d, 1,
                                           nullptr, (cudaStream_t)stream);
  return dfr::stage_impl<uint32_t, false>(d_keys_in, nullptr, d_keys_out, nullptr, n, d, 1,
                                          nullptr, (cudaStream_t)stream);
}

uint64_t dfr_launch_counter(void) { return dfr::g_launches.load(); }

#ifdef DFR_FPROF
int dfr_debug_fprof(uint64_t* out16) {
  return cudaMemcpyFromSymbol(out16, dfr::g_fprof, 16 * sizeof(uint64_t)) == cudaSuccess ? 0 : -3;
}
#endif
#ifdef DFR_LB_STATS
int dfr_debug_lb_stats(uint64_t* out4) {
  return cudaMemcpyFromSymbol(out4, dfr::g_lb_stats, 4 * sizeof(uint64_t)) == cudaSuccess ? 0 : -3;
}
#endif

int dfr_top_passes(size_t n, int key_bytes, uint32_t n_d) {
  if (n_d == 0) n_d = DFR_DEFAULT_ND;
  int p = dfr::est_top_passes(n, n_d);
  return p > key_bytes ? key_bytes : p;
}

size_t dfr_workspace_bytes(size_t n, int key_bytes, int val_bytes) {
  return dfr::make_layout(n, key_bytes, val_bytes, DFR_DEFAULT_ND).total;
}

const char* dfr_status_string(int status) {
  switch (status) {
    case DFR_OK: return "DFR_OK";
    case DFR_ERR_INVALID: return "DFR_ERR_INVALID";
    case DFR_ERR_ALLOC: return "DFR_ERR_ALLOC";
    case DFR_ERR_CUDA: return "DFR_ERR_CUDA";
    case DFR_ERR_TOO_LARGE: return "DFR_ERR_TOO_LARGE";
    default: return "DFR_ERR_UNKNOWN";
  }
}

}  // extern "C"
