/*
 * dfr.h — C ABI of the B200-native Diverting Fast Radix (DFR) sort.
 *
 * Method: PAPER.md (arXiv 2207.14334, "ThielSort") §3 Alg. 4:
 * estimate the top passes p (read as SPEC S:284: least p >= 0 with
 * n <= N_d * 256^p), run an LSD radix sort over those top p digits (
 * each pass = count -> exclusive prefix -> stable deal, §2),
 * scan for large buckets, divert runs of small buckets to a simple
 * stable sort (insertion-sort semantics P:194), recurse on
 * large buckets with the remaining digits.  Radix M = 256
 * (P:324), N_d = 64.  Every step is stable, so the result is
 * THE stable sort of the input by key.
 *
 * All entry points:
 *   - take DEVICE pointers owned by the caller (never freed by the library);
 *   - sort ascending, in place: on return-and-stream-sync the sorted data is
 *     in the caller's buffer(s);
 *   - are asynchronous and stream-ordered on `stream` (0 = legacy default
 *     stream); they perform no host<->device copy and no host synchronisation
 *     (except the _ex variants when `stats` is non-NULL, which synchronise
 *     `stream` to read the counters back);
 *   - allocate their scratch (a buffer the size of the input, Alg. 4
 *     l.2, plus counters/queues) with cudaMallocAsync/cudaFreeAsync on
 *     `stream` inside the call (the paper times allocation);
 *   - are reentrant: concurrent calls on distinct streams and buffers are safe.
 *
 * Errors: 0 (DFR_OK) or a negative code below.  Kernel execution faults
 * surface at the caller's next synchronisation (CUDA convention).  No C++
 * exception crosses the ABI.
 */
#ifndef DFR_H_
#define DFR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dfr_stream_t; /* == cudaStream_t */

enum {
  DFR_OK = 0,
  DFR_ERR_INVALID = -1,   /* NULL pointer with n > 0, misaligned element pointer,
                             overlapping keys/values, or a bad dfr_config field */
  DFR_ERR_ALLOC = -2,     /* scratch allocation failed (SPEC's "resource error") */
  DFR_ERR_CUDA = -3,      /* a CUDA launch/configuration error (cudaGetLastError) */
  DFR_ERR_TOO_LARGE = -4  /* n > 2^30 = 256^3.75, the paper's largest N: look-back
                             counts are packed in 30 bits and summed mod 2^30 */
};

/* Limits of this build. */
#define DFR_MAX_N ((size_t)1 << 30) /* inclusive */
#define DFR_RADIX_BITS 8            /* M = 256 */
#define DFR_DEFAULT_ND 64           /* diversion threshold N_d */

/* Optional configuration for the _ex entry points (NULL = defaults). */
typedef struct dfr_config {
  uint32_t n_d;         /* diversion threshold N_d: 0 = default 64, else 8 <= n_d <= 256
                           (other values: DFR_ERR_INVALID) */
  uint32_t skip_trivial_passes; /* 1 (default): skip a pass whose digit histogram has
                                   one non-empty bin — the identity permutation
                                   ("skipping unneeded passes"); 0: run every
                                   pass as Alg. 4 l.6 writes it.  Output identical. */
  void* const* phase_events; /* NULL, or 2*DFR_NUM_PHASES cudaEvent_t handles created by the
                                caller: events[2i] / events[2i+1] are recorded on `stream`
                                before / after phase i (see DFR_PHASE_*); a phase that does
                                not run records both back to back.  No synchronisation. */
  uint32_t fused_last_pass; /* 0 (default) or 1: a large keys-only top call (p = 3,
                               n >= 2^27) runs its last deal and the diversion of the
                               resulting buckets (Alg. 4 l.6 + l.7-14) as ONE kernel
                               over tiles made of whole runs of the two lower group
                               digits, through a second scratch buffer (A -> C -> B,
                               fused B -> A), so the keys move once instead of twice.
                               Same output; on the device it falls back to the
                               separate deal + diversion when a run is longer than a
                               tile (4608 keys) or a group pass was skipped.
                               2: always the separate deal and diversion kernels.
                               Other values: DFR_ERR_INVALID. */
  uint32_t full_lsd;        /* 0 (default).  1: ablation (SPEC AC7): the top call
                               runs a plain LSD radix sort over ALL D digits (p = D, no
                               diversion, no recursion).  u32 keys and u32 pairs only
                               (D = 4); DFR_ERR_INVALID for u64 keys.  Inputs of at most
                               4096 keys still run the on-chip DFR. */
  uint32_t fast_radix;      /* 0 (default).  1: Fast Radix estimation (§3, Alg. 3,
                               P:211-246) on the fused level-0 path (keys only, p = 3,
                               n >= 2^27; ignored elsewhere): the pass on the lowest group
                               digit deals into estimated buckets of ceil(n/256) keys
                               with overflow chunks instead of reading a histogram first,
                               counting the middle digit; the middle pass reads bucket by
                               bucket and counts the top digit (the top digit counted in the
                               penultimate pass, Alg. 3 l.5-6).  No pass is skipped.
                               Same output. */
  uint32_t stable_deals;    /* 0 (default): keys-only sorts rank the keys of equal digit in
                               any order inside a deal tile that is constant in the group
                               digits below the dealt one (always true for the group's
                               lowest digit) — shared-memory atomics instead of the stable
                               ballot multi-split.  Same output: equal keys are
                               indistinguishable, the group's later passes are stable and
                               every bucket is then sorted on all lower digits (DESIGN.md
                               R5).  1: every deal is the stable counting pass of P:118-120.
                               Pairs always deal stably.  Other values: DFR_ERR_INVALID. */
} dfr_config;

/* Phases timed through dfr_config.phase_events. */
enum {
  DFR_PHASE_HIST = 0,     /* k_init + k_hist: one read, p digit histograms (Alg. 4 l.4-5) */
  DFR_PHASE_PLAN = 1,     /* counts -> bucket offsets */
  DFR_PHASE_SCATTER0 = 2, /* stable deal of group pass j at DFR_PHASE_SCATTER0 + j, j < 4 */
  DFR_PHASE_DIVERT = 6,   /* scan for large buckets + small-bucket sort (Alg. 4 l.7-14) */
  DFR_PHASE_LEVELS = 7,   /* recursion levels >= 1 (Alg. 4 l.11) */
  DFR_PHASE_MID = 8,      /* buckets N_d < s <= 4096 finished on-chip */
  DFR_NUM_PHASES = 9
};

/* Optional device-side counters, read back (with a stream sync) by _ex. */
typedef struct dfr_stats {
  uint32_t level0_p;          /* top passes p at the top call (Alg. 4 l.4) */
  uint32_t level0_passes_run; /* of those, passes actually executed (not skipped) */
  uint64_t level0_large;      /* buckets > N_d found by the level-0 scan (l.8-9) */
  uint64_t mid_buckets;       /* buckets N_d < s <= 4096 finished on-chip (all levels) */
  uint64_t global_segments;   /* buckets > 4096 recursed through the global queue */
  uint32_t levels;            /* recursion levels executed after level 0 */
  uint32_t overflow;          /* device queue overflow flags (0 = none; non-zero = bug) */
  uint32_t fused;             /* 1: the top call ran the fused last deal + diversion */
  uint32_t fr_overflow;       /* Fast Radix: records the estimated pass dealt to overflow
                                 space (beyond their bucket's estimated capacity) */
} dfr_stats;

/*
 * Sort n uint32 keys at d_keys (4-byte aligned device pointer) in place.
 * Digits: D = 4 (u32).  Returns DFR_OK for n <= 1 without launching.
 */
int dfr_sort_u32(uint32_t* d_keys, size_t n, dfr_stream_t stream);

/* Sort n uint64 keys at d_keys (8-byte aligned device pointer) in place. D = 8. */
int dfr_sort_u64(uint64_t* d_keys, size_t n, dfr_stream_t stream);

/*
 * Stable sort of n (uint32 key, uint32 value) pairs held as two arrays
 * (SoA).  d_vals[i] moves with d_keys[i]; equal keys keep their input order
 * (stability).  Keys and values must not overlap.
 */
int dfr_sort_pairs_u32(uint32_t* d_keys, uint32_t* d_vals, size_t n, dfr_stream_t stream);

/*
 * Stable sort of n (uint64 key, uint64 value) records held as two arrays
 * (SoA; SPEC's 16-byte Record key + tag).  d_vals[i] moves with
 * d_keys[i]; equal keys keep their input order.  Keys and values must
 * not overlap; both 8-byte aligned.  The keys are sorted with their uint32
 * input positions as the payload (the pairs path), then the values follow that
 * permutation (a gather into scratch and a copy back).
 */
int dfr_sort_pairs_u64(uint64_t* d_keys, uint64_t* d_vals, size_t n, dfr_stream_t stream);

/* Same as above with a configuration and optional stats (stats != NULL
 * synchronises `stream`). */
int dfr_sort_u32_ex(uint32_t* d_keys, size_t n, dfr_stream_t stream, const dfr_config* cfg,
                    dfr_stats* stats);
int dfr_sort_u64_ex(uint64_t* d_keys, size_t n, dfr_stream_t stream, const dfr_config* cfg,
                    dfr_stats* stats);
int dfr_sort_pairs_u32_ex(uint32_t* d_keys, uint32_t* d_vals, size_t n, dfr_stream_t stream,
                          const dfr_config* cfg, dfr_stats* stats);
int dfr_sort_pairs_u64_ex(uint64_t* d_keys, uint64_t* d_vals, size_t n, dfr_stream_t stream,
                          const dfr_config* cfg, dfr_stats* stats);

/*
 * Stage entry points, exported so each kernel can be checked against the
 * oracle in isolation.  All take device pointers and run on `stream`.
 *
 * dfr_histogram_u32/u64: counts of digits digit_lo .. digit_lo+p-1 (radix 256,
 *   digit 0 least significant) over n keys into d_counts[p][256]
 *   (uint32, overwritten).  1 <= p <= 4, digit_lo + p <= D.
 * dfr_partition_pass_u64 / _pairs_u32: ONE stable counting-sort pass
 *    on digit d: d_in -> d_out (distinct buffers, n elements);
 *   d_vals_in/out may be NULL for keys-only u32 use of the pairs variant.
 */
int dfr_histogram_u32(const uint32_t* d_keys, size_t n, int digit_lo, int p, uint32_t* d_counts,
                      dfr_stream_t stream);
int dfr_histogram_u64(const uint64_t* d_keys, size_t n, int digit_lo, int p, uint32_t* d_counts,
                      dfr_stream_t stream);
int dfr_partition_pass_u64(const uint64_t* d_in, uint64_t* d_out, size_t n, int d,
                           dfr_stream_t stream);
int dfr_partition_pass_pairs_u32(const uint32_t* d_keys_in, const uint32_t* d_vals_in,
                                 uint32_t* d_keys_out, uint32_t* d_vals_out, size_t n, int d,
                                 dfr_stream_t stream);

/*
 * Monte Carlo of the Fast Radix overflow model (§3.1, P:292-306;
 * Alg. 3): each of `trials` experiments throws n records into m
 * buckets uniformly at random and writes its overflow against the estimated
 * capacity ceil(n/m),  sum_i max(0, count_i - ceil(n/m)),  to d_overflow[t]
 * (device array of `trials` uint64, caller-owned).  Random numbers: SplitMix64
 * counter-based: trial t's stream key is mix(key + (t+1)*GAMMA) and record b
 * goes to bucket hi32(mix(k_t + (b+1)*GAMMA)) * m >> 32 (GAMMA =
 * 0x9E3779B97F4A7C15).  1 <= m <= 16384; trials == 0 is a no-op.
 * Asynchronous on `stream`; DFR_ERR_INVALID for a NULL array or m out of range.
 */
int dfr_overflow_mc(uint64_t n, uint32_t m, uint32_t trials, uint64_t key, uint64_t* d_overflow,
                    dfr_stream_t stream);

/* Number of top passes the planner uses for n keys (Alg. 4 l.4), capped at D. */
int dfr_top_passes(size_t n, int key_bytes, uint32_t n_d);

/* Bytes of scratch one call allocates for n elements of the given widths. */
size_t dfr_workspace_bytes(size_t n, int key_bytes, int val_bytes);

/* Total kernel launches issued by this library in this process (monotonic). */
uint64_t dfr_launch_counter(void);

/* Static string for a status code. */
const char* dfr_status_string(int status);

#ifdef __cplusplus
}
#endif
#endif /* DFR_H_ */
