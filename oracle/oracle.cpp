// oracle — plain, slow, obviously-correct single-threaded CPU implementation
// of Diverting Fast Radix (DFR), arXiv 2207.14334 ("ThielSort").
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  It
// shares no code, header, table or helper with the CUDA product path
// (paper_2207_14334_b200/), and neither side includes the other.
//
// Citations: P:L = /root/reference/PAPER.md line L; S:L = SPEC.md line L.
//
// What it computes, step by step in the paper's order:
//   counting_sort_pass  P:118-120 §2 (count -> exclusive prefix -> stable deal
//                       "buff[index[N[i].key]++] = N") for one digit.
//   dfr_rec             P:252-275 §3 Alg. 4:
//     l.2  buffer the size of the input                     (allocated once)
//     l.4  estimate the top passes p  = least p >= 0 with len <= N_d * M^p
//          (integer arithmetic; reading E3/E4 in DESIGN.md), capped at
//          the remaining digits, re-estimated per call (reading E5)
//     l.6  LSD radix sort on those top p digits (Alg. 1), least
//          significant of the group first
//     l.7-13 scan for large buckets (size > N_d, reading E2); on a large
//          bucket first divert the pending run of small buckets (insertion
//          sort) then recurse on the large bucket with the
//          remaining digits
//     l.14 divert the trailing run of small buckets
//   Alg. 2 l.6-8: a bucket of size <= N_d is diverted at once
//     (reading E12: p = 0 means exactly this).
//   Alg. 2 l.17-18: digits exhausted => all keys of the bucket are
//     equal => already sorted.
//
// Every pass, shift and copy moves the payload with its key; every step is
// stable, so the result is THE stable sort of the input by key.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

extern "C" {
// Mirrors nothing in the product; plain counters for control-flow checks.
struct oracle_stats {
  uint64_t passes;            // counting-sort passes executed (all levels)
  uint64_t skippable_passes;  // of those, passes whose histogram had one non-empty bin
  uint64_t diversions;        // insertion-sort calls (bulk runs)
  uint64_t diverted_records;  // records sorted by insertion sort
  uint64_t large_buckets;     // recursive calls on large buckets
  uint64_t max_depth;         // deepest recursion level (top call = 0)
  uint64_t level0_p;          // top passes at the top call
  uint64_t level0_large;      // large buckets found at the top call
  uint64_t count_ops;         // per-record digit counts
  uint64_t deal_ops;          // per-record placements in counting passes
};
}

namespace {

template <typename K>
inline unsigned digit_of(K key, int d, int r) {
  return (unsigned)((key >> (d * r)) & (((K)1 << r) - 1));
}

// least p >= 0 with len <= n_d * M^p, evaluated in integers
int est_top_passes(uint64_t len, int r, uint64_t n_d) {
  int p = 0;
  unsigned __int128 cap = n_d;
  while ((unsigned __int128)len > cap) {
    cap <<= r;
    ++p;
  }
  return p;
}

template <typename K, typename V>
struct Dfr {
  K* key;
  V* val;  // may be null (keys only)
  K* skey;
  V* sval;
  int r;         // radix bits
  int D;         // digits per key
  uint64_t n_d;  // diversion threshold N_d
  oracle_stats* st;

  // insertion sort, strict '>' so equal keys keep their order (stable)
  void insertion_sort(uint64_t lo, uint64_t len) {
    for (uint64_t i = lo + 1; i < lo + len; ++i) {
      K x = key[i];
      V v = val ? val[i] : V();
      uint64_t j = i;
      while (j > lo && key[j - 1] > x) {
        key[j] = key[j - 1];
        if (val) val[j] = val[j - 1];
        --j;
      }
      key[j] = x;
      if (val) val[j] = v;
    }
    st->diversions++;
    st->diverted_records += len;
  }

  // one stable counting-sort pass on digit d over [lo, lo+len)
  void counting_sort_pass(uint64_t lo, uint64_t len, int d) {
    const unsigned M = 1u << r;
    std::vector<uint64_t> count(M, 0), index(M, 0);
    for (uint64_t i = lo; i < lo + len; ++i) count[digit_of(key[i], d, r)]++;  // count
    uint64_t nonempty = 0;
    for (unsigned b = 0; b < M; ++b) nonempty += count[b] != 0;
    uint64_t run = 0;  // convert counts into indices (exclusive prefix)
    for (unsigned b = 0; b < M; ++b) {
      index[b] = run;
      run += count[b];
    }
    for (uint64_t i = lo; i < lo + len; ++i) {  // deal: buff[index[key]++] = record
      uint64_t dst = lo + index[digit_of(key[i], d, r)]++;
      skey[dst] = key[i];
      if (val) sval[dst] = val[i];
    }
    std::memcpy(key + lo, skey + lo, len * sizeof(K));  // back into place
    if (val) std::memcpy(val + lo, sval + lo, len * sizeof(V));
    st->passes++;
    st->count_ops += len;
    st->deal_ops += len;
    if (nonempty == 1) st->skippable_passes++;
  }

  // Alg. 4 on [lo, lo+len) whose keys share all digits above `hi`
  void rec(uint64_t lo, uint64_t len, int hi, uint64_t depth) {
    if (depth > st->max_depth) st->max_depth = depth;
    if (len <= n_d) {  // Alg. 2 l.6-8 / reading E12
      if (len > 0) insertion_sort(lo, len);
      return;
    }
    if (hi < 0) return;  // digits exhausted: all keys equal (Alg. 2 l.17-18)
    int p = est_top_passes(len, r, n_d);  // Alg. 4 l.4
    if (p > hi + 1) p = hi + 1;
    for (int d = hi - p + 1; d <= hi; ++d) counting_sort_pass(lo, len, d);  // Alg. 4 l.6
    const int low = hi - p + 1;  // lowest digit of the group
    const int shift = r * low;
    uint64_t large_here = 0;
    // Alg. 4 l.7-14: scan buckets of equal top-p prefix
    uint64_t i = lo, run = lo;
    const uint64_t end = lo + len;
    while (i < end) {
      const K prefix = key[i] >> shift;
      uint64_t j = i + 1;
      while (j < end && (key[j] >> shift) == prefix) ++j;
      if (j - i > n_d) {                               // a large bucket
        if (run < i) insertion_sort(run, i - run);  // l.10: divert previous small buckets
        rec(i, j - i, low - 1, depth + 1);          // l.11: recurse on the large bucket
        st->large_buckets++;
        large_here++;
        run = j;
      }
      i = j;
    }
    if (run < end) insertion_sort(run, end - run);  // l.14
    if (depth == 0) {
      st->level0_p = (uint64_t)p;
      st->level0_large = large_here;
    }
  }
};

template <typename K, typename V>
int run_dfr(K* key, V* val, uint64_t n, int r, uint64_t n_d, oracle_stats* st) {
  if (r != 4 && r != 8 && r != 16) return -1;
  if ((int)(8 * sizeof(K)) % r) return -1;
  if (n_d < 1) return -1;
  oracle_stats local;
  if (!st) st = &local;
  std::memset(st, 0, sizeof(*st));
  // Alg. 4 l.2: a buffer the size of the input (inside the caller's timing)
  K* skey = n ? (K*)std::malloc(n * sizeof(K)) : nullptr;
  V* sval = (val && n) ? (V*)std::malloc(n * sizeof(V)) : nullptr;
  if (n && (!skey || (val && !sval))) {
    std::free(skey);
    std::free(sval);
    return -2;
  }
  Dfr<K, V> s{key, val, skey, sval, r, (int)(8 * sizeof(K)) / r, n_d, st};
  s.rec(0, n, s.D - 1, 0);
  std::free(skey);
  std::free(sval);
  return 0;
}

// counts of digits digit_lo .. digit_lo+p-1 (radix 8), out[p][256]
template <typename K>
void hist_impl(const K* keys, uint64_t n, int digit_lo, int p, uint32_t* out) {
  std::memset(out, 0, sizeof(uint32_t) * 256 * (size_t)p);
  for (uint64_t i = 0; i < n; ++i)
    for (int j = 0; j < p; ++j) out[j * 256 + digit_of(keys[i], digit_lo + j, 8)]++;
}
// the top-level group only: p = est(n) capped, LSD passes over digits
// hi-p+1..hi (radix 8), in place; returns p.  Values may be null.
template <typename K>
int group_impl(K* keys, uint32_t* vals, uint64_t n, uint64_t n_d, oracle_stats* st) {
  oracle_stats local;
  if (!st) st = &local;
  std::memset(st, 0, sizeof(*st));
  std::vector<K> sk(n);
  std::vector<uint32_t> sv(vals ? n : 0);
  Dfr<K, uint32_t> s{keys, vals, sk.data(), vals ? sv.data() : nullptr, 8, (int)sizeof(K), n_d,
                     st};
  int hi = s.D - 1;
  int p = est_top_passes(n, 8, n_d);
  if (p > hi + 1) p = hi + 1;
  for (int d = hi - p + 1; d <= hi; ++d) s.counting_sort_pass(0, n, d);
  return p;
}
}  // namespace

extern "C" {

int oracle_est_top_passes(uint64_t n, int radix_bits, uint64_t n_d) {
  return est_top_passes(n, radix_bits, n_d);
}

uint64_t oracle_extract_digit_u64(uint64_t key, int d, int radix_bits) {
  return digit_of<uint64_t>(key, d, radix_bits);
}

// exclusive prefix sum of m counts ("convert the count into indices")
void oracle_prefix_sum_exclusive(const uint64_t* counts, uint64_t* out, uint64_t m) {
  uint64_t run = 0;
  for (uint64_t b = 0; b < m; ++b) {
    out[b] = run;
    run += counts[b];
  }
}

int oracle_dfr_u32(uint32_t* keys, uint64_t n, int radix_bits, uint64_t n_d, oracle_stats* st) {
  return run_dfr<uint32_t, uint32_t>(keys, nullptr, n, radix_bits, n_d, st);
}
int oracle_dfr_u64(uint64_t* keys, uint64_t n, int radix_bits, uint64_t n_d, oracle_stats* st) {
  return run_dfr<uint64_t, uint32_t>(keys, nullptr, n, radix_bits, n_d, st);
}
int oracle_dfr_pairs_u32(uint32_t* keys, uint32_t* vals, uint64_t n, int radix_bits,
                         uint64_t n_d, oracle_stats* st) {
  return run_dfr<uint32_t, uint32_t>(keys, vals, n, radix_bits, n_d, st);
}
int oracle_dfr_pairs_u64(uint64_t* keys, uint64_t* vals, uint64_t n, int radix_bits,
                         uint64_t n_d, oracle_stats* st) {
  return run_dfr<uint64_t, uint64_t>(keys, vals, n, radix_bits, n_d, st);
}

// insertion sort alone (the diversion sort)
void oracle_insertion_sort_pairs_u64(uint64_t* keys, uint64_t* vals, uint64_t n) {
  oracle_stats st;
  std::memset(&st, 0, sizeof st);
  Dfr<uint64_t, uint64_t> s{keys, vals, nullptr, nullptr, 8, 8, 64, &st};
  if (n) s.insertion_sort(0, n);
}

// ---- stage API for incremental kernel parity ---------

void oracle_hist_u32(const uint32_t* k, uint64_t n, int digit_lo, int p, uint32_t* out) {
  hist_impl(k, n, digit_lo, p, out);
}
void oracle_hist_u64(const uint64_t* k, uint64_t n, int digit_lo, int p, uint32_t* out) {
  hist_impl(k, n, digit_lo, p, out);
}

int oracle_group_u32(uint32_t* k, uint32_t* v, uint64_t n, uint64_t n_d, oracle_stats* st) {
  return group_impl(k, v, n, n_d, st);
}
int oracle_group_u64(uint64_t* k, uint64_t n, uint64_t n_d, oracle_stats* st) {
  return group_impl<uint64_t>(k, nullptr, n, n_d, st);
}

// one stable counting pass on digit d (radix 8), in place
int oracle_pass_u64(uint64_t* k, uint64_t n, int d) {
  oracle_stats st;
  std::memset(&st, 0, sizeof st);
  std::vector<uint64_t> sk(n);
  Dfr<uint64_t, uint32_t> s{k, nullptr, sk.data(), nullptr, 8, 8, 64, &st};
  if (n) s.counting_sort_pass(0, n, d);
  return 0;
}
int oracle_pass_pairs_u32(uint32_t* k, uint32_t* v, uint64_t n, int d) {
  oracle_stats st;
  std::memset(&st, 0, sizeof st);
  std::vector<uint32_t> sk(n), sv(n);
  Dfr<uint32_t, uint32_t> s{k, v, sk.data(), sv.data(), 8, 4, 64, &st};
  if (n) s.counting_sort_pass(0, n, d);
  return 0;
}

// Classify the buckets of an array already grouped by the top-p-digit prefix
// (p digits ending at digit D-1) into small (<= n_d), mid (n_d < s <= cap)
// and large (> cap); out = {n_buckets, small, mid, large, records_in_mid,
// records_in_large}.
void oracle_level_buckets_u64(const uint64_t* k, uint64_t n, int p, uint64_t n_d, uint64_t cap,
                              uint64_t out[6]) {
  std::memset(out, 0, 6 * sizeof(uint64_t));
  const int shift = 8 * (8 - p);
  uint64_t i = 0;
  while (i < n) {
    uint64_t pre = shift >= 64 ? 0 : k[i] >> shift;
    uint64_t j = i + 1;
    while (j < n && (shift >= 64 ? 0 : k[j] >> shift) == pre) ++j;
    uint64_t s = j - i;
    out[0]++;
    if (s <= n_d)
      out[1]++;
    else if (s <= cap) {
      out[2]++;
      out[4] += s;
    } else {
      out[3]++;
      out[5] += s;
    }
    i = j;
  }
}

}  // extern "C"
