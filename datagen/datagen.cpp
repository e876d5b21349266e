// datagen — seeded synthetic inputs shared by the oracle tests, the GPU parity
// tests and bench.py.  This module holds NONE of the sorting method's
// arithmetic (no digits, counts, scans, deals or diversion): it only draws
// keys.  Layout/ordering helpers (sorted, reverse, nearly sorted, sorted runs)
// use the C++ standard library sort as a black-box primitive to build the
// input layouts that BASELINE.json names.
//
// Generator: SplitMix64 (Steele, Lea, Flood 2014).  The i-th output of a
// stream with initial state `k` is  mix(k + (i+1)*GAMMA)  — counter-based, so
// any draw can be produced independently (OpenMP-parallel fill).
//   GAMMA = 0x9E3779B97F4A7C15
//   mix(z): z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
//           z *= 0x94D049BB133111EB; z ^= z>>31
// Stream key for (seed, name): mix(seed*GAMMA ^ fnv1a64(name)).
// u01 = (draw >> 11) * 2^-53   (top 53 bits).
//
// Distribution recipes (DESIGN.md §"Input recipe"):
//   uniform u64     key_i = draw_i
//   uniform u32     key_i = draw_i >> 32
//   normal          Marsaglia polar method (§3.1 names it),
//                   key = clamp(mean + round(sd*z)) computed in integers
//   exponential     key = round(-scale * ln(1 - u01))
//   zipf            V[1..U] distinct draws; rank r by inverse CDF of r^-s
//   few-unique      T[0..k) distinct draws; key_i = T[draw_i mod-free index]
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <parallel/algorithm>
#include <string>
#include <unordered_set>
#include <vector>

namespace {
constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ull;

inline uint64_t mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
inline uint64_t draw(uint64_t key, uint64_t i) { return mix(key + (i + 1) * GAMMA); }
inline double u01(uint64_t d) { return (double)(d >> 11) * 0x1.0p-53; }

uint64_t fnv1a64(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ull;
  }
  return h;
}

// mean + round(delta) with saturation to [0, 2^64-1], delta a finite double.
uint64_t add_clamped(uint64_t mean, double delta) {
  double ad = std::nearbyint(std::fabs(delta));
  if (ad >= 0x1.0p64) return delta >= 0 ? ~0ull : 0ull;
  uint64_t a = (uint64_t)ad;
  if (delta >= 0) return (a > ~0ull - mean) ? ~0ull : mean + a;
  return (a > mean) ? 0ull : mean - a;
}
}  // namespace

extern "C" {

uint64_t dg_mix(uint64_t z) { return mix(z); }
uint64_t dg_stream_key(uint64_t seed, const char* name) { return mix(seed * GAMMA ^ fnv1a64(name)); }
uint64_t dg_draw(uint64_t key, uint64_t i) { return draw(key, i); }

void dg_uniform_u64(uint64_t* out, size_t n, uint64_t seed, const char* stream) {
  const uint64_t k = dg_stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) out[i] = draw(k, i);
}

void dg_uniform_u32(uint32_t* out, size_t n, uint64_t seed, const char* stream) {
  const uint64_t k = dg_stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)(draw(k, i) >> 32);
}

// keys uniform over [0, 2^bits)
void dg_lowbits_u64(uint64_t* out, size_t n, uint64_t seed, const char* stream, int bits) {
  const uint64_t k = dg_stream_key(seed, stream);
  const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) out[i] = draw(k, i) & mask;
}

// Marsaglia polar method: u,v uniform in (-1,1), s = u^2+v^2, reject s>=1 or
// s==0, z1 = u*sqrt(-2 ln s / s), z2 = v*sqrt(...); both outputs used in order.
void dg_normal_u64(uint64_t* out, size_t n, uint64_t seed, const char* stream, uint64_t mean,
                   double sd) {
  const uint64_t k = dg_stream_key(seed, stream);
  uint64_t c = 0;
  size_t i = 0;
  while (i < n) {
    double u = 2.0 * u01(draw(k, c++)) - 1.0;
    double v = 2.0 * u01(draw(k, c++)) - 1.0;
    double s = u * u + v * v;
    if (s >= 1.0 || s == 0.0) continue;
    double f = std::sqrt(-2.0 * std::log(s) / s);
    out[i++] = add_clamped(mean, sd * (u * f));
    if (i < n) out[i++] = add_clamped(mean, sd * (v * f));
  }
}

void dg_exponential_u64(uint64_t* out, size_t n, uint64_t seed, const char* stream, double scale) {
  const uint64_t k = dg_stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) {
    double x = -scale * std::log1p(-u01(draw(k, i)));
    out[i] = add_clamped(0, x);
  }
}

// Zipf over `universe` distinct random 64-bit values V[1..U] (stream
// "<stream>-values", duplicates rejected in draw order); rank r has
// probability r^-s / H; rank drawn by inverse CDF (binary search on the
// cumulative weights) with u01 from stream "<stream>".
void dg_zipf_u64(uint64_t* out, size_t n, uint64_t seed, const char* stream, double s,
                 size_t universe) {
  std::string vname = std::string(stream) + "-values";
  const uint64_t kv = dg_stream_key(seed, vname.c_str());
  std::vector<uint64_t> V;
  V.reserve(universe);
  std::unordered_set<uint64_t> seen;
  seen.reserve(universe * 2);
  for (uint64_t c = 0; V.size() < universe; ++c) {
    uint64_t x = draw(kv, c);
    if (seen.insert(x).second) V.push_back(x);
  }
  std::vector<double> cdf(universe);
  double acc = 0.0;
  for (size_t r = 0; r < universe; ++r) {
    acc += std::pow((double)(r + 1), -s);
    cdf[r] = acc;
  }
  const double total = acc;
  const uint64_t k = dg_stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) {
    double t = u01(draw(k, i)) * total;
    size_t r = (size_t)(std::upper_bound(cdf.begin(), cdf.end(), t) - cdf.begin());
    if (r >= universe) r = universe - 1;
    out[i] = V[r];
  }
}

// `distinct` distinct random u32 values T (stream "<stream>-values", dedup in
// draw order); key_i = T[(draw_i >> 32) * distinct >> 32]  (uniform choice).
void dg_few_unique_u32(uint32_t* out, size_t n, uint64_t seed, const char* stream,
                       uint32_t distinct) {
  std::string vname = std::string(stream) + "-values";
  const uint64_t kv = dg_stream_key(seed, vname.c_str());
  std::vector<uint32_t> T;
  std::unordered_set<uint32_t> seen;
  for (uint64_t c = 0; T.size() < distinct; ++c) {
    uint32_t x = (uint32_t)(draw(kv, c) >> 32);
    if (seen.insert(x).second) T.push_back(x);
  }
  const uint64_t k = dg_stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) out[i] = T[((draw(k, i) >> 32) * (uint64_t)distinct) >> 32];
}

void dg_const_u32(uint32_t* out, size_t n, uint64_t seed, const char* stream) {
  const uint32_t c = (uint32_t)(draw(dg_stream_key(seed, stream), 0) >> 32);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) out[i] = c;
}

void dg_iota_u32(uint32_t* out, size_t n) {
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)i;
}

// ---- layouts (library sort used as a primitive to build the layout) -------
void dg_sort_asc_u64(uint64_t* a, size_t n) { __gnu_parallel::sort(a, a + n); }
void dg_reverse_u64(uint64_t* a, size_t n) { std::reverse(a, a + n); }
// `swaps` random transpositions (i, j) drawn from the stream, applied in order.
void dg_transpose_u64(uint64_t* a, size_t n, uint64_t seed, const char* stream, size_t swaps) {
  if (n < 2) return;
  const uint64_t k = dg_stream_key(seed, stream);
  for (size_t t = 0; t < swaps; ++t) {
    size_t i = (size_t)(((unsigned __int128)draw(k, 2 * t) * n) >> 64);
    size_t j = (size_t)(((unsigned __int128)draw(k, 2 * t + 1) * n) >> 64);
    std::swap(a[i], a[j]);
  }
}
// sort each consecutive block of `run` keys ascending
void dg_sort_runs_u64(uint64_t* a, size_t n, size_t run) {
  const size_t nb = (n + run - 1) / run;
#pragma omp parallel for schedule(dynamic, 64)
  for (size_t b = 0; b < nb; ++b) {
    size_t lo = b * run, hi = std::min(n, lo + run);
    std::sort(a + lo, a + hi);
  }
}

// Order-independent multiset fingerprint: (sum h1(x), sum h2(x)) mod 2^64 over
// the `n` words of `elem_bytes` (4 or 8) bytes each.  Used only to check that
// a large output is a permutation of its input.
void dg_fingerprint(const void* p, size_t n, int elem_bytes, uint64_t out[2]) {
  uint64_t s1 = 0, s2 = 0;
#pragma omp parallel for schedule(static) reduction(+ : s1, s2)
  for (size_t i = 0; i < n; ++i) {
    uint64_t x = elem_bytes == 8 ? ((const uint64_t*)p)[i] : ((const uint32_t*)p)[i];
    s1 += mix(x ^ 0x243F6A8885A308D3ull);
    s2 += mix(x * 0x13198A2E03707344ull + 0xA4093822299F31D0ull);
  }
  out[0] = s1;
  out[1] = s2;
}

// 1 if non-decreasing, else 0
int dg_is_sorted_u64(const uint64_t* a, size_t n) {
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(& : ok)
  for (size_t i = 1; i < n; ++i) ok &= (a[i - 1] <= a[i]);
  return ok;
}
int dg_is_sorted_u32(const uint32_t* a, size_t n) {
  int ok = 1;
#pragma omp parallel for schedule(static) reduction(& : ok)
  for (size_t i = 1; i < n; ++i) ok &= (a[i - 1] <= a[i]);
  return ok;
}

}  // extern "C"
