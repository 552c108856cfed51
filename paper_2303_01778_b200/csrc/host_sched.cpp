// Host-side native runtime: greedy scheduler core and NumPy-compatible
// minibatch permutations.  Compiled with -ffp-contract=off (no FMA fusion of
// N*t + b), so plans are bit-identical to the reference's numba kernel
// (fedsim/schedule.py:88-126).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "parrot_b200.h"

namespace pb {
void set_error(const std::string& msg);
}

extern "C" int pb_greedy_assign(const double* sizes_desc, int64_t n, const double* t,
                                const double* b, int64_t k, int64_t* assign, double* loads) {
  if (n < 0 || k < 1 || (n > 0 && (!sizes_desc || !assign)) || !t || !b || !loads) {
    pb::set_error("pb_greedy_assign: bad arguments");
    return PB_ERR_INVALID;
  }
  const double inf = std::numeric_limits<double>::infinity();
  for (int64_t j = 0; j < k; ++j) loads[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    // top-two current loads (strict > keeps the lowest id on ties)
    double top = -inf, second = -inf;
    int64_t top_dev = -1;
    for (int64_t j = 0; j < k; ++j) {
      const double l = loads[j];
      if (l > top) {
        second = top;
        top = l;
        top_dev = j;
      } else if (l > second) {
        second = l;
      }
    }
    int64_t pick = -1;
    double pick_span = inf, pick_load = inf;
    for (int64_t j = 0; j < k; ++j) {
      volatile double prod = sizes_desc[i] * t[j];  // keep the product rounded
      double cost = prod + b[j];
      if (cost < 0.0) cost = 0.0;
      const double after = loads[j] + cost;
      const double others = (j == top_dev) ? second : top;
      const double span = after > others ? after : others;
      if (span < pick_span || (span == pick_span && after < pick_load)) {
        pick = j;
        pick_span = span;
        pick_load = after;
      }
    }
    assign[i] = pick;
    loads[pick] = pick_load;
  }
  return PB_OK;
}

// ---------------------------------------------------------------------------
// NumPy Generator(PCG64(SeedSequence(entropy))).permutation(n), bit-exact.
//   SeedSequence: numpy/random/bit_generator.pyx (mix_entropy, generate_state)
//   PCG64 XSL-RR 128/64: state = state*MULT + inc; output from the new state
//   permutation: Fisher-Yates from the top, j = random_interval(i) with a
//   power-of-two mask and rejection on buffered 32-bit draws.
// ---------------------------------------------------------------------------
namespace {

using u128 = unsigned __int128;

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

struct Pcg64 {
  u128 state = 0, inc = 0;
  bool has32 = false;
  uint32_t buf32 = 0;

  static constexpr u128 mult() {
    return (u128(0x2360ED051FC65DA4ull) << 64) | u128(0x4385DF649FCCF645ull);
  }
  void step() { state = state * mult() + inc; }
  uint64_t next64() {
    step();
    const uint64_t hi = uint64_t(state >> 64), lo = uint64_t(state);
    const unsigned rot = unsigned(state >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const uint64_t v = next64();
    has32 = true;
    buf32 = uint32_t(v >> 32);
    return uint32_t(v);
  }
  uint64_t interval(uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    uint64_t v;
    if (max <= 0xffffffffull) {
      do { v = next32() & mask; } while (v > max);
    } else {
      do { v = next64() & mask; } while (v > max);
    }
    return v;
  }
};

void entropy_words(const uint64_t* keys, int nkeys, std::vector<uint32_t>& out) {
  out.clear();
  for (int i = 0; i < nkeys; ++i) {
    uint64_t v = keys[i];
    if (v == 0) {
      out.push_back(0);
      continue;
    }
    while (v) {
      out.push_back(uint32_t(v & 0xffffffffu));
      v >>= 32;
    }
  }
}

Pcg64 seeded(const uint64_t* keys, int nkeys) {
  std::vector<uint32_t> ent;
  entropy_words(keys, nkeys, ent);
  uint32_t pool[4];
  uint32_t h = kInitA;
  auto hashmix = [&h](uint32_t v) {
    v ^= h;
    h *= kMultA;
    v *= h;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    return r ^ (r >> 16);
  };
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < int(ent.size()) ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (size_t s = 4; s < ent.size(); ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  // generate_state(4, uint64): 8 uint32 words, paired little-endian
  uint32_t w[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  uint64_t s64[4];
  for (int i = 0; i < 4; ++i) s64[i] = uint64_t(w[2 * i]) | (uint64_t(w[2 * i + 1]) << 32);
  const u128 initstate = (u128(s64[0]) << 64) | u128(s64[1]);
  const u128 initseq = (u128(s64[2]) << 64) | u128(s64[3]);
  Pcg64 g;
  g.state = 0;
  g.inc = (initseq << 1) | 1u;
  g.step();
  g.state += initstate;
  g.step();
  return g;
}

void client_rows(const uint64_t* key, int64_t n, int epochs, int64_t base, int32_t* out) {
  Pcg64 g = seeded(key, 4);
  std::vector<int64_t> perm(size_t(n > 0 ? n : 0));
  for (int e = 0; e < epochs; ++e) {
    for (int64_t j = 0; j < n; ++j) perm[size_t(j)] = j;
    for (int64_t i = n - 1; i >= 1; --i) {
      const int64_t j = int64_t(g.interval(uint64_t(i)));
      std::swap(perm[size_t(i)], perm[size_t(j)]);
    }
    int32_t* o = out + int64_t(e) * n;
    for (int64_t j = 0; j < n; ++j) o[j] = int32_t(base + perm[size_t(j)]);
  }
}

}  // namespace

extern "C" int pb_minibatch_rows(const uint64_t* keys, const int64_t* n, const int64_t* offset,
                                 const int64_t* row_base, int64_t g, int epochs, int32_t* out,
                                 int threads) {
  if (g < 0 || epochs < 1 || (g > 0 && (!keys || !n || !offset || !row_base || !out))) {
    pb::set_error("pb_minibatch_rows: bad arguments");
    return PB_ERR_INVALID;
  }
  for (int64_t i = 0; i < g; ++i)
    if (n[i] < 0 || row_base[i] + n[i] > int64_t(INT32_MAX)) {
      pb::set_error("pb_minibatch_rows: row ids exceed int32");
      return PB_ERR_INVALID;
    }
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) client_rows(keys + 4 * i, n[i], epochs, row_base[i], out + offset[i]);
  };
  int nt = threads > 0 ? threads : 1;
  if (nt > 64) nt = 64;
  if (nt == 1 || g < 2 * nt) {
    work(0, g);
    return PB_OK;
  }
  std::vector<std::thread> pool;
  const int64_t chunk = (g + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(g, lo + chunk);
    if (lo < hi) pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  return PB_OK;
}
