// SPSA direction draws for a block of batch rows (host side of
// vqc_spsa_signs, include/vqc.h). The reference gives every row its own
// generator, numpy.random.default_rng(mix_seed(seed, global_row))
// (batch.py:75-81, 197), and draws `rng.integers(0, 2, size=C)` once per
// sample (gradients.py:180-201). To stay bit-identical with it this file
// restates the published algorithms numpy pins for default_rng:
//   * SeedSequence (O'Neill's seed_seq_fe128 variant: 4-word pool, hashmix /
//     mix constants below) for an integer entropy with an empty spawn key,
//   * PCG64 (128-bit LCG, XSL-RR output), seeded with generate_state(4, u64),
//   * bounded integers through Lemire's multiply-shift on buffered 32-bit
//     draws; for the half-open range [0, 2) that is bit 31 of each draw and
//     the rejection threshold is 0.
// tests/test_methods.py compares it with numpy itself (CPU, no GPU).
#include <cstdint>

namespace {

using u128 = unsigned __int128;

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

inline uint32_t hashmix(uint32_t v, uint32_t* h) {
  v ^= *h;
  *h *= kMultA;
  v *= *h;
  return v ^ (v >> 16);
}

inline uint32_t mix(uint32_t x, uint32_t y) {
  const uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

struct Pcg64 {
  u128 state, inc;
  bool has32;
  uint32_t hold;

  void step() { state = state * ((u128(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull) + inc; }

  // default_rng(entropy): entropy is a non-negative integer < 2^64
  explicit Pcg64(uint64_t entropy) : has32(false), hold(0) {
    const uint32_t words[2] = {(uint32_t)entropy, (uint32_t)(entropy >> 32)};
    const int nw = words[1] != 0 ? 2 : 1;
    uint32_t pool[4], h = kInitA;
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nw ? words[i] : 0u, &h);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], &h));
    uint64_t v[4];
    uint32_t g = kInitB;
    for (int i = 0; i < 8; ++i) {
      uint32_t x = pool[i & 3] ^ g;
      g *= kMultB;
      x *= g;
      x ^= x >> 16;
      if (i & 1) v[i >> 1] |= (uint64_t)x << 32;
      else v[i >> 1] = x;
    }
    const u128 init = (u128(v[0]) << 64) | v[1], seq = (u128(v[2]) << 64) | v[3];
    state = 0;
    inc = (seq << 1) | 1;
    step();
    state += init;
    step();
  }

  uint64_t next64() {
    step();
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned r = (unsigned)(state >> 122);
    return (x >> r) | (x << ((64 - r) & 63));
  }

  uint32_t next32() {
    if (has32) {
      has32 = false;
      return hold;
    }
    const uint64_t n = next64();
    has32 = true;
    hold = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
};

inline uint64_t mix_seed(uint64_t seed, uint64_t index) {  // batch.py:75-81 (splitmix64 step)
  uint64_t z = seed + (index + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" int vqc_spsa_signs(uint64_t seed, int64_t row0, int64_t rows, int64_t samples, int64_t cols,
                              int per_row_seed, int8_t* out) {
  if (rows < 0 || samples < 0 || cols < 0 || row0 < 0 || (rows * samples * cols > 0 && out == nullptr)) return -1;
  const int64_t per = samples * cols;
  for (int64_t r = 0; r < rows; ++r) {
    Pcg64 g(per_row_seed ? mix_seed(seed, (uint64_t)(row0 + r)) : seed);
    int8_t* o = out + r * per;
    for (int64_t i = 0; i < per; ++i) o[i] = (g.next32() >> 31) ? 1 : -1;
  }
  return 0;
}
