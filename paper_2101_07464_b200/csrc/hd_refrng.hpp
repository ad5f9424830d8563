// Host-side restatement of the reference's RandomSource (random.hpp:21-112,
// random.cpp:10-188) for HD_DRAWS_REFERENCE operators and the hd_rs_* C-ABI:
// xoshiro256++ seeded by splitmix64, streams as 2^128 jumps, Marsaglia polar
// normal() and the 256-strip ziggurat normal_vector(). A reference user who
// switches gets the same Gaussian stream — hence the same matrix — for the
// same (seed, stream).
//
// The ziggurat stream is sequential (rejections consume a data-dependent
// number of words), so it runs on the host; normal_vector(a) followed by
// normal_vector(b) equals normal_vector(a + b) (test_random.cpp:90-98), which
// lets the operator treat the draws as one flat stream.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>

namespace hd {
namespace refrng {

inline uint64_t splitmix_next(uint64_t& x) {  // random.cpp:11-16
  uint64_t z = (x += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

inline uint64_t derive_seed(uint64_t base, uint64_t index) {  // random.cpp:73-76
  uint64_t s = base + index * 0x9e3779b97f4a7c15ULL;
  return splitmix_next(s);
}

inline double bits_to_double(uint64_t b) {
  double d;
  std::memcpy(&d, &b, sizeof d);
  return d;
}

inline uint64_t double_to_bits(double d) {
  uint64_t b;
  std::memcpy(&b, &d, sizeof b);
  return b;
}

class Source {
 public:
  Source(uint64_t seed, uint64_t stream) {  // random.cpp:78-81,101-104
    uint64_t x = seed;
    for (auto& w : s_) w = splitmix_next(x);
    for (uint64_t i = 0; i < stream; ++i) jump();
  }

  uint64_t next() {  // random.hpp:25-35
    const uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
  }

  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // [0, 1)

  // Defined in hd_refrng.cpp, compiled with the reference's own flags
  // (-O3 -mavx2 -mfma, CMakeLists.txt:7,24-41): GCC then contracts the same
  // multiply-adds into FMAs the reference binary does, keeping the stream
  // bit-identical.
  double normal();                               // random.cpp:106-121 (polar)
  void normal_fill(double* out, int64_t len);    // random.cpp:130-176 (ziggurat)
  // experiments.cpp:19-29: 0 with probability rho, else sigma_s * normal()
  void bernoulli_gaussian(double* out, int64_t n, double rho, double sigma_s);

 private:
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

  void jump() {  // random.cpp:83-99: advance 2^128 words
    static constexpr uint64_t J[4] = {0x180ec6d33cfd0abaULL, 0xd5a61266f0c9392cULL, 0xa9582618e03fc9aaULL,
                                      0x39abdc4529b1661cULL};
    uint64_t acc[4] = {0, 0, 0, 0};
    for (uint64_t word : J)
      for (int b = 0; b < 64; ++b) {
        if ((word >> b) & 1ULL)
          for (int i = 0; i < 4; ++i) acc[i] ^= s_[i];
        next();
      }
    for (int i = 0; i < 4; ++i) s_[i] = acc[i];
  }

  uint64_t s_[4];
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

}  // namespace refrng
}  // namespace hd
