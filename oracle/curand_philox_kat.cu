// oracle/curand_philox_kat.cu -- TEST INFRASTRUCTURE ONLY.
// Host-side run of cuRAND's own Philox4x32-10 block function
// (curand_philox4x32_x.h: curand_Philox4x32_10) to produce known-answer
// vectors that pin the oracle's and the product's independent Philox
// restatements.  Built and run by oracle/make_golden.py (nvcc, no GPU needed).
#define QUALIFIERS static __forceinline__ __host__ __device__
#include <curand_philox4x32_x.h>

#include <cstdint>
#include <cstdio>

static std::uint64_t sm(std::uint64_t& s) {  // splitmix64 to spread test inputs
  std::uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int main() {
  std::uint64_t s = 12345;
  // Random123's published vectors first, then 256 spread inputs.
  uint4 c0[3] = {{0, 0, 0, 0},
                 {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu},
                 {0x243f6a88u, 0x85a308d3u, 0x13198a2eu, 0x03707344u}};
  uint2 k0[3] = {{0, 0}, {0xffffffffu, 0xffffffffu}, {0xa4093822u, 0x299f31d0u}};
  for (int i = 0; i < 3 + 256; ++i) {
    uint4 c;
    uint2 k;
    if (i < 3) {
      c = c0[i];
      k = k0[i];
    } else {
      std::uint64_t a = sm(s), b = sm(s), e = sm(s);
      c = make_uint4(std::uint32_t(a), std::uint32_t(a >> 32), std::uint32_t(b),
                     std::uint32_t(b >> 32));
      k = make_uint2(std::uint32_t(e), std::uint32_t(e >> 32));
      if (i % 4 == 0) c.x = i, c.y = 0;  // small counters like the sampler's
    }
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%u %u %u %u %u %u %u %u %u %u\n", c.x, c.y, c.z, c.w, k.x, k.y, r.x, r.y,
                r.z, r.w);
  }
  return 0;
}
