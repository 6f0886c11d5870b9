// f2v_rng.h -- counter-based streams shared by host C++ and sm_100a device code.
//
// * SplitMix (the reference's own Rng, proj/core/include/force2vec/rng.hpp:12-53).
//   Its state after k draws is s0 + k*gamma, so draw k of a stream is the
//   closed form mix(s0 + (k+1)*gamma): any draw is O(1) on the device.
// * Philox4x32-10 (Salmon et al. SC'11), the BASELINE configs' negative
//   sampler.  Counter layout:
//     key = {lo32(seed), hi32(seed)}
//     ctr = {k, lo32(batch), epoch, hi16(batch)<<16 | shard}
//     index = hi64(u64(out.y:out.x) * n)
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define F2V_HD __host__ __device__ __forceinline__
#else
#define F2V_HD inline
#endif

namespace f2v {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;
constexpr uint64_t kStreamInit = 0x11;       // trainer.cpp:27
constexpr uint64_t kStreamPartition = 0x22;  // trainer.cpp:28
constexpr uint64_t kStreamSampling = 0x33;   // trainer.cpp:29

F2V_HD uint64_t mix64(uint64_t z) {  // rng.hpp:44-49
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

F2V_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Rng(seed, stream) initial state (rng.hpp:14-15)
F2V_HD uint64_t rng_init(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed) ^ mix64(stream ^ kGamma));
}
// Rng::keyed folding (rng.hpp:18-24), one key element at a time.
F2V_HD uint64_t rng_fold(uint64_t s, uint64_t k) { return mix64(s ^ mix64(k ^ kGamma)); }
F2V_HD uint64_t rng_keyed1(uint64_t seed, uint64_t a) { return rng_fold(mix64(seed), a); }
F2V_HD uint64_t rng_keyed2(uint64_t seed, uint64_t a, uint64_t b) {
  return rng_fold(rng_fold(mix64(seed), a), b);
}
F2V_HD uint64_t rng_keyed3(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return rng_fold(rng_fold(rng_fold(mix64(seed), a), b), c);
}
F2V_HD uint64_t rng_keyed4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return rng_fold(rng_keyed3(seed, a, b, c), d);
}
// draw k (0-based) of a stream whose state is s0 (rng.hpp:26-29 closed form)
F2V_HD uint64_t rng_draw(uint64_t s0, uint64_t k) { return mix64(s0 + (k + 1) * kGamma); }
// below(n) (rng.hpp:39-42)
F2V_HD uint64_t rng_below(uint64_t draw, uint64_t n) { return mulhi64(draw, n); }
// uniform() (rng.hpp:32)
F2V_HD double rng_uniform(uint64_t draw) { return (double)(draw >> 11) * 0x1.0p-53; }

struct Philox4 {
  uint32_t x, y, z, w;
};

F2V_HD Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c.z;
    Philox4 o;
    o.x = (uint32_t)(p1 >> 32) ^ c.y ^ k0;
    o.y = (uint32_t)p1;
    o.z = (uint32_t)(p0 >> 32) ^ c.w ^ k1;
    o.w = (uint32_t)p0;
    c = o;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Negative k of (epoch, batch, shard) under the Philox sampler.
F2V_HD uint32_t philox_negative(uint64_t seed, uint32_t epoch, uint64_t batch, uint32_t shard,
                                uint32_t k, uint32_t n) {
  Philox4 c{k, (uint32_t)batch, epoch, ((uint32_t)(batch >> 32) << 16) | (shard & 0xffffu)};
  const Philox4 r = philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t draw = ((uint64_t)r.y << 32) | r.x;
  return (uint32_t)mulhi64(draw, n);
}

// Negative k under the reference stream: build_minibatch's draw_negatives on
// Rng::keyed(seed, {0x33, epoch, batch}) (trainer.cpp:222-224,
// sampling.cpp:21-25); sharded runs (G > 1) add the shard as a 4th key.
F2V_HD uint32_t splitmix_negative(uint64_t seed, uint32_t epoch, uint64_t batch, uint32_t shard,
                                  uint32_t G, uint32_t k, uint32_t n) {
  const uint64_t s0 = G == 1 ? rng_keyed3(seed, kStreamSampling, epoch, batch)
                             : rng_keyed4(seed, kStreamSampling, epoch, batch, shard);
  return (uint32_t)rng_below(rng_draw(s0, k), n);
}

}  // namespace f2v
