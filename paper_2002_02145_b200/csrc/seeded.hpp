// Counter-based seeded generator shared by host and device code
// (SURVEY.md §7.2 step 1, §8d "Synthetic inputs"):
//   value(seed, i) = (int)(splitmix64(splitmix64(seed) ^ i) >> 40) * 2^-23 - 1
// i is the LOGICAL NCHW / KCRS index, so tensors do not depend on layout or on
// how the minibatch is sharded. Every value k*2^-23 - 1 (k < 2^24) is exact in
// fp32 and lies in [-1, 1).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define PSCONV_HD __host__ __device__ __forceinline__
#else
#define PSCONV_HD inline
#endif

namespace psconv {
namespace seeded {

PSCONV_HD uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
PSCONV_HD uint64_t mix(uint64_t seed) { return splitmix64(seed); }
// key = mix(seed)
PSCONV_HD float value(uint64_t key, uint64_t i) {
  const uint64_t z = splitmix64(key ^ i);
  return static_cast<float>(static_cast<int32_t>(z >> 40)) * (1.0f / 8388608.0f) - 1.0f;
}

}  // namespace seeded
}  // namespace psconv
