// Variational recurrent dropout mask (NEXT-3; "recurrent dropout"; DESIGN.md
// reading Q16b).  A counter-based hash of (seed, step, layer, sequence, unit), all
// arithmetic mod 2^32 -- the definition oracle/dropout.py implements independently:
//   mix32(x): x ^= x >> 16; x *= 0x7FEB352D; x ^= x >> 15; x *= 0x846CA68B; x ^= x >> 16
//   k1 = mix32(seed ^ mix32(step)); k2 = mix32(k1 ^ layer * 0x9E3779B9)
//   k3 = mix32(k2 ^ seq * 0x85EBCA6B); r = mix32(k3 ^ unit * 0xC2B2AE35); kept iff r < thr
#pragma once
#include <cstdint>

namespace hdp {

__host__ __device__ __forceinline__ uint32_t drop_mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}
// key of (seed, step, layer): one per launch
__host__ __device__ __forceinline__ uint32_t drop_layer_key(uint32_t seed, uint32_t step, uint32_t layer) {
  return drop_mix32(drop_mix32(seed ^ drop_mix32(step)) ^ (layer * 0x9E3779B9u));
}
// key of a sequence: one per batch row
__host__ __device__ __forceinline__ uint32_t drop_seq_key(uint32_t layer_key, uint32_t seq) {
  return drop_mix32(layer_key ^ (seq * 0x85EBCA6Bu));
}
__host__ __device__ __forceinline__ bool drop_kept(uint32_t seq_key, uint32_t unit, uint32_t thr) {
  return drop_mix32(seq_key ^ (unit * 0xC2B2AE35u)) < thr;
}

}  // namespace hdp
