// One-kernel NVLink exchange + fused average / update (see p2p_exchange.cu).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace hdp {

constexpr int P2P_MAX_RANKS = 8;
constexpr int P2P_MAX_BUCKETS = 16;
// per-rank flag block (unsigned words)
constexpr int P2P_FLAG_READY = 0;    // [8]: rank r's gradients of step s complete
constexpr int P2P_FLAG_DONE = 32;    // [8]: rank r's owned shards written everywhere
constexpr int P2P_CTR = 64;          // this rank's CTA completion counter (monotonic)
constexpr int P2P_STATUS = 96;       // [2] ints: non-finite count of step s in slot s & 1
constexpr int P2P_FLAG_WORDS = 128;

struct P2PArgs {
  // N = gradient contributions summed (and weight copies written); NR = ranks in the
  // flag protocol.  Across processes N = NR = world.  Loopback (world 1, N simulated
  // workers): the contributions are the local gradient slots, the weight copies local
  // buffers, and the protocol runs with NR = 1.
  int N = 1, NR = 1, rank = 0;
  unsigned step = 0;
  int nb = 0;
  long off[P2P_MAX_BUCKETS] = {}, shard[P2P_MAX_BUCKETS] = {}, moff[P2P_MAX_BUCKETS] = {};
  long vpre[P2P_MAX_BUCKETS + 1] = {};   // prefix sums of owned 8-element vectors per bucket
  const __half* g_peer[P2P_MAX_RANKS] = {};
  __half* w_peer[P2P_MAX_RANKS] = {};
  unsigned* flag_peer[P2P_MAX_RANKS] = {};
  int* status_peer[P2P_MAX_RANKS] = {};
  unsigned* flag_local = nullptr;
  float *W = nullptr, *S1 = nullptr, *S2 = nullptr;
  float inv_scale = 1.f, lam = 0.f, mom = 0.f;
  float b1 = 0.9f, omb1 = 0.1f, b2 = 0.999f, omb2 = 0.001f, c1 = 1.f, c2 = 1.f, eps = 1e-8f;
  float l2x2 = 0.f;  // fp32(2 * l2), see UpdateArgs
  const float* alpha_dev = nullptr;  // dynamic loss scaling, see UpdateArgs
  double n_workers = 1.0;
  const int* skip = nullptr;
};

cudaError_t launch_exch_update(const P2PArgs& a, int optimizer, int grid, cudaStream_t s);

}  // namespace hdp
