// One-kernel NVLink exchange + fused average / update (see p2p_exchange.cu).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace hdp {

constexpr int P2P_MAX_RANKS = 8;
constexpr int P2P_MAX_BUCKETS = 16;
// per-rank flag block (unsigned words)
constexpr int P2P_FLAG_READY = 0;    // [8]: contributor r's gradients of launch `seq` complete
constexpr int P2P_FLAG_DONE = 32;    // [8]: rank r's owned shards of launch `seq` written everywhere
constexpr int P2P_CTR = 64;          // this rank's CTA completion counter (monotonic)
constexpr int P2P_DECISION = 80;     // 2 words (8-byte aligned): (seq << 32) | contributor mask, from rank 0
constexpr int P2P_STATUS = 96;       // [2] ints: non-finite count of step s in slot s & 1
constexpr int P2P_FLAG_WORDS = 128;

struct P2PArgs {
  // N = gradient contributors summed (and weight copies written); NR = ranks in the
  // flag protocol.  Across processes N = NR = world and contributor r is rank r.
  // Loopback (world 1, N simulated workers): the contributions are the local gradient
  // slots, the weight copies local buffers, every READY flag is published by this
  // process (contributor r = slot r) and NR = 1.
  int N = 1, NR = 1, rank = 0;
  int loopback = 0;
  unsigned seq = 0;                      // launch sequence number (flags; monotonic, same on every rank)
  unsigned step = 0;                     // update count (non-finite status slot step & 1)
  unsigned ctr_target = 0;               // cumulative CTA count after this launch (last-CTA detection)
  int bk0 = 0, bk1 = 0;                  // buckets [bk0, bk1) of this launch
  int nb = 0;
  long off[P2P_MAX_BUCKETS] = {}, shard[P2P_MAX_BUCKETS] = {}, moff[P2P_MAX_BUCKETS] = {};
  long vpre[P2P_MAX_BUCKETS + 1] = {};   // prefix sums of owned 8-element vectors per bucket
  const void* g_peer[P2P_MAX_RANKS] = {};  // fp16 or fp32 gradient vectors (wire type)
  __half* w_peer[P2P_MAX_RANKS] = {};
  unsigned* flag_peer[P2P_MAX_RANKS] = {};
  int* status_peer[P2P_MAX_RANKS] = {};
  unsigned* flag_local = nullptr;
  float *W = nullptr, *S1 = nullptr, *S2 = nullptr;
  float inv_scale = 1.f, lam = 0.f, mom = 0.f;
  float b1 = 0.9f, omb1 = 0.1f, b2 = 0.999f, omb2 = 0.001f, c1 = 1.f, c2 = 1.f, eps = 1e-8f;
  float l2x2 = 0.f;  // fp32(2 * l2), see UpdateArgs
  int w_bf16 = 0;    // the weight copies hold bfloat16 (bf16 math mode)
  const float* alpha_dev = nullptr;  // dynamic loss scaling, see UpdateArgs
  double n_workers = 1.0;
  const int* skip = nullptr;
  // NEXT-2 partial collection: 0 < quorum < N makes rank 0
  // proceed once `quorum` contributors are ready and publish their set; every owner sums
  // exactly that set (rank order) and divides by its size.  0 = all N (lock-step).
  int quorum = 0;
  double alpha = 10.0;               // static alpha (partial collection descale in fp64)
  // test injection: contributors in straggler_mask publish READY straggler_ns late
  unsigned straggler_mask = 0;
  unsigned long long straggler_ns = 0;
};

// grad_f32: element type on the wire: 0 fp16, 1 fp32 (HDP_WIRE_FP32), 2 bf16 (bf16 math mode)
cudaError_t launch_exch_update(const P2PArgs& a, int optimizer, int grad_f32, int grid, cudaStream_t s);
// CTAs of the launch's instantiation that are co-resident on the whole GPU (the grid cap)
int exch_resident_ctas(const P2PArgs& a, int optimizer, int grad_f32);

}  // namespace hdp
