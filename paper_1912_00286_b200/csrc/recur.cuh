// Persistent fused LSTM recurrence kernels.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace hdp {

struct RecurFwdArgs {
  const __half* U = nullptr;  // [4hp][hp] gate rows interleaved (4j+g)
  const float* Gx = nullptr;  // [T][B][4hp] = X W^T + b
  __half* Hs = nullptr;       // [T+1][B][hp]; slot 0 = h_{-1} = 0 (read), slots 1..T written
  float* C = nullptr;         // [T][B][hp]
  __half* gates = nullptr;    // [T][B][4hp] activated gates, fp16 (R4)
  unsigned* counter = nullptr;  // grid-barrier counters, 16 x 32 uints (zeroed by the launcher)
  int T = 0, B = 0, hp = 0;
  unsigned long long* trace = nullptr;  // debug: per-step phase timestamps (T x 5), nullable
};

bool recur_fwd_supported(int B, int hp);
cudaError_t launch_recur_fwd(const RecurFwdArgs& a, cudaStream_t s);

struct RecurBwdArgs {
  const __half* U = nullptr;      // [4hp][hp]
  const float* dHa = nullptr;     // dH from above: [T][B][hp] (mode 0) or [B][hp] at t = T-1 only (mode 1)
  int dHa_last_only = 0;
  const __half* gates = nullptr;  // [T][B][4hp] saved fp16 gates
  const float* C = nullptr;       // [T][B][hp]
  __half* dA = nullptr;           // [T][B][4hp] output (fp16, R10)
  unsigned* counter = nullptr;    // 16 x 32 uints
  int T = 0, B = 0, hp = 0;
  unsigned long long* trace = nullptr;  // debug: per-step phase timestamps (T x 5), nullable
};
bool recur_bwd_supported(int B, int hp);
cudaError_t launch_recur_bwd(const RecurBwdArgs& a, cudaStream_t s);

}  // namespace hdp
