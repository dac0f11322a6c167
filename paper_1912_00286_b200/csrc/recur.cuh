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
  int T = 0, B = 0, hp = 0;
  unsigned long long* trace = nullptr;  // debug: per-step phase timestamps (T x 5), nullable
};
bool recur_bwd_supported(int B, int hp);

// Two stacked layers' forward recurrences as one wavefront (layer 1 one step
// behind layer 0); layer 1's input projection W1 h0_t + b1 is computed inside.
struct Recur2FwdArgs {
  const __half *U0 = nullptr, *W1 = nullptr, *U1 = nullptr, *b1 = nullptr;  // [4hp][hp], b1 [4hp]
  const float* Gx0 = nullptr;                 // [T][B][4hp] = X W0^T + b0
  __half *Hs0 = nullptr, *Hs1 = nullptr;      // [T+1][B][hp], slot 0 = 0
  float *C0 = nullptr, *C1 = nullptr;         // [T][B][hp]
  __half *gates0 = nullptr, *gates1 = nullptr;
  int T = 0, B = 0, hp = 0;
  unsigned long long* trace = nullptr;  // debug: [3 roles][T][5] timestamps, nullable
  float* a1x = nullptr;                 // [T][B][4hp] layer-1 G_x scratch (split-cluster variant)
  // fused layer-0 input projection (split variant, Ip0 <= 64): set X0 to have R0
  // compute X0 W0^T + b0 itself (Gx0 unused); leave X0 null to read Gx0
  const __half *X0 = nullptr, *W0 = nullptr, *b0 = nullptr;  // X0 [T][B][Ip0], W0 [4hp][Ip0]
  int Ip0 = 0;
  unsigned* flags = nullptr;            // >= 16*32 + 16*8*32 uints (split-cluster variant)
  // recurrent dropout (NEXT-3, reading Q16b; Ht0 == nullptr: off): the recurrent operand is
  // h~_t, written to Ht_l [T+1][B][hp] (slot 0 = h~_{-1} = 0, not written); masks from the
  // dropout.cuh hash of (seed, *drop_step, layer, drop_seq0 + b, unit)
  __half *Ht0 = nullptr, *Ht1 = nullptr;
  const int* drop_step = nullptr;
  uint32_t drop_seed = 0, drop_thr = 0, drop_seq0 = 0;
  float drop_scale = 1.f;
};
bool recur2_fwd_supported(int B, int hp);
bool recur2_fwd_fuses_x(int B, int hp, int Ip0);

// Two stacked layers' BPTT as one wavefront: layer-1 recurrence, the input
// gradient projection dX1 = dA1 W1, and the layer-0 recurrence (fed by dX1)
// run concurrently as three 4-CTA-cluster roles per batch group.
struct Recur2BwdArgs {
  const __half *U0 = nullptr, *U1 = nullptr, *W1 = nullptr;
  const float* dHtop = nullptr;  // dH above layer 1 ([T][B][hp], or [B][hp] at T-1 if last-only)
  int dHtop_last_only = 0;
  const __half *gates0 = nullptr, *gates1 = nullptr;
  const float *C0 = nullptr, *C1 = nullptr;
  __half *dA0 = nullptr, *dA1 = nullptr;  // separate [T][B][4hp] outputs
  float* dX1 = nullptr;                   // [T][B][hp] scratch
  unsigned* flags = nullptr;              // >= 2*16*32 + 16*8*32 uints
  int T = 0, B = 0, hp = 0;
  // weight-gradient role (A8 on idle SMs, overlapping the recurrences); gW[0] == nullptr: off
  const __half *Hs0 = nullptr, *Hs1 = nullptr;  // [T+1][B][hp] forward hidden states
  const __half* X0 = nullptr;                   // [T][B][Ip0] layer-0 input
  int Ip0 = 0;
  __half* gW[4] = {nullptr, nullptr, nullptr, nullptr};  // dU1, dW1, dU0, dW0
  __half* gb[2] = {nullptr, nullptr};                    // db1, db0
  unsigned long long* trace = nullptr;  // debug: [Q1, Q0, X][T][5] timestamps, nullable
  // recurrent dropout (Ht0 == nullptr: off): dh_rec of layer l is multiplied by its mask x
  // scale (the gradient of h~_{t-1}), and dU_l accumulates dA_t^T h~_{t-1} from Ht_l
  const __half *Ht0 = nullptr, *Ht1 = nullptr;
  const int* drop_step = nullptr;
  uint32_t drop_seed = 0, drop_thr = 0, drop_seq0 = 0;
  float drop_scale = 1.f;
};
bool recur2_bwd_supported(int B, int hp);
bool recur2_bwd_wgrad(int B, int hp, int Ip0);  // the launch can also produce the A8 weight gradients
cudaError_t launch_recur2_bwd(const Recur2BwdArgs& a, cudaStream_t s);
cudaError_t launch_recur2_fwd(const Recur2FwdArgs& a, cudaStream_t s);
cudaError_t launch_recur_bwd(const RecurBwdArgs& a, cudaStream_t s);

}  // namespace hdp
