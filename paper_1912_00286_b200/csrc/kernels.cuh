// Launchers for the non-GEMM kernels of the LSTM training step.
// Element type of activations / weights / gradients: fp16 in mixed mode,
// fp32 in FP32 mode (selected by an `f32` flag); cell state, gate
// pre-activations and all back-propagated hidden gradients are fp32.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace hdp {

// Element type of the working copy / activations / gradients, passed to the launchers
// in their `f32` / `x_f32` / `out_f32` arguments (0 and 1 keep their round-1 meaning).
enum ElemType { ET_F16 = 0, ET_F32 = 1, ET_BF16 = 2 };

// ---------------------------------------------------------------- K11
struct UpdateArgs {
  const void* g = nullptr;  // contribution r at g + r*g_stride (elements), rank order
  long g_stride = 0;
  int nsrc = 1;
  long count = 0;
  float* W = nullptr;       // fp32 master shard
  float* S1 = nullptr;      // momentum H (SGD-m) or first moment (Adam)
  float* S2 = nullptr;      // second moment (Adam)
  __half* w16 = nullptr;    // fp16 (or bf16, w_bf16) working copy (mixed modes), nullable
  int w_bf16 = 0;           // 1: w16 holds bfloat16 (bf16 math mode)
  float* w32 = nullptr;     // fp32 working copy (FP32 mode), nullable
  float inv_scale = 1.f, lam = 0.f, mom = 0.f;
  float b1 = 0.9f, omb1 = 0.1f, b2 = 0.999f, omb2 = 0.001f, c1 = 1.f, c2 = 1.f, eps = 1e-8f;
  int* nonfinite = nullptr;
  // L2 (reading Q16): g += fp32(2*l2) * w_work after the descale, w_work =
  // fp16(W) when a w16 copy is written (mixed mode, R1), else W
  float l2x2 = 0.f;
  // dynamic loss scaling (NEXT-3): alpha lives on the device; inv_scale is then
  // fp32(1 / (n_workers * alpha)) computed in fp64 like the host does, and the whole
  // update is skipped when *skip != 0 (the step's global non-finite count)
  const float* alpha_dev = nullptr;
  double n_workers = 1.0;
  const int* skip = nullptr;
};
// grad_is_f32: element type of the contributions (ET_F16 / ET_F32 / ET_BF16)
cudaError_t launch_avg_update(const UpdateArgs& a, int grad_is_f32, int optimizer, cudaStream_t s);
// *count += number of Inf/NaN values in g[0..n) (fp16, or fp32 if g_f32)
cudaError_t launch_count_nonfinite(const void* g, long n, int g_f32, int* count, cudaStream_t s);
// dynamic loss-scale rule after the (possibly skipped) update, one thread:
//   st[0] = global non-finite count of the step, st[1] = consecutive finite steps,
//   st[2] = skipped steps (total);  alpha /= factor (>= min_alpha) on a non-finite step,
//   alpha *= factor after `interval` finite steps
cudaError_t launch_loss_scale_update(int* st, float* alpha, int interval, float factor, float min_alpha,
                                     cudaStream_t s);

// ---------------------------------------------------------------- input
// x [B][T][I] (fp16 or fp32)  ->  X0 [T][B][Ip] (time-major, zero padded)
struct ZeroRows {  // regions zeroed by the input-packing launch (16-B vectors)
  uint4* base = nullptr;
  long stride = 0, nvec = 0;
  int count = 0;
};
cudaError_t launch_pack_input(const void* x, int x_f32, int B, int T, int I, int Ip, void* X0, int f32,
                              cudaStream_t s, ZeroRows z = ZeroRows());
// tokens [B][T] -> X0[t][b][:] = E[tok[b][t]][:]  (K10 gather); a token outside
// [0, vocab) reads row 0 and increments *bad
cudaError_t launch_embed_gather(const int32_t* tok, int B, int T, const void* E, int Ep, void* X0, int f32,
                                int vocab, int* bad, cudaStream_t s);

// recurrent dropout (NEXT-3, dropout.cuh): ht[b][u] = kept(seq0 + b, u) ? fp16(h * scale) : 0
cudaError_t launch_drop_mask(const void* h, void* ht, int B, int hp, const int* step, uint32_t seed, uint32_t layer,
                             uint32_t seq0, uint32_t thr, float scale, cudaStream_t s);
// *p += 1 (device counter, stream-ordered)
cudaError_t launch_increment(int* p, cudaStream_t s);

// ---------------------------------------------------------------- cell (K3 / K6)
// gate rows interleaved per unit: row 4*j + {i,f,g,o}
cudaError_t launch_cell_fwd(int f32, const float* Gx_t, const float* Gh, const float* c_prev, void* gates_t,
                            float* c_t, void* h_t, int B, int hp, cudaStream_t s);
cudaError_t launch_cell_bwd(int f32, const float* dHa_t, const float* dh_rec, const void* gates_t,
                            const float* c_t, const float* c_prev, float* dc, void* dA_t, int B, int hp,
                            int first, cudaStream_t s);

// ---------------------------------------------------------------- head (K4 / K5)
// y[r] = sum_k Z[r][k] wo[k] + bo; hinge (Eq. 6) -> dy[r], per-block partial sums.
// tgt_mode 0: row r = t*B + b <-> tgt[b*T + t];  1: row r = b <-> tgt[b]
int head_partials_count(int rows);
// dz (nullable): also writes dz = (Z > 0) * dy * wo (A5's ReLU', R9) for the FC head
cudaError_t launch_head_out(int f32, const void* Z, int rows, int Kd, long ldz, const void* wo, const void* bo,
                            const int8_t* tgt, int tgt_mode, int B, int T, float alpha, float inv_terms, float* y,
                            float* dy, float* partials, cudaStream_t s, void* dz = nullptr,
                            const float* alpha_dev = nullptr /* dynamic loss scale: alpha read on the device */);
// loss = (sum of partials) * inv_terms   (unscaled mean hinge), deterministic
// loss += l2 * sum(w[0..n)^2)  (deterministic; part: l2_partials_doubles() doubles)
cudaError_t launch_l2_loss(int f32, const void* w, long n, double* part, double l2, float* loss, cudaStream_t s);
size_t l2_partials_doubles();
cudaError_t launch_loss_final(const float* partials, int n, float inv_terms, float* loss, cudaStream_t s);
// dz[r][f] = (Z[r][f] > 0) ? dy[r]*wo[f] : 0   (ReLU', R9)
cudaError_t launch_relu_dz(int f32, const float* dy, const void* wo, const void* Z, void* dz, int rows, int Fp,
                           cudaStream_t s);
// dH[r][j] = dy[r] * wo[j]
cudaError_t launch_outer(int f32, const float* dy, const void* wo, float* dH, int rows, int hp, cudaStream_t s);

// ---------------------------------------------------------------- reductions
// out[c] = sum_r X[r*ldx + c] * (w ? w[r] : 1)   over rows in a fixed order.
// out is fp16 (RNE) when out_f32 == 0, else fp32.  partials: RS*cols floats.
size_t colreduce_partials_floats(int rows, int cols);
// FC head: dwo = Z^T dy, dfb = colsum(dz), dbo = sum(dy) in one fused pass (partials: (2F+1)*RS doubles)
cudaError_t launch_colreduce(int x_f32, const void* X, long ldx, int rows, int cols, const float* w,
                             float* partials, int out_f32, void* out, cudaStream_t s);
// pass 2 alone over rs rows of fp64 partials [rs][2F + 1] (the fused head's per-CTA sums)
cudaError_t launch_colreduce3_final(const double* partials, int rs, int F, int out_f32, void* dwo, void* dfb,
                                    void* dbo, cudaStream_t s);
cudaError_t launch_colreduce3(int x_f32, const void* Z, const void* dz, long ld, int rows, int F, const float* dy,
                              float* partials, int out_f32, void* dwo, void* dfb, void* dbo, cudaStream_t s);

// ---------------------------------------------------------------- embedding backward (K10)
// scratch of the library's own stable radix sort (per-tile digit histograms)
size_t embed_sort_temp_bytes(int n);
size_t embed_part_floats(int n, int Ep);
// dE[v][:] = sum over positions p (ascending, p = t*B+b) with tok = v of dX0[p][:]
cudaError_t launch_embed_backward(const int32_t* tok, int B, int T, int vocab, const float* dX0, int Ep,
                                  int32_t* keys_in, int32_t* keys_out, int32_t* vals_in, int32_t* vals_out,
                                  void* sort_temp, size_t sort_temp_bytes, float* part, void* dE, int out_f32, int32_t* range /* 2*vocab ints */,
                                  cudaStream_t s);

}  // namespace hdp
