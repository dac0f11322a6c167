// Gate-contraction GEMMs of the LSTM step (SURVEY.md §8(a) A1, A2, A4, A5,
// A7, A8; PAPER.md:82 fprop/bprop, :142 "Math: matrix ... multiplication").
//
//   C[m][n] = sum_k A(m,k) * B(n,k)        (fp32 accumulate)
//
// Operands are addressed either K-major (A stored [M][K], B stored [N][K])
// or MN-major (A stored [K][M], B stored [K][N]) so that every forward and
// backward contraction of the LSTM reads its operands where they already
// live -- no transposes.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace hdp {

enum EpiMode : int {
  EPI_F32 = 0,     // out32[m*ldo + n]
  EPI_F32_T = 1,   // out32[n*ldo + m]      (transposed store, coalesced for swap-AB)
  EPI_F16 = 2,     // out16[m*ldo + n]      (RNE, counts non-finite results)
  EPI_SPLITK = 3,  // internal: fp32 partials for the deterministic split-K reduction
  // A3 fused into K2 (mixed mode, gate-interleaved columns n = 4u + gate):
  //   a = acc + gx[m][n]; i,f,o = sigma, g = tanh; c = f c_prev + i g; h = o tanh(c)
  //   -> gates[m][n] fp16 (R4), cout[m][u] fp32 (R5), hout[m][u] fp16 (R6).  splits = 1.
  EPI_LSTM_FWD = 4,
  // A6 of step t-1 fused into K7 (acc = dh_rec[m][u], N = hp): the split-K reduction
  // adds dha[m][u] and runs the cell backward -> dA[m][4u..4u+3] fp16 (R10), dc[m][u].
  EPI_LSTM_BWD = 5,
};

struct Epilogue {
  int mode = EPI_F32;
  void* out = nullptr;
  long ldo = 0;
  const void* bias = nullptr;   // added before the activation (fp32, or fp16 if bias_f16)
  int bias_f16 = 0;
  int bias_on_m = 0;            // bias indexed by m (1) or by n (0)
  int relu = 0;
  int accumulate = 0;           // fp32 modes: out += result
  int* nonfinite = nullptr;     // EPI_F16: += number of non-finite outputs
  // EPI_LSTM_FWD / EPI_LSTM_BWD operands (row stride hp for [M][hp], 4 hp for [M][4hp])
  int hp = 0;
  const float* gx = nullptr;    // FWD: this step's G_x (bias included)
  const float* cprev = nullptr; // c_{t-1} (FWD) / c_{t-2} (BWD); nullptr = zeros
  float* cout = nullptr;        // FWD: c_t
  void* hout = nullptr;         // FWD: h_t (fp16)
  void* gates = nullptr;        // FWD: saved gates out; BWD: saved gates of step t-1 in
  const float* dha = nullptr;   // BWD: dH from the layer above at t-1 (nullable)
  const float* ct = nullptr;    // BWD: c_{t-1}
  float* dc = nullptr;          // BWD: cell-gradient carry (in/out)
  void* dA = nullptr;           // BWD: dA_{t-1} (fp16)
  // recurrent dropout (NEXT-3, dropout.cuh): active iff drop_step != nullptr.  FWD also
  // writes h~_t = fp16(fp32(h_t) * drop_scale) on kept units (0 elsewhere) to htout; BWD
  // multiplies dh_rec by the same mask * drop_scale.  Row m is sequence drop_seq0 + m.
  void* htout = nullptr;
  const int* drop_step = nullptr;  // device counter of completed updates
  uint32_t drop_seed = 0, drop_thr = 0, drop_layer = 0, drop_seq0 = 0;
  float drop_scale = 1.f;
  int bf16 = 0;                 // 16-bit operands / outputs are bfloat16 (bf16 math mode), else fp16
};

struct GemmPlan {
  bool tc = true;  // tcgen05 path (fp16) or fp32 SIMT path
  CUtensorMap ta, tb;
  const void* A = nullptr;
  const void* B = nullptr;
  long lda = 0, ldb = 0;
  int M = 0, N = 0, K = 0;
  int bn = 128, amn = 0, bmn = 0;
  int splits = 1, kbps = 0;
  int cn = 1;      // CTAs per cluster sharing (multicasting) the A tile
  int cg = 1;      // 2 = CTA pairs (cta_group::2) on 256-row tiles
  int cr = 1;      // 8: the fused cell backward's split-K partials reduced inside an 8-CTA cluster (DSMEM)
  Epilogue epi;
  float* ws = nullptr;
};

// Workspace (floats) an automatic plan may need for split-K.
size_t gemm_ws_floats(int M, int N, int K);

// fp16 tensor-core plan.  a_mn / b_mn select MN-major operands.
// force_bn / force_splits: 0 = automatic.  Returns 0 or a negative error.
int gemm_plan_tc(GemmPlan* p, const __half* A, long lda, int a_mn, const __half* B, long ldb, int b_mn, int M,
                 int N, int K, const Epilogue& epi, float* ws, size_t ws_floats, int force_bn = 0,
                 int force_splits = 0, int force_cg = 0 /* 0 auto, 1 single CTAs, 2 CTA pairs */);
// fp32 SIMT plan (FP32 mode, PAPER.md:147 baseline): same addressing.
int gemm_plan_f32(GemmPlan* p, const float* A, long lda, int a_mn, const float* B, long ldb, int b_mn, int M,
                  int N, int K, const Epilogue& epi);
cudaError_t gemm_run(const GemmPlan& p, cudaStream_t s);
// one-time per-device setup (dynamic smem opt-in for every instantiation);
// must precede stream capture
cudaError_t gemm_init();

const char* gemm_last_error();

// Generic 2-D tensor map (inner dimension contiguous); 0 on success.
int encode_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                   uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw);

}  // namespace hdp
