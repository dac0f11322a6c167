// Fused FC head of the per-step hinge loss (SURVEY.md §8(a) A4 + A5 except the dF GEMM;
// PAPER.md:80 "LSTM layers ... followed by a fully connected layer", :171 hinge loss per
// time step, :177-180 loss scale alpha).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace hdp {

struct HeadFusedArgs {
  const void* H = nullptr;       // top layer's h_t rows [rows][hp] fp16 (row r = t * B + b)
  const void* F = nullptr;       // FC weight [Fp][hp] fp16
  const void* fb = nullptr;      // FC bias [Fp] fp16
  const void* wo = nullptr;      // output weight [Fp] fp16
  const void* bo = nullptr;      // output bias [1] fp16
  const int8_t* tgt = nullptr;   // targets [B][T] in {-1, +1}
  void* dz = nullptr;            // out: dz [rows][Fp] fp16 (R9), read by the dF GEMM
  float* y = nullptr;            // out: y [rows]
  float* dy = nullptr;           // out: d(loss)/dy [rows]
  float* hinge = nullptr;        // scratch: per-CTA hinge sums [grid]
  double* colpart = nullptr;     // out: per-CTA column sums [grid][2 Fp + 1]: dwo | dfb | dbo
  float* loss = nullptr;         // out: mean hinge (written by the last CTA)
  unsigned* ticket = nullptr;    // zero-initialised counter; the last CTA resets it
  float* dH = nullptr;           // out: dH_top = dz F  [rows][hp] fp32
  int rows = 0, B = 0, T = 0, hp = 0, Fp = 0;
  float alpha = 10.f, inv_terms = 1.f;
  const float* alpha_dev = nullptr;  // dynamic loss scaling: device alpha (nullable)
  unsigned long long* trace = nullptr;  // phase trace (option recur_trace): [grid][8] %globaltimer
  int pdl = 0;  // launched as a programmatic dependent of the previous kernel (only H waits for it)
};

// Whether the fused kernel covers this shape (fp16 mixed mode only; hp, Fp <= 256).
bool head_fused_supported(int hp, int Fp);
int head_fused_grid(int rows);
cudaError_t launch_head_fused(const HeadFusedArgs& a, cudaStream_t s);

}  // namespace hdp
