// Elementwise / reduction kernels of the LSTM step (everything that is not a
// gate contraction): input packing, the fused LSTM cell forward (K3) and
// backward (K6), the head (K4/K5: Eq. 6 hinge x alpha), deterministic column
// reductions (bias / head gradients) and the embedding gather / scatter (K10).
//
// Cell equations (reading Q1, gate order i,f,g,o):
//   i,f,o = sigma(a), g = tanh(a);  c_t = f c_{t-1} + i g;  h_t = o tanh(c_t)
// Backward (BPTT):
//   dh = dH_above + dh_rec;  dc += dh o (1 - tanh^2 c_t)
//   dA = [dc g i(1-i), dc c_{t-1} f(1-f), dc i (1-g^2), dh tanh(c_t) o(1-o)]
//   dc_{t-1} = dc f
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <type_traits>
#include <utility>

#include "dropout.cuh"
#include "kernels.cuh"

namespace hdp {
namespace {

template <typename T>
__device__ __forceinline__ float ld(const T* p, long i);
template <>
__device__ __forceinline__ float ld<float>(const float* p, long i) { return p[i]; }
template <>
__device__ __forceinline__ float ld<__half>(const __half* p, long i) { return __half2float(p[i]); }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p, long i) { return __bfloat162float(p[i]); }

template <typename T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half cvt<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// one R12 output element of element type `et` (ET_F16 / ET_F32 / ET_BF16)
__device__ __forceinline__ void st_et(void* out, long i, float v, int et) {
  if (et == ET_F32) reinterpret_cast<float*>(out)[i] = v;
  else if (et == ET_BF16) reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
  else reinterpret_cast<__half*>(out)[i] = __float2half_rn(v);
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// 4 gate values of one unit: fp16 -> one 8-byte access, fp32 -> one 16-byte access
__device__ __forceinline__ void st4(__half* p, float a, float b, float c, float d) {
  __align__(8) __half2 v[2] = {__halves2half2(__float2half_rn(a), __float2half_rn(b)),
                               __halves2half2(__float2half_rn(c), __float2half_rn(d))};
  *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(v);
}
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ float4 ld4(const __half* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 x = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 y = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(x.x, x.y, y.x, y.y);
}
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(__nv_bfloat16* p, float a, float b, float c, float d) {
  __align__(8) __nv_bfloat162 v[2] = {__floats2bfloat162_rn(a, b), __floats2bfloat162_rn(c, d)};
  *reinterpret_cast<uint2*>(p) = *reinterpret_cast<const uint2*>(v);
}
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(x.x, x.y, y.x, y.y);
}

// ---------------------------------------------------------------- input
// the forward's h_{-1} rows (one per layer, `count` regions of `nvec` 16-B vectors, `stride`
// vectors apart) zeroed by the input-packing launch instead of one memset node per layer
__device__ __forceinline__ void zero_rows(const ZeroRows& z) {
  const long total = (long)z.count * z.nvec;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x)
    z.base[(i / z.nvec) * z.stride + i % z.nvec] = make_uint4(0u, 0u, 0u, 0u);
}

template <typename XT, typename T>
__global__ void pack_input_kernel(const XT* __restrict__ x, int B, int Tn, int I, int Ip, T* __restrict__ X0,
                                  ZeroRows z) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (PDL) the forward wavefront's prologue may start
  zero_rows(z);
  const long total = (long)Tn * B * Ip;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int k = (int)(idx % Ip);
    const long tb = idx / Ip;
    const int b = (int)(tb % B), t = (int)(tb / B);
    const float v = k < I ? ld<XT>(x, ((long)b * Tn + t) * I + k) : 0.f;
    X0[idx] = cvt<T>(v);
  }
}

// recurrent dropout (NEXT-3): h~ = fp16(fp32(h) * scale) on kept units, 0 elsewhere, for the
// step whose h the fused GEMM epilogue did not produce (t = 0)
__global__ void drop_mask_kernel(const __half* __restrict__ h, __half* __restrict__ ht, int B, int hp,
                                 const int* __restrict__ step, uint32_t seed, uint32_t layer, uint32_t seq0,
                                 uint32_t thr, float scale) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * hp) return;
  const int b = idx / hp, u = idx % hp;
  const uint32_t sk = drop_seq_key(drop_layer_key(seed, (uint32_t)*step, layer), seq0 + (uint32_t)b);
  ht[idx] = drop_kept(sk, (uint32_t)u, thr) ? __float2half_rn(__half2float(h[idx]) * scale) : __float2half_rn(0.f);
}

// same-type rows with I == Ip and 16-B aligned rows: one warp per (t, b) row, 16-B vectors
// (a pure row permutation [B][T] -> [T][B]; C4 moves 134 MB per step through here)
__global__ void pack_rows_kernel(const uint4* __restrict__ x, int B, int Tn, int vrow, uint4* __restrict__ X0,
                                 ZeroRows z) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  zero_rows(z);
  const long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (long)Tn * B) return;
  const int b = (int)(w % B), t = (int)(w / B);
  const uint4* src = x + ((long)b * Tn + t) * vrow;
  uint4* dst = X0 + w * vrow;
  for (int k = lane; k < vrow; k += 32) dst[k] = __ldcs(src + k);
}

template <typename T>
__global__ void embed_gather_kernel(const int32_t* __restrict__ tok, int B, int Tn, const T* __restrict__ E,
                                    int Ep, T* __restrict__ X0, int vocab, int* __restrict__ bad) {
  // one warp per position p = t*B + b; a token outside [0, vocab) reads row 0 and is
  // counted in *bad (reported as HDP_ERR_ARG by the next hdp_grad_average_update)
  const long p = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= (long)Tn * B) return;
  const int b = (int)(p % B), t = (int)(p / B);
  long row = tok[(long)b * Tn + t];
  if (row < 0 || row >= vocab) {
    if (lane == 0) atomicAdd(bad, 1);
    row = 0;
  }
  for (int k = lane; k < Ep; k += 32) X0[p * Ep + k] = E[row * Ep + k];
}

// ---------------------------------------------------------------- cell
template <typename T>
__global__ void cell_fwd_kernel(const float* __restrict__ Gx, const float* __restrict__ Gh,
                                const float* __restrict__ c_prev, T* __restrict__ gates, float* __restrict__ c_t,
                                T* __restrict__ h_t, int n) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  float4 a = reinterpret_cast<const float4*>(Gx)[idx];
  if (Gh) {
    const float4 r = reinterpret_cast<const float4*>(Gh)[idx];
    a.x += r.x; a.y += r.y; a.z += r.z; a.w += r.w;
  }
  const float i = sigmoidf_(a.x), f = sigmoidf_(a.y), g = tanhf(a.z), o = sigmoidf_(a.w);
  const float cp = c_prev ? c_prev[idx] : 0.f;
  const float c = f * cp + i * g;
  const float h = o * tanhf(c);
  st4(gates + 4L * idx, i, f, g, o);  // R4: saved gates (fp16 in mixed mode)
  c_t[idx] = c;                       // R5: fp32
  h_t[idx] = cvt<T>(h);               // R6: fp16 in mixed mode
}

template <typename T>
__global__ void cell_bwd_kernel(const float* __restrict__ dHa, const float* __restrict__ dh_rec,
                                const T* __restrict__ gates, const float* __restrict__ c_t,
                                const float* __restrict__ c_prev, float* __restrict__ dc, T* __restrict__ dA, int n,
                                int first) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  float dh = 0.f;
  if (dHa) dh += dHa[idx];
  if (dh_rec) dh += dh_rec[idx];
  const float4 G = ld4(gates + 4L * idx);
  const float i = G.x, f = G.y, g = G.z, o = G.w;
  const float c = c_t[idx];
  const float cp = c_prev ? c_prev[idx] : 0.f;
  const float tc = tanhf(c);
  const float d = (first ? 0.f : dc[idx]) + dh * o * (1.f - tc * tc);
  st4(dA + 4L * idx, d * g * i * (1.f - i), d * cp * f * (1.f - f), d * i * (1.f - g * g),
      dh * tc * o * (1.f - o));  // R10
  dc[idx] = d * f;
}

// ---------------------------------------------------------------- head
constexpr int HEAD_WARPS = 8;

// dy of row r as head_out computed it (valid on lane 0, which holds the row's sum path)
__device__ __forceinline__ float margin_dy(int lane, float hinge, float alpha, float inv_terms, const int8_t* tgt,
                                           int tgt_mode, int r, int B, int Tn) {
  if (lane != 0) return 0.f;
  const int8_t tv = tgt_mode == 0 ? tgt[(long)(r % B) * Tn + r / B] : tgt[r];
  return hinge > 0.f ? -alpha * (float)tv * inv_terms : 0.f;
}

template <typename T>
__global__ void __launch_bounds__(HEAD_WARPS * 32)
    head_out_kernel(const T* __restrict__ Z, int rows, int Kd, long ldz, const T* __restrict__ wo,
                    const T* __restrict__ bo, const int8_t* __restrict__ tgt, int tgt_mode, int B, int Tn,
                    float alpha, float inv_terms, float* __restrict__ y, float* __restrict__ dy,
                    float* __restrict__ partials, T* __restrict__ dz, const float* __restrict__ alpha_dev) {
  __shared__ float part[HEAD_WARPS];
  if (alpha_dev) alpha = *alpha_dev;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * HEAD_WARPS + warp;
  float hinge = 0.f;
  // fp16 rows of <= 256 elements (multiple of 8): one 16-B vector per lane, kept for dz
  const bool vec = std::is_same<T, __half>::value && (Kd & 7) == 0 && Kd <= 256 && (ldz & 7) == 0;
  if (r < rows && vec) {
    float acc = 0.f;
    float zv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, wv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int k0 = lane * 8;
    if (k0 < Kd) {
      const uint4 zu = *reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(Z) + (long)r * ldz + k0);
      const uint4 wu = *reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(wo) + k0);
      const __half2* zh = reinterpret_cast<const __half2*>(&zu);
      const __half2* wh = reinterpret_cast<const __half2*>(&wu);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 zf = __half22float2(zh[q]), wf = __half22float2(wh[q]);
        zv[2 * q] = zf.x;
        zv[2 * q + 1] = zf.y;
        wv[2 * q] = wf.x;
        wv[2 * q + 1] = wf.y;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += zv[q] * wv[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const float yy = acc + ld<T>(bo, 0);
    const int8_t tv = tgt_mode == 0 ? tgt[(long)(r % B) * Tn + r / B] : tgt[r];
    const float tf = (float)tv;
    const float margin = 1.f - tf * yy;
    const float dyr = margin > 0.f ? -alpha * tf * inv_terms : 0.f;
    if (lane == 0) {
      y[r] = yy;
      dy[r] = dyr;  // subgradient 0 at the kink (reading Q5)
      hinge = margin > 0.f ? margin : 0.f;
    }
    if (dz && k0 < Kd) {  // A5's ReLU' (R9), the same fp32 product relu_dz forms
      __align__(16) __half o[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] = __float2half_rn(zv[q] > 0.f ? dyr * wv[q] : 0.f);
      *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(dz) + (long)r * ldz + k0) = *reinterpret_cast<const uint4*>(o);
    }
  } else if (r < rows) {
    float acc = 0.f;
    for (int k = lane; k < Kd; k += 32) acc += ld<T>(Z, (long)r * ldz + k) * ld<T>(wo, k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float yy = acc + ld<T>(bo, 0);
      int8_t tv;
      if (tgt_mode == 0) {
        const int b = r % B, t = r / B;
        tv = tgt[(long)b * Tn + t];
      } else {
        tv = tgt[r];
      }
      const float tf = (float)tv;
      const float margin = 1.f - tf * yy;
      y[r] = yy;
      // d/dy alpha*mean(max(0, 1 - t y)) ; subgradient 0 at the kink (reading Q5)
      dy[r] = margin > 0.f ? -alpha * tf * inv_terms : 0.f;
      hinge = margin > 0.f ? margin : 0.f;
    }
    if (dz) {
      // A5's ReLU' (R9) fused here: dz = (z > 0) dy wo, the same fp32 product relu_dz forms
      const float dyr = __shfl_sync(0xffffffffu, margin_dy(lane, hinge, alpha, inv_terms, tgt, tgt_mode, r, B, Tn), 0);
      for (int k = lane; k < Kd; k += 32) {
        const float z = ld<T>(Z, (long)r * ldz + k);
        dz[(long)r * ldz + k] = cvt<T>(z > 0.f ? dyr * ld<T>(wo, k) : 0.f);
      }
    }
  }
  if (lane == 0) part[warp] = hinge;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < HEAD_WARPS; ++w) s += part[w];
    partials[blockIdx.x] = s;
  }
}

__global__ void loss_final_kernel(const float* __restrict__ partials, int n, float inv_terms, float* loss) {
  __shared__ float sm[256];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += 256) s += partials[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = sm[0] * inv_terms;
}

// L2 penalty of the reported loss: loss += l2 * sum(w^2) over the
// working weights; fixed grid + fp64 partials summed in block order (deterministic)
constexpr int L2_BLOCKS = 296;
template <typename T>
__global__ void __launch_bounds__(256) sumsq_partial_kernel(const T* __restrict__ w, long n, double* part) {
  __shared__ double sm[256];
  double s = 0.0;
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n; i += (long)gridDim.x * 256) {
    const double v = (double)ld<T>(w, i);
    s += v * v;
  }
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) sm[threadIdx.x] += sm[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}
__global__ void l2_loss_final_kernel(const double* __restrict__ part, int n, double l2, float* loss) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *loss = (float)((double)*loss + l2 * s);
  }
}

template <typename T>
__global__ void relu_dz_kernel(const float* __restrict__ dy, const T* __restrict__ wo, const T* __restrict__ Z,
                               T* __restrict__ dz, int rows, int Fp) {
  const long total = (long)rows * Fp;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int f = (int)(idx % Fp);
    const long r = idx / Fp;
    const float z = ld<T>(Z, idx);
    dz[idx] = cvt<T>(z > 0.f ? dy[r] * ld<T>(wo, f) : 0.f);  // R9
  }
}

template <typename T>
__global__ void outer_kernel(const float* __restrict__ dy, const T* __restrict__ wo, float* __restrict__ dH,
                             int rows, int hp) {
  const long total = (long)rows * hp;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total; idx += (long)gridDim.x * blockDim.x) {
    const int j = (int)(idx % hp);
    dH[idx] = dy[idx / hp] * ld<T>(wo, j);
  }
}

// ---------------------------------------------------------------- deterministic column reduction
constexpr int CR_WARPS = 8;

int cr_splits(int rows) {
  int rs = (rows + 127) / 128;  // row chunks of 128 (16 rows per warp): enough blocks to fill the GPU
  if (rs > 128) rs = 128;
  if (rs < 1) rs = 1;
  return rs;
}

// fp64 accumulation: these sums (bias / head gradients) cancel strongly over
// B*T terms; double accumulation keeps the reduction itself exact to fp32
template <typename XT>
__global__ void __launch_bounds__(CR_WARPS * 32)
    colreduce_pass1(const XT* __restrict__ X, long ldx, int rows, int cols, const float* __restrict__ w, int rs,
                    double* __restrict__ partials) {
  __shared__ double sm[CR_WARPS][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + lane;
  const int per = (rows + rs - 1) / rs;
  const int r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  double acc = 0.0;
  if (c < cols)
    for (int r = r0 + warp; r < r1; r += CR_WARPS) {
      const float v = ld<XT>(X, (long)r * ldx + c);
      acc += w ? (double)v * (double)w[r] : (double)v;
    }
  sm[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && c < cols) {
    double s = 0.0;
    for (int q = 0; q < CR_WARPS; ++q) s += sm[q][lane];
    partials[(long)blockIdx.y * cols + c] = s;
  }
}

// FC head (A5): dwo = Z^T dy, dfb = colsum(dz), dbo = sum(dy) in one pass over Z and dz:
// combined columns [0, F) -> Z*dy, [F, 2F) -> dz, 2F -> dy; same fp64 fixed-order sums
// as colreduce_pass1 (rows r0 + warp, r0 + warp + 8, ... then the 8 warps in order)
template <typename XT>
__global__ void __launch_bounds__(CR_WARPS * 32)
    colreduce3_pass1(const XT* __restrict__ Z, const XT* __restrict__ dz, long ldx, int rows, int F,
                     const float* __restrict__ dy, int rs, double* __restrict__ partials) {
  __shared__ double sm[CR_WARPS][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cols = 2 * F + 1;
  const int c = blockIdx.x * 32 + lane;
  const int per = (rows + rs - 1) / rs;
  const int r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  double acc = 0.0;
  if (c < F) {
    for (int r = r0 + warp; r < r1; r += CR_WARPS) acc += (double)ld<XT>(Z, (long)r * ldx + c) * (double)dy[r];
  } else if (c < 2 * F) {
    for (int r = r0 + warp; r < r1; r += CR_WARPS) acc += (double)ld<XT>(dz, (long)r * ldx + c - F);
  } else if (c == 2 * F) {
    for (int r = r0 + warp; r < r1; r += CR_WARPS) acc += (double)dy[r];
  }
  sm[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && c < cols) {
    double s = 0.0;
    for (int q = 0; q < CR_WARPS; ++q) s += sm[q][lane];
    partials[(long)blockIdx.y * cols + c] = s;
  }
}
// pass 2: one warp per column, lane-strided partial sums then a fixed xor-butterfly
// (deterministic order), so the up to 128 partials of a column are not one serial chain
__device__ __forceinline__ double warp_col_sum(const double* __restrict__ partials, int rs, int cols, int c, int lane) {
  double s = 0.0;
  for (int q = lane; q < rs; q += 32) s += partials[(long)q * cols + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__global__ void colreduce3_pass2(const double* __restrict__ partials, int rs, int F, int out_f32, void* dwo, void* dfb,
                                 void* dbo) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int cols = 2 * F + 1;
  if (c >= cols) return;
  const double s = warp_col_sum(partials, rs, cols, c, lane);
  if (lane != 0) return;
  void* out = c < F ? dwo : c < 2 * F ? dfb : dbo;
  const int i = c < F ? c : c < 2 * F ? c - F : 0;
  st_et(out, i, (float)s, out_f32);  // R12: fp32 value, one RNE
}

__global__ void colreduce_pass2(const double* __restrict__ partials, int rs, int cols, int out_f32, void* out) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= cols) return;
  const double s = warp_col_sum(partials, rs, cols, c, lane);
  if (lane != 0) return;
  st_et(out, c, (float)s, out_f32);  // R12: fp32 value, one RNE
}

// ---------------------------------------------------------------- embedding backward
__global__ void embed_keys_kernel(const int32_t* __restrict__ tok, int B, int Tn, int vocab, int32_t* keys,
                                  int32_t* vals) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= B * Tn) return;
  const int b = p % B, t = p / B;
  const int k = tok[(long)b * Tn + t];
  keys[p] = (k < 0 || k >= vocab) ? 0 : k;  // as the gather did (the forward counted it)
  vals[p] = p;
}

// Stable LSD radix sort of the (token, position) pairs by token, 8-bit digits
// (ceil(log2 vocab) / 8 passes; C3's vocab 20000 -> 2).  One pass:
//   radix_hist_kernel    per tile of RS_TILE positions, the 256-bin digit histogram,
//                        stored bin-major: hist[bin][tile];
//   radix_scatter_kernel per tile: its (bin, tile) output offsets from the bin-major
//                        exclusive scan of hist (computed in-block), the rank of each element among the elements of its
//                        tile with the same digit and a smaller position (in-warp:
//                        __match_any_sync + popc of the lower lanes; across warps:
//                        per-warp bin counts scanned in warp order), written to
//                        offset[bin][tile] + rank.
// Element order inside a tile is position order, tiles are visited in order and the
// scan is bin-major, so every pass is stable and the sort is deterministic.
constexpr int RS_TILE = 1024;

__global__ void __launch_bounds__(RS_TILE) radix_hist_kernel(const int32_t* __restrict__ keys, int n, int shift,
                                                            int ntiles, int32_t* __restrict__ hist) {
  __shared__ int h[256];
  if (threadIdx.x < 256) h[threadIdx.x] = 0;
  __syncthreads();
  const int p = blockIdx.x * RS_TILE + threadIdx.x;
  if (p < n) atomicAdd(&h[(keys[p] >> shift) & 255], 1);
  __syncthreads();
  if (threadIdx.x < 256) hist[(long)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// The scatter computes its tiles' global offsets itself (no separate scan launch): for its
// tile and every bin, offset = (elements of all smaller bins) + (elements of this bin in
// earlier tiles) -- the bin-major exclusive scan evaluated at (bin, tile), exact integers.
__global__ void __launch_bounds__(RS_TILE) radix_scatter_kernel(const int32_t* __restrict__ kin,
                                                               const int32_t* __restrict__ vin, int n, int shift,
                                                               int ntiles, const int32_t* __restrict__ hist,
                                                               int32_t* __restrict__ kout,
                                                               int32_t* __restrict__ vout) {
  __shared__ int wc[RS_TILE / 32][256];
  __shared__ int offs[256];
  __shared__ int wsum[8];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < (RS_TILE / 32) * 256; i += RS_TILE) (&wc[0][0])[i] = 0;
  if (tid < 256) {  // bin tid: total over all tiles, and over the tiles before mine
    const int32_t* hb = hist + (long)tid * ntiles;
    int tot = 0, before = 0;
    for (int j = 0; j < ntiles; ++j) {
      const int c = hb[j];
      tot += c;
      if (j < (int)blockIdx.x) before += c;
    }
    int x = tot;  // exclusive scan of the bin totals over the 256 bins (8 warps)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    offs[tid] = x - tot + before;
  }
  __syncthreads();
  if (tid < 256) {
    int add = 0;
    for (int j = 0; j < w; ++j) add += wsum[j];
    offs[tid] += add;
  }
  __syncthreads();
  const int p = blockIdx.x * RS_TILE + tid;
  const bool valid = p < n;
  const int key = valid ? kin[p] : 0;
  const int d = (key >> shift) & 255;
  const unsigned same = __match_any_sync(0xffffffffu, valid ? d : -1);
  const unsigned lower = (1u << lane) - 1u;
  const int rank = __popc(same & lower);
  if (valid && rank == 0) wc[w][d] = __popc(same);
  __syncthreads();
  if (tid < 256) {  // per-bin exclusive scan over the warps, in warp (= position) order
    int run = 0;
    for (int j = 0; j < RS_TILE / 32; ++j) {
      const int c = wc[j][tid];
      wc[j][tid] = run;
      run += c;
    }
  }
  __syncthreads();
  if (valid) {
    const int dst = offs[d] + wc[w][d] + rank;
    kout[dst] = key;
    vout[dst] = vin[p];
  }
}

// Deterministic two-level segmented sum over the token-sorted positions:
// (1) one warp per fixed chunk of EMB_CHUNK sorted positions sums each run of
//     equal tokens inside its chunk (ascending position order) and stores the
//     partial at the run's first index; the chunk's keys / positions come in
//     with one coalesced load and the dX rows of EMB_BATCH positions are
//     loaded before they are accumulated (independent loads in flight);
// (2) one warp per vocabulary row adds its partials (at its first index and
//     at every chunk start inside its range) in index order; the row's range
//     [first, last) of sorted positions was recorded by embed_range_kernel.
// No atomics; load-balanced for Zipf-frequent tokens.
constexpr int EMB_CHUNK = 32;
constexpr int EMB_BATCH = 32;  // dX rows in flight per warp (the whole chunk; 8 left the chunk pass latency-bound)

__global__ void embed_range_kernel(const int32_t* __restrict__ keys, int n, int32_t* __restrict__ first,
                                   int32_t* __restrict__ last) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = keys[i];
  if (i == 0 || keys[i - 1] != k) first[k] = i;
  if (i == n - 1 || keys[i + 1] != k) last[k] = i + 1;
}

__global__ void embed_chunk_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ vals, int n,
                                   const float* __restrict__ dX0, int Ep, float* __restrict__ part) {
  const long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long i0 = w * EMB_CHUNK;
  if (i0 >= n) return;
  const int cnt = (int)min((long)EMB_CHUNK, (long)n - i0);
  const int my_key = lane < cnt ? keys[i0 + lane] : -1;
  const int my_val = lane < cnt ? vals[i0 + lane] : 0;
  for (int k0 = 0; k0 < Ep; k0 += 128) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    int start = 0;
    int cur = __shfl_sync(0xffffffffu, my_key, 0);
    for (int j0 = 0; j0 < cnt; j0 += EMB_BATCH) {
      float rv[EMB_BATCH][4];
#pragma unroll
      for (int b = 0; b < EMB_BATCH; ++b) {
        const int val = __shfl_sync(0xffffffffu, my_val, (j0 + b) & 31);
        const float* row = dX0 + (long)val * Ep;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = k0 + lane + 32 * q;
          rv[b][q] = (j0 + b < cnt && k < Ep) ? row[k] : 0.f;
        }
      }
#pragma unroll
      for (int b = 0; b < EMB_BATCH; ++b) {
        const int key = __shfl_sync(0xffffffffu, my_key, (j0 + b) & 31);
        if (j0 + b >= cnt) break;
        if (key != cur) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k = k0 + lane + 32 * q;
            if (k < Ep) part[(i0 + start) * Ep + k] = acc[q];
            acc[q] = 0.f;
          }
          start = j0 + b;
          cur = key;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += rv[b][q];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = k0 + lane + 32 * q;
      if (k < Ep) part[(i0 + start) * Ep + k] = acc[q];
    }
  }
}

// one warp per (vocabulary row, 32-column slice); a Zipf-frequent token spans ~200 chunk
// partials: 16 independent chains, combined in a fixed order (deterministic).  (A warp per
// row with 4 columns per lane measured slower: 32 -> 56 us cold-cache at C3, fewer
// independent loads in flight.)
__global__ void embed_segsum_kernel(const int32_t* __restrict__ first, const int32_t* __restrict__ last, int vocab,
                                    const float* __restrict__ part, int Ep, int out_f32, void* dE) {
  constexpr int CH = 16;
  const long w = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int slices = (Ep + 31) >> 5;
  const long v = w / slices;
  const int k = (int)(w % slices) * 32 + lane;
  if (v >= vocab || k >= Ep) return;
  const int lo = first[v], hi = last[v];  // [0, 0) for tokens that do not occur
  float s = 0.f;
  if (lo < hi) {
    float a[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) a[j] = 0.f;
    long c = ((long)lo / EMB_CHUNK + 1) * EMB_CHUNK;
    for (; c + (CH - 1) * EMB_CHUNK < hi; c += CH * EMB_CHUNK) {
#pragma unroll
      for (int j = 0; j < CH; ++j) a[j] += part[(c + j * EMB_CHUNK) * Ep + k];
    }
#pragma unroll
    for (int j = 0; j < CH; ++j)
      if (c + j * EMB_CHUNK < hi) a[j] += part[(c + j * EMB_CHUNK) * Ep + k];
#pragma unroll
    for (int m = CH / 2; m > 0; m >>= 1)
#pragma unroll
      for (int j = 0; j < m; ++j) a[j] += a[j + m];
    s = part[(long)lo * Ep + k] + a[0];
  }
  st_et(dE, v * Ep + k, s, out_f32);  // R12
}

// element-type dispatch of the launchers: et = ET_F16 (0), ET_F32 (1) or ET_BF16 (2)
#define HDP_ET(et, T, ...)                                   \
  do {                                                       \
    if ((et) == ET_F32) {                                    \
      using T = float;                                       \
      __VA_ARGS__;                                           \
    } else if ((et) == ET_BF16) {                            \
      using T = __nv_bfloat16;                               \
      __VA_ARGS__;                                           \
    } else {                                                 \
      using T = __half;                                      \
      __VA_ARGS__;                                           \
    }                                                        \
  } while (0)

inline int grid_for(long n, int threads, int cap = 148 * 16) {
  long b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

// ============================================================== launchers
cudaError_t launch_pack_input(const void* x, int x_f32, int B, int T, int I, int Ip, void* X0, int f32,
                              cudaStream_t s, ZeroRows z) {
  const long n = (long)T * B * Ip;
  const int g = grid_for(n, 256);
  const int esz = f32 == ET_F32 ? 4 : 2;
  if (I == Ip && x_f32 == f32 && (I * esz) % 16 == 0 && !(reinterpret_cast<uintptr_t>(x) & 15) &&
      !(reinterpret_cast<uintptr_t>(X0) & 15)) {
    const long threads = (long)T * B * 32;
    pack_rows_kernel<<<(int)((threads + 255) / 256), 256, 0, s>>>((const uint4*)x, B, T, I * esz / 16, (uint4*)X0, z);
    return cudaGetLastError();
  }
  if (f32 == ET_BF16) {
    if (x_f32 != ET_BF16) return cudaErrorInvalidValue;
    pack_input_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, s>>>((const __nv_bfloat16*)x, B, T, I, Ip,
                                                                      (__nv_bfloat16*)X0, z);
  } else if (f32) {
    if (x_f32) pack_input_kernel<float, float><<<g, 256, 0, s>>>((const float*)x, B, T, I, Ip, (float*)X0, z);
    else pack_input_kernel<__half, float><<<g, 256, 0, s>>>((const __half*)x, B, T, I, Ip, (float*)X0, z);
  } else {
    if (x_f32) pack_input_kernel<float, __half><<<g, 256, 0, s>>>((const float*)x, B, T, I, Ip, (__half*)X0, z);
    else pack_input_kernel<__half, __half><<<g, 256, 0, s>>>((const __half*)x, B, T, I, Ip, (__half*)X0, z);
  }
  return cudaGetLastError();
}

cudaError_t launch_drop_mask(const void* h, void* ht, int B, int hp, const int* step, uint32_t seed, uint32_t layer,
                             uint32_t seq0, uint32_t thr, float scale, cudaStream_t s) {
  const int n = B * hp;
  drop_mask_kernel<<<(n + 255) / 256, 256, 0, s>>>((const __half*)h, (__half*)ht, B, hp, step, seed, layer, seq0, thr,
                                                   scale);
  return cudaGetLastError();
}

__global__ void incr_kernel(int* p) { *p += 1; }
cudaError_t launch_increment(int* p, cudaStream_t s) {
  incr_kernel<<<1, 1, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_embed_gather(const int32_t* tok, int B, int T, const void* E, int Ep, void* X0, int f32,
                                int vocab, int* bad, cudaStream_t s) {
  const long warps = (long)B * T;
  const int g = (int)((warps * 32 + 255) / 256);
  HDP_ET(f32, TT, (embed_gather_kernel<TT><<<g, 256, 0, s>>>(tok, B, T, (const TT*)E, Ep, (TT*)X0, vocab, bad)));
  return cudaGetLastError();
}

cudaError_t launch_cell_fwd(int f32, const float* Gx_t, const float* Gh, const float* c_prev, void* gates_t,
                            float* c_t, void* h_t, int B, int hp, cudaStream_t s) {
  const int n = B * hp;
  const int g = (n + 127) / 128;
  HDP_ET(f32, TT, (cell_fwd_kernel<TT><<<g, 128, 0, s>>>(Gx_t, Gh, c_prev, (TT*)gates_t, c_t, (TT*)h_t, n)));
  return cudaGetLastError();
}

cudaError_t launch_cell_bwd(int f32, const float* dHa_t, const float* dh_rec, const void* gates_t,
                            const float* c_t, const float* c_prev, float* dc, void* dA_t, int B, int hp,
                            int first, cudaStream_t s) {
  const int n = B * hp;
  const int g = (n + 127) / 128;
  HDP_ET(f32, TT, (cell_bwd_kernel<TT><<<g, 128, 0, s>>>(dHa_t, dh_rec, (const TT*)gates_t, c_t, c_prev, dc,
                                                         (TT*)dA_t, n, first)));
  return cudaGetLastError();
}

int head_partials_count(int rows) { return (rows + HEAD_WARPS - 1) / HEAD_WARPS; }

cudaError_t launch_head_out(int f32, const void* Z, int rows, int Kd, long ldz, const void* wo, const void* bo,
                            const int8_t* tgt, int tgt_mode, int B, int T, float alpha, float inv_terms, float* y,
                            float* dy, float* partials, cudaStream_t s, void* dz, const float* alpha_dev) {
  const int g = head_partials_count(rows);
  HDP_ET(f32, TT, (head_out_kernel<TT><<<g, HEAD_WARPS * 32, 0, s>>>((const TT*)Z, rows, Kd, ldz, (const TT*)wo,
                                                                    (const TT*)bo, tgt, tgt_mode, B, T, alpha,
                                                                    inv_terms, y, dy, partials, (TT*)dz, alpha_dev)));
  return cudaGetLastError();
}

cudaError_t launch_loss_final(const float* partials, int n, float inv_terms, float* loss, cudaStream_t s) {
  loss_final_kernel<<<1, 256, 0, s>>>(partials, n, inv_terms, loss);
  return cudaGetLastError();
}

cudaError_t launch_l2_loss(int f32, const void* w, long n, double* part, double l2, float* loss, cudaStream_t s) {
  HDP_ET(f32, TT, (sumsq_partial_kernel<TT><<<L2_BLOCKS, 256, 0, s>>>((const TT*)w, n, part)));
  l2_loss_final_kernel<<<1, 32, 0, s>>>(part, L2_BLOCKS, l2, loss);
  return cudaGetLastError();
}
size_t l2_partials_doubles() { return L2_BLOCKS; }

cudaError_t launch_relu_dz(int f32, const float* dy, const void* wo, const void* Z, void* dz, int rows, int Fp,
                           cudaStream_t s) {
  const int g = grid_for((long)rows * Fp, 256);
  HDP_ET(f32, TT, (relu_dz_kernel<TT><<<g, 256, 0, s>>>(dy, (const TT*)wo, (const TT*)Z, (TT*)dz, rows, Fp)));
  return cudaGetLastError();
}

cudaError_t launch_outer(int f32, const float* dy, const void* wo, float* dH, int rows, int hp, cudaStream_t s) {
  const int g = grid_for((long)rows * hp, 256);
  HDP_ET(f32, TT, (outer_kernel<TT><<<g, 256, 0, s>>>(dy, (const TT*)wo, dH, rows, hp)));
  return cudaGetLastError();
}

size_t colreduce_partials_floats(int rows, int cols) { return (size_t)cr_splits(rows) * cols * 2; }

cudaError_t launch_colreduce(int x_f32, const void* X, long ldx, int rows, int cols, const float* w,
                             float* partials, int out_f32, void* out, cudaStream_t s) {
  const int rs = cr_splits(rows);
  dim3 g1((cols + 31) / 32, rs);
  double* part = reinterpret_cast<double*>(partials);
  HDP_ET(x_f32, TT, (colreduce_pass1<TT><<<g1, CR_WARPS * 32, 0, s>>>((const TT*)X, ldx, rows, cols, w, rs, part)));
  colreduce_pass2<<<(cols * 32 + 255) / 256, 256, 0, s>>>(part, rs, cols, out_f32, out);
  return cudaGetLastError();
}

cudaError_t launch_colreduce3(int x_f32, const void* Z, const void* dz, long ld, int rows, int F, const float* dy,
                              float* partials, int out_f32, void* dwo, void* dfb, void* dbo, cudaStream_t s) {
  const int rs = cr_splits(rows);
  const int cols = 2 * F + 1;
  dim3 g1((cols + 31) / 32, rs);
  double* part = reinterpret_cast<double*>(partials);
  HDP_ET(x_f32, TT, (colreduce3_pass1<TT><<<g1, CR_WARPS * 32, 0, s>>>((const TT*)Z, (const TT*)dz, ld, rows, F, dy,
                                                                       rs, part)));
  colreduce3_pass2<<<(cols * 32 + 255) / 256, 256, 0, s>>>(part, rs, F, out_f32, dwo, dfb, dbo);
  return cudaGetLastError();
}

cudaError_t launch_colreduce3_final(const double* partials, int rs, int F, int out_f32, void* dwo, void* dfb,
                                    void* dbo, cudaStream_t s) {
  const int cols = 2 * F + 1;
  colreduce3_pass2<<<(cols * 32 + 255) / 256, 256, 0, s>>>(partials, rs, F, out_f32, dwo, dfb, dbo);
  return cudaGetLastError();
}

size_t embed_sort_temp_bytes(int n) {
  const size_t ntiles = ((size_t)n + RS_TILE - 1) / RS_TILE;
  return 256 * ntiles * sizeof(int32_t);
}

size_t embed_part_floats(int n, int Ep) { return (size_t)n * Ep; }

cudaError_t launch_embed_backward(const int32_t* tok, int B, int T, int vocab, const float* dX0, int Ep,
                                  int32_t* keys_in, int32_t* keys_out, int32_t* vals_in, int32_t* vals_out,
                                  void* sort_temp, size_t sort_temp_bytes, float* part, void* dE, int out_f32,
                                  int32_t* range, cudaStream_t s) {
  const int n = B * T;
  const int ntiles = (n + RS_TILE - 1) / RS_TILE;
  if (sort_temp_bytes < embed_sort_temp_bytes(n)) return cudaErrorInvalidValue;
  embed_keys_kernel<<<(n + 255) / 256, 256, 0, s>>>(tok, B, T, vocab, keys_in, vals_in);
  int bits = 1;
  while ((1 << bits) < vocab) ++bits;
  int32_t* hist = (int32_t*)sort_temp;
  int32_t *ka = keys_in, *va = vals_in, *kb = keys_out, *vb = vals_out;
  for (int shift = 0; shift < bits; shift += 8) {
    radix_hist_kernel<<<ntiles, RS_TILE, 0, s>>>(ka, n, shift, ntiles, hist);
    radix_scatter_kernel<<<ntiles, RS_TILE, 0, s>>>(ka, va, n, shift, ntiles, hist, kb, vb);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  // (ka, va) = the sorted keys / positions
  cudaError_t e = cudaMemsetAsync(range, 0, (size_t)2 * vocab * sizeof(int32_t), s);
  if (e != cudaSuccess) return e;
  embed_range_kernel<<<(n + 255) / 256, 256, 0, s>>>(ka, n, range, range + vocab);
  const long cw = ((long)n + EMB_CHUNK - 1) / EMB_CHUNK * 32;
  embed_chunk_kernel<<<(int)((cw + 255) / 256), 256, 0, s>>>(ka, va, n, dX0, Ep, part);
  const long threads = (long)vocab * ((Ep + 31) / 32) * 32;
  embed_segsum_kernel<<<(int)((threads + 255) / 256), 256, 0, s>>>(range, range + vocab, vocab, part, Ep, out_f32,
                                                                   dE);
  return cudaGetLastError();
}

}  // namespace hdp
