// K11: fused gradient average + global weight update (PAPER.md:94-95 steps
// 4-5, Eqs. 1-2 :101-102; loss-scale removal :177, reading Q6).
//
// Per owned element, in this exact fp32 operation order (R14/R15):
//   s  = fp32(g_0) + fp32(g_1) + ... + fp32(g_{N-1})     rank order, each add RNE
//   g  = s * inv_scale                                  inv_scale = fp32(1/(N*alpha))
//   g  = g + l2x2 * w_work     (only if l2 > 0; w_work = fp16(W) in mixed mode)
//   SGD-m:  H = m*H - lam*g ;  W = W + H                (each op separately RNE, no FMA)
//   Adam :  m1 = b1*m1 + (1-b1)*g ; v = b2*v + (1-b2)*g*g ;
//           W  = W - lam * (m1*c1) / (sqrt(v*c2) + eps)
//   w16 = RNE_fp16(W)    (or w32 = W in FP32 mode)
//   nonfinite += number of Inf/NaN contributions
// HBM traffic per element: N*sizeof(g) + 4+4 (W,H read) + 4+4 (W,H write) + 2 (w16).
// 128-bit loads/stores, grid-stride over 8-element vectors.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hdp {
namespace {

template <typename GT>
struct Vec8;
template <>
struct Vec8<__half> {
  __device__ static void load(const __half* p, float (&o)[8], int& nf) {
    const uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));  // streamed once
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(h[i]);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      nf += ((w[i] & 0x7C00u) == 0x7C00u);
      nf += ((w[i] & 0x7C000000u) == 0x7C000000u);
    }
  }
};
template <>
struct Vec8<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, float (&o)[8], int& nf) {
    const uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // bf16 = the upper half of a binary32
      o[2 * i] = __uint_as_float(w[i] << 16);
      o[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      nf += ((w[i] & 0x7F80u) == 0x7F80u) + ((w[i] & 0x7F800000u) == 0x7F800000u);
    }
  }
};
template <>
struct Vec8<float> {
  __device__ static void load(const float* p, float (&o)[8], int& nf) {
    const float4 a = __ldcs(reinterpret_cast<const float4*>(p));
    const float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
#pragma unroll
    for (int i = 0; i < 8; ++i) nf += !isfinite(o[i]);
  }
};

__device__ __forceinline__ float upd_sgdm(const UpdateArgs& a, float g, float& W, float& H) {
  const float t1 = __fmul_rn(a.mom, H);
  const float t2 = __fmul_rn(a.lam, g);
  H = __fsub_rn(t1, t2);
  W = __fadd_rn(W, H);
  return W;
}
__device__ __forceinline__ float upd_adam(const UpdateArgs& a, float g, float& W, float& m1, float& v) {
  m1 = __fadd_rn(__fmul_rn(a.b1, m1), __fmul_rn(a.omb1, g));
  const float gg = __fmul_rn(g, g);
  v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(a.omb2, gg));
  const float mhat = __fmul_rn(m1, a.c1);
  const float vhat = __fmul_rn(v, a.c2);
  const float den = __fadd_rn(__fsqrt_rn(vhat), a.eps);
  const float u = __fdiv_rn(mhat, den);
  W = __fsub_rn(W, __fmul_rn(a.lam, u));
  return W;
}

// the working weight of this step: fp16(W) / bf16(W) (mixed modes, R1) or W
__device__ __forceinline__ float w_work(const UpdateArgs& a, float W) {
  if (!a.w16) return W;
  return a.w_bf16 ? __bfloat162float(__float2bfloat16_rn(W)) : __half2float(__float2half_rn(W));
}
__device__ __forceinline__ float l2_term(const UpdateArgs& a, float g, float W) {
  if (a.l2x2 == 0.f) return g;
  return __fadd_rn(g, __fmul_rn(a.l2x2, w_work(a, W)));
}

// EXT = 0: the plain SGD-m / Adam step (the hot configuration); EXT = 1 adds the L2 term and
// the dynamic-loss-scale skip / device alpha (NEXT-3).  Separate instantiations keep the
// plain kernel's code exactly as lean as before the options existed (measured: folding the
// option checks into one kernel cost ~9 % of its HBM rate at 1 GiB).
template <typename GT, int OPT, bool EXT>
__global__ void __launch_bounds__(256) avg_update_kernel(UpdateArgs a) {
  if (EXT) {
    if (a.skip && *a.skip) return;  // dynamic loss scaling: non-finite step, nothing changes
    if (a.alpha_dev) a.inv_scale = (float)(1.0 / (a.n_workers * (double)*a.alpha_dev));  // R14
  }
  const GT* __restrict__ g = static_cast<const GT*>(a.g);
  const long nvec = a.count >> 3;
  int nf = 0;
  for (long v = blockIdx.x * (long)blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.x * blockDim.x) {
    const long e = v << 3;
    float s[8];
    Vec8<GT>::load(g + e, s, nf);
    for (int r = 1; r < a.nsrc; ++r) {
      float t[8];
      Vec8<GT>::load(g + (long)r * a.g_stride + e, t, nf);
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] = __fadd_rn(s[i], t[i]);
    }
    float4 W0 = *reinterpret_cast<const float4*>(a.W + e), W1 = *reinterpret_cast<const float4*>(a.W + e + 4);
    float4 S0 = *reinterpret_cast<const float4*>(a.S1 + e), S1 = *reinterpret_cast<const float4*>(a.S1 + e + 4);
    float w[8] = {W0.x, W0.y, W0.z, W0.w, W1.x, W1.y, W1.z, W1.w};
    float h[8] = {S0.x, S0.y, S0.z, S0.w, S1.x, S1.y, S1.z, S1.w};
    if (EXT) {
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] = l2_term(a, __fmul_rn(s[i], a.inv_scale), w[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] = __fmul_rn(s[i], a.inv_scale);
    }
    if (OPT == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) upd_sgdm(a, s[i], w[i], h[i]);
    } else {
      float4 V0 = *reinterpret_cast<const float4*>(a.S2 + e), V1 = *reinterpret_cast<const float4*>(a.S2 + e + 4);
      float vv[8] = {V0.x, V0.y, V0.z, V0.w, V1.x, V1.y, V1.z, V1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) upd_adam(a, s[i], w[i], h[i], vv[i]);
      *reinterpret_cast<float4*>(a.S2 + e) = make_float4(vv[0], vv[1], vv[2], vv[3]);
      *reinterpret_cast<float4*>(a.S2 + e + 4) = make_float4(vv[4], vv[5], vv[6], vv[7]);
    }
    *reinterpret_cast<float4*>(a.W + e) = make_float4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<float4*>(a.W + e + 4) = make_float4(w[4], w[5], w[6], w[7]);
    *reinterpret_cast<float4*>(a.S1 + e) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(a.S1 + e + 4) = make_float4(h[4], h[5], h[6], h[7]);
    if (a.w16 && a.w_bf16) {
      __align__(16) __nv_bfloat162 o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = __floats2bfloat162_rn(w[2 * i], w[2 * i + 1]);
      *reinterpret_cast<uint4*>(a.w16 + e) = *reinterpret_cast<const uint4*>(o);
    } else if (a.w16) {
      __align__(16) __half2 o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = __halves2half2(__float2half_rn(w[2 * i]), __float2half_rn(w[2 * i + 1]));
      *reinterpret_cast<uint4*>(a.w16 + e) = *reinterpret_cast<const uint4*>(o);
    }
    if (a.w32) {
      *reinterpret_cast<float4*>(a.w32 + e) = make_float4(w[0], w[1], w[2], w[3]);
      *reinterpret_cast<float4*>(a.w32 + e + 4) = make_float4(w[4], w[5], w[6], w[7]);
    }
  }
  // scalar tail (count not a multiple of 8)
  for (long e = (nvec << 3) + blockIdx.x * (long)blockDim.x + threadIdx.x; e < a.count;
       e += (long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int r = 0; r < a.nsrc; ++r) {
      const float t = static_cast<float>(g[(long)r * a.g_stride + e]);
      nf += !isfinite(t);
      s = r == 0 ? t : __fadd_rn(s, t);
    }
    float w = a.W[e], h = a.S1[e];
    s = __fmul_rn(s, a.inv_scale);
    if (EXT) s = l2_term(a, s, w);
    if (OPT == 0) {
      upd_sgdm(a, s, w, h);
    } else {
      float vv = a.S2[e];
      upd_adam(a, s, w, h, vv);
      a.S2[e] = vv;
    }
    a.W[e] = w;
    a.S1[e] = h;
    if (a.w16 && a.w_bf16) reinterpret_cast<__nv_bfloat16*>(a.w16)[e] = __float2bfloat16_rn(w);
    else if (a.w16) a.w16[e] = __float2half_rn(w);
    if (a.w32) a.w32[e] = w;
  }
  if (a.nonfinite) {
    nf = __reduce_add_sync(0xffffffffu, nf);
    if ((threadIdx.x & 31) == 0 && nf) atomicAdd(a.nonfinite, nf);
  }
}

template <typename GT>
__global__ void __launch_bounds__(256) count_nonfinite_kernel(const GT* __restrict__ g, long n, int* count) {
  int nf = 0;
  const long nvec = n >> 3;
  for (long v = blockIdx.x * (long)blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.x * blockDim.x) {
    float t[8];
    Vec8<GT>::load(g + (v << 3), t, nf);
  }
  for (long e = (nvec << 3) + blockIdx.x * (long)blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
    nf += !isfinite(static_cast<float>(g[e]));
  nf = __reduce_add_sync(0xffffffffu, nf);
  if ((threadIdx.x & 31) == 0 && nf) atomicAdd(count, nf);
}

__global__ void loss_scale_update_kernel(int* st, float* alpha, int interval, float factor, float min_alpha) {
  if (threadIdx.x != 0) return;
  if (st[0] > 0) {
    *alpha = fmaxf(*alpha / factor, min_alpha);
    st[1] = 0;
    st[2] += 1;
  } else if (++st[1] >= interval) {
    *alpha = *alpha * factor;
    st[1] = 0;
  }
}

}  // namespace

cudaError_t launch_count_nonfinite(const void* g, long n, int g_f32, int* count, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  long blocks = ((n >> 3) + 255) / 256;
  if (blocks > 148L * 8) blocks = 148L * 8;
  if (blocks < 1) blocks = 1;
  if (g_f32 == ET_F32) count_nonfinite_kernel<float><<<(int)blocks, 256, 0, s>>>((const float*)g, n, count);
  else if (g_f32 == ET_BF16)
    count_nonfinite_kernel<__nv_bfloat16><<<(int)blocks, 256, 0, s>>>((const __nv_bfloat16*)g, n, count);
  else count_nonfinite_kernel<__half><<<(int)blocks, 256, 0, s>>>((const __half*)g, n, count);
  return cudaGetLastError();
}

cudaError_t launch_loss_scale_update(int* st, float* alpha, int interval, float factor, float min_alpha,
                                     cudaStream_t s) {
  loss_scale_update_kernel<<<1, 32, 0, s>>>(st, alpha, interval, factor, min_alpha);
  return cudaGetLastError();
}

cudaError_t launch_avg_update(const UpdateArgs& a, int grad_is_f32, int optimizer, cudaStream_t s) {
  if (a.count <= 0) return cudaSuccess;
  long nvec = (a.count + 7) >> 3;
  long blocks = (nvec + 255) / 256;
  if (blocks > 148L * 8) blocks = 148L * 8;
  if (blocks < 1) blocks = 1;
  const bool ext = a.l2x2 != 0.f || a.alpha_dev || a.skip;
  const int g = (int)blocks;
#define HDP_AVG_LAUNCH(GT, OPT)                                                         \
  (ext ? (avg_update_kernel<GT, OPT, true><<<g, 256, 0, s>>>(a), 0)                     \
       : (avg_update_kernel<GT, OPT, false><<<g, 256, 0, s>>>(a), 0))
  if (grad_is_f32 == ET_F32) {
    if (optimizer == 0) HDP_AVG_LAUNCH(float, 0);
    else HDP_AVG_LAUNCH(float, 1);
  } else if (grad_is_f32 == ET_BF16) {
    if (optimizer == 0) HDP_AVG_LAUNCH(__nv_bfloat16, 0);
    else HDP_AVG_LAUNCH(__nv_bfloat16, 1);
  } else {
    if (optimizer == 0) HDP_AVG_LAUNCH(__half, 0);
    else HDP_AVG_LAUNCH(__half, 1);
  }
#undef HDP_AVG_LAUNCH
  return cudaGetLastError();
}

}  // namespace hdp
