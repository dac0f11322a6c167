// NEXT-2: the gradient exchange and the fused average + update (A9 + K11 + A11,
// PAPER.md:94-96 steps 4-6) as ONE kernel over NVLink peer memory.
//
// Every rank exposes (CUDA IPC) its fp16 gradient vector, its fp16 working
// weights and a small flag / counter block.  Owner r of each bucket shard:
//   A. publishes "my gradients of step s are complete" to every peer (st.release.sys)
//      and waits until all N ranks have published step s (ld.acquire.sys);
//   B. reads the N contributions of its shard straight from the peers' gradient
//      vectors over NVLink (16-B loads, rank order), sums them in fp32 (R14 order,
//      identical to K11), applies SGD-m / Adam to its fp32 master shard, rounds
//      to fp16 and stores the result into EVERY rank's weight vector (16-B peer
//      stores) -- the all-to-all, the update and the all-gather in one pass;
//   C. the last CTA to finish (threadfence-reduction pattern, system scope)
//      publishes "my shards are written" and waits for all N ranks' publication,
//      so that kernel completion means: every weight everywhere is final and no
//      peer still reads my gradients (the next step may overwrite them).
// Non-finite contribution counts are added into every rank's per-step counter.
// Flags hold monotonically increasing step numbers: no resets between steps.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "p2p_exchange.cuh"

namespace hdp {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_all(const unsigned* f, int n, unsigned step) {
  const long long t0 = clock64();
  for (int r = 0; r < n; ++r)
    while (ld_acquire_sys(f + r) < step) {
      if (clock64() - t0 > 40000000000ll) __trap();  // ~20 s: a peer died or the protocol broke
    }
}

__device__ __forceinline__ void load8h(const __half* p, float (&o)[8], int& nf) {
  const uint4 u = __ldcv(reinterpret_cast<const uint4*>(p));  // peer memory: no stale L1 / L2 lines
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(h[i]);
    o[2 * i] = f.x;
    o[2 * i + 1] = f.y;
  }
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) nf += ((w[i] & 0x7C00u) == 0x7C00u) + ((w[i] & 0x7C000000u) == 0x7C000000u);
}

template <int OPT>
__global__ void __launch_bounds__(256) exch_update_kernel(const __grid_constant__ P2PArgs a) {
  __shared__ int s_nf;
  __shared__ int s_last;
  const int N = a.N, NR = a.NR;
  // ---- A: my gradients are complete (stream order: this kernel runs after the backward)
  if (blockIdx.x == 0 && threadIdx.x < NR) {
    __threadfence_system();
    st_release_sys(a.flag_peer[threadIdx.x] + P2P_FLAG_READY + a.rank, a.step);
  }
  if (threadIdx.x == 0) {
    s_nf = 0;
    wait_all(a.flag_local + P2P_FLAG_READY, NR, a.step);
  }
  __syncthreads();
  // ---- B: owned 8-element vectors of every bucket (none on a skipped step)
  int nf = 0;
  const long total = (a.skip && *a.skip) ? 0 : a.vpre[a.nb];
  const float inv_scale = a.alpha_dev ? (float)(1.0 / (a.n_workers * (double)*a.alpha_dev)) : a.inv_scale;
  for (long v = blockIdx.x * (long)blockDim.x + threadIdx.x; v < total; v += (long)gridDim.x * blockDim.x) {
    int bi = 0;
    while (v >= a.vpre[bi + 1]) ++bi;
    const long k = (v - a.vpre[bi]) << 3;
    const long e = a.off[bi] + (long)a.rank * a.shard[bi] + k;  // element in the parameter vector
    const long m = a.moff[bi] + k;                              // element in my master shard
    float s[8];
    load8h(a.g_peer[0] + e, s, nf);
    for (int r = 1; r < N; ++r) {
      float t[8];
      load8h(a.g_peer[r] + e, t, nf);
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] = __fadd_rn(s[i], t[i]);
    }
    float4 W0 = *reinterpret_cast<const float4*>(a.W + m), W1 = *reinterpret_cast<const float4*>(a.W + m + 4);
    float4 H0 = *reinterpret_cast<const float4*>(a.S1 + m), H1 = *reinterpret_cast<const float4*>(a.S1 + m + 4);
    float w[8] = {W0.x, W0.y, W0.z, W0.w, W1.x, W1.y, W1.z, W1.w};
    float h[8] = {H0.x, H0.y, H0.z, H0.w, H1.x, H1.y, H1.z, H1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s[i] = __fmul_rn(s[i], inv_scale);
      // L2 (reading Q16): + fp32(2 l2) * fp16(W), the working weight of this step
      if (a.l2x2 != 0.f) s[i] = __fadd_rn(s[i], __fmul_rn(a.l2x2, __half2float(__float2half_rn(w[i]))));
    }
    if (OPT == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float g = s[i];
        h[i] = __fsub_rn(__fmul_rn(a.mom, h[i]), __fmul_rn(a.lam, g));
        w[i] = __fadd_rn(w[i], h[i]);
      }
    } else {
      float4 V0 = *reinterpret_cast<const float4*>(a.S2 + m), V1 = *reinterpret_cast<const float4*>(a.S2 + m + 4);
      float vv[8] = {V0.x, V0.y, V0.z, V0.w, V1.x, V1.y, V1.z, V1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float g = s[i];
        h[i] = __fadd_rn(__fmul_rn(a.b1, h[i]), __fmul_rn(a.omb1, g));
        vv[i] = __fadd_rn(__fmul_rn(a.b2, vv[i]), __fmul_rn(a.omb2, __fmul_rn(g, g)));
        const float den = __fadd_rn(__fsqrt_rn(__fmul_rn(vv[i], a.c2)), a.eps);
        w[i] = __fsub_rn(w[i], __fmul_rn(a.lam, __fdiv_rn(__fmul_rn(h[i], a.c1), den)));
      }
      *reinterpret_cast<float4*>(a.S2 + m) = make_float4(vv[0], vv[1], vv[2], vv[3]);
      *reinterpret_cast<float4*>(a.S2 + m + 4) = make_float4(vv[4], vv[5], vv[6], vv[7]);
    }
    *reinterpret_cast<float4*>(a.W + m) = make_float4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<float4*>(a.W + m + 4) = make_float4(w[4], w[5], w[6], w[7]);
    *reinterpret_cast<float4*>(a.S1 + m) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(a.S1 + m + 4) = make_float4(h[4], h[5], h[6], h[7]);
    __align__(16) __half2 o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = __halves2half2(__float2half_rn(w[2 * i]), __float2half_rn(w[2 * i + 1]));
    const uint4 ov = *reinterpret_cast<const uint4*>(o);
    for (int r = 0; r < N; ++r) __stcg(reinterpret_cast<uint4*>(a.w_peer[r] + e), ov);  // all-gather by peer stores
  }
  // ---- C: completion
  if (nf) atomicAdd(&s_nf, nf);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_nf)
      for (int r = 0; r < NR; ++r) atomicAdd_system(a.status_peer[r] + (a.step & 1), s_nf);
    __threadfence_system();
    const unsigned prev = atomicAdd(a.flag_local + P2P_CTR, 1u);
    s_last = prev == a.step * gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x < NR) {
    __threadfence_system();
    st_release_sys(a.flag_peer[threadIdx.x] + P2P_FLAG_DONE + a.rank, a.step);
  }
  if (s_last && threadIdx.x == 0) wait_all(a.flag_local + P2P_FLAG_DONE, NR, a.step);
}

}  // namespace

cudaError_t launch_exch_update(const P2PArgs& a, int optimizer, int grid, cudaStream_t s) {
  if (optimizer == 0)
    exch_update_kernel<0><<<grid, 256, 0, s>>>(a);
  else
    exch_update_kernel<1><<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace hdp
