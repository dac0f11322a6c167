// NEXT-2: the gradient exchange and the fused average + update (A9 + K11 + A11,
// PAPER.md:94-96 steps 4-6) as ONE kernel over NVLink peer memory, launched once per
// bucket group as soon as the group's gradients are complete (the update of the top
// layers overlaps the BPTT of the lower ones, north_star "overlapped with BPTT").
//
// Every rank exposes (CUDA IPC) its gradient vector (fp16, or fp32 on the fp32 wire),
// its fp16 working weights and a small flag / counter block.  One launch, owner r of
// each shard of the launch's buckets:
//   A. publishes "my gradients for launch `seq` are complete" to every peer
//      (st.release.sys) and waits until every contributor has published `seq`
//      (ld.acquire.sys); with partial collection rank 0 instead waits
//      for `quorum` contributors, publishes that set, and every owner uses it;
//   B. reads the contributions of its shard straight from the peers' gradient vectors
//      over NVLink (all loads of a vector issued before the sum), sums them in fp32 in
//      rank order (R14, identical to K11), applies SGD-m / Adam to its fp32 master
//      shard, rounds to fp16 and stores the result into EVERY rank's weight vector --
//      the all-to-all, the update and the all-gather in one pass;
//   C. the last CTA to finish (threadfence-reduction pattern, system scope) publishes
//      "my shards are written" and waits for all ranks, so kernel completion means:
//      every weight of the launch's buckets is final everywhere and no peer still reads
//      my gradients of those buckets.
// Non-finite contribution counts are added into every rank's per-step counter.
// Flags hold monotonically increasing launch numbers: no resets between steps.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "p2p_exchange.cuh"

namespace hdp {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys64(unsigned* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// ~20 s without progress: a peer died or the protocol broke
__device__ __forceinline__ void check_timeout(unsigned long long t0) {
  if (gtimer() - t0 > 20000000000ull) __trap();
}
__device__ __forceinline__ void wait_all(const unsigned* f, int n, unsigned seq) {
  const unsigned long long t0 = gtimer();
  for (int r = 0; r < n; ++r)
    while (ld_acquire_sys(f + r) < seq) check_timeout(t0);
}
__device__ __forceinline__ void spin_ns(unsigned long long ns) {
  const unsigned long long t0 = gtimer();
  while (gtimer() - t0 < ns) {
  }
}

// 8 consecutive contributions of one contributor: raw registers, then fp32
template <typename GT>
struct PV;
template <>
struct PV<__half> {
  struct raw_t { uint4 u; };
  __device__ static raw_t load(const void* base, long e) {
    return {__ldcg(reinterpret_cast<const uint4*>(static_cast<const __half*>(base) + e))};
  }
  __device__ static void cvt(const raw_t& r, float (&o)[8], int& nf) {
    const __half2* h = reinterpret_cast<const __half2*>(&r.u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(h[i]);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
    const uint32_t w[4] = {r.u.x, r.u.y, r.u.z, r.u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) nf += ((w[i] & 0x7C00u) == 0x7C00u) + ((w[i] & 0x7C000000u) == 0x7C000000u);
  }
};
template <>
struct PV<__nv_bfloat16> {  // bf16 wire (bf16 math mode): the upper halves of binary32 values
  struct raw_t { uint4 u; };
  __device__ static raw_t load(const void* base, long e) {
    return {__ldcg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + e))};
  }
  __device__ static void cvt(const raw_t& r, float (&o)[8], int& nf) {
    const uint32_t w[4] = {r.u.x, r.u.y, r.u.z, r.u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[2 * i] = __uint_as_float(w[i] << 16);
      o[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      nf += ((w[i] & 0x7F80u) == 0x7F80u) + ((w[i] & 0x7F800000u) == 0x7F800000u);
    }
  }
};
template <>
struct PV<float> {
  struct raw_t { float4 a, b; };
  __device__ static raw_t load(const void* base, long e) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + e);
    return {__ldcg(p), __ldcg(p + 1)};
  }
  __device__ static void cvt(const raw_t& r, float (&o)[8], int& nf) {
    o[0] = r.a.x; o[1] = r.a.y; o[2] = r.a.z; o[3] = r.a.w;
    o[4] = r.b.x; o[5] = r.b.y; o[6] = r.b.z; o[7] = r.b.w;
#pragma unroll
    for (int i = 0; i < 8; ++i) nf += !isfinite(o[i]);
  }
};

// EXT = 0: plain SGD-m / Adam with every contributor (the hot configuration);
// EXT = 1: L2 term, dynamic-loss-scale skip / device alpha, partial collection.
// NMAX >= N: register arrays sized for at most NMAX contributions (2 / 4 / 8), so a
// 2-rank exchange keeps occupancy (every contribution's load is in flight at once).
template <typename GT, int OPT, bool EXT, int NMAX>
__global__ void __launch_bounds__(256, NMAX <= 2 ? 4 : NMAX <= 4 ? 3 : 2) exch_update_kernel(const __grid_constant__ P2PArgs a) {
  __shared__ int s_nf;
  __shared__ int s_last;
  __shared__ unsigned s_mask;
  const int N = a.N, NR = a.NR, tid = threadIdx.x;
  // ---- A: my gradients are complete (stream order: this kernel runs after them)
  if (blockIdx.x == 0 && a.loopback && (tid < 32 || (tid >= 64 && tid < 96))) {
    // contributor lane = gradient slot lane: on time from warp 0, injected stragglers late from
    // warp 2 (a separate warp, so the on-time lanes do not wait for the spinning ones)
    const int r = tid & 31;
    const bool late = EXT && ((a.straggler_mask >> r) & 1u);
    if (r < N && late == (tid >= 64)) {
      if (late) spin_ns(a.straggler_ns);
      __threadfence_system();
      st_release_sys(a.flag_local + P2P_FLAG_READY + r, a.seq);
    }
  } else if (blockIdx.x == 0 && tid < 32) {
    if (tid < NR) {
      if (EXT && ((a.straggler_mask >> a.rank) & 1u)) spin_ns(a.straggler_ns);
      __threadfence_system();
      st_release_sys(a.flag_peer[tid] + P2P_FLAG_READY + a.rank, a.seq);
    }
  }
  if (EXT && a.quorum > 0 && a.rank == 0 && blockIdx.x == 0 && tid == 32) {
    // partial collection, rank 0 decides: the first `quorum` contributors seen ready
    const unsigned long long t0 = gtimer();
    unsigned m = 0;
    for (;;) {
      m = 0;
      for (int r = 0; r < N; ++r)
        if (ld_acquire_sys(a.flag_local + P2P_FLAG_READY + r) >= a.seq) m |= 1u << r;
      if (__popc(m) >= a.quorum) break;
      check_timeout(t0);
    }
    const unsigned long long dec = ((unsigned long long)a.seq << 32) | m;
    for (int r = 0; r < NR; ++r)
      st_release_sys64((a.loopback ? a.flag_local : a.flag_peer[r]) + P2P_DECISION, dec);
  }
  if (tid == 0) {
    s_nf = 0;
    if (EXT && a.quorum > 0) {
      const unsigned long long t0 = gtimer();
      unsigned long long dec;
      while (((dec = ld_acquire_sys64(a.flag_local + P2P_DECISION)) >> 32) < a.seq) check_timeout(t0);
      s_mask = (unsigned)(dec & 0xffffffffu);
    } else {
      wait_all(a.flag_local + P2P_FLAG_READY, N, a.seq);
      s_mask = (N >= 32) ? 0xffffffffu : ((1u << N) - 1u);
    }
  }
  __syncthreads();
  // ---- B: owned 8-element vectors of the launch's buckets (none on a skipped step)
  const unsigned mask = s_mask;
  int nf = 0;
  const long v0 = a.vpre[a.bk0];
  const long total = (EXT && a.skip && *a.skip) ? 0 : a.vpre[a.bk1] - v0;
  float inv_scale = a.inv_scale;
  if (EXT) {
    if (a.quorum > 0) inv_scale = (float)(1.0 / ((double)__popc(mask) * a.alpha));  // divide by the actual count
    else if (a.alpha_dev) inv_scale = (float)(1.0 / (a.n_workers * (double)*a.alpha_dev));
  }
  int bi = a.bk0;
  for (long v = blockIdx.x * (long)blockDim.x + tid; v < total; v += (long)gridDim.x * blockDim.x) {
    const long vg = v0 + v;
    while (vg >= a.vpre[bi + 1]) ++bi;
    const long k = (vg - a.vpre[bi]) << 3;
    const long e = a.off[bi] + (long)a.rank * a.shard[bi] + k;  // element in the parameter vector
    const long m = a.moff[bi] + k;                              // element in my master shard
    // every contribution's load in flight before the first add
    typename PV<GT>::raw_t raw[NMAX];
#pragma unroll
    for (int r = 0; r < NMAX; ++r)
      if (r < N && ((mask >> r) & 1u)) raw[r] = PV<GT>::load(a.g_peer[r], e);
    const float4 W0 = *reinterpret_cast<const float4*>(a.W + m), W1 = *reinterpret_cast<const float4*>(a.W + m + 4);
    const float4 H0 = *reinterpret_cast<const float4*>(a.S1 + m), H1 = *reinterpret_cast<const float4*>(a.S1 + m + 4);
    float s[8];
    bool first = true;
#pragma unroll
    for (int r = 0; r < NMAX; ++r) {
      if (r < N && ((mask >> r) & 1u)) {
        float t[8];
        PV<GT>::cvt(raw[r], t, nf);
        if (first) {
#pragma unroll
          for (int i = 0; i < 8; ++i) s[i] = t[i];
          first = false;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) s[i] = __fadd_rn(s[i], t[i]);  // rank order (R14)
        }
      }
    }
    float w[8] = {W0.x, W0.y, W0.z, W0.w, W1.x, W1.y, W1.z, W1.w};
    float h[8] = {H0.x, H0.y, H0.z, H0.w, H1.x, H1.y, H1.z, H1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s[i] = __fmul_rn(s[i], inv_scale);
      // L2 (reading Q16): + fp32(2 l2) * fp16(W) (bf16(W) in bf16 mode), the working weight of this step
      if (EXT && a.l2x2 != 0.f)
        s[i] = __fadd_rn(s[i], __fmul_rn(a.l2x2, a.w_bf16 ? __bfloat162float(__float2bfloat16_rn(w[i]))
                                                            : __half2float(__float2half_rn(w[i]))));
    }
    if (OPT == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        h[i] = __fsub_rn(__fmul_rn(a.mom, h[i]), __fmul_rn(a.lam, s[i]));
        w[i] = __fadd_rn(w[i], h[i]);
      }
    } else {
      const float4 V0 = *reinterpret_cast<const float4*>(a.S2 + m), V1 = *reinterpret_cast<const float4*>(a.S2 + m + 4);
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
    uint4 ov;
    if (a.w_bf16) {
      __align__(16) __nv_bfloat162 o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = __floats2bfloat162_rn(w[2 * i], w[2 * i + 1]);
      ov = *reinterpret_cast<const uint4*>(o);
    } else {
      __align__(16) __half2 o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = __halves2half2(__float2half_rn(w[2 * i]), __float2half_rn(w[2 * i + 1]));
      ov = *reinterpret_cast<const uint4*>(o);
    }
#pragma unroll
    for (int r = 0; r < NMAX; ++r)
      if (r < N) __stcg(reinterpret_cast<uint4*>(a.w_peer[r] + e), ov);  // all-gather by peer stores
  }
  // ---- C: completion
  nf = __reduce_add_sync(0xffffffffu, nf);
  if ((tid & 31) == 0 && nf) atomicAdd(&s_nf, nf);
  __syncthreads();
  if (tid == 0) {
    if (s_nf)
      for (int r = 0; r < NR; ++r) atomicAdd_system(a.status_peer[r] + (a.step & 1), s_nf);
    __threadfence_system();
    const unsigned prev = atomicAdd(a.flag_local + P2P_CTR, 1u);
    s_last = prev == a.ctr_target - 1;
  }
  __syncthreads();
  if (s_last && tid < NR) {
    __threadfence_system();
    st_release_sys(a.flag_peer[tid] + P2P_FLAG_DONE + a.rank, a.seq);
  }
  if (s_last && tid == 0) wait_all(a.flag_local + P2P_FLAG_DONE, NR, a.seq);
}

}  // namespace

template <typename GT, int OPT, bool EXT>
const void* exch_fn_n(int N) {
  return N <= 2 ? (const void*)exch_update_kernel<GT, OPT, EXT, 2>
       : N <= 4 ? (const void*)exch_update_kernel<GT, OPT, EXT, 4> : (const void*)exch_update_kernel<GT, OPT, EXT, 8>;
}
const void* exch_fn(const P2PArgs& a, int optimizer, int grad_f32) {
  const bool ext = a.l2x2 != 0.f || a.alpha_dev || a.skip || a.quorum > 0 || a.straggler_mask;
#define HDP_EXCH(GT, OPT) (ext ? exch_fn_n<GT, OPT, true>(a.N) : exch_fn_n<GT, OPT, false>(a.N))
  if (grad_f32 == 2) return optimizer == 0 ? HDP_EXCH(__nv_bfloat16, 0) : HDP_EXCH(__nv_bfloat16, 1);
  if (grad_f32) return optimizer == 0 ? HDP_EXCH(float, 0) : HDP_EXCH(float, 1);
  return optimizer == 0 ? HDP_EXCH(__half, 0) : HDP_EXCH(__half, 1);
#undef HDP_EXCH
}

cudaError_t launch_exch_update(const P2PArgs& a, int optimizer, int grad_f32, int grid, cudaStream_t s) {
  void* args[] = {const_cast<P2PArgs*>(&a)};
  return cudaLaunchKernel(exch_fn(a, optimizer, grad_f32), dim3(grid), dim3(256), args, 0, s);
}

int exch_resident_ctas(const P2PArgs& a, int optimizer, int grad_f32) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, exch_fn(a, optimizer, grad_f32), 256, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

}  // namespace hdp
