// Persistent fused LSTM recurrences for small h: one launch
// runs all T steps of a layer (per-layer cluster kernels) or of both layers of a
// two-layer model (the wavefronts, recur2f_kernel / recur2_bwd_kernel).
//
//   a_t = G_x[t] + h_{t-1} U^T ;  i,f,o = sigma(a), g = tanh(a)
//   c_t = f c_{t-1} + i g ;  h_t = o tanh(c_t)          (reading Q1)
//
// One thread-block cluster per batch group: each CTA keeps its U (or U^T) slice
// resident in shared memory / TMEM for all T steps, runs the step's tcgen05.mma into
// TMEM, applies the cell in the epilogue, and pushes its slice of h_t (dA_t backward)
// into every peer's operand buffer by cp.async.bulk shared::cta -> shared::cluster,
// completing on the peer's mbarrier (double-buffered by step parity).
// Layout conventions are those of hdp_api.cpp (gate row 4j+g).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <algorithm>

#include "gemm.cuh"
#include "options.h"
#include "ptx.cuh"
#include "dropout.cuh"
#include "recur.cuh"

namespace hdp {
namespace {


// sigma(x) with the SFU exponential; relative error ~1e-6, far below the
// fp16 rounding (R4, R6) applied to everything this kernel stores.
__device__ __forceinline__ float sigm_fast(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
// tanh(c) and 1 - tanh(c)^2 from s = sigma(2c): tanh = s - (1 - s), sech^2 = 4 s (1 - s)
// (no cancellation in sech^2; |c| clamped to 15 where both are exact in fp32)
__device__ __forceinline__ void tanh_sech2(float c, float& th, float& sech2) {
  const float cc = fminf(fmaxf(c, -15.f), 15.f);
  const float e = __expf(-2.f * cc);
  const float sg = __fdividef(1.f, 1.f + e);
  const float om = e * sg;  // 1 - sigma(2c)
  th = sg - om;
  sech2 = 4.f * sg * om;
}
// branch-free gate activation: tanh(a) = 2 sigma(2a) - 1 for the g gate
__device__ __forceinline__ float act_gate(float a, float s) { return fmaf(s, sigm_fast(s * a), 1.f - s); }

__device__ __forceinline__ void release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned acquire_ld(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// named CTA barrier 1..15 (barrier 0 is __syncthreads): arrive without waiting / wait
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// spin (one thread) until a release/acquire counter reaches target; trap after 10 s
__device__ __forceinline__ void spin_until(const unsigned* f, unsigned target) {
  if (acquire_ld(f) >= target) return;
  const uint64_t t0 = ptx::globaltimer_ns();
  while (acquire_ld(f) < target) {
    if (ptx::globaltimer_ns() - t0 > 10000000000ull) __trap();
  }
}

// smem: [U: nkb x 16 KB][H: nkb x Bc*128 B][act: nwarps x 16 x ACT_LD fp32][barriers]
constexpr int ACT_LD = 40;  // 32 rows + 8 pad: conflict-free float4 reads (see epilogue)

size_t fwd_smem(int hp, int Bc, int nwarps) {
  const int nkb = (hp + 63) / 64;
  return 1024 + (size_t)nkb * 16384 + (size_t)nkb * Bc * 128 + (size_t)nwarps * 16 * ACT_LD * 4 + 128;
}

struct FwdPlan {
  int nbg = 1, Bc = 0, cgN = 1, nci = 1, G = 1;
};

bool plan_fwd(int B, int hp, FwdPlan* p) {
  if (B < 16 || (B & 15) || (hp & 15)) return false;
  p->G = (4 * hp + 127) / 128;
  int force = 0;
  force = opt(OPT_RECUR_NBG);
  int best = 0;
  for (int nbg = 16; nbg >= 1; nbg >>= 1) {
    if (force && nbg != force) continue;
    if (B % nbg) continue;
    const int Bc = B / nbg;
    if ((Bc & 15) || Bc < 16 || Bc > 256) continue;
    if (p->G * nbg > 148) continue;
    best = nbg;  // largest batch-group count that fits: most SMs, shortest per-step critical path
    break;
  }
  if (!best) return false;
  p->nbg = best;
  p->Bc = B / best;
  const int nchunk = p->Bc / 16;
  p->cgN = nchunk < 4 ? nchunk : 4;
  p->nci = (nchunk + p->cgN - 1) / p->cgN;
  if (p->nci > 4) return false;
  return fwd_smem(hp, p->Bc, 4 * p->cgN) <= 227 * 1024;
}


// ============================================================== backward
size_t bwd_smem(int hp, int Bc) {
  const int nkb = 4 * hp / 64;
  return 1024 + (size_t)nkb * 8192 + (size_t)nkb * Bc * 128 + 128;
}

bool plan_bwd(int B, int hp, int* Bc_out, int* nbg_out) {
  if (B < 16 || (B & 15) || (hp & 15)) return false;
  const int G = (hp + 63) / 64;
  int force = 0;
  force = opt(OPT_RECUR_NBG);
  for (int nbg = 16; nbg >= 1; nbg >>= 1) {
    if (force && nbg != force) continue;
    if (B % nbg) continue;
    const int Bc = B / nbg;
    if ((Bc & 15) || Bc < 16 || Bc > 64) continue;
    if (G * nbg > 148) continue;
    if (bwd_smem(hp, Bc) > 227 * 1024) continue;
    *Bc_out = Bc;
    *nbg_out = nbg;
    return true;
  }
  return false;
}


// ============================================================== per-layer cluster kernels
// One thread-block cluster per batch group (cluster = all row / unit tiles of
// the layer, <= 8 CTAs).  The per-step exchange never leaves the chip: each
// CTA pushes its slice of h_t (forward) or dA_t (backward) into every peer's
// shared-memory operand buffer (double-buffered by step parity).  Global copies
// (needed by later kernels) are still written, off the critical path.
// (Round 1's grid-barrier variants -- an L2 counter barrier per step and a TMA
// reload of h_{t-1} -- were superseded by these and removed in round 2.)

// CTA = 64 units = 256 interleaved gate rows (two M=128 MMAs per K-step) =
// one full 64-wide K-block of h, so its h_t slice is one contiguous region of
// every peer's operand buffer.  Warps: 4 lane quarters x 2 row halves x cgN
// column groups.
template <int NCI>
__global__ void __launch_bounds__(512, 1)
    recur_fwd_cl_kernel(const __grid_constant__ CUtensorMap tmU, const float* __restrict__ Gx, int T, int B, int Bc,
                        int hp, __half* __restrict__ Hs, float* __restrict__ Cst, __half* __restrict__ gates,
                        unsigned long long* __restrict__ trace) {
  const bool tr = trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nkb = (hp + 63) / 64;             // == cluster size
  const int nk16 = (hp + 15) / 16;
  const int nwarps = blockDim.x >> 5;
  const int cgN = nwarps >> 3;
  const int hbuf = nkb * Bc * 128;            // one h operand buffer (K-major SW128)
  uint8_t* sU = smem;                         // [2 halves][nkb][16 KB]
  uint8_t* sH = sU + 2 * nkb * 16384;         // [2][hbuf], filled by the peers' bulk copies
  uint8_t* sX = sH + 2 * hbuf;                // [2][Bc][128 B] my h_t K-block (destination layout)
  float* sAct = reinterpret_cast<float*>(sX + 2 * Bc * 128);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAct + nwarps * 16 * ACT_LD);
  uint64_t* barU = bars;
  uint64_t* barM = bars + 1;
  uint64_t* fullH = bars + 2;                 // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, hf = (warp >> 2) & 1, cg = warp >> 3;
  const int G = gridDim.x;                    // == cluster size
  const int rank = blockIdx.x;
  const int row0 = rank * 256;
  const int col0 = blockIdx.y * Bc;
  const int r = hf * 128 + quarter * 32 + lane;  // tile row in [0, 256)
  const int grow = row0 + r;
  const int gate = r & 3;
  const int unit = grow >> 2;
  const bool unit_ok = unit < hp;
  const int fourhp = 4 * hp;
  const int nacc = Bc <= 32 ? 4 : Bc <= 64 ? 2 : 1;
  const int nis = min(nacc, nk16);            // issuing warps
  const int ac = 2 * nacc * Bc;               // [half][acc][Bc] fp32 columns
  const uint32_t tcols = ac <= 32 ? 32 : ac <= 64 ? 64 : ac <= 128 ? 128 : ac <= 256 ? 256 : 512;
  const int total_bytes = nkb * Bc * 128;     // every consumer receives all of h_{t-1}

  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tmU);
    ptx::mbar_init(barU, 1);
    ptx::mbar_init(barM, nis);
    ptx::mbar_init(fullH, 1);
    ptx::mbar_init(fullH + 1, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tslot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(fullH, total_bytes);
    ptx::mbar_arrive_expect_tx(fullH + 1, total_bytes);
    ptx::mbar_arrive_expect_tx(barU, 2 * nkb * 16384);
    for (int h2 = 0; h2 < 2; ++h2)
      for (int kb = 0; kb < nkb; ++kb)
        ptx::tma_load_2d(sU + (h2 * nkb + kb) * 16384, &tmU, barU, kb * 64, row0 + h2 * 128);
    ptx::mbar_wait(barU, 0);
  }
  ptx::cluster_arrive();  // all CTAs resident, barriers initialised and armed
  ptx::cluster_wait();

  float creg[NCI * 4];
#pragma unroll
  for (int i = 0; i < NCI * 4; ++i) creg[i] = 0.f;
  const uint32_t idesc = ptx::idesc_f16_f32(128, Bc, 0, 0);
  const int nchunk = Bc / 16;
  float* myAct = sAct + warp * 16 * ACT_LD;
  const float gsc = gate == 2 ? 2.f : 1.f;
  const uint32_t sH_addr = ptx::smem_u32(sH), sX_addr = ptx::smem_u32(sX);
  uint32_t fphase[2] = {0u, 0u};

  for (int t = 0; t < T; ++t) {
    if (tr) trace[t * 5 + 0] = ptx::globaltimer_ns();
    float gx[NCI][16];
#pragma unroll
    for (int ci = 0; ci < NCI; ++ci) {
      const int ch = ci * cgN + cg;
      const bool ok = ch < nchunk && grow < fourhp;
      const float* gp = Gx + ((size_t)t * B + col0 + ch * 16) * fourhp + grow;
#pragma unroll
      for (int k = 0; k < 16; ++k) gx[ci][k] = ok ? __ldg(gp + (size_t)k * fourhp) : 0.f;
    }
    if (t > 0) {
      const int p = (t - 1) & 1;
      if (lane == 0 && warp < nis) {
        ptx::mbar_wait(fullH + p, fphase[p]);  // every peer's h_{t-1} K-block landed in sH[p]
        ptx::tc_fence_after();
        if (tr) trace[t * 5 + 1] = ptx::globaltimer_ns();
        const uint32_t aU = ptx::smem_u32(sU), aH = sH_addr + p * hbuf;
        const uint64_t ad0 = ptx::smem_desc_sw128(aU, 0, 1024), bd0 = ptx::smem_desc_sw128(aH, 0, 1024);
        for (int k = warp; k < nk16; k += nis) {
          const int kb = k >> 2, kk = k & 3;  // start-address field is in 16-B units
          const uint64_t bd = bd0 + (uint64_t)((kb * Bc * 128 + kk * 32) >> 4);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const uint64_t ad = ad0 + (uint64_t)(((h2 * nkb + kb) * 16384 + kk * 32) >> 4);
            ptx::mma_f16(tbase + (h2 * nacc + warp) * Bc, ad, bd, idesc, k >= nis ? 1u : 0u);
          }
        }
        ptx::mma_commit(barM);
      }
      __syncwarp();
      ptx::mbar_wait_relaxed(barM, (t - 1) & 1);
      ptx::tc_fence_after();
      fphase[p] ^= 1u;
      if (threadIdx.x == 0 && t + 2 <= T - 1) ptx::mbar_arrive_expect_tx(fullH + p, total_bytes);
    }
    if (tr) trace[t * 5 + 2] = ptx::globaltimer_ns();
    __half* hout = Hs + (size_t)(t + 1) * B * hp;
    float* cout = Cst + (size_t)t * B * hp;
    __half* gout = gates + (size_t)t * B * fourhp;
    uint8_t* stg = sX + (t & 1) * Bc * 128;
#pragma unroll
    for (int ci = 0; ci < NCI; ++ci) {
      const int ch = ci * cgN + cg;
      if (ch >= nchunk) break;
      const int c0 = ch * 16;
      float v[16];
      if (t > 0) {
        const uint32_t ta = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + hf * nacc * Bc + c0;
        ptx::tmem_ld16(ta, v);
        for (int a = 1; a < nis; ++a) {
          float w[16];
          ptx::tmem_ld16(ta + a * Bc, w);
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] += w[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) myAct[k * ACT_LD + lane] = act_gate(v[k] + gx[ci][k], gsc);
      __syncwarp();
      if (unit_ok) {
        const int u = lane >> 2;
        const int ul = (r >> 2);              // unit within my 64-unit slice
        const int c = ul >> 3;                // 16-B chunk of the K-block row
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col = 4 * q + gate;
          const float4 a4 = *reinterpret_cast<const float4*>(myAct + col * ACT_LD + 4 * u);
          const int bl = c0 + col;
          const size_t b = (size_t)col0 + bl;
          const float i = a4.x, f = a4.y, g = a4.z, o = a4.w;
          const float cv = f * creg[ci * 4 + q] + i * g;
          creg[ci * 4 + q] = cv;
          const __half hh = __float2half_rn(o * act_gate(cv, 2.f));
          cout[b * hp + unit] = cv;                   // R5
          hout[b * hp + unit] = hh;                   // R6
          *reinterpret_cast<__half*>(stg + bl * 128 + ((c ^ (bl & 7)) << 4) + (ul & 7) * 2) = hh;
          __align__(8) __half2 gg[2] = {__halves2half2(__float2half_rn(i), __float2half_rn(f)),
                                        __halves2half2(__float2half_rn(g), __float2half_rn(o))};
          *reinterpret_cast<uint2*>(gout + b * fourhp + 4 * unit) = *reinterpret_cast<const uint2*>(gg);  // R4
        }
      }
      __syncwarp();
    }
    ptx::tc_fence_before();
    ptx::fence_async_smem();  // staging writes (generic) -> bulk copy reads (async proxy)
    __syncthreads();
    if (tr) trace[t * 5 + 3] = ptx::globaltimer_ns();
    // push h_t (consumed at step t+1): my K-block rows into every peer's sH[t & 1], one copy per peer
    if (t < T - 1 && threadIdx.x < G) {
      const int dst = threadIdx.x;
      const uint32_t dsta = ptx::mapa(sH_addr + (t & 1) * hbuf + rank * Bc * 128, dst);
      const uint32_t mb = ptx::mapa(ptx::smem_u32(fullH + (t & 1)), dst);
      ptx::bulk_copy_to_peer(dsta, sX_addr + (t & 1) * Bc * 128, Bc * 128, mb);
    }
    if (tr) trace[t * 5 + 4] = ptx::globaltimer_ns();
  }
  ptx::cluster_arrive();  // nobody leaves while a peer may still read my staging / write my sH
  ptx::cluster_wait();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tbase, tcols);
}

size_t fwd_cl_smem(int hp, int Bc, int nwarps) {
  const int nkb = (hp + 63) / 64;
  return 1024 + 2 * (size_t)nkb * 16384 + 2 * (size_t)nkb * Bc * 128 + 2 * (size_t)Bc * 128 +
         (size_t)nwarps * 16 * ACT_LD * 4 + 128;
}

template <int NC>
__global__ void __launch_bounds__(128, 1)
    recur_bwd_cl_kernel(const __grid_constant__ CUtensorMap tmU, const float* __restrict__ dHa, int dHa_last_only,
                        const __half* __restrict__ gates, const float* __restrict__ Cst, __half* __restrict__ dA,
                        int T, int B, int hp, unsigned long long* __restrict__ trace) {
  constexpr int Bc = 16 * NC;
  // optional phase trace (CTA (0,0), thread 0): [t][5] globaltimer stamps
  const bool tr = trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int fourhp = 4 * hp;
  const int nkb = fourhp / 64;
  const int abuf = nkb * Bc * 128;
  constexpr int SX = 4 * Bc * 128;             // my 4 K-blocks (256 gate rows) in destination layout
  uint8_t* sU = smem;                          // nkb x 8 KB (U^T slice, MN-major)
  uint8_t* sA = sU + nkb * 8192;               // [2][abuf] B operand (dA_{t+1}), filled by peers
  uint8_t* sX = sA + 2 * abuf;                 // [2][SX] staging of my dA_t slice, swizzled like sA
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + 2 * SX);
  uint64_t* barU = bars;
  uint64_t* barM = bars + 1;
  uint64_t* fullA = bars + 2;                  // [2]: peers' bulk copies into sA[p]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int rank = blockIdx.x;
  const int j0 = rank * 64;
  const int col0 = blockIdx.y * Bc;
  const int jl = lane & 15;
  const int half = lane >> 4;
  const int ul = warp * 16 + jl;               // unit within my 64-unit slice
  const int unit = j0 + ul;
  const bool unit_ok = unit < hp;
  constexpr int NACC = Bc <= 32 ? 8 : 4;
  constexpr int AC = NACC * Bc;
  constexpr uint32_t tcols = AC <= 32 ? 32 : AC <= 64 ? 64 : AC <= 128 ? 128 : 256;
  // bytes every consumer receives per step: all producers' valid K-blocks
  int total_bytes = 0;
  for (int r = 0; r < G; ++r) total_bytes += max(0, min(64, hp - 64 * r)) / 16 * Bc * 128;
  const int my_kblocks = max(0, min(64, hp - j0)) / 16;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tmU);
    ptx::mbar_init(barU, 1);
    ptx::mbar_init(barM, 4);  // one commit per issuing warp
    ptx::mbar_init(fullA, 1);
    ptx::mbar_init(fullA + 1, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tslot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) {
    // arm both operand slots for their first use before any peer can deliver
    ptx::mbar_arrive_expect_tx(fullA, total_bytes);
    ptx::mbar_arrive_expect_tx(fullA + 1, total_bytes);
    ptx::mbar_arrive_expect_tx(barU, nkb * 8192);
    for (int kb = 0; kb < nkb; ++kb) ptx::tma_load_2d(sU + kb * 8192, &tmU, barU, j0, kb * 64);
    ptx::mbar_wait(barU, 0);
  }
  ptx::cluster_arrive();  // all CTAs resident, barriers initialised and armed
  ptx::cluster_wait();

  float dcr[NC * 8];
#pragma unroll
  for (int i = 0; i < NC * 8; ++i) dcr[i] = 0.f;
  const uint32_t idesc = ptx::idesc_f16_f32(64, Bc, 1, 0);
  const uint32_t sA_addr = ptx::smem_u32(sA), sX_addr = ptx::smem_u32(sX);
  uint32_t fphase[2] = {0u, 0u};

  for (int t = T - 1; t >= 0; --t) {
    if (tr) trace[t * 5 + 0] = ptx::globaltimer_ns();
    float dh0[NC * 8], cc[NC * 8], cp[NC * 8];
    uint2 gq[NC * 8];
#pragma unroll
    for (int ch = 0; ch < NC; ++ch)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = ch * 8 + k;
        const size_t b = (size_t)col0 + ch * 16 + half * 8 + k;
        float d = 0.f, c1 = 0.f, c0 = 0.f;
        uint2 gg = make_uint2(0u, 0u);
        if (unit_ok) {
          if (dHa_last_only) {
            if (t == T - 1) d = __ldg(dHa + b * hp + unit);
          } else {
            d = __ldg(dHa + ((size_t)t * B + b) * hp + unit);
          }
          c1 = __ldg(Cst + ((size_t)t * B + b) * hp + unit);
          if (t > 0) c0 = __ldg(Cst + ((size_t)(t - 1) * B + b) * hp + unit);
          gg = __ldg(reinterpret_cast<const uint2*>(gates + ((size_t)t * B + b) * fourhp + 4 * unit));
        }
        dh0[idx] = d;
        cc[idx] = c1;
        cp[idx] = c0;
        gq[idx] = gg;
      }
    if (t < T - 1) {
      const int p = (t + 1) & 1;
      if (lane == 0) {
        ptx::mbar_wait(fullA + p, fphase[p]);  // every peer's dA_{t+1} slice landed in sA[p]
        ptx::tc_fence_after();
        if (tr) trace[t * 5 + 1] = ptx::globaltimer_ns();
        // lane 0 of each warp issues K-steps k = warp, warp + 4, ... (barM counts 4 commits)
        const uint32_t aU = ptx::smem_u32(sU), aA = sA_addr + p * abuf;
        const uint64_t ad0 = ptx::smem_desc_sw128(aU, 8192, 1024), bd0 = ptx::smem_desc_sw128(aA, 0, 1024);
        for (int k = warp; k < nkb * 4; k += 4) {
          const int kb = k >> 2, kk = k & 3;  // start-address field is in 16-B units
          const uint64_t ad = ad0 + (uint64_t)((kb * 8192 + kk * 2048) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((kb * Bc * 128 + kk * 32) >> 4);
          ptx::mma_f16(tbase + (k % NACC) * Bc, ad, bd, idesc, k >= NACC ? 1u : 0u);
        }
        ptx::mma_commit(barM);
      }
      __syncwarp();
      ptx::mbar_wait_relaxed(barM, (T - 2 - t) & 1);
      ptx::tc_fence_after();
      fphase[p] ^= 1u;
      // re-arm slot p for its next use (peers can deliver into it only after
      // they consumed my dA_t, i.e. after this point -- see the WAR note below)
      if (threadIdx.x == 0 && t >= 2) ptx::mbar_arrive_expect_tx(fullA + p, total_bytes);
    }
    if (tr) trace[t * 5 + 2] = ptx::globaltimer_ns();
    __half* dAout = dA + (size_t)t * B * fourhp;
    uint8_t* stg = sX + (t & 1) * SX;
#pragma unroll
    for (int ch = 0; ch < NC; ++ch) {
      float v[16];
      if (t < T - 1) {
        const uint32_t ta = tbase + (static_cast<uint32_t>(warp * 32) << 16) + ch * 16;
        ptx::tmem_ld16(ta, v);
#pragma unroll
        for (int a = 1; a < NACC; ++a) {
          if (a >= nkb * 4) break;  // accumulator never written (tiny K)
          float w[16];
          ptx::tmem_ld16(ta + a * Bc, w);
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] += w[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.f;
      }
      float rec[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float hi = __shfl_sync(0xffffffffu, v[8 + k], jl);
        rec[k] = half ? hi : v[k];
      }
      if (unit_ok) {
        // staging position of my unit's 4 gate rows (local gate row 4*ul) in row bl:
        // K-block j = ul/16, 16-B chunk c = (4ul % 64)/8, byte (4ul % 8)*2
        const int j = ul >> 4, c = (ul & 15) >> 1, byo = (ul & 1) * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int idx = ch * 8 + k;
          const int bl = ch * 16 + half * 8 + k;
          const size_t b = (size_t)col0 + bl;
          const float dh = dh0[idx] + rec[k];
          const float2 if2 = __half22float2(*reinterpret_cast<const __half2*>(&gq[idx].x));
          const float2 go2 = __half22float2(*reinterpret_cast<const __half2*>(&gq[idx].y));
          const float i = if2.x, f = if2.y, g = go2.x, o = go2.y;
          float tc, sech2;
          tanh_sech2(cc[idx], tc, sech2);
          const float d = dcr[idx] + dh * o * sech2;
          __align__(8) __half2 q2[2] = {
              __halves2half2(__float2half_rn(d * g * i * (1.f - i)), __float2half_rn(d * cp[idx] * f * (1.f - f))),
              __halves2half2(__float2half_rn(d * i * (1.f - g * g)), __float2half_rn(dh * tc * o * (1.f - o)))};
          const uint2 pk = *reinterpret_cast<const uint2*>(q2);
          *reinterpret_cast<uint2*>(dAout + b * fourhp + 4 * unit) = pk;  // R10 (for K8 / K9)
          *reinterpret_cast<uint2*>(stg + j * Bc * 128 + bl * 128 + ((c ^ (bl & 7)) << 4) + byo) = pk;
          dcr[idx] = d * f;
        }
      }
    }
    ptx::tc_fence_before();
    ptx::fence_async_smem();  // staging writes (generic) -> bulk copy reads (async proxy)
    __syncthreads();
    if (tr) trace[t * 5 + 3] = ptx::globaltimer_ns();
    // push dA_t (consumed by step t-1) into every peer's sA[t & 1]: one bulk copy per peer.
    // WAR: a peer writes sA[p] of step s only after consuming my dA_{s+1}, which I produce
    // after my MMA that read sA[p] for step s+2 -- the double buffers need no extra barrier.
    if (t > 0 && threadIdx.x < G && my_kblocks > 0) {
      const int dst = threadIdx.x;
      const uint32_t dsta = ptx::mapa(sA_addr + (t & 1) * abuf + 4 * rank * Bc * 128, dst);
      const uint32_t mb = ptx::mapa(ptx::smem_u32(fullA + (t & 1)), dst);
      ptx::bulk_copy_to_peer(dsta, sX_addr + (t & 1) * SX, my_kblocks * Bc * 128, mb);
    }
    if (tr) trace[t * 5 + 4] = ptx::globaltimer_ns();
  }
  // nobody leaves while a peer may still read my staging / write my sA
  ptx::cluster_arrive();
  ptx::cluster_wait();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tbase, tcols);
}


// ============================================================== 2-layer wavefront (backward)
struct BwdRoleParams {
  const float* dHa;
  int last_only;
  const __half* gates;
  const float* C;
  __half* dA;
};
struct __align__(64) Bwd2Params {
  CUtensorMap tmU[2];  // MN-major U^T slices: [0] U1 (role 0), [1] U0 (role 2)
  CUtensorMap tmW1;    // MN-major W1^T slice (role 1)
  CUtensorMap tmA1;    // dA1 rows [T*B][4hp], K-major (role 1)
  BwdRoleParams q[2];  // [0] layer 1, [1] layer 0
  float* dX1;          // [T][B][hp] = dA1 W1  (dH_above of layer 0)
  unsigned* q1done;    // [nbg][32]: layer-1 steps published (x G CTAs)
  unsigned* xdone;     // [nbg][8][32]: projection steps published per unit slice
  int T, B, hp, nbg;
  // ---- weight-gradient role (K8 on otherwise idle SMs; wtiles == 0: off)
  CUtensorMap tmdA[2];  // dA1 / dA0 rows [T*B][4hp], MN-major A operand boxes (64 rows, 64 batch)
  CUtensorMap tmHs[2];  // Hs1 / Hs0 rows [(T+1)*B][hp], MN-major B operand boxes (64, 64)
  CUtensorMap tmX0;     // X0 rows [T*B][Ip0] (Ip0 <= 256)
  __half* gW[4];        // dU1, dW1, dU0, dW0 (fp16 grads, row-major [4hp][N])
  __half* gb[2];        // db1, db0
  unsigned* q0done;     // [nbg][32]: layer-0 steps published (x G CTAs)
  int Ip0, wtiles;
  int wstages;          // W role TMA ring depth (2..4, as the launch's shared memory allows)
  unsigned long long* trace;  // debug: [Q1, Q0, X][T][5] stamps of CTA 0 / group 0, nullable
  CUtensorMap tmdAo[2];       // dA1 / dA0 rows [T*B][4hp], SWIZZLE_128B box (64, Bc): TMA stores from the push staging
  CUtensorMap tmDX;           // dX1 rows [T*B][hp] fp32, box (64, Bc): Q0's dH_above prefetch (TSQ)
  CUtensorMap tmGq[2];        // gates_1 / gates_0 rows [T*B][4hp] fp16, box (256, Bc) (TSQ prefetch)
  CUtensorMap tmCq[2];        // C_1 / C_0 rows [T*B][hp] fp32, box (64, Bc) (TSQ prefetch)
  CUtensorMap tmDXo;          // dX1 rows [T*B][hp] fp32, box (64, Bc): X's TMA stores (TSQ)
  // recurrent dropout (reading Q16b): mask x scale on dh_rec; dU from Hst (tmHt = tmHs when off)
  CUtensorMap tmHt[2];        // Hst1 / Hst0 rows [(T+1)*B][hp], MN-major B operand boxes (64, 64)
  int drop;
  const int* drop_step;
  uint32_t drop_seed, drop_thr, drop_seq0;
  float drop_scale;
};

// Weight-gradient role: one CTA per (matrix, 128-gate-row tile[, column half]) accumulates
// over all (t, b) in TMEM as the recurrence roles publish dA_t (A8 of the paper's step):
//   mat 0: dU1 = sum dA1_t^T h1_{t-1}   mat 1: dW1 = sum dA1_t^T h0_t
//   mat 2: dU0 = sum dA0_t^T h0_{t-1}   mat 3: dW0 = sum dA0_t^T x_t
// plus db1 / db0 (= sum dA_t, an MMA against a block of ones) on the dU tiles.  The dU
// tiles can be split into two column halves (two CTAs, wg_usplit) so the heaviest tiles
// keep pace with the layer-0 chain (the trace shows the dU0 tiles finishing ~30 us after
// Q0 at C2).
// (measured: at C2 the split needs 35 co-resident 4-CTA clusters, more than the GPU holds,
// so the plan fell back to the K8 GEMMs -- the split is off until a plan can choose it)
__host__ __device__ inline int wg_usplit(int hp) { return (void)hp, 1; }
__host__ __device__ inline int wg_tiles(int hp) { return (2 + 2 * wg_usplit(hp)) * ((4 * hp + 127) / 128); }
// Items = (t, 64-wide batch chunk) in descending t; a TMA ring of P.wstages stages (as
// deep as the launch's shared memory -- sized for the Q roles -- allows: the W role is a
// throughput role whose item loads are latency-bound; with 2 stages it trailed the Q0
// chain by ~90 us at C2 B = 128): thread 0 acquires the dA_t flags and loads, thread 32
// issues the MMAs.
constexpr int WG_STAGE = 2 * 8192 + 4 * 8192;  // A: 2 m-atoms x 64 b; B: up to 4 n-atoms x 64 b
constexpr int WG_MAX_STAGES = 4;
constexpr size_t WG_FIXED = 1024 + 2048 + 256;  // align slack, ones block, barriers
size_t wgrad_smem() { return WG_FIXED + 2 * (size_t)WG_STAGE; }
int wgrad_stages(size_t smem) {
  const int n = (int)((smem - WG_FIXED) / WG_STAGE);
  return n < 2 ? 2 : n > WG_MAX_STAGES ? WG_MAX_STAGES : n;
}

__device__ __forceinline__ void bwd_wgrad_role(const Bwd2Params& P, int tile) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int T = P.T, B = P.B, hp = P.hp, fourhp = 4 * hp;
  const int ntile = (fourhp + 127) / 128;
  if (tile >= wg_tiles(hp)) return;  // padding CTA of the last cluster
  // job = (matrix, column half): dU1 halves, dW1, dU0 halves, dW0
  const int us = wg_usplit(hp);
  const int job = tile / ntile, m0 = (tile % ntile) * 128;
  const int mat = job < us ? 0 : job == us ? 1 : job < 2 * us + 1 ? 2 : 3;
  const int uhalf = mat == 0 ? job : mat == 2 ? job - us - 1 : 0;
  const int layer = mat < 2 ? 1 : 0;           // whose dA
  const int ai = mat < 2 ? 0 : 1;              // tmdA / tmHs index: [0] layer 1, [1] layer 0
  const int nfull = mat == 3 ? 16 * ((P.Ip0 + 15) / 16) : hp;
  const int ucols = (mat == 0 || mat == 2) && us == 2 ? 128 : nfull;  // column-half width
  const int n0 = uhalf * ucols;                                        // first output column
  const int N = (mat == 0 || mat == 2) ? min(ucols, hp - n0) : nfull;
  const int natom = (N + 63) / 64;
  const bool withb = (mat == 0 || mat == 2) && uhalf == 0;
  const int NS = P.wstages;
  uint8_t* sones = smem + NS * WG_STAGE;       // [16 rows][128 B] fp16 ones, K-major B operand (N = 16)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sones + 2048);
  uint64_t* full = bars;                       // [NS]
  uint64_t* empty = bars + WG_MAX_STAGES;      // [NS]
  uint64_t* done = bars + 2 * WG_MAX_STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * WG_MAX_STAGES + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned* flags = layer == 1 ? P.q1done : P.q0done;
  const int G = gridDim.x;
  const int nbc = (B + 63) / 64;               // 64-wide batch chunks per step
  const int nitems = T * nbc;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&P.tmdA[ai]);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(full + i, 1);
      ptx::mbar_init(empty + i, 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 2048 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sones)[i] = 0x3C003C00u;
  ptx::fence_async_smem();
  if (warp == 2) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;               // [0, N): weight grad; [256, 272): bias grad
  if (warp == 0) {
    // ---- producer (lane 0 issues; the whole warp polls the batch groups' dA_t flags)
    // dU: h~_{t-1} (Hst with recurrent dropout, else Hs); dW1: the unmasked h0_t; dW0: x_t
    const CUtensorMap* tb = mat == 3 ? &P.tmX0 : mat == 1 ? &P.tmHs[1] : &P.tmHt[mat == 0 ? 0 : 1];
    // minimum over the batch groups of the published counts seen so far: a step whose
    // target it already covers needs no poll.  (Round 1 acquired the nbg flags one after
    // the other for every step: nbg sequential L2 round trips per step made this role the
    // tail of the launch.)
    unsigned minpub = 0;
    for (int it = 0; it < nitems; ++it) {
      const int t = T - 1 - it / nbc, bc = it % nbc;
      const int s = it % NS;
      if (bc == 0) {
        const unsigned target = (unsigned)(G * (T - t));
        if (minpub < target) {
          const uint64_t t0 = ptx::globaltimer_ns();
          for (;;) {
            const unsigned v = lane < P.nbg ? acquire_ld(flags + lane * 32) : 0xFFFFFFFFu;
            minpub = __reduce_min_sync(0xffffffffu, v);
            if (minpub >= target) break;
            if (ptx::globaltimer_ns() - t0 > 10000000000ull) __trap();
            // back off: the flag lines are the ones the recurrence roles release-add to every
            // step, and this is a throughput role -- polling them flat out slows those atomics
            __nanosleep(128);
          }
        }
        __syncwarp();  // the lanes' acquires happen-before lane 0's TMA reads (memory ordering of the warp barrier)
        fence_proxy_async();
        if (P.trace && t == 0 && lane == 0) {  // phase trace: the last step's dA seen (W slots after the CTA stamps)
          unsigned long long* w = P.trace + (size_t)6 * T * 5 + 3 * 148 + 3 * (blockIdx.y * gridDim.x + blockIdx.x);
          w[0] = ptx::globaltimer_ns();
          w[2] = 1 + mat;
        }
      }
      if (lane != 0) continue;
      ptx::mbar_wait(empty + s, ((it / NS) & 1) ^ 1);
      uint8_t* sa = smem + s * WG_STAGE;
      uint8_t* sb = sa + 2 * 8192;
      ptx::mbar_arrive_expect_tx(full + s, 2 * 8192 + natom * 8192);
      const int brow = t * B + bc * 64;        // dA_t / x_t rows
      ptx::tma_load_2d(sa, &P.tmdA[ai], full + s, m0, brow);
      ptx::tma_load_2d(sa + 8192, &P.tmdA[ai], full + s, m0 + 64, brow);
      // B rows: h_{t-1} = Hs slot t (dU), h0_t = Hs0 slot t+1 (dW1), x_t (dW0)
      const int hrow = mat == 1 ? (t + 1) * B + bc * 64 : mat == 3 ? brow : t * B + bc * 64;
      for (int a = 0; a < natom; ++a) ptx::tma_load_2d(sb + a * 8192, tb, full + s, n0 + a * 64, hrow);
    }
  } else if (threadIdx.x == 32) {
    // ---- MMA issuer
    const uint32_t idesc = ptx::idesc_f16_f32(128, natom * 64, 1, 1);  // whole 64-wide MN atoms
    const uint32_t idb = ptx::idesc_f16_f32(128, 16, 1, 0);
    for (int it = 0; it < nitems; ++it) {
      const int s = it % NS;
      ptx::mbar_wait(full + s, (it / NS) & 1);
      ptx::tc_fence_after();
      const uint32_t sa = ptx::smem_u32(smem + s * WG_STAGE), sb = sa + 2 * 8192;
      const int bc = it % nbc;
      const int kvalid = min(64, B - bc * 64);
#pragma unroll 1
      for (int k = 0; k < kvalid / 16; ++k) {
        const uint64_t ad = ptx::smem_desc_sw128(sa + k * 2048, 8192, 1024);
        const uint64_t bd = ptx::smem_desc_sw128(sb + k * 2048, 8192, 1024);
        const uint32_t acc = (it > 0 || k > 0) ? 1u : 0u;
        ptx::mma_f16(tbase, ad, bd, idesc, acc);
        if (withb) ptx::mma_f16(tbase + 256, ad, ptx::smem_desc_sw128(ptx::smem_u32(sones) + k * 32, 0, 1024), idb, acc);
      }
      ptx::mma_commit(empty + s);
    }
    ptx::mma_commit(done);
  }
  __syncwarp();
  ptx::mbar_wait(done, 0);
  ptx::tc_fence_after();
  if (P.trace && threadIdx.x == 0)
    P.trace[(size_t)6 * T * 5 + 3 * 148 + 3 * (blockIdx.y * gridDim.x + blockIdx.x) + 1] = ptx::globaltimer_ns();
  // ---- epilogue: TMEM lane = tile row; fp32 sums rounded once to fp16 (R13), staged as a
  // [128][N] fp16 tile in the (now idle) TMA ring and written as whole 16-B row chunks.
  // (Round 2 stored 2-byte values lane-per-row: 32 scattered sectors per instruction, a
  // 28 us tail of the launch after the layer-0 chain at C2.)
  const int row = m0 + warp * 32 + lane;
  __half* gout = P.gW[mat];
  const int ld = mat == 3 ? P.Ip0 : hp;
  const int lds = natom * 64 + 8;              // staging row stride (halves): conflict-free 16-B rows
  __half* stile = reinterpret_cast<__half*>(smem);
  for (int c = 0; c < N; c += 16) {
    float v[16];
    ptx::tmem_ld16(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
    __align__(16) __half hv[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) hv[q] = __float2half_rn(v[q]);
    uint4* dst = reinterpret_cast<uint4*>(stile + (size_t)(warp * 32 + lane) * lds + c);
    dst[0] = reinterpret_cast<const uint4*>(hv)[0];
    dst[1] = reinterpret_cast<const uint4*>(hv)[1];
  }
  __syncthreads();
  {
    const int ncol = min(N, ld - n0);            // valid output columns of this tile
    const int nch = (ncol + 7) / 8;              // 8-half chunks per row
    for (int i = threadIdx.x; i < 128 * nch; i += blockDim.x) {
      const int r = i / nch, ch = i % nch;
      const int grow = m0 + r, col = ch * 8;
      if (grow >= fourhp) continue;
      const __half* src = stile + (size_t)r * lds + col;
      __half* o = gout + (size_t)grow * ld + n0 + col;
      if (col + 8 <= ncol && (((size_t)grow * ld + n0 + col) & 7) == 0) {
        *reinterpret_cast<uint4*>(o) = *reinterpret_cast<const uint4*>(src);
      } else {
        for (int q = 0; q < 8 && col + q < ncol; ++q) o[q] = src[q];
      }
    }
  }
  if (withb) {
    float v[16];
    ptx::tmem_ld16(tbase + (static_cast<uint32_t>(warp * 32) << 16) + 256, v);
    if (row < fourhp) P.gb[mat == 0 ? 0 : 1][row] = __float2half_rn(v[0]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

// Projection role: dX1_t[b][unit] = sum_r dA1_t[b][r] W1[r][unit] for my 64 units
// (swap-AB tcgen05, A = W1^T slice MN-major resident, B = dA1_t rows via TMA).
// Projection role, A-from-TMEM variant (h_p = 208): W1^T slice copied from SMEM into TMEM
// (M = 64 layout), dA1_t operands TMA-prefetched into a 3-slot ring (reusing the W1 slice's
// SMEM) as Q1 publishes them, 2 issuing warps, dX1_t staged and written by TMA stores,
// xdone published lazily once a store group is complete.
template <int NC, int NKQ>
__device__ __forceinline__ void bwd_proj_role_ts(const Bwd2Params& P, int grp) {
  constexpr int Bc = 16 * NC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int T = P.T, B = P.B, hp = P.hp;
  const int fourhp = 4 * hp;
  const int nkb = fourhp / 64;
  const int abytes = nkb * Bc * 128;
  uint8_t* sW = smem;                              // nkb x 8 KB, then (after the TMEM copy) the dA1 ring
  uint8_t* sRing = sW;                             // [3][abytes]
  float* sO = reinterpret_cast<float*>(sW + nkb * 8192);  // [2][Bc][64] dX1 staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(sW + nkb * 8192 + 2 * Bc * 64 * 4);
  uint64_t* barU = bars;
  uint64_t* barM = bars + 1;
  uint64_t* barA = bars + 2;                       // [3]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = blockIdx.x, G = gridDim.x;
  const int j0 = rank * 64, col0 = grp * Bc;
  const int jl = lane & 15, half = lane >> 4;
  const int ul = warp * 16 + jl;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&P.tmW1);
    ptx::tma_prefetch(&P.tmA1);
    ptx::mbar_init(barU, 1);
    ptx::mbar_init(barM, 2);
    for (int i = 0; i < 3; ++i) ptx::mbar_init(barA + i, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tA = tbase + 64;
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(barU, nkb * 8192);
    for (int kb = 0; kb < nkb; ++kb) ptx::tma_load_2d(sW + kb * 8192, &P.tmW1, barU, j0, kb * 64);
  }
  ptx::mbar_wait(barU, 0);
  {
    // W1^T slice -> TMEM: unit 16q + i -> lane 32q + i, two gate rows per column
    const int i = lane & 15;
    const int u = warp * 16 + i;
    const uint32_t tq = tA + (static_cast<uint32_t>(warp * 32) << 16);
    int off[8];  // swizzled offsets repeat every 8 rows (see the Q roles' copy)
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) off[r8] = r8 * 128 + (((u >> 3) ^ r8) << 4) + (u & 7) * 2;
    for (int c0 = 0; c0 < 2 * hp; c0 += 16) {
      const uint8_t* base = sW + (size_t)c0 * 256;
      uint32_t v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint8_t* g8 = base + ((2 * j) & ~7) * 128;
        const uint32_t lo = *reinterpret_cast<const uint16_t*>(g8 + off[(2 * j) & 7]);
        const uint32_t hi = *reinterpret_cast<const uint16_t*>(g8 + off[(2 * j + 1) & 7]);
        v[j] = lane < 16 ? (lo | (hi << 16)) : 0u;
      }
      ptx::tmem_st16(tq + c0, v);
    }
    ptx::tmem_wait_st();
  }
  ptx::tc_fence_before();
  ptx::fence_async_smem();  // generic reads of sW before the TMA writes of the ring that reuses it
  __syncthreads();
  ptx::tc_fence_after();

  const int pf_thr = 97, st_thr = 96;
  const unsigned* q1f = P.q1done + grp * 32;
  auto fetch = [&](int tt, bool known_ready = false) {  // pf thread
    if (!known_ready) spin_until(q1f, (unsigned)(G * (T - tt)));
    fence_proxy_async();
    ptx::mbar_arrive_expect_tx(barA + tt % 3, abytes);
    for (int kb = 0; kb < nkb; ++kb)
      ptx::tma_load_2d(sRing + (tt % 3) * abytes + kb * Bc * 128, &P.tmA1, barA + tt % 3, kb * 64, tt * B + col0);
  };
  int nf = T - 1;
  if (threadIdx.x == pf_thr) {
    fetch(nf--);
    if (nf >= 0 && nf >= T - 2) fetch(nf--);
  }
  unsigned long long* xtr = (P.trace && rank == 0 && grp == 0 && threadIdx.x == 0) ? P.trace + (size_t)2 * T * 5 : nullptr;
  unsigned* xf = P.xdone + (grp * 8 + rank) * 32;
  uint32_t mph = 0;
  for (int t = T - 1; t >= 0; --t) {
    if (xtr) xtr[t * 5 + 0] = ptx::globaltimer_ns();
    if (threadIdx.x == pf_thr)
      while (nf >= t) fetch(nf--);  // due now
    if (warp < 2) {
      ptx::mbar_wait(barA + t % 3, ((T - 1 - t) / 3) & 1);
      ptx::tc_fence_after();
      if (xtr) xtr[t * 5 + 1] = ptx::globaltimer_ns();
      const uint64_t bd0 = ptx::smem_desc_sw128(ptx::smem_u32(sRing + (t % 3) * abytes), 0, 1024);
      const uint32_t idesc = ptx::idesc_f16_f32(64, Bc, 0, 0);
#pragma unroll
      for (int k = 0; k < NKQ; k += 2) {
        const int kw = k + warp;
        const uint64_t bd = bd0 + (uint64_t)(((kw >> 2) * Bc * 128 + (kw & 3) * 32) >> 4);
        if (ptx::elect_one_sync()) ptx::mma_f16_ts(tbase + warp * Bc, tA + kw * 8, bd, idesc, k > 0 ? 1u : 0u);
      }
      if (ptx::elect_one_sync()) ptx::mma_commit(barM);
      __syncwarp();
    }
    // publish dX1_{t+1} inside the MMA wait (the store thread issues no MMAs): step t+1's
    // store group is the latest, so a full wait completes it -- one step of hand-off lag to
    // the layer-0 chain instead of two
    if (threadIdx.x == st_thr && t < T - 1) {
      ptx::bulk_wait_group0();
      fence_proxy_async();
      release_add(xf, 1u);
      if (P.trace && rank == 0 && grp == 0) P.trace[(size_t)4 * T * 5 + (t + 1) * 5 + 1] = ptx::globaltimer_ns();
    }
    {
      ptx::mbar_wait_relaxed(barM, mph);
    }
    mph ^= 1u;
    ptx::tc_fence_after();
    if (xtr) xtr[t * 5 + 2] = ptx::globaltimer_ns();
    float* so = sO + (t & 1) * Bc * 64;
#pragma unroll
    for (int ch = 0; ch < NC; ++ch) {
      float v[16], w[16];
      const uint32_t ta = tbase + (static_cast<uint32_t>(warp * 32) << 16) + ch * 16;
      ptx::tmem_ld16(ta, v);
      ptx::tmem_ld16(ta + Bc, w);
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] += w[q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float hi = __shfl_sync(0xffffffffu, v[8 + q], jl);
        so[(ch * 16 + half * 8 + q) * 64 + ul] = half ? hi : v[q];  // R11 (fp32)
      }
    }
    if (threadIdx.x == st_thr) ptx::bulk_wait_group_read0();  // earlier stores finished reading sO
    ptx::tc_fence_before();
    ptx::fence_async_smem();
    __syncthreads();  // MMA reads of the ring slot done (barM), staging complete
    if (xtr) xtr[t * 5 + 3] = ptx::globaltimer_ns();
    if (threadIdx.x == st_thr) {
      ptx::tma_store_2d(&P.tmDXo, so, j0, t * B + col0);
      ptx::bulk_commit_group();
      if (t == 0) {  // step 0 (steps T-1 .. 1 were published in the MMA waits of steps T-2 .. 0)
        ptx::bulk_wait_group0();
        fence_proxy_async();
        release_add(xf, 1u);
      }
    }
    // ring slot (t-2) % 3 = (t+1) % 3 was read by step t+1's MMAs (complete): prefetch ahead
    if (threadIdx.x == pf_thr && nf >= 0 && nf >= t - 2 && acquire_ld(q1f) >= (unsigned)(G * (T - nf))) fetch(nf--, true);
    if (xtr) xtr[t * 5 + 4] = ptx::globaltimer_ns();
  }
  ptx::tc_fence_after();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tbase, 512);
}

template <int NC>
__device__ __forceinline__ void bwd_proj_role(const Bwd2Params& P, int grp) {
  constexpr int Bc = 16 * NC;
  constexpr int NACC = Bc <= 32 ? 8 : 4;
  constexpr int AC = NACC * Bc;
  constexpr uint32_t tcols = AC <= 32 ? 32 : AC <= 64 ? 64 : AC <= 128 ? 128 : 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int T = P.T, B = P.B, hp = P.hp;
  const int fourhp = 4 * hp;
  const int nkb = fourhp / 64;
  uint8_t* sW = smem;                 // nkb x 8 KB
  uint8_t* sA = sW + nkb * 8192;      // nkb x Bc*128 (single buffer)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + nkb * Bc * 128);
  uint64_t* barU = bars;
  uint64_t* barM = bars + 1;
  uint64_t* barA = bars + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = blockIdx.x, G = gridDim.x;
  const int j0 = rank * 64, col0 = grp * Bc;
  const int jl = lane & 15, half = lane >> 4;
  const int unit = j0 + warp * 16 + jl;
  const bool unit_ok = unit < hp;
  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&P.tmW1);
    ptx::tma_prefetch(&P.tmA1);
    ptx::mbar_init(barU, 1);
    ptx::mbar_init(barM, 4);
    ptx::mbar_init(barA, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tslot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(barU, nkb * 8192);
    for (int kb = 0; kb < nkb; ++kb) ptx::tma_load_2d(sW + kb * 8192, &P.tmW1, barU, j0, kb * 64);
    ptx::mbar_wait(barU, 0);
  }
  __syncthreads();
  const uint32_t idesc = ptx::idesc_f16_f32(64, Bc, 1, 0);
  uint32_t ph = 0;
  unsigned long long* xtr = (P.trace && rank == 0 && grp == 0 && threadIdx.x == 0) ? P.trace + (size_t)2 * T * 5 : nullptr;
  for (int t = T - 1; t >= 0; --t) {
    if (xtr) xtr[t * 5 + 0] = ptx::globaltimer_ns();
    if (threadIdx.x == 0) {
      // dA1_t published by every layer-1 CTA of my batch group
      const unsigned* f = P.q1done + grp * 32;
      const unsigned target = (unsigned)(G * (T - t));
      if (acquire_ld(f) < target) {
        const uint64_t t0 = ptx::globaltimer_ns();
        while (acquire_ld(f) < target) {
          if (ptx::globaltimer_ns() - t0 > 10000000000ull) __trap();
        }
      }
      fence_proxy_async();
      ptx::mbar_arrive_expect_tx(barA, nkb * Bc * 128);
      for (int kb = 0; kb < nkb; ++kb) ptx::tma_load_2d(sA + kb * Bc * 128, &P.tmA1, barA, kb * 64, t * B + col0);
    }
    if (lane == 0) {
      ptx::mbar_wait(barA, ph);
      ptx::tc_fence_after();
      const uint32_t aW = ptx::smem_u32(sW), aA = ptx::smem_u32(sA);
      const uint64_t ad0 = ptx::smem_desc_sw128(aW, 8192, 1024), bd0 = ptx::smem_desc_sw128(aA, 0, 1024);
      for (int k = warp; k < nkb * 4; k += 4) {
        const int kb = k >> 2, kq = k & 3;
        const uint64_t ad = ad0 + (uint64_t)((kb * 8192 + kq * 2048) >> 4);
        const uint64_t bd = bd0 + (uint64_t)((kb * Bc * 128 + kq * 32) >> 4);
        ptx::mma_f16(tbase + (k % NACC) * Bc, ad, bd, idesc, k >= NACC ? 1u : 0u);
      }
      ptx::mma_commit(barM);
    }
    __syncwarp();
    if (xtr) xtr[t * 5 + 1] = ptx::globaltimer_ns();
    ptx::mbar_wait_relaxed(barM, ph);
    ph ^= 1u;
    ptx::tc_fence_after();
    if (xtr) xtr[t * 5 + 2] = ptx::globaltimer_ns();
    float* out = P.dX1 + (size_t)t * B * hp;
#pragma unroll
    for (int ch = 0; ch < NC; ++ch) {
      float v[16];
      const uint32_t ta = tbase + (static_cast<uint32_t>(warp * 32) << 16) + ch * 16;
      ptx::tmem_ld16(ta, v);
#pragma unroll
      for (int a = 1; a < NACC; ++a) {
        if (a >= nkb * 4) break;
        float w[16];
        ptx::tmem_ld16(ta + a * Bc, w);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] += w[q];
      }
      if (unit_ok) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float hi = __shfl_sync(0xffffffffu, v[8 + q], jl);
          const float val = half ? hi : v[q];
          out[((size_t)col0 + ch * 16 + half * 8 + q) * hp + unit] = val;  // R11 (fp32)
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) (void)__shfl_sync(0xffffffffu, v[8 + q], jl);
      }
    }
    ptx::tc_fence_before();
    __syncthreads();  // MMA reads of sA done (barM) and all dX1 stores issued
    if (xtr) xtr[t * 5 + 3] = ptx::globaltimer_ns();
    if (threadIdx.x == 0) {
      release_add(P.xdone + (grp * 8 + rank) * 32, 1u);
    }
    if (xtr) xtr[t * 5 + 4] = ptx::globaltimer_ns();
  }
  ptx::tc_fence_after();
  __syncthreads();
  if (warp == 2) ptx::tmem_dealloc(tbase, tcols);
}

// phase trace (option recur_trace): per-CTA entry / exit stamps and role after the [6][T][5]
// per-step stamps -- where a launch's time goes outside the recurrence chains
__device__ __forceinline__ void cta_stamp(const Bwd2Params& P, int slot, unsigned long long role) {
  if (!P.trace || threadIdx.x != 0) return;
  unsigned long long* b = P.trace + (size_t)6 * P.T * 5 + 3 * (blockIdx.y * gridDim.x + blockIdx.x);
  b[slot] = ptx::globaltimer_ns();
  b[2] = role;
}

template <int NC, int NKQ>
__global__ void __launch_bounds__(128, 1)
    recur2_bwd_kernel(const __grid_constant__ Bwd2Params P) {
  const int T = P.T, B = P.B, hp = P.hp;
  if ((int)blockIdx.y >= 3 * P.nbg) {
    cta_stamp(P, 0, 3);
    bwd_wgrad_role(P, (blockIdx.y - 3 * P.nbg) * gridDim.x + blockIdx.x);
    cta_stamp(P, 1, 3);
    return;
  }
  const int role = blockIdx.y / P.nbg, grp = blockIdx.y % P.nbg;
  cta_stamp(P, 0, role);  // 0 Q1, 1 X, 2 Q0, 3 W
  if (role == 1) {
    // (the TMEM-A projection needs 64 + 2 h_p <= 512 columns: h_p = 208 yes, 256 no)
    if constexpr (NKQ != 0 && 64 + NKQ * 8 <= 512)
      bwd_proj_role_ts<NC, (NKQ != 0 ? NKQ : 52)>(P, grp);
    else
      bwd_proj_role<NC>(P, grp);
    cta_stamp(P, 1, 1);
    return;
  }
  const int qi = role == 0 ? 0 : 1;  // 0: layer 1 (Q1), 1: layer 0 (Q0)
  const CUtensorMap& tmU = P.tmU[qi];
  const float* __restrict__ dHa = P.q[qi].dHa;
  const int dHa_last_only = P.q[qi].last_only;
  const __half* __restrict__ gates = P.q[qi].gates;
  const float* __restrict__ Cst = P.q[qi].C;
  __half* __restrict__ dA = P.q[qi].dA;
  unsigned long long* __restrict__ trace = P.trace ? P.trace + (size_t)qi * T * 5 : nullptr;
  constexpr int Bc = 16 * NC;
  // optional phase trace (CTA 0 of batch group 0, thread 0): [t][5] globaltimer stamps
  const bool tr = trace != nullptr && blockIdx.x == 0 && grp == 0 && threadIdx.x == 0;
  unsigned long long* trq = (tr && qi == 1) ? P.trace + (size_t)3 * T * 5 : nullptr;  // Q0 epilogue sub-phases
  unsigned long long* trw = (P.trace && qi == 1 && blockIdx.x == 0 && grp == 0) ? P.trace + (size_t)3 * T * 5 : nullptr;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int fourhp = 4 * hp;
  const int nkb = fourhp / 64;
  const int abuf = nkb * Bc * 128;
  constexpr int SX = 4 * Bc * 128;             // my 4 K-blocks (256 gate rows) in destination layout
  uint8_t* sU = smem;                          // nkb x 8 KB (U^T slice, MN-major)
  uint8_t* sA = sU + nkb * 8192;               // [2][abuf] B operand (dA_{t+1}), filled by peers
  uint8_t* sX = sA + 2 * abuf;                 // [2][SX] staging of my dA_t slice, swizzled like sA
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + 2 * SX);
  uint64_t* barU = bars;
  uint64_t* barM = bars + 1;
  uint64_t* fullA = bars + 2;                  // [2]: peers' bulk copies into sA[p]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  uint64_t* barD = bars + 5;                   // [3] TSQ, Q0: dX1_t slice landed in sD[t % 3]
  constexpr int RG = 5;                        // gates / c ring depth (fetched RG-1 steps ahead)
  uint64_t* barP = bars + 8;                   // [RG] TSQ: gates_t + C_t tiles landed in ring slot t % RG

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int rank = blockIdx.x;
  const int j0 = rank * 64;
  const int col0 = grp * Bc;
  const int jl = lane & 15;
  const int half = lane >> 4;
  const int ul = warp * 16 + jl;               // unit within my 64-unit slice
  const int unit = j0 + ul;
  const bool unit_ok = unit < hp;
  // NKQ != 0 (h_p = 208): U^T slice in TMEM (A operand, M = 64 layout), 2 issuing warps x
  // 1 accumulator each; dA_t written by TMA stores from the push staging; warps 2 / 3
  // push and store (async copies from an MMA-issuing thread delay its commits)
  constexpr bool TSQ = NKQ != 0;
  // K-steps whose A (U^T slice) lives in TMEM: all of them while 64 + 8 NKQ <= 512 columns
  // (h_p = 208); at h_p = 256 the last NKQ - NKT K-steps read A from the SMEM copy (MN-major)
  constexpr int NKT = TSQ ? (64 + NKQ * 8 <= 512 ? NKQ : (512 - 64) / 8) : 0;
  // TSQ accumulators: the 2 issuing warps alternate over QACC / 2 accumulators each
  // (QACC * Bc <= 64 columns: tA at 64).  Measured at C2: 4 accumulators (13-MMA chains)
  // leave the step's MMA phase at ~1.0 us like 2 (26-MMA chains) -- the chain length is
  // not what separates it from the 0.38 us of tools/micro/mma_floor.cu -- so 2.
  constexpr int QACC = 2;
  constexpr int NACC = TSQ ? QACC : (Bc <= 32 ? 8 : 4);
  static_assert(!TSQ || QACC * Bc <= 64, "TSQ accumulators must stay below the TMEM A slice");
  constexpr int AC = NACC * Bc;
  constexpr uint32_t tcols = TSQ ? 512u : (AC <= 32 ? 32u : AC <= 64 ? 64u : AC <= 128 ? 128u : 256u);
  constexpr int NISQ = TSQ ? 2 : 4;
  // bytes every consumer receives per step: all producers' valid K-blocks
  int total_bytes = 0;
  for (int r = 0; r < G; ++r) total_bytes += max(0, min(64, hp - 64 * r)) / 16 * Bc * 128;
  const int my_kblocks = max(0, min(64, hp - j0)) / 16;

  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tmU);
    ptx::mbar_init(barU, 1);
    ptx::mbar_init(barM, NISQ);  // one commit per issuing warp
    ptx::mbar_init(fullA, 1);
    ptx::mbar_init(fullA + 1, 1);
    ptx::mbar_init(barD, 1);
    ptx::mbar_init(barD + 1, 1);
    ptx::mbar_init(barD + 2, 1);
    for (int i = 0; i < RG; ++i) ptx::mbar_init(barP + i, 1);
    ptx::fence_mbar_init();
  }
  // phase trace: prologue stamps of CTA 0 / group 0 (after the W-role slots)
  unsigned long long* tpro = (P.trace && blockIdx.x == 0 && grp == 0 && threadIdx.x == 0)
                                 ? P.trace + (size_t)6 * T * 5 + 6 * 148 + qi * 8 : nullptr;
  if (tpro) tpro[0] = ptx::globaltimer_ns();
  if (warp == 2) ptx::tmem_alloc(tslot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (tpro) tpro[1] = ptx::globaltimer_ns();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) {
    // arm both operand slots for their first use before any peer can deliver
    ptx::mbar_arrive_expect_tx(fullA, total_bytes);
    ptx::mbar_arrive_expect_tx(fullA + 1, total_bytes);
    ptx::mbar_arrive_expect_tx(barU, nkb * 8192);
    for (int kb = 0; kb < nkb; ++kb) ptx::tma_load_2d(sU + kb * 8192, &tmU, barU, j0, kb * 64);
    ptx::mbar_wait(barU, 0);
  }
  if (tpro) tpro[2] = ptx::globaltimer_ns();
  ptx::cluster_arrive();  // all CTAs resident, barriers initialised and armed
  ptx::cluster_wait();
  if (tpro) tpro[3] = ptx::globaltimer_ns();
  const uint32_t tA = tbase + 64;  // TSQ: A = U^T slice, columns [64, 64 + 2 h_p)
  if (TSQ) {
    // sU (MN-major SWIZZLE_128B: row k = 128 B of 64 units, 16-B chunk (unit/8) ^ (k%8)) -> TMEM:
    // unit 16q + i -> lane 32q + i (i < 16), two K-elements (gate rows) per column
    const int i = lane & 15;
    const int u = warp * 16 + i;
    const uint32_t tq = tA + (static_cast<uint32_t>(warp * 32) << 16);
    // gate row kk of unit u sits at sU + kk * 128 + 16 * ((u / 8) ^ (kk % 8)) + 2 * (u % 8)
    // (8 KB K blocks of 64 rows are contiguous): the swizzled offsets repeat every 8 rows,
    // so they are computed once (the per-element address arithmetic made this copy 5 us)
    int off[8];
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) off[r8] = r8 * 128 + (((u >> 3) ^ r8) << 4) + (u & 7) * 2;
    for (int c0 = 0; c0 < 8 * NKT; c0 += 16) {     // (K-steps >= NKT stay in sU)
      const uint8_t* base = sU + (size_t)c0 * 256;  // gate row 2 c0
      uint32_t v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint8_t* g8 = base + ((2 * j) & ~7) * 128;
        const uint32_t lo = *reinterpret_cast<const uint16_t*>(g8 + off[(2 * j) & 7]);
        const uint32_t hi = *reinterpret_cast<const uint16_t*>(g8 + off[(2 * j + 1) & 7]);
        v[j] = lane < 16 ? (lo | (hi << 16)) : 0u;
      }
      ptx::tmem_st16(tq + c0, v);
    }
    ptx::tmem_wait_st();
    ptx::tc_fence_before();
    ptx::fence_async_smem();  // generic reads of sU before the TMA writes that reuse it (Q0's dX1 prefetch)
    __syncthreads();
    ptx::tc_fence_after();
  }
  if (tpro) tpro[4] = ptx::globaltimer_ns();
  const int st_thr = 96;  // TSQ: TMA stores + publication (warp 3, no MMA issue)
  // TSQ, Q0: dH_above = dX1 slices prefetched by TMA one step ahead into the (now free) sU
  // region, by a thread that issues no MMAs; the flag acquire leaves the step's chain
  const bool dpf = TSQ && qi == 1;
  float* sD = reinterpret_cast<float*>(sU);    // [3][Bc][64] fp32 (two steps ahead)
  const int pf_thr = 97;
  unsigned long long* tr4 = (P.trace && qi == 1 && blockIdx.x == 0 && grp == 0) ? P.trace + (size_t)4 * T * 5 : nullptr;
  auto fetch_dx = [&](int tt, bool known_ready = false) {  // pf thread: wait for X's slice of step tt, then TMA it
    if (!known_ready) spin_until(P.xdone + (grp * 8 + rank) * 32, (unsigned)(T - tt));
    fence_proxy_async();
    ptx::mbar_arrive_expect_tx(barD + tt % 3, Bc * 64 * 4);
    ptx::tma_load_2d(sD + (tt % 3) * Bc * 64, &P.tmDX, barD + tt % 3, j0, tt * B + col0);
  };
  // next step whose dX1 slice is still to be fetched (descending); the pf thread fetches
  // ahead only when X has already published (non-blocking), and blocks only when due
  int nf = T - 1;
  if (dpf && threadIdx.x == pf_thr) {
    fetch_dx(nf--);
    if (nf >= 0 && nf >= T - 2) fetch_dx(nf--);
  }
  // TSQ: the step's saved gates and c (written by the forward kernel, usually no longer in L2)
  // arrive by TMA two steps ahead into a 3-slot ring, instead of per-thread loads whose HBM
  // latency the epilogue waited for
  // (measured: these loads take ~4 us to land -- far-die HBM under the wavefront's traffic)
  __half* sGp = reinterpret_cast<__half*>(sU + 3 * Bc * 64 * 4);                  // [RG][Bc][256]
  float* sCp = reinterpret_cast<float*>(sU + 3 * Bc * 64 * 4 + RG * Bc * 256 * 2);  // [RG][Bc][64]
  auto fetch_gc = [&](int tt) {
    if (tr4) tr4[tt * 5 + 0] = ptx::globaltimer_ns();
    ptx::mbar_arrive_expect_tx(barP + tt % RG, Bc * 256 * 2 + Bc * 64 * 4);
    ptx::tma_load_2d(sGp + (tt % RG) * Bc * 256, &P.tmGq[qi], barP + tt % RG, j0 * 4, tt * B + col0);
    ptx::tma_load_2d(sCp + (tt % RG) * Bc * 64, &P.tmCq[qi], barP + tt % RG, j0, tt * B + col0);
  };
  if (TSQ && threadIdx.x == pf_thr)
    for (int tt = T - 1; tt >= 0 && tt >= T - (RG - 1); --tt) fetch_gc(tt);

  float dcr[NC * 8];
#pragma unroll
  for (int i = 0; i < NC * 8; ++i) dcr[i] = 0.f;
  // recurrent dropout: dh_rec (the gradient of h~_{t-1}) x mask x scale, per (unit, column)
  float dsc[NC * 8];
#pragma unroll
  for (int i = 0; i < NC * 8; ++i) dsc[i] = 1.f;
  if (P.drop) {
    const uint32_t lk = drop_layer_key(P.drop_seed, (uint32_t)*P.drop_step, qi == 0 ? 1u : 0u);
#pragma unroll
    for (int ch = 0; ch < NC; ++ch)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t seq = P.drop_seq0 + (uint32_t)(col0 + ch * 16 + half * 8 + k);
        dsc[ch * 8 + k] = unit_ok && drop_kept(drop_seq_key(lk, seq), (uint32_t)unit, P.drop_thr) ? P.drop_scale : 0.f;
      }
  }
  const uint32_t idesc = ptx::idesc_f16_f32(64, Bc, 1, 0);
  const uint32_t sA_addr = ptx::smem_u32(sA), sX_addr = ptx::smem_u32(sX);
  uint32_t fphase[2] = {0u, 0u};

  for (int t = T - 1; t >= 0; --t) {
    if (tr) trace[t * 5 + 0] = ptx::globaltimer_ns();
    if (qi == 1 && !dpf) {
      // dH_above[t] of layer 0 = dX1_t, produced in this kernel by the projection CTA of my units
      if (threadIdx.x == 0) {
        const unsigned* f = P.xdone + (grp * 8 + rank) * 32;
        const unsigned target = (unsigned)(T - t);
        if (acquire_ld(f) < target) {
          const uint64_t t0 = ptx::globaltimer_ns();
          while (acquire_ld(f) < target) {
            if (ptx::globaltimer_ns() - t0 > 10000000000ull) __trap();
          }
        }
      }
      __syncthreads();
    }
    float dh0[NC * 8], cc[NC * 8], cp[NC * 8];
    uint2 gq[NC * 8];
#pragma unroll
    for (int ch = 0; ch < NC; ++ch)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = ch * 8 + k;
        const size_t b = (size_t)col0 + ch * 16 + half * 8 + k;
        float d = 0.f, c1 = 0.f, c0 = 0.f;
        uint2 gg = make_uint2(0u, 0u);
        if (unit_ok) {
          if (dHa_last_only) {
            if (t == T - 1) d = __ldg(dHa + b * hp + unit);
          } else if (qi == 1) {
            if (!dpf) d = __ldcg(dHa + ((size_t)t * B + b) * hp + unit);  // written in-kernel: L2-coherent load
          } else {
            d = __ldg(dHa + ((size_t)t * B + b) * hp + unit);
          }
          if (!TSQ) {
            c1 = __ldg(Cst + ((size_t)t * B + b) * hp + unit);
            if (t > 0) c0 = __ldg(Cst + ((size_t)(t - 1) * B + b) * hp + unit);
            gg = __ldg(reinterpret_cast<const uint2*>(gates + ((size_t)t * B + b) * fourhp + 4 * unit));
          }
        }
        dh0[idx] = d;
        cc[idx] = c1;
        cp[idx] = c0;
        gq[idx] = gg;
      }
    if (t < T - 1) {
      const int p = (t + 1) & 1;
      if (TSQ) {
        if (warp < 2) {
          ptx::mbar_wait(fullA + p, fphase[p]);  // every peer's dA_{t+1} slice landed in sA[p]
          ptx::tc_fence_after();
          if (tr) trace[t * 5 + 1] = ptx::globaltimer_ns();
          const uint64_t bd0 = ptx::smem_desc_sw128(sA_addr + p * abuf, 0, 1024);
#pragma unroll
          for (int k = 0; k < (TSQ ? NKQ : 1); k += 2) {
            const int kw = k + warp;  // this warp's K-steps: warp, warp + 2, ...
            const int slot = (k >> 1) % (QACC / 2);  // this warp's accumulators round-robin
            const uint32_t dacc = tbase + (warp + 2 * slot) * Bc;
            const uint32_t acc = (k >> 1) >= QACC / 2 ? 1u : 0u;
            const uint64_t bd = bd0 + (uint64_t)(((kw >> 2) * Bc * 128 + (kw & 3) * 32) >> 4);
            // (A from TMEM is K-major: the MN-major bit of the SMEM variant's idesc must be clear)
            if (kw < NKT) {
              if (ptx::elect_one_sync()) ptx::mma_f16_ts(dacc, tA + kw * 8, bd, ptx::idesc_f16_f32(64, Bc, 0, 0), acc);
            } else {  // A from the SMEM copy of the slice: MN-major, 8 KB per 64-row K block
              const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(sU) + (kw >> 2) * 8192 + (kw & 3) * 2048, 8192, 1024);
              if (ptx::elect_one_sync()) ptx::mma_f16(dacc, ad, bd, ptx::idesc_f16_f32(64, Bc, 1, 0), acc);
            }
          }
          if (ptx::elect_one_sync()) ptx::mma_commit(barM);
          __syncwarp();
        }
        // Q0 publishes dA_{t+2} (for the weight-gradient role only, off the critical path)
        // here, inside the MMA wait every warp sits in anyway: the store-group wait + the
        // gpu-scope release cost ~0.7 us, which at the end of the step held the epilogue
        // barrier of the hosting warp back (measured: warp 3 +0.7 us behind warps 0-2)
        if (qi == 1 && threadIdx.x == st_thr && (qi == 0 || P.wtiles) && t + 2 <= T - 1) {
          ptx::bulk_wait_group1();  // all but step t+1's store group complete
          fence_proxy_async();
          release_add(P.q0done + grp * 32, 1u);
        }
        // Q1 publishes dA1_{t+1} (for X, on the layer-0 chain's path) in the same window:
        // step t+1's store group is the latest one, so a full wait completes it -- one step
        // of hand-off lag instead of two
        if (qi == 0 && threadIdx.x == st_thr) {
          ptx::bulk_wait_group0();
          fence_proxy_async();
          release_add(P.q1done + grp * 32, 1u);
        }
      } else if (lane == 0) {
        ptx::mbar_wait(fullA + p, fphase[p]);  // every peer's dA_{t+1} slice landed in sA[p]
        ptx::tc_fence_after();
        if (tr) trace[t * 5 + 1] = ptx::globaltimer_ns();
        // lane 0 of each warp issues K-steps k = warp, warp + 4, ... (barM counts 4 commits)
        const uint32_t aU = ptx::smem_u32(sU), aA = sA_addr + p * abuf;
        const uint64_t ad0 = ptx::smem_desc_sw128(aU, 8192, 1024), bd0 = ptx::smem_desc_sw128(aA, 0, 1024);
        for (int k = warp; k < nkb * 4; k += 4) {
          const int kb = k >> 2, kk = k & 3;  // start-address field is in 16-B units
          const uint64_t ad = ad0 + (uint64_t)((kb * 8192 + kk * 2048) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((kb * Bc * 128 + kk * 32) >> 4);
          ptx::mma_f16(tbase + (k % NACC) * Bc, ad, bd, idesc, k >= NACC ? 1u : 0u);
        }
        ptx::mma_commit(barM);
      }
      __syncwarp();
      {
        ptx::mbar_wait_relaxed(barM, (T - 2 - t) & 1);
      }
      ptx::tc_fence_after();
      fphase[p] ^= 1u;
      // re-arm slot p for its next use (peers can deliver into it only after
      // they consumed my dA_t, i.e. after this point -- see the WAR note below)
      if (threadIdx.x == 0 && t >= 2) ptx::mbar_arrive_expect_tx(fullA + p, total_bytes);
    }
    if (tr) trace[t * 5 + 2] = ptx::globaltimer_ns();
    if (TSQ) {
      if (tr4 && threadIdx.x == 0) tr4[t * 5 + 2] = ptx::globaltimer_ns();
      ptx::mbar_wait(barP + t % RG, ((T - 1 - t) / RG) & 1);
      if (tr4 && threadIdx.x == 0) tr4[t * 5 + 3] = ptx::globaltimer_ns();
      if (t > 0) ptx::mbar_wait(barP + (t - 1) % RG, ((T - t) / RG) & 1);  // c_{t-1} (fetched one step later)
      if (tr4 && threadIdx.x == 0) tr4[t * 5 + 4] = ptx::globaltimer_ns();
#pragma unroll
      for (int ch = 0; ch < NC; ++ch)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int bl = ch * 16 + half * 8 + k;
          cc[ch * 8 + k] = sCp[((t % RG) * Bc + bl) * 64 + ul];
          cp[ch * 8 + k] = t > 0 ? sCp[(((t + RG - 1) % RG) * Bc + bl) * 64 + ul] : 0.f;  // slot of step t-1
          gq[ch * 8 + k] = *reinterpret_cast<const uint2*>(sGp + ((t % RG) * Bc + bl) * 256 + 4 * ul);
        }
    }
    if (dpf) {

      if (threadIdx.x == pf_thr) {
        const unsigned long long w0 = trw ? ptx::globaltimer_ns() : 0;
        while (nf >= t) fetch_dx(nf--);  // due now: blocking
        if (trw) trw[t * 5 + 4] = ptx::globaltimer_ns() - w0;
      }
      ptx::mbar_wait(barD + t % 3, ((T - 1 - t) / 3) & 1);
      if (trq) trq[t * 5 + 0] = ptx::globaltimer_ns();
#pragma unroll
      for (int ch = 0; ch < NC; ++ch)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          dh0[ch * 8 + k] = sD[((t % 3) * Bc + ch * 16 + half * 8 + k) * 64 + ul];
    }
    __half* dAout = dA + (size_t)t * B * fourhp;
    uint8_t* stg = sX + (t & 1) * SX;
#pragma unroll
    for (int ch = 0; ch < NC; ++ch) {
      float v[16];
      if (t < T - 1) {
        const uint32_t ta = tbase + (static_cast<uint32_t>(warp * 32) << 16) + ch * 16;
        ptx::tmem_ld16(ta, v);
#pragma unroll
        for (int a = 1; a < NACC; ++a) {
          if (a >= nkb * 4) break;  // accumulator never written (tiny K)
          float w[16];
          ptx::tmem_ld16(ta + a * Bc, w);
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] += w[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = 0.f;
      }
      float rec[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float hi = __shfl_sync(0xffffffffu, v[8 + k], jl);
        rec[k] = half ? hi : v[k];
      }
      if (trq) trq[t * 5 + 1] = ptx::globaltimer_ns();
      if (unit_ok) {
        // staging position of my unit's 4 gate rows (local gate row 4*ul) in row bl:
        // K-block j = ul/16, 16-B chunk c = (4ul % 64)/8, byte (4ul % 8)*2
        const int j = ul >> 4, c = (ul & 15) >> 1, byo = (ul & 1) * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int idx = ch * 8 + k;
          const int bl = ch * 16 + half * 8 + k;
          const size_t b = (size_t)col0 + bl;
          const float dh = dh0[idx] + (P.drop ? rec[k] * dsc[idx] : rec[k]);
          const float2 if2 = __half22float2(*reinterpret_cast<const __half2*>(&gq[idx].x));
          const float2 go2 = __half22float2(*reinterpret_cast<const __half2*>(&gq[idx].y));
          const float i = if2.x, f = if2.y, g = go2.x, o = go2.y;
          float tc, sech2;
          tanh_sech2(cc[idx], tc, sech2);
          const float d = dcr[idx] + dh * o * sech2;
          __align__(8) __half2 q2[2] = {
              __halves2half2(__float2half_rn(d * g * i * (1.f - i)), __float2half_rn(d * cp[idx] * f * (1.f - f))),
              __halves2half2(__float2half_rn(d * i * (1.f - g * g)), __float2half_rn(dh * tc * o * (1.f - o)))};
          const uint2 pk = *reinterpret_cast<const uint2*>(q2);
          if (!TSQ) *reinterpret_cast<uint2*>(dAout + b * fourhp + 4 * unit) = pk;  // R10 (for K8 / K9)
          *reinterpret_cast<uint2*>(stg + j * Bc * 128 + bl * 128 + ((c ^ (bl & 7)) << 4) + byo) = pk;
          dcr[idx] = d * f;
        }
      }
    }
    if (trq) trq[t * 5 + 2] = ptx::globaltimer_ns();
    if (tr4 && lane == 0) P.trace[(size_t)5 * T * 5 + t * 5 + warp] = ptx::globaltimer_ns();  // per-warp arrival
    if (TSQ && threadIdx.x == st_thr) {
      const unsigned long long w0 = trw ? ptx::globaltimer_ns() : 0;
      ptx::bulk_wait_group_read0();  // all earlier stores finished reading their staging
      if (trw) trw[t * 5 + 3] = ptx::globaltimer_ns() - w0;
    }
    ptx::tc_fence_before();
    ptx::fence_async_smem();  // staging writes (generic) -> bulk copy / TMA store reads (async proxy)
    __syncthreads();
    const bool publish = qi == 0 || P.wtiles;
    if (!TSQ) {
      // publish dA_t to the projection / weight-gradient roles: one release (cumulative over
      // the CTA's stores via the barrier); the consumers order their TMA reads after their
      // acquire with a consumer-side fence.proxy.async
      if (threadIdx.x == 64 && publish) release_add((qi == 0 ? P.q1done : P.q0done) + grp * 32, 1u);
    } else if (threadIdx.x == st_thr) {
      unsigned* pubf = (qi == 0 ? P.q1done : P.q0done) + grp * 32;
      // (Q1 publishes step t+1 inside step t's MMA wait, Q0 step t+2 -- see above)
      for (int kb = 0; kb < 4; ++kb)
        if (j0 * 4 + kb * 64 < fourhp) ptx::tma_store_2d(&P.tmdAo[qi], stg + kb * Bc * 128, j0 * 4 + kb * 64, t * B + col0);
      ptx::bulk_commit_group();
      if (t == 0) {
        ptx::bulk_wait_group0();
        if (publish) {  // Q1: step 0; Q0: steps min(1, T-1) .. 0
          fence_proxy_async();
          release_add(pubf, qi == 0 ? 1u : (T >= 2 ? 2u : 1u));
        }
      }
    }
    if (tr) trace[t * 5 + 3] = ptx::globaltimer_ns();
    // ring slot (t-2) % 3 = (t+1) % 3 was last read by the epilogues of steps t+1 and t+2
    // (steps read slots t % 3 and (t-1) % 3), i.e. before the barrier above
    // slot (t-(RG-1)) % RG = (t+1) % RG was last read by steps t+1 and t+2
    if (TSQ && threadIdx.x == pf_thr && t >= RG - 1) fetch_gc(t - (RG - 1));
    if (dpf && threadIdx.x == pf_thr && nf >= 0 && nf >= t - 2 &&
        acquire_ld(P.xdone + (grp * 8 + rank) * 32) >= (unsigned)(T - nf))
      fetch_dx(nf--, true);
    // push dA_t (consumed by step t-1) into every peer's sA[t & 1]: one bulk copy per peer.
    // WAR: a peer writes sA[p] of step s only after consuming my dA_{s+1}, which I produce
    // after my MMA that read sA[p] for step s+2 -- the double buffers need no extra barrier.
    const int pt = TSQ ? (int)threadIdx.x - 64 : (int)threadIdx.x;  // TSQ: warp 2 pushes
    if (t > 0 && pt >= 0 && pt < G && my_kblocks > 0) {
      const int dst = pt;
      const uint32_t dsta = ptx::mapa(sA_addr + (t & 1) * abuf + 4 * rank * Bc * 128, dst);
      const uint32_t mb = ptx::mapa(ptx::smem_u32(fullA + (t & 1)), dst);
      ptx::bulk_copy_to_peer(dsta, sX_addr + (t & 1) * SX, my_kblocks * Bc * 128, mb);
    }
    if (tr) trace[t * 5 + 4] = ptx::globaltimer_ns();
  }
  // nobody leaves while a peer may still read my staging / write my sA
  ptx::cluster_arrive();
  ptx::cluster_wait();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tbase, tcols);
  cta_stamp(P, 1, role);
}

size_t bwd_cl_smem(int hp, int Bc) {
  const int nkb = 4 * hp / 64;
  return 1024 + (size_t)nkb * 8192 + 2 * (size_t)nkb * Bc * 128 + 2 * (size_t)4 * Bc * 128 + 128;
}

cudaError_t launch_cluster(const void* fn, dim3 grid, dim3 block, size_t smem, int cluster_x, cudaStream_t s,
                           void** args, bool pdl = false) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster_x;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (the kernel griddep-waits before its inputs)
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}




// ============================================================== 2-layer wavefront (forward, split clusters)
// Three G-CTA clusters per batch group (G = ceil(hp/64)), one per role:
//   role 0 (R0_k): layer-0 recurrence, units [64k, 64k+64)        (cluster-local h exchange)
//   role 1 (P_k) : a1x_t = W1 h0_t + b1 for gate rows [256k, 256k+256)
//   role 2 (R1_k): layer-1 recurrence, units [64k, 64k+64), gate inputs a1x from P_k
// Cross-role hand-offs go through global memory (every step has its own slot, so
// no back-pressure is needed) with release/acquire counters:
//   R0 -> P : h0_t (the Hs0 stores R0 makes anyway), r0done[g] += 1 per CTA
//   P  -> R1: a1x_t fp32 rows, pdone[g][k] += 1
// Layer 1 trails layer 0 by a couple of steps; both recurrences run at the
// single-layer step rate with 8 warps per CTA at Bc = 16.
struct __align__(64) Fwd2Params {
  CUtensorMap tmA[3];  // resident A slices (K-major, box 64 x 128): U0, W1, U1
  CUtensorMap tmH0;    // Hs0 rows [(T+1)B][hp], box (64, Bc): P's B operand
  CUtensorMap tmW0;    // W0 [4hp][Ip0], box 64 x 128 (fused layer-0 input projection)
  CUtensorMap tmX0;    // X0 rows [T B][Ip0], box (64, Bc)
  CUtensorMap tmG1;    // a1x rows [T B][4hp] fp32, box (256, Bc): R1's gate inputs (r1_tma)
  // R roles' per-step outputs written by TMA stores from shared staging (TSA variant):
  CUtensorMap tmCo[2];  // C_l rows [T B][hp] fp32, box (64, Bc)
  CUtensorMap tmHo[2];  // Hs_l rows [(T+1) B][hp] fp16, box (64, Bc), SWIZZLE_128B (= the push staging)
  CUtensorMap tmGo[2];  // gates_l rows [T B][4hp] fp16, box (256, Bc)
  const float* Gx0;    // [T][B][4hp]
  float* a1x;          // [T][B][4hp]
  const __half* b1;
  const __half* b0;    // fused input projection: G_x0 = X0 W0^T + b0 inside R0 (fuse_x)
  __half* Hs[2];
  float* C[2];
  __half* gates[2];
  unsigned* r0done;    // [16][32]
  unsigned* pdone;     // [16][8][32]
  unsigned long long* trace;
  int T, B, Bc, hp, nbg, fuse_x, r1_tma;
  int region;          // the 32 KB + 2 x Bc x 128 B region (fused projection / R1 staging) exists
  const __half* Ag[3]; // row-major U0, W1, U1 [4hp][hp] (A operands copied into TMEM, NKS != 0)
  const __half* W0g;   // W0 [4hp][Ip0] (fused projection, TMEM copy)
  int Ip0;
  // recurrent dropout (NEXT-3, reading Q16b): the recurrent operand pushed to the peers is
  // h~_t = fp16(fp32(h_t) * scale) on kept units, 0 elsewhere, and is stored to Ht[l]
  // (the W role's dU operand); Hs keeps the unmasked h_t (next layer, head)
  int drop;
  CUtensorMap tmHt[2];  // Hst_l rows [(T+1) B][hp] fp16, box (64, Bc), SWIZZLE_128B (TMA stores)
  __half* Ht[2];
  const int* drop_step;
  uint32_t drop_seed, drop_thr, drop_seq0;
  float drop_scale;
};

// Copy rows [row0 + half*128 + 32*quadrant + lane] of a row-major fp16 matrix (ncols K
// elements, ld elements) into TMEM columns [col, col + ceil(K/32)*16) of this warp's lane
// quadrant: two K-elements per 32-bit column, zero padded (tcgen05.mma A-operand layout).
__device__ __forceinline__ void tmem_load_rows(uint32_t taddr_quadrant_col, const __half* __restrict__ src, int row,
                                               int nrows, int K, int ld) {
  const bool ok = row < nrows;
  for (int c0 = 0; c0 < (K + 31) / 32 * 16; c0 += 16) {
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int kk = 2 * (c0 + j);
      const uint32_t lo = (ok && kk < K) ? __half_as_ushort(src[(size_t)row * ld + kk]) : 0u;
      const uint32_t hi = (ok && kk + 1 < K) ? __half_as_ushort(src[(size_t)row * ld + kk + 1]) : 0u;
      v[j] = lo | (hi << 16);
    }
    ptx::tmem_st16(taddr_quadrant_col + c0, v);
  }
  ptx::tmem_wait_st();
}


// Same columns from the SWIZZLE_128B K-major SMEM copy a TMA load made of the rows (64-wide
// K-blocks of `kbstride` bytes, 128-B rows, 16-B chunk c of row r at ((c ^ (r & 7)) << 4));
// row r_local of the block, K elements (zero beyond the tensor: TMA out-of-bounds fill).
__device__ __forceinline__ void tmem_load_rows_sw(uint32_t taddr_quadrant_col, const uint8_t* sbase, int r_local,
                                                  int K, int kbstride) {
  for (int c0 = 0; c0 < (K + 31) / 32 * 16; c0 += 16) {
    uint32_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int kk = 2 * (c0 + j), kb = kk >> 6, w = kk & 63;
      v[j] = *reinterpret_cast<const uint32_t*>(sbase + kb * kbstride + r_local * 128 +
                                                ((((w >> 3) ^ (r_local & 7))) << 4) + (w & 7) * 2);
    }
    ptx::tmem_st16(taddr_quadrant_col + c0, v);
  }
  ptx::tmem_wait_st();
}

// Forward roles' per-step MMAs for issuing warp W of 4, K-steps known at compile time:
// warp-uniform, fully unrolled, one elected lane issues (k = W, W+4, ... < NKS; both
// M=128 halves of the 256-row A slice; accumulator (half, W)).
// A in TMEM (tA: half h2's rows at columns tA + h2*KCP, 8 columns per K-step of 16).
template <int NKS, int W, int NIS>
__device__ __forceinline__ void fwd_issue_unrolled(uint32_t tbase, uint32_t tA, int KCP, uint32_t aH, int Bc,
                                                   int nacc, uint32_t idesc, bool acc0, uint64_t* barM) {
  const uint64_t bd0 = ptx::smem_desc_sw128(aH, 0, 1024);
#pragma unroll
  for (int k = W; k < NKS; k += NIS) {
    const int kb = k >> 2, kk = k & 3;
    const uint64_t bd = bd0 + (uint64_t)((kb * Bc * 128 + kk * 32) >> 4);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      if (ptx::elect_one_sync())
        ptx::mma_f16_ts(tbase + (h2 * nacc + W) * Bc, tA + h2 * KCP + k * 8, bd, idesc,
                        (k >= NIS || (W == 0 && acc0)) ? 1u : 0u);
    }
  }
  if (ptx::elect_one_sync()) ptx::mma_commit(barM);
  __syncwarp();
}

template <int NCI, int NKS, bool DROP>
__global__ void __launch_bounds__(512, 1) recur2f_kernel(const __grid_constant__ Fwd2Params P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int T = P.T, B = P.B, Bc = P.Bc, hp = P.hp;
  const int role = blockIdx.y / P.nbg, grp = blockIdx.y % P.nbg;
  // phase trace: per-CTA entry / exit stamps and role (0 R0, 1 P, 2 R1) after the step stamps
  unsigned long long* ctas = (P.trace && threadIdx.x == 0)
                                 ? P.trace + (size_t)6 * T * 5 + 3 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (ctas) {
    ctas[0] = ptx::globaltimer_ns();
    ctas[2] = (unsigned long long)role;
  }
  const int nkb = (hp + 63) / 64;             // == cluster size
  const int nk16 = (hp + 15) / 16;
  const int nwarps = blockDim.x >> 5;
  const int cgN = nwarps >> 3;
  const int hbuf = nkb * Bc * 128;
  uint8_t* sU = smem;                         // [2 halves][nkb][16 KB]
  uint8_t* sH = sU + 2 * nkb * 16384;         // [2][hbuf]
  uint8_t* sX = sH + 2 * hbuf;                // [2][Bc][128 B]
  uint8_t* sW0 = sX + 2 * Bc * 128;           // R0, fuse_x: [2 halves][16 KB] W0 slice (Ip0 <= 64)
                                              // R1, r1_tma: [2][Bc][256] fp32 a1x staging
  uint8_t* sXin = sW0 + (P.region ? 32768 : 0);  // R0, fuse_x: [2][Bc][128 B] x_t operand
  float* sAct = reinterpret_cast<float*>(sXin + (P.region ? 2 * Bc * 128 : 0));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sAct + nwarps * 16 * ACT_LD);
  uint64_t* barU = bars;
  uint64_t* barM = bars + 1;
  uint64_t* fullH = bars + 2;                 // [2]
  uint64_t* barX = bars + 4;                  // [2] x_t landed (fuse_x)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 6);
  // recurrent dropout: [2][Bc][128 B] staging of the UNMASKED h_t for the Hs TMA store (the
  // push staging sX then holds h~_t); 1024-aligned for SWIZZLE_128B
  uint8_t* sXu = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(bars + 16) + 1023) & ~uintptr_t(1023));
  const bool fx = role == 0 && P.fuse_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quarter = warp & 3, hf = (warp >> 2) & 1, cg = warp >> 3;
  const int G = gridDim.x;
  const int rank = blockIdx.x;
  const int row0 = rank * 256;
  const int col0 = grp * Bc;
  const int r = hf * 128 + quarter * 32 + lane;
  const int grow = row0 + r;
  const int gate = r & 3;
  const int unit = grow >> 2;
  const bool unit_ok = unit < hp;
  const int fourhp = 4 * hp;
  // with the A slice in TMEM (NKS != 0) two issuing warps reach the MMA floor; two
  // accumulators per half also halve the epilogue's TMEM reads
  const int nacc = NKS != 0 ? 2 : (Bc <= 32 ? 4 : Bc <= 64 ? 2 : 1);
  const int nis = min(nacc, nk16);
  const int ac = 2 * nacc * Bc;
  // NKS != 0: the role's A slice lives in TMEM (columns [TA, TA + 2*KCP)), fused W0 at TW0
  constexpr bool TSA = NKS != 0;
  const int KCP = (hp + 31) / 32 * 16;
  const uint32_t tcols = TSA ? 512u : (ac <= 32 ? 32u : ac <= 64 ? 64u : ac <= 128 ? 128u : ac <= 256 ? 256u : 512u);
  const int total_bytes = nkb * Bc * 128;
  const bool tr = P.trace != nullptr && rank == 0 && grp == 0 && threadIdx.x == 0;
  unsigned long long* trr = P.trace ? P.trace + (size_t)role * T * 5 : nullptr;
#define TR(t, i) \
  if (tr) trr[(t) * 5 + (i)] = ptx::globaltimer_ns()

  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&P.tmA[role]);
    ptx::mbar_init(barU, 1);
    ptx::mbar_init(barM, nis);
    ptx::mbar_init(fullH, 1);
    ptx::mbar_init(fullH + 1, 1);
    ptx::mbar_init(barX, 1);
    ptx::mbar_init(barX + 1, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tslot, tcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tA = tbase + 256, tW0 = tbase + 256 + 2 * KCP;
  if (TSA) {
    // A slice (and the fused W0 slice) by TMA into the otherwise unused sU / sW0 regions,
    // then SMEM -> TMEM: warp (quarter, hf) owns gate rows hf*128 + 32*quarter + lane.
    // (Round 1 gathered the rows from global memory with strided 2-byte loads: ~20 us of
    // every forward launch before its first step.)
    if (threadIdx.x == 0) {
      ptx::mbar_arrive_expect_tx(barU, 2 * nkb * 16384 + (fx ? 32768 : 0));
      for (int h2 = 0; h2 < 2; ++h2)
        for (int kb = 0; kb < nkb; ++kb)
          ptx::tma_load_2d(sU + (h2 * nkb + kb) * 16384, &P.tmA[role], barU, kb * 64, row0 + h2 * 128);
      if (fx)
        for (int h2 = 0; h2 < 2; ++h2) ptx::tma_load_2d(sW0 + h2 * 16384, &P.tmW0, barU, 0, row0 + h2 * 128);
    }
    ptx::mbar_wait(barU, 0);
    if (cg == 0) {
      const uint32_t tq = (static_cast<uint32_t>(quarter * 32) << 16);
      const int rl = quarter * 32 + lane;
      tmem_load_rows_sw(tA + tq + hf * KCP, sU + hf * nkb * 16384, rl, hp, 16384);
      if (fx) tmem_load_rows_sw(tW0 + tq + hf * 16, sW0 + hf * 16384, rl, P.Ip0, 16384);  // 16 columns per half
    }
    ptx::fence_async_smem();  // generic reads of sU / sW0 before the async-proxy writes that reuse them
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) {
    // (PDL, option fwd_pdl) everything above reads weights only; the activations this
    // launch reads (x_t, G_x) were written by the previous kernel: wait for it here -- the
    // cluster barrier below orders every other thread's reads after this wait
    ptx::griddep_wait();
    if (role != 1) {
      ptx::mbar_arrive_expect_tx(fullH, total_bytes);
      ptx::mbar_arrive_expect_tx(fullH + 1, total_bytes);
    }
    if (!TSA) {
      ptx::mbar_arrive_expect_tx(barU, 2 * nkb * 16384 + (fx ? 32768 : 0));
      for (int h2 = 0; h2 < 2; ++h2)
        for (int kb = 0; kb < nkb; ++kb)
          ptx::tma_load_2d(sU + (h2 * nkb + kb) * 16384, &P.tmA[role], barU, kb * 64, row0 + h2 * 128);
      if (fx)
        for (int h2 = 0; h2 < 2; ++h2) ptx::tma_load_2d(sW0 + h2 * 16384, &P.tmW0, barU, 0, row0 + h2 * 128);
    }
    if (fx) {
      ptx::mbar_arrive_expect_tx(barX, Bc * 128);
      ptx::tma_load_2d(sXin, &P.tmX0, barX, 0, col0);
    }
    if (!TSA) ptx::mbar_wait(barU, 0);
  }
  ptx::cluster_arrive();
  ptx::cluster_wait();
  ptx::griddep_launch();  // (PDL) every CTA resident: the next kernel (the head) may start its prologue

  const uint32_t idesc = ptx::idesc_f16_f32(128, Bc, 0, 0);
  const int nchunk = Bc / 16;
  const uint32_t sH_addr = ptx::smem_u32(sH), sX_addr = ptx::smem_u32(sX);
  uint32_t fphase[2] = {0u, 0u};
  auto issue_mma = [&](int p) {  // fx: accumulator 0 already holds x_t W0^T
    const uint32_t aU = ptx::smem_u32(sU), aH = sH_addr + p * hbuf;
    const uint64_t ad0 = ptx::smem_desc_sw128(aU, 0, 1024), bd0 = ptx::smem_desc_sw128(aH, 0, 1024);
    for (int k = warp; k < nk16; k += nis) {
      const int kb = k >> 2, kk = k & 3;
      const uint64_t bd = bd0 + (uint64_t)((kb * Bc * 128 + kk * 32) >> 4);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const uint64_t ad = ad0 + (uint64_t)(((h2 * nkb + kb) * 16384 + kk * 32) >> 4);
        ptx::mma_f16(tbase + (h2 * nacc + warp) * Bc, ad, bd, idesc, (k >= nis || (fx && warp == 0)) ? 1u : 0u);
      }
    }
    ptx::mma_commit(barM);
  };
  int t_cur = 0;  // (phase trace only)
  // wait for the step's B operand in slot p, then this warp's share of the MMAs
  auto issue_step = [&](int p, bool acc0) {
    if (NKS == nk16 && nis == 2) {
      ptx::mbar_wait(fullH + p, fphase[p]);
      ptx::tc_fence_after();
      if (lane == 0) TR(t_cur, 1);
      const uint32_t aH = sH_addr + p * hbuf;
      if (warp == 0)
        fwd_issue_unrolled<NKS, 0, 2>(tbase, tA, KCP, aH, Bc, nacc, idesc, acc0, barM);
      else
        fwd_issue_unrolled<NKS, 1, 2>(tbase, tA, KCP, aH, Bc, nacc, idesc, acc0, barM);
    } else if (lane == 0) {
      ptx::mbar_wait(fullH + p, fphase[p]);
      ptx::tc_fence_after();
      TR(t_cur, 1);
      issue_mma(p);
    }
  };
  auto load_acc = [&](float (&v)[16], int c0, int nacc_used) {
    const uint32_t ta = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + hf * nacc * Bc + c0;
    ptx::tmem_ld16(ta, v);
    for (int a = 1; a < nacc_used; ++a) {
      float w[16];
      ptx::tmem_ld16(ta + a * Bc, w);
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] += w[k];
    }
  };

  if (role == 1) {
    // ------------------------------------------------------------ projection P_k
    const float bias = unit_ok ? __half2float(P.b1[grow]) : 0.f;
    const unsigned* r0f = P.r0done + grp * 32;
    auto load_h0 = [&](int t) {  // thread 0: h0_t of every R0_k (all stored) -> sH[t & 1]
      fence_proxy_async();
      ptx::mbar_arrive_expect_tx(fullH + (t & 1), total_bytes);
      for (int kb = 0; kb < nkb; ++kb)
        ptx::tma_load_2d(sH + (t & 1) * hbuf + kb * Bc * 128, &P.tmH0, fullH + (t & 1), kb * 64,
                         (t + 1) * B + col0);
    };
    bool pending = false;
    if (threadIdx.x == 0) {
      spin_until(r0f, (unsigned)G);
      load_h0(0);
    }
    for (int t = 0; t < T; ++t) {
      const int p = t & 1;
      t_cur = t;
      TR(t, 0);
      if (warp < nis) issue_step(p, false);
      // prefetch h0_{t+1} now if R0 already published it (sH[p^1] was read by MMA t-1, complete)
      if (threadIdx.x == 0 && t + 1 < T) {
        if (acquire_ld(r0f) >= (unsigned)(G * (t + 2))) load_h0(t + 1);
        else pending = true;
      }
      __syncwarp();
      ptx::mbar_wait_relaxed(barM, t & 1);
      ptx::tc_fence_after();
      fphase[p] ^= 1u;
      TR(t, 2);
#pragma unroll
      for (int ci = 0; ci < NCI; ++ci) {
        const int ch = ci * cgN + cg;
        if (ch >= nchunk) break;
        float v[16];
        load_acc(v, ch * 16, nis);
        if (grow < fourhp) {
          float* out = P.a1x + ((size_t)t * B + col0 + ch * 16) * fourhp + grow;
#pragma unroll
          for (int k = 0; k < 16; ++k) out[(size_t)k * fourhp] = v[k] + bias;  // layer-1 G_x (R3)
        }
      }
      ptx::tc_fence_before();
      fence_proxy_async();  // a1x stores -> R1's TMA reads
      __syncthreads();
      TR(t, 3);
      if (threadIdx.x == 0) {
        release_add(P.pdone + (grp * 8 + rank) * 32, 1u);
        if (pending) {
          spin_until(r0f, (unsigned)(G * (t + 2)));
          load_h0(t + 1);
          pending = false;
        }
      }
      TR(t, 4);
    }
  } else {
    // ------------------------------------------------------------ recurrence R0_k / R1_k
    const int li = role == 0 ? 0 : 1;
    __half* Hs = P.Hs[li];
    float* Cst = P.C[li];
    __half* gts = P.gates[li];
    const float* Gx = li == 0 ? P.Gx0 : P.a1x;
    const unsigned* pf = P.pdone + (grp * 8 + rank) * 32;
    // r1_tma: a1x_t (my 256 gate rows x Bc) staged by TMA into the (otherwise unused)
    // fused-projection region, double-buffered, barX[t & 1] -- one thread acquires
    const bool gt = li == 1 && P.r1_tma;
    const float* sG1 = reinterpret_cast<const float*>(sW0);
    auto fetch_a1x = [&](int t) {  // one thread
      spin_until(pf, (unsigned)(t + 1));
      fence_proxy_async();
      ptx::mbar_arrive_expect_tx(barX + (t & 1), Bc * 256 * 4);
      ptx::tma_load_2d(sW0 + (t & 1) * Bc * 1024, &P.tmG1, barX + (t & 1), row0, t * B + col0);
    };
    if (gt && threadIdx.x == 128) fetch_a1x(0);
    float creg[NCI * 4];
#pragma unroll
    for (int i = 0; i < NCI * 4; ++i) creg[i] = 0.f;
    float* myAct = sAct + warp * 16 * ACT_LD;
    const float gsc = gate == 2 ? 2.f : 1.f;
    const float bias0 = fx && unit_ok ? __half2float(P.b0[grow]) : 0.f;
    // recurrent dropout: mask x scale of this lane's (unit, column) pairs, fixed over t
    float dsc[NCI * 4];
#pragma unroll
    for (int i = 0; i < NCI * 4; ++i) dsc[i] = 1.f;
    if (DROP) {
      const uint32_t lk = drop_layer_key(P.drop_seed, (uint32_t)*P.drop_step, (uint32_t)li);
#pragma unroll
      for (int ci = 0; ci < NCI; ++ci)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t seq = P.drop_seq0 + (uint32_t)(col0 + (ci * cgN + cg) * 16 + 4 * q + gate);
          dsc[ci * 4 + q] = unit_ok && drop_kept(drop_seq_key(lk, seq), (uint32_t)unit, P.drop_thr) ? P.drop_scale : 0.f;
        }
    }
    // debug sub-phase stamps of the epilogue (R0 CTA 0 / group 0, thread 0) in trace role slot 3
    unsigned long long* trx = (tr && li == 0) ? P.trace + (size_t)3 * T * 5 : nullptr;
    // TSA: the SMEM A region is free -> stage c_t and the gates there and let one thread
    // (no MMA issue, no push) write them -- and h_t from the push staging -- by TMA stores
    constexpr bool TST = TSA;
    float* sCo = reinterpret_cast<float*>(sU);                          // [2][Bc][64] fp32
    __half* sGo = reinterpret_cast<__half*>(sU + 2 * Bc * 64 * 4);      // [2][Bc][256] fp16
    const int st_thr = blockDim.x - 32;
    uint32_t mph = 0;
    // gate inputs of step t (layer 0: G_x0 rows from K1, or the bias when the projection
    // is fused; layer 1: a1x rows from P_k once published), loaded one step ahead so
    // the flag acquire and the L2 latency overlap the previous step's MMA
    float gx[NCI][16], gxn[NCI][16];
    auto load_gx = [&](int t, float (&dst)[NCI][16]) {
      if (gt) return;
      if (li == 1) {
        if (lane == 0) spin_until(pf, (unsigned)(t + 1));  // a1x_t of my gate rows stored by P_k
        __syncwarp();
      }
#pragma unroll
      for (int ci = 0; ci < NCI; ++ci) {
        const int ch = ci * cgN + cg;
        const bool ok = ch < nchunk && grow < fourhp;
        const float* gp = Gx + ((size_t)t * B + col0 + ch * 16) * fourhp + grow;
        if (fx) {
#pragma unroll
          for (int k = 0; k < 16; ++k) dst[ci][k] = bias0;
        } else if (li == 0) {
#pragma unroll
          for (int k = 0; k < 16; ++k) dst[ci][k] = ok ? __ldg(gp + (size_t)k * fourhp) : 0.f;
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) dst[ci][k] = ok ? __ldcg(gp + (size_t)k * fourhp) : 0.f;
        }
      }
    };
    // layer 0 with G_x0 from K1: loads one step ahead (NCI = 1; the 512-thread variant's
    // register budget keeps them in-step)
    const bool PIPE = false;  // (measured slower: the loads sit between MMA issue and the barM wait)
    if (PIPE) load_gx(0, gx);
    // operand prefetch for step t+1 (x_{t+1} for the fused projection, a1x_{t+1} for layer 1)
    // by a thread that issues no MMAs: TMA issued by an MMA issuer measurably delays its commit
    const int pf_thr = 128;
    for (int t = 0; t < T; ++t) {
      t_cur = t;
      TR(t, 0);
      if (!PIPE) load_gx(t, gx);
      if (threadIdx.x == pf_thr && t + 1 < T) {
        // slots (t+1)&1 were last read by step t-1 (x MMA complete at its barM; sG1 in its epilogue)
        if (fx) {
          ptx::mbar_arrive_expect_tx(barX + ((t + 1) & 1), Bc * 128);
          ptx::tma_load_2d(sXin + ((t + 1) & 1) * Bc * 128, &P.tmX0, barX + ((t + 1) & 1), 0, (t + 1) * B + col0);
        }
        if (gt) fetch_a1x(t + 1);
      }
      if (fx && warp == 0 && lane == 0) {
        // x_t W0^T into accumulator 0 (both halves) -- off the recurrence's critical path
        ptx::mbar_wait(barX + (t & 1), (t >> 1) & 1);
        ptx::tc_fence_after();
        const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(sXin + (t & 1) * Bc * 128), 0, 1024);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          if (TSA)
            ptx::mma_f16_ts(tbase + (h2 * nacc) * Bc, tW0 + h2 * 16, bd, idesc, 0u);
          else
            ptx::mma_f16(tbase + (h2 * nacc) * Bc, ptx::smem_desc_sw128(ptx::smem_u32(sW0 + h2 * 16384), 0, 1024), bd,
                         idesc, 0u);
        }
        if (t == 0) ptx::mma_commit(barM);
      }
      if (fx && t == 0 && lane == 0 && warp > 0 && warp < nis) ptx::mbar_arrive(barM);
      if (t > 0) {
        const int p = (t - 1) & 1;
        if (warp < nis) issue_step(p, fx);
        if (PIPE && t + 1 < T) load_gx(t + 1, gxn);
        __syncwarp();
        ptx::mbar_wait_relaxed(barM, mph);
        mph ^= 1u;
        ptx::tc_fence_after();
        fphase[p] ^= 1u;
        if (threadIdx.x == 0 && t + 2 <= T - 1) ptx::mbar_arrive_expect_tx(fullH + p, total_bytes);
      } else {
        if (PIPE && t + 1 < T) load_gx(t + 1, gxn);
        if (fx) {
          __syncwarp();
          ptx::mbar_wait_relaxed(barM, mph);
          mph ^= 1u;
          ptx::tc_fence_after();
        }
      }
      TR(t, 2);
      if (gt) {
        ptx::mbar_wait(barX + (t & 1), (t >> 1) & 1);
        const float* g = sG1 + (t & 1) * Bc * 256;
#pragma unroll
        for (int ci = 0; ci < NCI; ++ci)
#pragma unroll
          for (int k = 0; k < 16; ++k) gx[ci][k] = g[((ci * cgN + cg) * 16 + k) * 256 + r];
      }
      __half* hout = Hs + (size_t)(t + 1) * B * hp;
      float* cout = Cst + (size_t)t * B * hp;
      __half* gout = gts + (size_t)t * B * fourhp;
      uint8_t* stg = sX + (t & 1) * Bc * 128;
#pragma unroll
      for (int ci = 0; ci < NCI; ++ci) {
        const int ch = ci * cgN + cg;
        if (ch >= nchunk) break;
        const int c0 = ch * 16;
        float v[16];
        if (t > 0 || fx) {
          load_acc(v, c0, t > 0 ? nis : 1);
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = 0.f;
        }
        if (trx) trx[t * 5 + 0] = ptx::globaltimer_ns();
#pragma unroll
        for (int k = 0; k < 16; ++k) myAct[k * ACT_LD + lane] = act_gate(v[k] + gx[ci][k], gsc);
        __syncwarp();
        if (trx) trx[t * 5 + 1] = ptx::globaltimer_ns();
        if (unit_ok) {
          const int u = lane >> 2;
          const int ul = (r >> 2);
          const int c = ul >> 3;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int col = 4 * q + gate;
            const float4 a4 = *reinterpret_cast<const float4*>(myAct + col * ACT_LD + 4 * u);
            const int bl = c0 + col;
            const size_t b = (size_t)col0 + bl;
            const float i = a4.x, f = a4.y, g = a4.z, o = a4.w;
            const float cv = f * creg[ci * 4 + q] + i * g;
            creg[ci * 4 + q] = cv;
            const __half hh = __float2half_rn(o * act_gate(cv, 2.f));
            // the recurrent operand: h_t, or h~_t = fp16(fp32(h_t) * scale) / 0 (R6d)
            const __half hm = DROP ? __float2half_rn(__half2float(hh) * dsc[ci * 4 + q]) : hh;
            const int so = bl * 128 + ((c ^ (bl & 7)) << 4) + (ul & 7) * 2;
            if (!TST) {
              cout[b * hp + unit] = cv;                 // R5
              hout[b * hp + unit] = hh;                 // R6
              if (DROP) P.Ht[li][(size_t)(t + 1) * B * hp + b * hp + unit] = hm;
            } else {
              sCo[((t & 1) * Bc + bl) * 64 + ul] = cv;
              if (DROP) *reinterpret_cast<__half*>(sXu + (t & 1) * Bc * 128 + so) = hh;
            }
            *reinterpret_cast<__half*>(stg + so) = hm;
            __align__(8) __half2 gg[2] = {__halves2half2(__float2half_rn(i), __float2half_rn(f)),
                                          __halves2half2(__float2half_rn(g), __float2half_rn(o))};
            if (!TST)
              *reinterpret_cast<uint2*>(gout + b * fourhp + 4 * unit) = *reinterpret_cast<const uint2*>(gg);  // R4
            else
              *reinterpret_cast<uint2*>(sGo + ((t & 1) * Bc + bl) * 256 + 4 * ul) = *reinterpret_cast<const uint2*>(gg);
          }
        }
        __syncwarp();
      }
      if (trx) trx[t * 5 + 2] = ptx::globaltimer_ns();
      if (TST && threadIdx.x == st_thr) {
        // step t-1's stores must have finished reading their staging (rewritten at step t+1)
        ptx::bulk_wait_group_read0();
      }
      ptx::tc_fence_before();
      ptx::fence_async_smem();
      __syncthreads();
      if (trx) trx[t * 5 + 3] = ptx::globaltimer_ns();
      TR(t, 3);
      if (PIPE) {
#pragma unroll
        for (int ci = 0; ci < NCI; ++ci)
#pragma unroll
          for (int k = 0; k < 16; ++k) gx[ci][k] = gxn[ci][k];
      }
      // pushers: warp 5 (issues no MMAs: async copies from an MMA-issuing thread delay its commits)
      if (t < T - 1 && threadIdx.x >= 160 && threadIdx.x < 160 + G) {
        const int dst = threadIdx.x - 160;
        const uint32_t dsta = ptx::mapa(sH_addr + (t & 1) * hbuf + rank * Bc * 128, dst);
        const uint32_t mb = ptx::mapa(ptx::smem_u32(fullH + (t & 1)), dst);
        ptx::bulk_copy_to_peer(dsta, sX_addr + (t & 1) * Bc * 128, Bc * 128, mb);
      }
      if (TST) {
        if (threadIdx.x == st_thr) {
          // c_t, h_t (the swizzled push staging = Hs' SWIZZLE_128B box) and the gates of step t
          if (li == 0 && t > 0) {
            // h0_{t-1}'s store (previous group) complete -> publish it to the projection role
            ptx::bulk_wait_group0();
            fence_proxy_async();
            release_add(P.r0done + grp * 32, 1u);
          }
          ptx::tma_store_2d(&P.tmCo[li], sCo + (t & 1) * Bc * 64, rank * 64, t * B + col0);
          if (DROP) {  // h~_t (the push staging) -> Hst, unmasked h_t -> Hs
            ptx::tma_store_2d(&P.tmHt[li], stg, rank * 64, (t + 1) * B + col0);
            ptx::tma_store_2d(&P.tmHo[li], sXu + (t & 1) * Bc * 128, rank * 64, (t + 1) * B + col0);
          } else {
            ptx::tma_store_2d(&P.tmHo[li], stg, rank * 64, (t + 1) * B + col0);
          }
          ptx::tma_store_2d(&P.tmGo[li], sGo + (t & 1) * Bc * 256, rank * 256, t * B + col0);
          ptx::bulk_commit_group();
          if (li == 0 && t == T - 1) {
            ptx::bulk_wait_group0();
            fence_proxy_async();
            release_add(P.r0done + grp * 32, 1u);
          }
        }
      } else if (li == 0) {
        // publish h0_t to the projection role after the push (off the recurrence's critical
        // path): every thread's Hs0 stores -> async proxy, then one release
        fence_proxy_async();
        if (warp == nwarps - 1) {
          named_bar_sync(1, blockDim.x);
          if (lane == 0) release_add(P.r0done + grp * 32, 1u);
        } else {
          named_bar_arrive(1, blockDim.x);
        }
      }
      TR(t, 4);
    }
    if (TST && threadIdx.x == st_thr) ptx::bulk_wait_group0();  // all stores done before exit
  }
#undef TR
  ptx::cluster_arrive();
  ptx::cluster_wait();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tbase, tcols);
  if (ctas) ctas[1] = ptx::globaltimer_ns();
}


}  // namespace

bool recur_fwd_supported(int B, int hp) {
  FwdPlan p;
  if (!plan_fwd(B, hp, &p)) return false;
  const int nw = 8 * p.cgN;
  return (hp + 63) / 64 <= 8 && nw <= 16 && fwd_cl_smem(hp, p.Bc, nw) <= 227 * 1024;  // one cluster per group
}

cudaError_t launch_recur_fwd(const RecurFwdArgs& a, cudaStream_t s) {
  FwdPlan p;
  if (!recur_fwd_supported(a.B, a.hp) || !plan_fwd(a.B, a.hp, &p)) return cudaErrorInvalidConfiguration;
  const int Gc = (a.hp + 63) / 64;  // CTAs of 64 units = cluster size
  const int nw = 8 * p.cgN;
  CUtensorMap mU;
  if (encode_tmap_2d(&mU, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.U, a.hp, 4 * a.hp, a.hp * 2, 64, 128,
                     CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const float* gx = a.Gx;
  int T = a.T, B = a.B, Bc = p.Bc, hp = a.hp;
  __half* hs = a.Hs;
  float* cst = a.C;
  __half* gt = a.gates;
  unsigned long long* trace = a.trace;
  void* args[] = {&mU, &gx, &T, &B, &Bc, &hp, &hs, &cst, &gt, &trace};
  const void* fn = p.nci == 1 ? (const void*)recur_fwd_cl_kernel<1>
                 : p.nci == 2 ? (const void*)recur_fwd_cl_kernel<2> : (const void*)recur_fwd_cl_kernel<4>;
  return launch_cluster(fn, dim3(Gc, p.nbg), dim3(32 * nw), fwd_cl_smem(a.hp, p.Bc, nw), Gc, s, args);
}

}  // namespace hdp

namespace hdp {

bool recur_bwd_supported(int B, int hp) {
  int Bc, nbg;
  if (!plan_bwd(B, hp, &Bc, &nbg)) return false;
  return pow2ceil((hp + 63) / 64) <= 8 && bwd_cl_smem(hp, Bc) <= 227 * 1024;  // one cluster per group
}

cudaError_t launch_recur_bwd(const RecurBwdArgs& a, cudaStream_t s) {
  int Bc = 0, nbg = 0;
  if (!recur_bwd_supported(a.B, a.hp) || !plan_bwd(a.B, a.hp, &Bc, &nbg)) return cudaErrorInvalidConfiguration;
  const int Gc = pow2ceil((a.hp + 63) / 64);
  CUtensorMap mU;
  if (encode_tmap_2d(&mU, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.U, a.hp, 4 * a.hp, a.hp * 2, 64, 64,
                     CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const float* dha = a.dHa;
  int last = a.dHa_last_only, T = a.T, B = a.B, hp = a.hp;
  const __half* gt = a.gates;
  const float* cst = a.C;
  __half* da = a.dA;
  unsigned long long* trace = a.trace;
  void* args[] = {&mU, &dha, &last, &gt, &cst, &da, &T, &B, &hp, &trace};
  const void* fn = Bc == 16 ? (const void*)recur_bwd_cl_kernel<1>
                 : Bc == 32 ? (const void*)recur_bwd_cl_kernel<2>
                 : Bc == 48 ? (const void*)recur_bwd_cl_kernel<3> : (const void*)recur_bwd_cl_kernel<4>;
  return launch_cluster(fn, dim3(Gc, nbg), dim3(128), bwd_cl_smem(a.hp, Bc), Gc, s, args);
}

}  // namespace hdp

namespace hdp {

// split-cluster forward wavefront plan: largest batch-group count whose 3 x G x nbg
// CTAs fit on the GPU as co-resident clusters (cached per shape)
// extra shared memory of the fused layer-0 input projection (W0 slice + x_t double buffer)
size_t w2f_fuse_bytes(int Bc) { return 32768 + 2 * (size_t)Bc * 128; }
// the dropout staging sXu behind the barriers (reserved whether or not dropout is on)
size_t w2f_drop_bytes(int Bc) { return 1024 + 128 + 2 * (size_t)Bc * 128; }

struct W2Plan {
  int Bc = 0, nbg = 0, cgN = 0, nci = 0, fuse = 0;
};
// K-step counts with an unrolled MMA-issue instantiation (h_p = 208, 256); others generic
// DROP: the recurrent-dropout instantiation (its epilogue differs; kept out of the plain one)
template <int NCI, bool DROP>
const void* recur2f_fn_nks(int nk16) {
  return nk16 == 13 ? (const void*)recur2f_kernel<NCI, 13, DROP>
       : nk16 == 16 ? (const void*)recur2f_kernel<NCI, 16, DROP> : (const void*)recur2f_kernel<NCI, 0, DROP>;
}
const void* recur2f_fn(int nci, int hp, bool drop = false) {
  const int nk16 = opt(OPT_WAVEFRONT_TMEM) == 0 ? -1 : (hp + 15) / 16;  // -1: the generic (SMEM-A) instantiation
  if (drop) return nci == 1 ? recur2f_fn_nks<1, true>(nk16) : nci == 2 ? recur2f_fn_nks<2, true>(nk16) : nullptr;
  return nci == 1 ? recur2f_fn_nks<1, false>(nk16) : nci == 2 ? recur2f_fn_nks<2, false>(nk16) : nullptr;
}
bool plan_w2f(int B, int hp, W2Plan* out) {
  static std::map<std::pair<int, int>, W2Plan> cache;
  auto key = std::make_pair(B, hp);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return out->nbg > 0;
  }
  W2Plan best;
  const int G = (hp + 63) / 64;
  if (B >= 16 && !(B & 15) && !(hp & 15) && G <= 8) {
    for (int nbg = 16; nbg >= 1 && !best.nbg; nbg >>= 1) {
      if (B % nbg) continue;
      const int Bc = B / nbg;
      if ((Bc & 15) || Bc > 32 || 3 * G * nbg > 148) continue;
      W2Plan p;
      p.Bc = Bc;
      p.nbg = nbg;
      p.cgN = Bc / 16;
      p.nci = 1;
      size_t smem = fwd_cl_smem(hp, Bc, 8 * p.cgN) + w2f_drop_bytes(Bc);
      if (smem > 227 * 1024) continue;
      if (opt(OPT_WAVEFRONT_FUSEX) != 0 && smem + w2f_fuse_bytes(Bc) <= 227 * 1024) {
        smem += w2f_fuse_bytes(Bc);
        p.fuse = 1;
      }
      const void* fn = recur2f_fn(p.nci, hp);
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) break;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G, 3 * nbg);
      cfg.blockDim = dim3(256 * p.cgN);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        continue;
      }
      if (ncl >= 3 * nbg) best = p;
    }
  }
  cache[key] = best;
  *out = best;
  return best.nbg > 0;
}

bool recur2_fwd_fuses_x(int B, int hp, int Ip0) {
  W2Plan p;
  // (with the A slices in TMEM, columns [256, 256 + 2*KCP) + 2 x 16 for W0 must fit in 512)
  return recur2_fwd_supported(B, hp) && plan_w2f(B, hp, &p) && p.fuse && Ip0 <= 16 &&
         256 + 2 * ((hp + 31) / 32 * 16) + 32 <= 512 &&
         opt(OPT_WAVEFRONT_FUSEX) != 0;
}

bool recur2_fwd_supported(int B, int hp) {
  if (opt(OPT_WAVEFRONT) == 0) return false;
  W2Plan p;
  return plan_w2f(B, hp, &p);
}

cudaError_t launch_recur2_fwd(const Recur2FwdArgs& a, cudaStream_t s) {
  if (!recur2_fwd_supported(a.B, a.hp)) return cudaErrorInvalidConfiguration;
  {
    W2Plan pl;
    plan_w2f(a.B, a.hp, &pl);
    const int G = (a.hp + 63) / 64;
    const uint64_t hp = a.hp;
    Fwd2Params P;
    memset(&P, 0, sizeof P);
    const __half* As[3] = {a.U0, a.W1, a.U1};
    for (int i = 0; i < 3; ++i)
      if (encode_tmap_2d(&P.tmA[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, As[i], hp, 4 * hp, hp * 2, 64, 128,
                         CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    if (encode_tmap_2d(&P.tmH0, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.Hs0, hp, (uint64_t)(a.T + 1) * a.B, hp * 2, 64,
                       pl.Bc, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    P.Gx0 = a.Gx0;
    P.a1x = a.a1x;
    P.b1 = a.b1;
    P.Hs[0] = a.Hs0;
    P.Hs[1] = a.Hs1;
    P.C[0] = a.C0;
    P.C[1] = a.C1;
    P.gates[0] = a.gates0;
    P.gates[1] = a.gates1;
    P.r0done = a.flags;
    P.pdone = a.flags + 16 * 32;
    P.trace = a.trace;
    P.T = a.T;
    P.B = a.B;
    P.Bc = pl.Bc;
    P.hp = a.hp;
    P.nbg = pl.nbg;
    P.fuse_x = a.X0 != nullptr;
    if (P.fuse_x) {
      if (!recur2_fwd_fuses_x(a.B, a.hp, a.Ip0) || !a.W0 || !a.b0) return cudaErrorInvalidValue;
      if (encode_tmap_2d(&P.tmW0, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.W0, a.Ip0, 4 * hp, (uint64_t)a.Ip0 * 2, 64, 128,
                         CU_TENSOR_MAP_SWIZZLE_128B) ||
          encode_tmap_2d(&P.tmX0, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.X0, a.Ip0, (uint64_t)a.T * a.B,
                         (uint64_t)a.Ip0 * 2, 64, pl.Bc, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
      P.b0 = a.b0;
    } else if (!a.Gx0) {
      return cudaErrorInvalidValue;
    }
    if (!a.a1x || !a.flags) return cudaErrorInvalidValue;
    {
      const uint64_t TB = (uint64_t)a.T * a.B, TB1 = (uint64_t)(a.T + 1) * a.B;
      __half* hs[2] = {a.Hs0, a.Hs1};
      float* cs[2] = {a.C0, a.C1};
      __half* gs[2] = {a.gates0, a.gates1};
      for (int l = 0; l < 2; ++l)
        if (encode_tmap_2d(&P.tmCo[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cs[l], hp, TB, hp * 4, 64, pl.Bc,
                           CU_TENSOR_MAP_SWIZZLE_NONE) ||
            encode_tmap_2d(&P.tmHo[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, hs[l], hp, TB1, hp * 2, 64, pl.Bc,
                           CU_TENSOR_MAP_SWIZZLE_128B) ||
            encode_tmap_2d(&P.tmGo[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, gs[l], 4 * hp, TB, 4 * hp * 2, 256, pl.Bc,
                           CU_TENSOR_MAP_SWIZZLE_NONE))
          return cudaErrorInvalidValue;
    }
    P.region = pl.fuse;
    P.Ag[0] = a.U0;
    P.Ag[1] = a.W1;
    P.Ag[2] = a.U1;
    P.W0g = a.W0;
    P.Ip0 = a.Ip0;
    P.r1_tma = pl.fuse && (size_t)2 * pl.Bc * 1024 <= w2f_fuse_bytes(pl.Bc);
    if (P.r1_tma && encode_tmap_2d(&P.tmG1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.a1x, 4 * hp, (uint64_t)a.T * a.B,
                                   4 * hp * 4, 256, pl.Bc, CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
    if (a.Ht0) {  // recurrent dropout
      if (!a.Ht1 || !a.drop_step) return cudaErrorInvalidValue;
      const uint64_t TB1 = (uint64_t)(a.T + 1) * a.B;
      __half* ht[2] = {a.Ht0, a.Ht1};
      for (int l = 0; l < 2; ++l)
        if (encode_tmap_2d(&P.tmHt[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, ht[l], hp, TB1, hp * 2, 64, pl.Bc,
                           CU_TENSOR_MAP_SWIZZLE_128B))
          return cudaErrorInvalidValue;
      P.drop = 1;
      P.Ht[0] = a.Ht0;
      P.Ht[1] = a.Ht1;
      P.drop_step = a.drop_step;
      P.drop_seed = a.drop_seed;
      P.drop_thr = a.drop_thr;
      P.drop_seq0 = a.drop_seq0;
      P.drop_scale = a.drop_scale;
    }
    cudaError_t e = cudaMemsetAsync(a.flags, 0, (16 * 32 + 16 * 8 * 32) * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    void* args[] = {&P};
    return launch_cluster(recur2f_fn(pl.nci, a.hp, P.drop != 0), dim3(G, 3 * pl.nbg), dim3(256 * pl.cgN),
                          fwd_cl_smem(a.hp, pl.Bc, 8 * pl.cgN) + w2f_drop_bytes(pl.Bc) +
                              (pl.fuse ? w2f_fuse_bytes(pl.Bc) : 0),
                          G, s, args, opt(OPT_FWD_PDL) == 1);
  }
}

}  // namespace hdp

namespace hdp {

// U^T slice in TMEM: all of it needs 64 + 2 h_p <= 512 columns (h_p = 208); at h_p = 256
// (4 h_p / 16 = 64 K-steps) 56 K-steps come from TMEM and 8 from the SMEM copy; everything
// else runs the SMEM-A variant (option wavefront_tmem = 0 forces it)
template <int NC>
const void* recur2b_fn_nk(int hp) {
  // (TMEM-A layout: the accumulators of Bc = 16 NC columns must fit below the slice at column 64)
  if constexpr (NC > 2) {
    return (void)hp, (const void*)recur2_bwd_kernel<NC, 0>;
  } else {
    if (opt(OPT_WAVEFRONT_TMEM) == 0) return (const void*)recur2_bwd_kernel<NC, 0>;
    return 4 * hp / 16 == 52   ? (const void*)recur2_bwd_kernel<NC, 52>
           : 4 * hp / 16 == 64 ? (const void*)recur2_bwd_kernel<NC, 64>
                               : (const void*)recur2_bwd_kernel<NC, 0>;
  }
}
const void* recur2b_fn(int Bc, int hp) {
  return Bc == 16 ? recur2b_fn_nk<1>(hp) : Bc == 32 ? recur2b_fn_nk<2>(hp) : Bc == 48 ? recur2b_fn_nk<3>(hp)
                                                                                        : recur2b_fn_nk<4>(hp);
}

// backward wavefront plan: largest batch-group count whose 3 x G x nbg CTAs are
// co-resident as G-CTA clusters (every role waits on the others); cached per shape
// plan: largest batch-group count whose 3 x G x nbg role CTAs (plus, when wanted,
// the weight-gradient clusters) are co-resident as G-CTA clusters; cached per shape
struct W2BPlan {
  int Bc = 0, nbg = 0, wrows = 0;  // wrows: extra cluster rows of weight-gradient CTAs (0: off)
};
int wgrad_rows(int hp) {
  const int G = (hp + 63) / 64;
  return (wg_tiles(hp) + G - 1) / G;
}
bool plan_w2b(int B, int hp, bool want_wgrad, W2BPlan* out) {
  static std::map<std::tuple<int, int, bool>, W2BPlan> cache;
  auto key = std::make_tuple(B, hp, want_wgrad);
  auto it = cache.find(key);
  if (it == cache.end()) {
    W2BPlan best;
    const int G = (hp + 63) / 64;
    if (B >= 16 && !(B & 15) && !(hp & 15) && G <= 8) {
      for (int nbg = 16; nbg >= 1 && !best.nbg; nbg >>= 1) {
        if (B % nbg) continue;
        const int Bc = B / nbg;
        if ((Bc & 15) || Bc > 64) continue;
        const size_t smem = std::max(bwd_cl_smem(hp, Bc), wgrad_smem());
        if (smem > 227 * 1024) continue;
        const void* fn = recur2b_fn(Bc, hp);
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) break;
        for (int w = want_wgrad ? 1 : 0; w >= 0 && !best.nbg; --w) {
          const int wrows = w ? wgrad_rows(hp) : 0;
          const int rows = 3 * nbg + wrows;
          if (G * rows > 148) continue;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(G, rows);
          cfg.blockDim = dim3(128);
          cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = G;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          int ncl = 0;
          if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess) {
            (void)cudaGetLastError();
            continue;
          }
          if (ncl >= rows) {
            best.Bc = Bc;
            best.nbg = nbg;
            best.wrows = wrows;
          }
        }
      }
    }
    it = cache.emplace(key, best).first;
  }
  *out = it->second;
  return it->second.nbg > 0;
}

bool wgrad_wanted(int Ip0) {
  return opt(OPT_WAVEFRONT_WGRAD) != 0 && Ip0 > 0 && Ip0 <= 256 && !(Ip0 & 15);
}

bool recur2_bwd_supported(int B, int hp) {
  if (opt(OPT_WAVEFRONT) == 0) return false;
  W2BPlan p;
  return plan_w2b(B, hp, false, &p);
}

bool recur2_bwd_wgrad(int B, int hp, int Ip0) {
  if (!recur2_bwd_supported(B, hp) || !wgrad_wanted(Ip0)) return false;
  W2BPlan p;
  return plan_w2b(B, hp, true, &p) && p.wrows > 0;
}

cudaError_t launch_recur2_bwd(const Recur2BwdArgs& a, cudaStream_t s) {
  if (!recur2_bwd_supported(a.B, a.hp)) return cudaErrorInvalidConfiguration;
  const bool wg = a.gW[0] != nullptr;
  if (wg && !recur2_bwd_wgrad(a.B, a.hp, a.Ip0)) return cudaErrorInvalidConfiguration;
  W2BPlan pl;
  if (!plan_w2b(a.B, a.hp, wg, &pl)) return cudaErrorInvalidConfiguration;
  const int Bc = pl.Bc, nbg = pl.nbg;
  const int G = (a.hp + 63) / 64;
  const uint64_t hp = a.hp;
  Bwd2Params P;
  memset(&P, 0, sizeof P);
  if (encode_tmap_2d(&P.tmU[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.U1, hp, 4 * hp, hp * 2, 64, 64,
                     CU_TENSOR_MAP_SWIZZLE_128B) ||
      encode_tmap_2d(&P.tmU[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.U0, hp, 4 * hp, hp * 2, 64, 64,
                     CU_TENSOR_MAP_SWIZZLE_128B) ||
      encode_tmap_2d(&P.tmW1, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.W1, hp, 4 * hp, hp * 2, 64, 64,
                     CU_TENSOR_MAP_SWIZZLE_128B) ||
      encode_tmap_2d(&P.tmA1, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.dA1, 4 * hp, (uint64_t)a.T * a.B, 4 * hp * 2, 64,
                     Bc, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  P.q[0] = {a.dHtop, a.dHtop_last_only, a.gates1, a.C1, a.dA1};
  P.q[1] = {a.dX1, 0, a.gates0, a.C0, a.dA0};
  P.dX1 = a.dX1;
  P.q1done = a.flags;
  P.xdone = a.flags + 16 * 32;
  P.q0done = a.flags + 16 * 32 + 16 * 8 * 32;
  P.T = a.T;
  P.B = a.B;
  P.hp = a.hp;
  P.nbg = nbg;
  if (wg) {
    const uint64_t TB = (uint64_t)a.T * a.B, TB1 = (uint64_t)(a.T + 1) * a.B;
    if (encode_tmap_2d(&P.tmdA[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.dA1, 4 * hp, TB, 4 * hp * 2, 64, 64,
                       CU_TENSOR_MAP_SWIZZLE_128B) ||
        encode_tmap_2d(&P.tmdA[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.dA0, 4 * hp, TB, 4 * hp * 2, 64, 64,
                       CU_TENSOR_MAP_SWIZZLE_128B) ||
        encode_tmap_2d(&P.tmHs[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.Hs1, hp, TB1, hp * 2, 64, 64,
                       CU_TENSOR_MAP_SWIZZLE_128B) ||
        encode_tmap_2d(&P.tmHs[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.Hs0, hp, TB1, hp * 2, 64, 64,
                       CU_TENSOR_MAP_SWIZZLE_128B) ||
        encode_tmap_2d(&P.tmX0, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.X0, a.Ip0, TB, (uint64_t)a.Ip0 * 2, 64, 64,
                       CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    if (a.Ht0) {
      if (encode_tmap_2d(&P.tmHt[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.Ht1, hp, TB1, hp * 2, 64, 64,
                         CU_TENSOR_MAP_SWIZZLE_128B) ||
          encode_tmap_2d(&P.tmHt[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.Ht0, hp, TB1, hp * 2, 64, 64,
                         CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    } else {
      P.tmHt[0] = P.tmHs[0];
      P.tmHt[1] = P.tmHs[1];
    }
    for (int i = 0; i < 4; ++i) P.gW[i] = a.gW[i];
    P.gb[0] = a.gb[0];
    P.gb[1] = a.gb[1];
    P.Ip0 = a.Ip0;
    P.wtiles = wg_tiles(a.hp);
    P.wstages = wgrad_stages(std::max(bwd_cl_smem(a.hp, Bc), wgrad_smem()));
  }
  P.trace = a.trace;
  {
    const __half* gsrc[2] = {a.gates1, a.gates0};
    const float* csrc[2] = {a.C1, a.C0};
    for (int l = 0; l < 2; ++l)
      if (encode_tmap_2d(&P.tmGq[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, gsrc[l], 4 * hp, (uint64_t)a.T * a.B, 4 * hp * 2,
                         256, Bc, CU_TENSOR_MAP_SWIZZLE_NONE) ||
          encode_tmap_2d(&P.tmCq[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, csrc[l], hp, (uint64_t)a.T * a.B, hp * 4, 64, Bc,
                         CU_TENSOR_MAP_SWIZZLE_NONE))
        return cudaErrorInvalidValue;
  }
  if (encode_tmap_2d(&P.tmDXo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.dX1, hp, (uint64_t)a.T * a.B, hp * 4, 64, Bc,
                     CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  if (encode_tmap_2d(&P.tmDX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.dX1, hp, (uint64_t)a.T * a.B, hp * 4, 64, Bc,
                     CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  if (encode_tmap_2d(&P.tmdAo[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.dA1, 4 * hp, (uint64_t)a.T * a.B, 4 * hp * 2, 64,
                     Bc, CU_TENSOR_MAP_SWIZZLE_128B) ||
      encode_tmap_2d(&P.tmdAo[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.dA0, 4 * hp, (uint64_t)a.T * a.B, 4 * hp * 2, 64,
                     Bc, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (a.Ht0) {
    if (!a.Ht1 || !a.drop_step) return cudaErrorInvalidValue;
    P.drop = 1;
    P.drop_step = a.drop_step;
    P.drop_seed = a.drop_seed;
    P.drop_thr = a.drop_thr;
    P.drop_seq0 = a.drop_seq0;
    P.drop_scale = a.drop_scale;
  }
  cudaError_t e = cudaMemsetAsync(a.flags, 0, (2 * 16 * 32 + 16 * 8 * 32) * sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  void* args[] = {&P};
  const int rows = 3 * nbg + (wg ? pl.wrows : 0);
  return launch_cluster(recur2b_fn(Bc, a.hp), dim3(G, rows), dim3(128), std::max(bwd_cl_smem(a.hp, Bc), wgrad_smem()), G,
                        s, args);
}

}  // namespace hdp
