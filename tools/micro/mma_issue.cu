// Microbenchmark: cost of issuing a chain of small tcgen05.mma (M=64, N=16, K=16)
// from (a) one lane inside `if (lane == 0)` vs (b) a warp-uniform loop with
// elect.sync, with 1 or 4 issuing warps.  Prints ns from first issue to the
// commit's mbarrier completion, averaged over reps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1912_00286_b200/csrc/ptx.cuh"
using namespace hdp;

__device__ __forceinline__ uint32_t elect_sync() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
  return pred;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int nk, int nwarps, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;              // 13 x 8 KB  (MN-major A, 64 x 64 per kb)
  uint8_t* sB = sA + 13 * 8192;    // 13 x 2 KB  (K-major B, 16 rows x 128 B)
  uint64_t* barM = reinterpret_cast<uint64_t*>(sB + 13 * 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(barM + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (13 * 8192 + 13 * 2048) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(barM, nwarps); ptx::fence_mbar_init(); }
  ptx::fence_async_smem();
  if (warp == 2) ptx::tmem_alloc(tslot, 128);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t idesc = ptx::idesc_f16_f32(64, 16, 1, 0);
  const uint32_t aA = ptx::smem_u32(sA), aB = ptx::smem_u32(sB);
  unsigned long long tsum = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const unsigned long long t0 = ptx::globaltimer_ns();
    if (warp < nwarps) {
      if (MODE == 0) {
        if (lane == 0) {
          const uint64_t ad0 = ptx::smem_desc_sw128(aA, 8192, 1024), bd0 = ptx::smem_desc_sw128(aB, 0, 1024);
          for (int kk = warp; kk < nk; kk += nwarps) {
            const int kb = kk >> 2, kq = kk & 3;
            const uint64_t ad = ad0 + (uint64_t)((kb * 8192 + kq * 2048) >> 4);
            const uint64_t bd = bd0 + (uint64_t)((kb * 2048 + kq * 32) >> 4);
            ptx::mma_f16(tbase + (kk % 8) * 16, ad, bd, idesc, kk >= 8 ? 1u : 0u);
          }
          ptx::mma_commit(barM);
        }
      } else {
        const uint64_t ad0 = ptx::smem_desc_sw128(aA, 8192, 1024), bd0 = ptx::smem_desc_sw128(aB, 0, 1024);
        for (int kk = warp; kk < nk; kk += nwarps) {
          const int kb = kk >> 2, kq = kk & 3;
          const uint64_t ad = ad0 + (uint64_t)((kb * 8192 + kq * 2048) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((kb * 2048 + kq * 32) >> 4);
          if (elect_sync()) ptx::mma_f16(tbase + (kk % 8) * 16, ad, bd, idesc, kk >= 8 ? 1u : 0u);
        }
        if (elect_sync()) ptx::mma_commit(barM);
      }
      __syncwarp();
    }
    ptx::mbar_wait(barM, r & 1);
    ptx::tc_fence_after();
    const unsigned long long t1 = ptx::globaltimer_ns();
    tsum += t1 - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tsum / reps;
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 128); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  const int smem = 13 * 8192 + 13 * 2048 + 2048;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 1; ++mode)
    for (int nw : {1, 2, 4, 8, 16})
      for (int nk : {13, 26, 52}) {
        if (mode == 0) k<0><<<1, 512, smem>>>(nk, nw, 200, d); else k<1><<<1, 512, smem>>>(nk, nw, 200, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %s warps %d mmas %2d : %llu ns (%s)\n", mode ? "elect-uniform" : "lane0-branch", nw, nk, h, cudaGetErrorString(e));
      }
  return 0;
}
