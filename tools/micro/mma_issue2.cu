// Issue-cost microbenchmark: 13 / 26 / 52 tcgen05.mma (M=128, N=16, K=16, SS) from ONE warp:
//  mode 0: `if (lane == 0)` loop (divergent issue, descriptors in regular registers)
//  mode 1: warp-uniform loop from 0, elect.sync around the MMA only
//  mode 2: mode 1 with the trip count a template constant (fully unrolled)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1912_00286_b200/csrc/ptx.cuh"
using namespace hdp;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <int MODE, int NKT>
__global__ void __launch_bounds__(128, 1) k(int nk, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint64_t* barM = reinterpret_cast<uint64_t*>(smem + 7 * 16384 + 7 * 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(barM + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (7 * 16384 + 7 * 2048) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(barM, 1); ptx::fence_mbar_init(); }
  ptx::fence_async_smem();
  if (warp == 2) ptx::tmem_alloc(tslot, 128);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t idesc = ptx::idesc_f16_f32(128, 16, 0, 0);
  const uint32_t aA = ptx::smem_u32(smem), aB = aA + 7 * 16384;
  unsigned long long tsum = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const unsigned long long t0 = ptx::globaltimer_ns();
    if (warp == 0) {
      const uint64_t ad0 = ptx::smem_desc_sw128(aA, 0, 1024), bd0 = ptx::smem_desc_sw128(aB, 0, 1024);
      if (MODE == 0) {
        if (lane == 0) {
          for (int kk = 0; kk < nk; ++kk) {
            const int kb = (kk >> 2) % 7, kq = kk & 3;
            ptx::mma_f16(tbase + (kk & 3) * 16, ad0 + (uint64_t)((kb * 16384 + kq * 32) >> 4),
                         bd0 + (uint64_t)((kb * 2048 + kq * 32) >> 4), idesc, kk >= 4 ? 1u : 0u);
          }
          ptx::mma_commit(barM);
        }
      } else if (MODE == 1) {
        for (int kk = 0; kk < nk; ++kk) {
          const int kb = (kk >> 2) % 7, kq = kk & 3;
          const uint64_t ad = ad0 + (uint64_t)((kb * 16384 + kq * 32) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((kb * 2048 + kq * 32) >> 4);
          if (elect_one()) ptx::mma_f16(tbase + (kk & 3) * 16, ad, bd, idesc, kk >= 4 ? 1u : 0u);
          __syncwarp();
        }
        if (elect_one()) ptx::mma_commit(barM);
      } else {
#pragma unroll
        for (int kk = 0; kk < NKT; ++kk) {
          const int kb = (kk >> 2) % 7, kq = kk & 3;
          const uint64_t ad = ad0 + (uint64_t)((kb * 16384 + kq * 32) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((kb * 2048 + kq * 32) >> 4);
          if (elect_one()) ptx::mma_f16(tbase + (kk & 3) * 16, ad, bd, idesc, kk >= 4 ? 1u : 0u);
          __syncwarp();
        }
        if (elect_one()) ptx::mma_commit(barM);
      }
      __syncwarp();
    }
    ptx::mbar_wait(barM, r & 1);
    ptx::tc_fence_after();
    tsum += ptx::globaltimer_ns() - t0;
  }
  if (threadIdx.x == 0) out[0] = tsum / reps;
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 2) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 128); }
}

template <int MODE, int NKT>
void run(const char* name, int nk, unsigned long long* d) {
  const int smem = 7 * 16384 + 7 * 2048 + 2048;
  cudaFuncSetAttribute(k<MODE, NKT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE, NKT><<<1, 128, smem>>>(nk, 200, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-34s mmas %2d : %5llu ns (%s)\n", name, nk, h, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  for (int nk : {13, 26, 52}) run<0, 1>("lane0 branch", nk, d);
  for (int nk : {13, 26, 52}) run<1, 1>("uniform loop + elect", nk, d);
  run<2, 13>("uniform unrolled + elect", 13, d);
  run<2, 26>("uniform unrolled + elect", 26, d);
  run<2, 52>("uniform unrolled + elect", 52, d);
  return 0;
}
