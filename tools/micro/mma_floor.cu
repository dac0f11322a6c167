// Throughput floor of small tcgen05.mma chains (N = 16, K = 16 per MMA):
// NK MMAs split over NW issuing warps (warp-uniform, unrolled, elect.sync),
// accumulators k % 8, A from SMEM (SS) or TMEM (TS), M = 64 or 128.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1912_00286_b200/csrc/ptx.cuh"
using namespace hdp;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}

template <int M, int TS, int NK, int W, int NW>
__device__ __forceinline__ void issue(uint32_t tbase, uint32_t aA, uint32_t aB, uint32_t idesc, uint64_t* bar) {
  const uint64_t ad0 = ptx::smem_desc_sw128(aA, 0, 1024), bd0 = ptx::smem_desc_sw128(aB, 0, 1024);
#pragma unroll
  for (int k = W; k < NK; k += NW) {
    const int kb = (k >> 2) % 4, kq = k & 3;
    const uint64_t bd = bd0 + (uint64_t)((kb * 2048 + kq * 32) >> 4);
    if (ptx::elect_one_sync()) {
      if (TS) mma_ts(tbase + (k % 8) * 16, tbase + 256 + (k % 26) * 8, bd, idesc, k >= 8);
      else ptx::mma_f16(tbase + (k % 8) * 16, ad0 + (uint64_t)((kb * (M * 128) + kq * 32) >> 4), bd, idesc, k >= 8);
    }
  }
  if (ptx::elect_one_sync()) ptx::mma_commit(bar);
  __syncwarp();
}

template <int M, int TS, int NK, int NW>
__global__ void __launch_bounds__(256, 1) k(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem; uint8_t* sB = sA + 4 * M * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + 4 * 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (4 * M * 128 + 4 * 2048) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { ptx::mbar_init(bar, NW); ptx::fence_mbar_init(); }
  ptx::fence_async_smem();
  if (warp == 0) ptx::tmem_alloc(tslot, 512);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t idesc = ptx::idesc_f16_f32(M, 16, 0, 0);
  unsigned long long tsum = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const unsigned long long t0 = ptx::globaltimer_ns();
    if (warp < NW) {
      const uint32_t aA = ptx::smem_u32(sA), aB = ptx::smem_u32(sB);
      switch (warp) {
        case 0: issue<M, TS, NK, 0, NW>(tbase, aA, aB, idesc, bar); break;
        case 1: if (NW > 1) issue<M, TS, NK, 1, NW>(tbase, aA, aB, idesc, bar); break;
        case 2: if (NW > 2) issue<M, TS, NK, 2, NW>(tbase, aA, aB, idesc, bar); break;
        case 3: if (NW > 3) issue<M, TS, NK, 3, NW>(tbase, aA, aB, idesc, bar); break;
        case 4: if (NW > 4) issue<M, TS, NK, 4, NW>(tbase, aA, aB, idesc, bar); break;
        case 5: if (NW > 5) issue<M, TS, NK, 5, NW>(tbase, aA, aB, idesc, bar); break;
        case 6: if (NW > 6) issue<M, TS, NK, 6, NW>(tbase, aA, aB, idesc, bar); break;
        default: if (NW > 7) issue<M, TS, NK, 7, NW>(tbase, aA, aB, idesc, bar); break;
      }
    }
    ptx::mbar_wait(bar, r & 1);
    ptx::tc_fence_after();
    tsum += ptx::globaltimer_ns() - t0;
  }
  if (threadIdx.x == 0) out[0] = tsum / reps;
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 512); }
}

template <int M, int TS, int NK, int NW>
void run(unsigned long long* d) {
  const int smem = 4 * M * 128 + 4 * 2048 + 2048;
  cudaFuncSetAttribute(k<M, TS, NK, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<M, TS, NK, NW><<<1, 256, smem>>>(200, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("M=%3d %s NK=%2d issuers=%d : %5llu ns  (%s)\n", M, TS ? "TS" : "SS", NK, NW, h, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  run<64, 0, 52, 1>(d); run<64, 0, 52, 4>(d); run<64, 0, 52, 8>(d);
  run<64, 1, 52, 1>(d); run<64, 1, 52, 2>(d); run<64, 1, 52, 4>(d); run<64, 1, 52, 8>(d);
  run<128, 0, 26, 1>(d); run<128, 0, 26, 2>(d); run<128, 0, 26, 4>(d);
  run<128, 1, 26, 1>(d); run<128, 1, 26, 2>(d); run<128, 1, 26, 4>(d);
  run<128, 0, 52, 4>(d); run<128, 1, 52, 4>(d); run<128, 1, 52, 8>(d);
  return 0;
}
