// Latency of the recurrence kernels' per-step hand-off: a cp.async.bulk copy of S bytes
// from one CTA's shared memory into a cluster peer's shared memory, completing on the
// peer's mbarrier (complete_tx), observed by the peer's mbar wait.  Two CTAs of a
// G-CTA cluster ping-pong R times; one hop = total time / R.  Also the bare
// remote mbarrier arrive -> wait hop (no payload).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 push_rt.cu -o push_rt
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1912_00286_b200/csrc/ptx.cuh"
using namespace hdp;

template <int MODE>  // 0: bulk copy to the partner; 2: remote arrive only
__global__ void __launch_bounds__(128, 1) pingpong(int reps, int bytes, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* src = buf;                 // [bytes]
  uint8_t* dst = buf + 16384;         // [G][bytes/G...] landing zone (peers write here)
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 2 * 16384);
  const uint32_t me = ptx::cluster_ctarank();
  const uint32_t G = gridDim.x;
  const uint32_t partner = me ^ 1u;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(src)[i] = i;
  // the receiver's mbarrier counts one arrival (its own expect_tx) per round; the bytes of
  // the sender's copy complete it
  (void)G;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, MODE == 2 ? 2 : 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_async_smem();
  __syncthreads();
  ptx::cluster_arrive();
  ptx::cluster_wait();
  if (me > 1) {  // bystanders: only the cluster shape of the real kernels
    ptx::cluster_arrive();
    ptx::cluster_wait();
    return;
  }
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) {
    if (MODE != 2) ptx::mbar_arrive_expect_tx(bar, bytes);  // arm round 0
    t0 = ptx::globaltimer_ns();
    for (int r = 0; r < reps; ++r) {
      const bool my_turn = ((r & 1) == (int)me);
      if (my_turn) {
        if (MODE == 2) {
          ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(bar), partner));
        } else {
          ptx::bulk_copy_to_peer(ptx::mapa(ptx::smem_u32(dst), partner), ptx::smem_u32(src), bytes,
                                 ptx::mapa(ptx::smem_u32(bar), partner));
        }
      } else {
        if (MODE == 2) {
          ptx::mbar_arrive(bar);           // my own arrival; the partner's remote one completes the phase
          ptx::mbar_wait_cluster(bar, (r >> 1) & 1);
        } else {
          ptx::mbar_wait(bar, (r >> 1) & 1);
          if (r + 2 < reps) ptx::mbar_arrive_expect_tx(bar, bytes);  // arm my next receive
        }
      }
    }
    out[me] = (ptx::globaltimer_ns() - t0) / reps;  // = one hop
  }
  ptx::cluster_arrive();
  ptx::cluster_wait();
}

template <int MODE>
void run(const char* name, int G, int bytes, unsigned long long* d) {
  const int smem = 2 * 16384 + 1024 + 64;
  cudaFuncSetAttribute(pingpong<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (G > 8) cudaFuncSetAttribute(pingpong<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int reps = 2000;
  void* args[] = {&reps, &bytes, &d};
  cudaError_t e = cudaLaunchKernelExC(&cfg, (const void*)pingpong<MODE>, args);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("{\"case\": \"%s\", \"cluster\": %d, \"bytes\": %d, \"hop_ns\": %llu, \"status\": \"%s\"}\n", name, G, bytes,
         (h[0] + h[1]) / 2, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  run<2>("remote mbarrier arrive (no payload)", 2, 0, d);
  for (int b : {2048, 8192, 16384}) run<0>("bulk copy to one peer", 4, b, d);
  run<0>("bulk copy to one peer", 2, 8192, d);
  return 0;
}
