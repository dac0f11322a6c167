// Correctness + timing of tcgen05.mma with the A operand in TMEM (".ts"):
// D[128 x 16] = A[128 x K] * B[16 x K]^T, K = 208, fp16 -> fp32.
// A is written to TMEM by tcgen05.st (lane i = row i, 2 fp16 per 32-bit column);
// B is K-major SWIZZLE_128B in shared memory (built by hand).  Compared with
// a host reference; also times 26 MMAs (2 x 13 K-steps) SS vs TS.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../../paper_1912_00286_b200/csrc/ptx.cuh"
using namespace hdp;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                  "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}

constexpr int M = 128, N = 16, K = 208, NK = K / 16, KB = (K + 63) / 64;  // (M=64 modes use rows 0..63)

// A: row-major [M][K] fp16; B: row-major [N][K] fp16
__global__ void __launch_bounds__(128, 1) k(const __half* A, const __half* B, float* D, int mode, int reps,
                                          unsigned long long* tout) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // KB x 16 KB : K-major SW128, 128 rows x 128 B per k-block
  uint8_t* sB = sA + KB * 16384;      // KB x 2 KB  : 16 rows x 128 B per k-block
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + KB * 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // manual SW128 K-major fill: element (r, k) of a k-block at row r, byte (k%64)*2,
  // 16-B chunk c = (k%64)/8 stored at chunk c ^ (r & 7)
  for (int i = threadIdx.x; i < M * KB * 64; i += blockDim.x) {
    const int r = i / (KB * 64), kk = i % (KB * 64), kb = kk / 64, kc = kk % 64;
    const __half v = kk < K ? A[r * K + kk] : __float2half(0.f);
    const int c = kc / 8, e = kc % 8;
    *reinterpret_cast<__half*>(sA + kb * 16384 + r * 128 + ((c ^ (r & 7)) << 4) + e * 2) = v;
  }
  for (int i = threadIdx.x; i < N * KB * 64; i += blockDim.x) {
    const int r = i / (KB * 64), kk = i % (KB * 64), kb = kk / 64, kc = kk % 64;
    const __half v = kk < K ? B[r * K + kk] : __float2half(0.f);
    const int c = kc / 8, e = kc % 8;
    *reinterpret_cast<__half*>(sB + kb * 2048 + r * 128 + ((c ^ (r & 7)) << 4) + e * 2) = v;
  }
  ptx::fence_async_smem();
  if (threadIdx.x == 0) { ptx::mbar_init(bar, (mode == 2 || mode == 3) ? 4 : 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(tslot, 256);
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t tbase = *tslot;                 // cols [0,16): D ; [128, 128+K/2): A
  const uint32_t tA = tbase + 128;
  // A rows into TMEM: thread = row (lane quadrant = warp), 2 fp16 per column
  // mode 6: M=64 with row 16q+i placed in lane 32q+i (the M=64 accumulator layout)
  {
    int r = warp * 32 + lane;
    if (mode == 6) r = (lane < 16) ? warp * 16 + lane : 1000;  // lanes 16..31 of each quadrant unused
    for (int c0 = 0; c0 < (K / 2 + 15) / 16 * 16; c0 += 16) {
      uint32_t v[16];
      for (int j = 0; j < 16; ++j) {
        const int kk = 2 * (c0 + j);
        const bool okr = r < M;
        const __half lo = (okr && kk < K) ? A[r * K + kk] : __float2half(0.f);
        const __half hi = (okr && kk + 1 < K) ? A[r * K + kk + 1] : __float2half(0.f);
        v[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tmem_st16(tA + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
    }
    tmem_st_wait();
  }
  ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
  const uint32_t idesc = ptx::idesc_f16_f32(mode >= 4 ? 64 : M, N, 0, 0);
  unsigned long long tsum = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncthreads();
    const unsigned long long t0 = ptx::globaltimer_ns();
    const int nis = (mode == 2 || mode == 3) ? 4 : 1;      // issuing warps (each its own accumulator set)
    const int halves = (mode == 2 || mode == 3) ? 2 : 1;   // 2 x M=128 (the forward's 256 gate rows: A reused)
    if (lane == 0 && warp < nis) {
      for (int s = warp; s < NK; s += nis) {
        const int kb = s / 4, kq = s % 4;
        const uint64_t bd = ptx::smem_desc_sw128(ptx::smem_u32(sB) + kb * 2048 + kq * 32, 0, 1024);
        for (int h2 = 0; h2 < halves; ++h2) {
          const uint32_t dacc = tbase + (h2 * 4 + (nis > 1 ? warp : 0)) * 16;
          const uint32_t acc = s >= nis;
          if (mode == 0 || mode == 2 || mode == 4) {
            const uint64_t ad = ptx::smem_desc_sw128(ptx::smem_u32(sA) + kb * 16384 + kq * 32, 0, 1024);
            ptx::mma_f16(dacc, ad, bd, idesc, acc);
          } else {
            mma_ts(dacc, tA + s * 8, bd, idesc, acc);
          }
        }
      }
      ptx::mma_commit(bar);
    }
    __syncwarp();
    ptx::mbar_wait(bar, rep & 1);
    ptx::tc_fence_after();
    tsum += ptx::globaltimer_ns() - t0;
  }
  float v[16];
  ptx::tmem_ld16(tbase + (static_cast<uint32_t>(warp * 32) << 16), v);
  if (mode >= 4) {
    if (lane < 16) for (int j = 0; j < 16; ++j) D[(warp * 16 + lane) * N + j] = v[j];
  } else {
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + j] = v[j];
  }
  if (threadIdx.x == 0) *tout = tsum / reps;
  ptx::tc_fence_before(); __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 256); }
}

int main() {
  std::vector<__half> hA(M * K), hB(N * K);
  std::vector<double> ref(M * N, 0.0);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2half(((i * 37) % 101 - 50) / 64.f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2half(((i * 53) % 97 - 48) / 64.f);
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) for (int kk = 0; kk < K; ++kk)
    ref[m * N + n] += (double)__half2float(hA[m * K + kk]) * __half2float(hB[n * K + kk]);
  __half *dA, *dB; float* dD; unsigned long long* dt;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dt, 8);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = KB * 16384 + KB * 2048 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 7; ++mode) {
    cudaMemset(dD, 0, M * N * 4);
    k<<<1, 128, smem>>>(dA, dB, dD, mode, 200, dt);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> hD(M * N); unsigned long long t = 0;
    cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&t, dt, 8, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    const int rows = mode >= 4 ? 64 : M;
    for (int i = 0; i < rows * N; ++i) { err = fmax(err, fabs(hD[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); }
    const char* names[7] = {"SS 1 issuer", "TS 1 issuer", "SS 4 issuers x 2 halves", "TS 4 issuers x 2 halves",
                            "SS M=64", "TS M=64 row i->lane i", "TS M=64 row 16q+i->lane 32q+i"};
    printf("mode %s: %s  max err %.3e (max |ref| %.3e)  %d MMAs in %llu ns\n", names[mode],
           cudaGetErrorString(e), (mode == 2 || mode == 3) ? -1.0 : err, mx, NK * ((mode == 2 || mode == 3) ? 2 : 1), t);
  }
  return 0;
}
