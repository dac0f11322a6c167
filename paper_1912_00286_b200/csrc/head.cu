// Fused FC head (A4 + A5 except the dF GEMM): one launch per forward replaces the FC GEMM,
// head_out, loss_final, the head's column reductions (colreduce3 pass 1) and the
// dH_top = dz F GEMM of the backward.
//
// Per 128-row tile (one CTA; row r = t * B + b, PAPER.md:171 per-step loss):
//   z   = fp16(relu(H F^T + fb))                          R7   (tcgen05, TMEM accumulator)
//   y   = sum_j wo_j z_j + bo                             fp32
//   dy  = -alpha t / rows  if 1 - t y > 0, else 0         (hinge, subgradient 0 at the kink; Q5)
//   dz  = fp16(dy wo_j) where z_j > 0, else 0             R9
//   dH  = dz F                                            fp32 (tcgen05; F re-read MN-major from
//                                                         the same shared-memory bytes)
//   column sums over the tile's rows of dy z_j (dwo), dz_j (dfb), dy (dbo) and the hinge
//   -> per-CTA partials; the last CTA to finish sums the hinge partials into the loss.
// The per-CTA column partials are fp64 [grid][2 Fp + 1] in the layout of the column
// reduction's pass 1, so the backward finishes them with the same fixed-order pass 2.
//
// Warp roles (320 threads): warp 0 lane 0 TMA + MMA issue; warp 1 TMEM allocation (512
// columns: z accumulator at 0, dH accumulator at 256); warps 2..9 epilogue, warp w owns
// TMEM lane quadrant w % 4 = tile rows 32 (w % 4) .. +32, one row per thread, and one
// half of the columns (8 warps: two per SM sub-partition, the latency-bound element math
// of 4 warps measured 26 us per launch at C2).
#include <cuda_fp16.h>

#include <cstdio>

#include "gemm.cuh"
#include "head.cuh"
#include "ptx.cuh"

namespace hdp {
namespace {

constexpr int HM = 128;                 // rows per CTA
constexpr int KB_BYTES = HM * 128;      // one 64-wide K block of a 128-row SW128 tile
constexpr int EPI_LD = 36;              // fp32 staging row stride (conflict-free float4 rows)

struct HeadSmem {
  static constexpr int TILE = 4 * KB_BYTES;             // H tile, later the dz tile (64 KB)
  static constexpr int F_MAX = 4 * 256 * 128;            // F: 4 K blocks x Fp rows x 128 B
  static constexpr int VEC = 2 * 256 * 4;                // fb, wo as fp32
  static constexpr int YP = 2 * HM * 4;                  // the two column halves' partial y
  static constexpr int RED = 4 * 2 * 256 * 4 + 16 * 4;   // per-quadrant column sums [4][2][256] + scalars [4][2]
  static constexpr int BARS = 64;                        // 4 mbarriers + the TMEM slot
  static constexpr int BYTES = 1024 + TILE + F_MAX + VEC + YP + RED + BARS;
  static_assert(8 * 32 * EPI_LD * 4 <= F_MAX / 2, "dH staging fits in F's bytes");
};

__device__ __forceinline__ float h2f(uint16_t b) { return __half2float(__ushort_as_half(b)); }

// Column sums over the warp's 32 rows: on entry v[k] is this lane's (row's) value of column
// k of a 32-column group; on exit v[0] holds the warp sum of column `lane` (a fixed binary
// tree: deterministic).
__device__ __forceinline__ void transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int k = 0; k < m; ++k) {
      const float send = up ? v[k] : v[k + m];
      const float keep = up ? v[k + m] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__global__ void __launch_bounds__(320, 1)
    head_fused_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmF,
                      const __grid_constant__ CUtensorMap tmDz, HeadFusedArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sT = base;                                   // H tile, then dz tile
  uint8_t* sF = sT + HeadSmem::TILE;
  float* sfb = reinterpret_cast<float*>(sF + HeadSmem::F_MAX);
  float* swo = sfb + 256;
  float* ypart = swo + 256;                             // [2][128]
  float* red = ypart + 2 * HM;                          // [4 quadrants][2][256]: dy z | dz
  float* scal = red + 4 * 2 * 256;                      // [4 quadrants][2]: dy, hinge
  uint64_t* bars = reinterpret_cast<uint64_t*>(scal + 16);
  uint64_t* bar_ld = bars;       // TMA of H and F landed
  uint64_t* bar_z = bars + 1;    // z accumulator complete
  uint64_t* bar_dz = bars + 2;   // dz tile written (4 epilogue warps)
  uint64_t* bar_h = bars + 3;    // dH accumulator complete
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hp = a.hp, Fp = a.Fp;
  const int m0 = blockIdx.x * HM;
  const int nkH = (hp + 63) / 64, nkF = (Fp + 63) / 64;  // 64-wide K blocks of the two MMAs

  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tmH);
    ptx::tma_prefetch(&tmF);
    ptx::tma_prefetch(&tmDz);
    ptx::mbar_init(bar_ld, 1);
    ptx::mbar_init(bar_z, 1);
    ptx::mbar_init(bar_dz, 8);
    ptx::mbar_init(bar_h, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tslot, 512);
  // output-layer vectors as fp32 (broadcast reads in the epilogue)
  for (int j = threadIdx.x; j < 256; j += blockDim.x) {
    sfb[j] = j < Fp ? h2f(reinterpret_cast<const uint16_t*>(a.fb)[j]) : 0.f;
    swo[j] = j < Fp ? h2f(reinterpret_cast<const uint16_t*>(a.wo)[j]) : 0.f;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tZ = tbase, tD = tbase + 256;
  unsigned long long* tr = a.trace ? a.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = ptx::globaltimer_ns();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA: H tile (K-major A) and all of F (K-major B of z = H F^T)
      ptx::mbar_arrive_expect_tx(bar_ld, nkH * (KB_BYTES + Fp * 128));
      for (int kb = 0; kb < nkH; ++kb) ptx::tma_load_2d(sF + kb * Fp * 128, &tmF, bar_ld, kb * 64, 0);
      // (PDL) only H is the previous kernel's output: F and the setup above overlap its tail;
      // everything else this launch reads was written before the forward began
      ptx::griddep_wait();
      for (int kb = 0; kb < nkH; ++kb) ptx::tma_load_2d(sT + kb * KB_BYTES, &tmH, bar_ld, kb * 64, m0);
      // ---------------- z = H F^T: M = 128, N = Fp, K = hp
      ptx::mbar_wait(bar_ld, 0);
      ptx::tc_fence_after();
      if (tr) tr[1] = ptx::globaltimer_ns();
      const uint32_t idz = ptx::idesc_f16_f32(HM, Fp, 0, 0);
      const uint32_t aT = ptx::smem_u32(sT), aF = ptx::smem_u32(sF);
      for (int kb = 0; kb < nkH; ++kb)
        for (int k = 0; k < 4 && kb * 64 + k * 16 < hp; ++k)
          ptx::mma_f16(tZ, ptx::smem_desc_sw128(aT + kb * KB_BYTES + k * 32, 0, 1024),
                       ptx::smem_desc_sw128(aF + kb * Fp * 128 + k * 32, 0, 1024), idz, (kb | k) ? 1u : 0u);
      ptx::mma_commit(bar_z);
      // ---------------- dH = dz F: M = 128, N = hp, K = Fp.  A = the dz tile (K-major, same
      // SW128 layout as H), B = F read MN-major: row j of F's K block i is K-row j of the
      // 64-wide N atom i (LBO = Fp * 128 B between atoms, SBO = 1024 B per 8 K-rows)
      ptx::mbar_wait(bar_dz, 0);
      ptx::tc_fence_after();
      const uint32_t idh = ptx::idesc_f16_f32(HM, hp, 0, 1);
      for (int kb = 0; kb < nkF; ++kb)
        for (int k = 0; k < 4 && kb * 64 + k * 16 < Fp; ++k)
          ptx::mma_f16(tD, ptx::smem_desc_sw128(aT + kb * KB_BYTES + k * 32, 0, 1024),
                       ptx::smem_desc_sw128(aF + (kb * 64 + k * 16) * 128, (uint32_t)Fp * 128, 1024), idh,
                       (kb | k) ? 1u : 0u);
      ptx::mma_commit(bar_h);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: one tile row per thread; the two warps of a lane quadrant
    // split the columns by 32-wide groups (half 0: the first ceil(n/2) groups)
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int te = (warp - 2) * 32 + lane;  // 0..255
    const int rl = q * 32 + lane;
    const int m = m0 + rl;
    const bool valid = m < a.rows;
    const uint32_t tq = static_cast<uint32_t>(q * 32) << 16;
    const int ngz = (Fp + 31) / 32, ngh = (hp + 31) / 32;
    const int gz0 = half ? (ngz + 1) / 2 : 0, gz1 = half ? ngz : (ngz + 1) / 2;
    const int gh0 = half ? (ngh + 1) / 2 : 0, gh1 = half ? ngh : (ngh + 1) / 2;
    float alpha = a.alpha;
    if (a.alpha_dev) alpha = *a.alpha_dev;
    int8_t tv = 0;
    if (valid) tv = a.tgt[(long)(m % a.B) * a.T + m / a.B];
    const float bo = h2f(*reinterpret_cast<const uint16_t*>(a.bo));
    ptx::mbar_wait(bar_z, 0);
    ptx::tc_fence_after();
    if (tr && te == 0) tr[2] = ptx::globaltimer_ns();
    // pass 1: y (this half's columns, then the two halves in order)
    float acc = 0.f;
    for (int c = gz0 * 32; c < gz1 * 32 && c < Fp; c += 16) {
      float v[16];
      ptx::tmem_ld16(tZ + tq + c, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float z = __half2float(__float2half_rn(fmaxf(v[j] + sfb[c + j], 0.f)));  // R7
        acc = fmaf(z, swo[c + j], acc);
      }
    }
    ypart[half * HM + rl] = acc;
    asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 epilogue warps
    if (tr && te == 0) tr[3] = ptx::globaltimer_ns();
    const float yy = (ypart[rl] + ypart[HM + rl]) + bo;
    const float tf = (float)tv;
    const float margin = 1.f - tf * yy;
    const float dyr = valid && margin > 0.f ? -alpha * tf * a.inv_terms : 0.f;
    const float hinge = valid && margin > 0.f ? margin : 0.f;
    if (valid && half == 0) {
      a.y[m] = yy;
      a.dy[m] = dyr;
    }
    // pass 2: dz into the (now free) H tile's bytes + the column sums of dy z and dz
    float* rw = red + q * 2 * 256;
    for (int g = gz0 * 32; g < gz1 * 32; g += 32) {
      float v[32];
      ptx::tmem_ld16_nowait(tZ + tq + g, *reinterpret_cast<float(*)[16]>(v));
      ptx::tmem_ld16_nowait(tZ + tq + g + 16, *reinterpret_cast<float(*)[16]>(v + 16));
      ptx::tmem_wait_ld();
      float zd[32], dzf[32];
      __align__(16) uint16_t hz[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = g + j;
        const float z = __half2float(__float2half_rn(fmaxf(v[j] + sfb[col & 255], 0.f)));
        const __half d = __float2half_rn(z > 0.f ? dyr * swo[col & 255] : 0.f);  // R9
        const bool in = valid && col < Fp;
        hz[j] = in ? __half_as_ushort(d) : (uint16_t)0;
        zd[j] = in ? z * dyr : 0.f;
        dzf[j] = in ? __half2float(d) : 0.f;
      }
      // 4 16-byte chunks into the SW128 tile: K block g / 64, chunk (g % 64) / 8 + i
      uint8_t* rowp = sT + (g >> 6) * KB_BYTES + rl * 128;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ch = ((g & 63) >> 3) + i;
        *reinterpret_cast<uint4*>(rowp + ((ch ^ (rl & 7)) << 4)) = reinterpret_cast<const uint4*>(hz)[i];
      }
      transpose_reduce32(zd, lane);
      transpose_reduce32(dzf, lane);
      if (g + lane < Fp) {
        rw[g + lane] = zd[0];
        rw[256 + g + lane] = dzf[0];
      }
    }
    // dz tile -> async proxy (MMA, TMA store), then hand it to the MMA issuer
    ptx::fence_async_smem();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(bar_dz);
    if (half == 0) {
      const float sdy = warp_sum(dyr), sh = warp_sum(hinge);
      if (lane == 0) {
        scal[q * 2] = sdy;
        scal[q * 2 + 1] = sh;
      }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (tr && te == 0) tr[4] = ptx::globaltimer_ns();
    // dz tile -> global (clipped to [rows][Fp] by the tensor map)
    if (te == 0) {
      for (int kb = 0; kb < nkF; ++kb) ptx::tma_store_2d(&tmDz, sT + kb * KB_BYTES, kb * 64, m0);
      ptx::bulk_commit_group();
    }
    // per-CTA partials: lane quadrants in fixed order 0..3, fp64 across them
    const int ncol = 2 * Fp + 1;
    double* cp = a.colpart + (size_t)blockIdx.x * ncol;
    for (int col = te; col < ncol; col += 256) {
      double sum = 0.0;
      if (col < 2 * Fp) {
        const int off = col < Fp ? col : 256 + col - Fp;
#pragma unroll
        for (int w = 0; w < 4; ++w) sum += (double)red[w * 2 * 256 + off];
      } else {
#pragma unroll
        for (int w = 0; w < 4; ++w) sum += (double)scal[w * 2];
      }
      cp[col] = sum;
    }
    if (te == 32) {
      a.hinge[blockIdx.x] = ((scal[1] + scal[3]) + scal[5]) + scal[7];
      __threadfence();
    }
    // pass 3: dH rows through a 32 x 32 staging block per warp (coalesced 128-B rows); the
    // staging lives in F's bytes, free once the dH MMA (its last reader) completed
    ptx::mbar_wait(bar_h, 0);
    ptx::tc_fence_after();
    if (tr && te == 0) tr[5] = ptx::globaltimer_ns();
    float* st = reinterpret_cast<float*>(sF) + (warp - 2) * 32 * EPI_LD;
    for (int c = gh0 * 32; c < gh1 * 32; c += 32) {
      float v[32];
      ptx::tmem_ld16_nowait(tD + tq + c, *reinterpret_cast<float(*)[16]>(v));
      ptx::tmem_ld16_nowait(tD + tq + c + 16, *reinterpret_cast<float(*)[16]>(v + 16));
      ptx::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(st + lane * EPI_LD + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = i * 4 + (lane >> 3), cc = (lane & 7) * 4;
        const int mr = m0 + q * 32 + r, n = c + cc;
        if (mr < a.rows && n < hp)  // hp is a multiple of 8: whole float4s
          *reinterpret_cast<float4*>(a.dH + (size_t)mr * hp + n) =
              *reinterpret_cast<const float4*>(st + r * EPI_LD + cc);
      }
      __syncwarp();
    }
    if (tr && te == 0) tr[6] = ptx::globaltimer_ns();
    if (te == 0) ptx::bulk_wait_group_read0();  // dz tile read before exit
  }
  // ---------------- last CTA: the loss (hinge partials in CTA order, fp64)
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {  // (block-uniform) all threads: lane-strided loads, fixed-order fp64 tree
    __threadfence();
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += (double)__ldcg(a.hinge + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    double* wsum = reinterpret_cast<double*>(red);  // (the column sums are written out)
    if (lane == 0) wsum[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 10; ++w) t += wsum[w];
      *a.loss = (float)t * a.inv_terms;
      *a.ticket = 0u;
    }
  }
  if (tr && threadIdx.x == 0) tr[7] = ptx::globaltimer_ns();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

}  // namespace

bool head_fused_supported(int hp, int Fp) {
  return hp >= 16 && Fp >= 16 && hp <= 256 && Fp <= 256 && (hp % 16) == 0 && (Fp % 16) == 0;
}

int head_fused_grid(int rows) { return (rows + HM - 1) / HM; }

cudaError_t launch_head_fused(const HeadFusedArgs& a, cudaStream_t s) {
  if (!head_fused_supported(a.hp, a.Fp) || a.rows <= 0) return cudaErrorInvalidValue;
  CUtensorMap mH, mF, mDz;
  if (encode_tmap_2d(&mH, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.H, a.hp, a.rows, (uint64_t)a.hp * 2, 64, HM,
                     CU_TENSOR_MAP_SWIZZLE_128B) ||
      encode_tmap_2d(&mF, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.F, a.hp, a.Fp, (uint64_t)a.hp * 2, 64, a.Fp,
                     CU_TENSOR_MAP_SWIZZLE_128B) ||
      encode_tmap_2d(&mDz, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.dz, a.Fp, a.rows, (uint64_t)a.Fp * 2, 64, HM,
                     CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(head_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         HeadSmem::BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(head_fused_grid(a.rows));
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = HeadSmem::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, head_fused_kernel, mH, mF, mDz, a);
}

}  // namespace hdp
