// tcgen05 / TMEM / TMA GEMM for sm_100a, plus the fp32 SIMT GEMM of FP32 mode.
//
// One CTA computes a 128 x BN output tile (UMMA M=128, N=BN, K=16 steps):
//   warp 0 lane 0 : TMA producer, STAGES-deep smem ring (SWIZZLE_128B tiles)
//   warp 1 lane 0 : tcgen05.mma issuer, accumulator in TMEM (BN fp32 columns)
//   warp 2        : TMEM allocation / deallocation
//   all 4 warps   : epilogue, tcgen05.ld 32 lanes x 16 columns at a time
// Split-K writes fp32 partials that a deterministic reduction kernel sums in
// split order (no atomics), so results do not depend on scheduling.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>

#include "dropout.cuh"
#include "gemm.cuh"
#include "options.h"
#include "ptx.cuh"

namespace hdp {

static thread_local char g_gemm_err[256];
const char* gemm_last_error() { return g_gemm_err; }

namespace {

constexpr int BM = 128;
constexpr int BK = 64;

template <int BN, int CG = 1>
struct TileCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;  // a CTA pair splits the B tile along N
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // as deep as the 227 KB allow
  static constexpr int STAGES = STAGE >= 49152 ? 3 : (STAGE >= 32768 ? 5 : 7);
  static constexpr int EPI_LD = 36;  // staging row stride (floats): conflict-free float4 rows
  static constexpr int EPI_WARPS = 8;  // 2 per TMEM lane quadrant, each half of the columns
  static constexpr int EPI_BYTES = EPI_WARPS * 32 * EPI_LD * 4;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align slack*/ + 256 /*barriers*/ + EPI_BYTES;
};

// 16-bit working type of the operands / outputs: fp16, or bfloat16 (Epilogue::bf16, the
// bf16 math mode).  Values travel as their bit patterns (uint16_t).
__device__ __forceinline__ uint16_t cvt16(float v, int bf) {
  return bf ? __bfloat16_as_ushort(__float2bfloat16_rn(v)) : __half_as_ushort(__float2half_rn(v));
}
__device__ __forceinline__ float f16v(uint32_t bits, int bf) {
  bits &= 0xFFFFu;
  return bf ? __uint_as_float(bits << 16) : __half2float(__ushort_as_half((unsigned short)bits));
}
__device__ __forceinline__ int nonfinite16(uint16_t b, int bf) {
  return bf ? (b & 0x7F80u) == 0x7F80u : (b & 0x7C00u) == 0x7C00u;
}

__device__ __forceinline__ float bias_at(const Epilogue& e, long i) {
  return e.bias_f16 ? f16v(reinterpret_cast<const uint16_t*>(e.bias)[i], e.bf16)
                    : reinterpret_cast<const float*>(e.bias)[i];
}

// Store 16 consecutive columns [n, n+16) of row m.
__device__ __forceinline__ void epi_store16(const Epilogue& epi, float* ws, int M, int N, int m, int n,
                                            float (&v)[16], int& nf) {
  if (m >= M) return;
  if (epi.mode == EPI_SPLITK) {
    float* o = ws + (size_t)blockIdx.z * M * N + (size_t)m * N;
    if (n + 16 <= N && (N & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(o + n + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
      for (int j = 0; j < 16; ++j)
        if (n + j < N) o[n + j] = v[j];
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float b = 0.f;
    if (epi.bias) b = epi.bias_on_m ? bias_at(epi, m) : ((n + j < N) ? bias_at(epi, n + j) : 0.f);
    float x = v[j] + b;
    if (epi.relu) x = fmaxf(x, 0.f);
    v[j] = x;
  }
  if (epi.mode == EPI_F32) {
    float* o = reinterpret_cast<float*>(epi.out) + (size_t)m * epi.ldo;
    if (n + 16 <= N && (epi.ldo & 3) == 0) {
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        float4 w = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if (epi.accumulate) {
          float4 q = *reinterpret_cast<const float4*>(o + n + j);
          w.x += q.x; w.y += q.y; w.z += q.z; w.w += q.w;
        }
        *reinterpret_cast<float4*>(o + n + j) = w;
      }
    } else {
      for (int j = 0; j < 16; ++j)
        if (n + j < N) o[n + j] = epi.accumulate ? o[n + j] + v[j] : v[j];
    }
  } else if (epi.mode == EPI_F32_T) {
    float* o = reinterpret_cast<float*>(epi.out);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (n + j < N) {
        float* p = o + (size_t)(n + j) * epi.ldo + m;
        *p = epi.accumulate ? *p + v[j] : v[j];
      }
  } else {  // EPI_F16 (fp16, or bf16 in the bf16 mode)
    uint16_t* o = reinterpret_cast<uint16_t*>(epi.out) + (size_t)m * epi.ldo;
    if (n + 16 <= N && (epi.ldo & 7) == 0) {
#pragma unroll
      for (int j = 0; j < 16; j += 8) {
        __align__(16) uint16_t hv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          hv[q] = cvt16(v[j + q], epi.bf16);
          nf += nonfinite16(hv[q], epi.bf16);
        }
        *reinterpret_cast<uint4*>(o + n + j) = *reinterpret_cast<const uint4*>(hv);
      }
    } else {
      for (int j = 0; j < 16; ++j)
        if (n + j < N) {
          const uint16_t h = cvt16(v[j], epi.bf16);
          nf += nonfinite16(h, epi.bf16);
          o[n + j] = h;
        }
    }
  }
}

// ---------------------------------------------------------------- fused cell epilogues
// Same cell as K3 / K6 (lstm_kernels.cu; PAPER.md:60-62 cell, :82 BPTT) with the SFU
// activations of the persistent recurrence kernels (recur.cu): sigma via __expf, tanh(x) =
// 2 sigma(2x) - 1; relative error ~1e-6, far below the fp16 rounding of everything stored.
__device__ __forceinline__ float lstm_sigmoid(float x) { return __fdividef(1.f, 1.f + __expf(-x)); }
__device__ __forceinline__ float lstm_tanh(float x) {
  const float xc = fminf(fmaxf(x, -15.f), 15.f);
  return fmaf(2.f, lstm_sigmoid(2.f * xc), -1.f);
}

// recurrent dropout: the masked copy h~ of 8 units of row m (R6d: fp16 of fp32(h) * scale)
__device__ __forceinline__ void lstm_drop_store(const Epilogue& e, int m, int u0, const uint16_t (&hh)[8]) {
  const uint32_t sk = drop_seq_key(drop_layer_key(e.drop_seed, (uint32_t)*e.drop_step, e.drop_layer),
                                   e.drop_seq0 + (uint32_t)m);
  __align__(16) uint16_t ht[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    ht[j] = drop_kept(sk, (uint32_t)(u0 + j), e.drop_thr) ? cvt16(f16v(hh[j], e.bf16) * e.drop_scale, e.bf16)
                                                          : (uint16_t)0;
  *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(e.htout) + (size_t)m * e.hp + u0) =
      *reinterpret_cast<const uint4*>(ht);
}

// A3 for 8 units of row m: columns [n, n+32) of the gate pre-activation (n = 4 u0).
__device__ __forceinline__ void lstm_fwd_chunk(const Epilogue& e, int m, int n, const float (&v)[32]) {
  const int u0 = n >> 2;
  const float4* gx = reinterpret_cast<const float4*>(e.gx + (size_t)m * 4 * e.hp + n);
  float cp[8];
  if (e.cprev) {
    const float4* p = reinterpret_cast<const float4*>(e.cprev + (size_t)m * e.hp + u0);
    const float4 a = p[0], b = p[1];
    cp[0] = a.x; cp[1] = a.y; cp[2] = a.z; cp[3] = a.w; cp[4] = b.x; cp[5] = b.y; cp[6] = b.z; cp[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) cp[j] = 0.f;
  }
  __align__(16) uint16_t gh[32];
  __align__(16) uint16_t hh[8];
  float cn[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 g4 = gx[j];
    const float i = lstm_sigmoid(g4.x + v[4 * j]), f = lstm_sigmoid(g4.y + v[4 * j + 1]);
    const float g = lstm_tanh(g4.z + v[4 * j + 2]), o = lstm_sigmoid(g4.w + v[4 * j + 3]);
    const float c = f * cp[j] + i * g;
    cn[j] = c;
    hh[j] = cvt16(o * lstm_tanh(c), e.bf16);  // R6
    gh[4 * j] = cvt16(i, e.bf16);         // R4
    gh[4 * j + 1] = cvt16(f, e.bf16);
    gh[4 * j + 2] = cvt16(g, e.bf16);
    gh[4 * j + 3] = cvt16(o, e.bf16);
  }
  uint4* go = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(e.gates) + (size_t)m * 4 * e.hp + n);
#pragma unroll
  for (int q = 0; q < 4; ++q) go[q] = reinterpret_cast<const uint4*>(gh)[q];
  float4* co = reinterpret_cast<float4*>(e.cout + (size_t)m * e.hp + u0);
  co[0] = make_float4(cn[0], cn[1], cn[2], cn[3]);
  co[1] = make_float4(cn[4], cn[5], cn[6], cn[7]);
  *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(e.hout) + (size_t)m * e.hp + u0) =
      *reinterpret_cast<const uint4*>(hh);
  if (e.drop_step) lstm_drop_store(e, m, u0, hh);
}

// Same, with G_x and c_{t-1} already in registers.
__device__ __forceinline__ void lstm_fwd_chunk_reg(const Epilogue& e, int m, int n, const float (&v)[32],
                                                   const float4 (&gx)[8], const float4 (&cp4)[2]) {
  const int u0 = n >> 2;
  const float cp[8] = {cp4[0].x, cp4[0].y, cp4[0].z, cp4[0].w, cp4[1].x, cp4[1].y, cp4[1].z, cp4[1].w};
  __align__(16) uint16_t gh[32];
  __align__(16) uint16_t hh[8];
  float cn[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float i = lstm_sigmoid(gx[j].x + v[4 * j]), f = lstm_sigmoid(gx[j].y + v[4 * j + 1]);
    const float g = lstm_tanh(gx[j].z + v[4 * j + 2]), o = lstm_sigmoid(gx[j].w + v[4 * j + 3]);
    const float c = f * cp[j] + i * g;
    cn[j] = c;
    hh[j] = cvt16(o * lstm_tanh(c), e.bf16);  // R6
    gh[4 * j] = cvt16(i, e.bf16);         // R4
    gh[4 * j + 1] = cvt16(f, e.bf16);
    gh[4 * j + 2] = cvt16(g, e.bf16);
    gh[4 * j + 3] = cvt16(o, e.bf16);
  }
  uint4* go = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(e.gates) + (size_t)m * 4 * e.hp + n);
#pragma unroll
  for (int q = 0; q < 4; ++q) go[q] = reinterpret_cast<const uint4*>(gh)[q];
  float4* co = reinterpret_cast<float4*>(e.cout + (size_t)m * e.hp + u0);
  co[0] = make_float4(cn[0], cn[1], cn[2], cn[3]);
  co[1] = make_float4(cn[4], cn[5], cn[6], cn[7]);
  *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(e.hout) + (size_t)m * e.hp + u0) =
      *reinterpret_cast<const uint4*>(hh);
  if (e.drop_step) lstm_drop_store(e, m, u0, hh);
}

// A6 for unit idx = m * hp + u given dh_rec (the reduced K7 result).
__device__ __forceinline__ void lstm_bwd_unit(const Epilogue& e, size_t idx, float dh_rec) {
  float dh = 0.f;
  if (e.dha) dh += e.dha[idx];
  if (e.drop_step) {  // dh_rec is the gradient of h~_{t-1}: back through the mask and scale
    const uint32_t mrow = (uint32_t)(idx / e.hp), u = (uint32_t)(idx % e.hp);
    const uint32_t sk = drop_seq_key(drop_layer_key(e.drop_seed, (uint32_t)*e.drop_step, e.drop_layer),
                                     e.drop_seq0 + mrow);
    dh_rec = drop_kept(sk, u, e.drop_thr) ? dh_rec * e.drop_scale : 0.f;
  }
  dh += dh_rec;
  const uint2 gu = reinterpret_cast<const uint2*>(e.gates)[idx];
  const float i = f16v(gu.x, e.bf16), f = f16v(gu.x >> 16, e.bf16);
  const float g = f16v(gu.y, e.bf16), o = f16v(gu.y >> 16, e.bf16);
  const float c = e.ct[idx];
  const float cp = e.cprev ? e.cprev[idx] : 0.f;
  const float tc = lstm_tanh(c);
  const float d = e.dc[idx] + dh * o * (1.f - tc * tc);
  __align__(8) uint16_t hv[4] = {cvt16(d * g * i * (1.f - i), e.bf16), cvt16(d * cp * f * (1.f - f), e.bf16),
                                 cvt16(d * i * (1.f - g * g), e.bf16), cvt16(dh * tc * o * (1.f - o), e.bf16)};
  reinterpret_cast<uint2*>(e.dA)[idx] = *reinterpret_cast<const uint2*>(hv);  // R10
  e.dc[idx] = d * f;
}

// Persistent, warp-specialised: each CTA walks tiles blockIdx.x, +gridDim.x, ...
//   warp 0 (one lane): TMA producer over a continuous k-block stream (STAGES ring)
//   warp 1           : TMEM allocation; one lane issues tcgen05.mma into one of two
//                      TMEM accumulators (2 x BN columns) per tile
//   warps 2..9       : epilogue of tile i (TMEM -> registers -> smem -> coalesced
//                      global stores) while the MMAs of tile i+1 run; warp w drains
//                      TMEM lane quadrant w % 4, column half (w - 2) / 4
//
// CN > 1 (K-major A only): clusters of CN CTAs walk tile groups that share the M tile and
// the K range (consecutive N tiles); every CTA TMA-loads 1/CN of the A rows and multicasts
// them to the whole cluster, so A (the operand every N tile re-reads) leaves L2 once per
// cluster.  A slot is refilled only after all CN CTAs' MMAs consumed it (each commit
// arrives on every CTA's empty barrier).
//
// CG = 2: CTA pairs (cta_group::2).  A pair owns a 256 x BN tile: each CTA loads its 128
// A rows and half of the B tile, the leader (rank 0) issues M = 256 MMAs over both CTAs'
// shared memory, and each CTA's TMEM receives its 128 rows -- per SM half the B bytes of
// a 128 x BN tile for the same flops.  Both CTAs' TMA loads complete on the leader's
// full barrier; the leader's commits arrive on both CTAs' empty / accumulator barriers;
// both epilogues arrive on the leader's drain barrier.
//
// CR = 8 (the fused cell backward, EPI_LSTM_BWD, 8 K-splits, one tile per CTA): the 8 splits
// of an output tile form one cluster; after every split's accumulator is complete (cluster
// barrier: all shared-memory rings idle) each CTA sends the 32-column slice d of its fp32
// partial into CTA d's ring through DSMEM, and after a second cluster barrier CTA d sums the
// 8 partials of its slice in split order -- the same fp32 operation order as
// splitk_reduce_kernel, so bit-identical -- and runs the cell backward on them.  No partial
// planes in global memory, no second launch.
template <int BN, int AMN, int BMN, int CN = 1, int CG = 1, int CR = 1>
__global__ void __launch_bounds__(320, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, int M, int N,
                   int K, int kbps, int splits, Epilogue epi, float* ws) {
  static_assert(CN == 1 || AMN == 0, "A multicast needs K-major A");
  static_assert(CG == 1 || CN == 1, "CTA pairs: no multicast");
  static_assert(CR == 1 || (CN == 1 && CG == 1 && BN == 256), "cluster split-K reduction: single CTAs, BN = 256");
  static_assert(CR == 1 || CR * 128 * 36 * 4 <= TileCfg<BN, CG>::STAGES * TileCfg<BN, CG>::STAGE,
                "the partials fit in the ring");
  using C = TileCfg<BN, CG>;
  constexpr int CL = CN * CG;  // cluster size
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;  // [2] accumulator b complete
  uint64_t* acce = accf + 2;           // [2] accumulator b drained (8 epilogue warps)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acce + 2);
  float* epi_stage = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE + 256);  // [8 warps][32][EPI_LD]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = (M + BM * CG - 1) / (BM * CG), nt = (N + BN - 1) / BN;
  const int ngr = (nt + CN - 1) / CN;               // N-tile groups (one per cluster pass)
  const int ntiles = mt * ngr * splits;             // = tiles when CN == 1
  const int kb_total = (K + BK - 1) / BK;
  const int crank = CN > 1 ? (int)(blockIdx.x % CN) : 0;
  const int prank = CG > 1 ? (int)(blockIdx.x % CG) : 0;  // 0 = pair leader
  // CR > 1: cluster c's CTA z computes split z of output tile c (one tile per CTA)
  const int tile0 = CR > 1 ? (int)(blockIdx.x % CR) * mt * ngr + (int)(blockIdx.x / CR)
                           : CL > 1 ? (int)(blockIdx.x / CL) : (int)blockIdx.x;
  const int tstep = CR > 1 ? ntiles : CL > 1 ? (int)(gridDim.x / CL) : (int)gridDim.x;
  auto decode = [&](int tile, int& m0, int& n0, int& z, int& kb0, int& nkb) {
    z = tile / (mt * ngr);
    const int r = tile % (mt * ngr);
    m0 = (r % mt) * BM * CG + prank * BM;  // this CTA's 128 rows of the (pair) tile
    n0 = ((r / mt) * CN + crank) * BN;
    kb0 = z * kbps;
    nkb = min(kb_total, kb0 + kbps) - kb0;
  };
  constexpr uint16_t cmask = (uint16_t)((1u << CN) - 1u);

  if (threadIdx.x == 0) {
    ptx::tma_prefetch(&tma);
    ptx::tma_prefetch(&tmb);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, CN);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(accf + b, 1);
      ptx::mbar_init(acce + b, C::EPI_WARPS * CG);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (CG > 1) ptx::tmem_alloc2(tslot, 2 * BN);
    else ptx::tmem_alloc(tslot, 2 * BN);
  }
  ptx::tc_fence_before();
  if constexpr (CL > 1) ptx::cluster_sync_all();  // peers' barriers exist before any multicast
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tslot;
  ptx::griddep_wait();  // (PDL) the setup above overlapped the previous kernel's tail
  ptx::griddep_launch();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep) {
        int m0, n0, z, kb0, nkb;
        decode(tile, m0, n0, z, kb0, nkb);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          ptx::mbar_wait(empty + s, ph ^ 1);
          uint8_t* sa = smem + s * C::STAGE;
          uint8_t* sb = sa + C::A_BYTES;
          const int k0 = (kb0 + i) * BK;
          if constexpr (CG > 1) {
            // both CTAs' bytes complete on the leader's full barrier
            if (prank == 0) ptx::mbar_arrive_expect_tx(full + s, 2 * C::STAGE);
            if (AMN == 0) {
              ptx::tma_load_2d_cg2(sa, &tma, full + s, k0, m0);
            } else {  // MN-major A: this CTA's 128 M columns as two 64-wide atoms
              ptx::tma_load_2d_cg2(sa, &tma, full + s, m0, k0);
              ptx::tma_load_2d_cg2(sa + 8192, &tma, full + s, m0 + 64, k0);
            }
            if (BMN == 0) {
              ptx::tma_load_2d_cg2(sb, &tmb, full + s, k0, n0 + prank * (BN / 2));
            } else {
#pragma unroll
              for (int j = 0; j < BN / 128; ++j)
                ptx::tma_load_2d_cg2(sb + j * 8192, &tmb, full + s, n0 + prank * (BN / 2) + 64 * j, k0);
            }
            continue;
          }
          ptx::mbar_arrive_expect_tx(full + s, C::STAGE);
          if (CN > 1) {
            ptx::tma_load_2d_mc(sa + crank * (BM / CN) * 128, &tma, full + s, k0, m0 + crank * (BM / CN), cmask);
          } else if (AMN == 0) {
            ptx::tma_load_2d(sa, &tma, full + s, k0, m0);
          } else {
            ptx::tma_load_2d(sa, &tma, full + s, m0, k0);
            ptx::tma_load_2d(sa + 8192, &tma, full + s, m0 + 64, k0);
          }
          if (BMN == 0) {
            ptx::tma_load_2d(sb, &tmb, full + s, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) ptx::tma_load_2d(sb + j * 8192, &tmb, full + s, n0 + 64 * j, k0);
          }
        }
      }
      if (CL > 1)  // drain: every slot's last use consumed by all the MMAs (their commits have
        for (int i = 0; i < C::STAGES; ++i, ++it)  // landed here) before the cluster may exit
          ptx::mbar_wait(empty + it % C::STAGES, ((it / C::STAGES) & 1) ^ 1);
    }
    if constexpr (CR > 1) {  // the epilogue's two cluster barriers (every thread of the cluster)
      __syncwarp();
      ptx::cluster_arrive();
      ptx::cluster_wait();
      ptx::cluster_arrive();
      ptx::cluster_wait();
    }
  } else if (warp == 1) {
    if (lane == 0 && prank == 0) {
      // ---------------- MMA issuer (the pair leader for CG = 2)
      // operand format bits [7, 10) / [10, 13): 0 = fp16, 1 = bf16 (the bf16 math mode)
      const uint32_t idesc = ptx::idesc_f16_f32(BM * CG, BN, AMN, BMN) | (epi.bf16 ? (1u << 7) | (1u << 10) : 0u);
      constexpr uint16_t pmask = 3;
      int it = 0, lt = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep, ++lt) {
        int m0, n0, z, kb0, nkb;
        decode(tile, m0, n0, z, kb0, nkb);
        const int b = lt & 1;
        ptx::mbar_wait(acce + b, ((lt >> 1) & 1) ^ 1);  // accumulator b drained by the epilogue
        ptx::tc_fence_after();
        const uint32_t tacc = tbase + b * BN;
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          ptx::mbar_wait(full + s, ph);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + s * C::STAGE);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 16 elements = 32 B inside the 128 B swizzled row.
            // MN-major: advance 16 K-rows = 2048 B (two 8-row atoms of 1024 B);
            //   LBO = 8192 B between 64-wide MN atoms, SBO = 1024 B between 8-row K groups.
            const uint64_t ad = AMN ? ptx::smem_desc_sw128(sa + k * 2048, 8192, 1024)
                                    : ptx::smem_desc_sw128(sa + k * 32, 0, 1024);
            const uint64_t bd = BMN ? ptx::smem_desc_sw128(sb + k * 2048, 8192, 1024)
                                    : ptx::smem_desc_sw128(sb + k * 32, 0, 1024);
            if constexpr (CG > 1) ptx::mma_f16_cg2(tacc, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
            else ptx::mma_f16(tacc, ad, bd, idesc, (i > 0 || k > 0) ? 1u : 0u);
          }
          if (CG > 1) ptx::mma_commit_cg2_mc(empty + s, pmask);      // both CTAs' slot s
          else if (CN > 1) ptx::mma_commit_mc(empty + s, cmask);  // every CTA's slot s was written by all
          else ptx::mma_commit(empty + s);  // frees the smem slot once these MMAs retire
        }
        if (CG > 1) ptx::mma_commit_cg2_mc(accf + b, pmask);  // both CTAs' accumulators complete
        else ptx::mma_commit(accf + b);     // accumulator b complete
      }
    }
    if constexpr (CR > 1) {
      __syncwarp();
      ptx::cluster_arrive();
      ptx::cluster_wait();
      ptx::cluster_arrive();
      ptx::cluster_wait();
    }
  } else if (CR > 1) {
    // ---------------- cluster split-K reduction + fused cell backward (one tile per CTA)
    const int q = warp & 3;
    const int ch = (warp - 2) >> 2;
    int m0, n0, z, kb0, nkb;
    decode(tile0, m0, n0, z, kb0, nkb);
    ptx::mbar_wait(accf, 0);
    ptx::tc_fence_after();
    ptx::cluster_arrive();  // every split's MMAs are complete: all rings are idle
    ptx::cluster_wait();
    float* rbuf = reinterpret_cast<float*>(smem);  // [CR][128 rows][36] fp32 partial slices
    const int row = q * 32 + lane;
    const uint32_t tq = tbase + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t my_slot = ptx::smem_u32(rbuf + ((size_t)z * 128 + row) * 36);
#pragma unroll 1
    for (int j = 0; j < BN / 64; ++j) {
      const int c = ch * (BN / 2) + 32 * j;  // 32-column slice owned by CTA c / 32 of the cluster
      float v[32];
      ptx::tmem_ld16_nowait(tq + c, *reinterpret_cast<float(*)[16]>(v));
      ptx::tmem_ld16_nowait(tq + c + 16, *reinterpret_cast<float(*)[16]>(v + 16));
      ptx::tmem_wait_ld();
      const uint32_t dst = ptx::mapa(my_slot, (uint32_t)(c >> 5));
#pragma unroll
      for (int k = 0; k < 8; ++k)
        ptx::st_cluster_v4(dst + 16 * k, make_uint4(__float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                                                    __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3])));
    }
    ptx::tc_fence_before();
    ptx::cluster_arrive();  // release: every slice delivered
    ptx::cluster_wait();
    // my slice: columns n0 + 32 z + lane; warp e takes rows e, e + 8, ...; splits summed in order
    const int n = n0 + 32 * z + lane;
#pragma unroll 1
    for (int rr = warp - 2; rr < BM; rr += 8) {
      const int m = m0 + rr;
      float s = rbuf[(size_t)rr * 36 + lane];
#pragma unroll
      for (int z2 = 1; z2 < CR; ++z2) s += rbuf[((size_t)z2 * 128 + rr) * 36 + lane];
      if (m < M && n < N) lstm_bwd_unit(epi, (size_t)m * N + n, s);
    }
  } else {
    // ---------------- epilogue warps 2..9: TMEM lane quadrant q = warp % 4, column half ch
    const int q = warp & 3;
    const int ch = (warp - 2) >> 2;
    const int c_lo = ch * (BN / 2), c_hi = c_lo + BN / 2;
    float* st = epi_stage + (warp - 2) * 32 * C::EPI_LD;
    const bool f16 = epi.mode == EPI_F16;
    const bool fast = !epi.accumulate && (epi.mode == EPI_F32 || epi.mode == EPI_SPLITK || f16);
    uint16_t* o16 = reinterpret_cast<uint16_t*>(epi.out);
    const bool post = epi.mode != EPI_SPLITK;  // bias / relu belong to the reduction for split-K
    // accumulator b drained: the MMA issuer's (leader's) barrier
    auto drained = [&](int b) {
      if (CG > 1 && prank != 0) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(acce + b), 0));
      else ptx::mbar_arrive(acce + b);
    };
    int nf = 0, lt = 0;
    for (int tile = tile0; tile < ntiles; tile += tstep, ++lt) {
      int m0, n0, z, kb0, nkb;
      decode(tile, m0, n0, z, kb0, nkb);
      const int b = lt & 1;
      const int m = m0 + q * 32 + lane;
      if constexpr (BN <= 128) {
        if (epi.mode == EPI_LSTM_FWD) {
          // fused cell: this lane's G_x and c_{t-1} are loaded while the MMAs run
          constexpr int NCH = BN / 64;  // 32-column chunks per warp
          float4 gx[NCH][8], cp[NCH][2];
#pragma unroll
          for (int h = 0; h < NCH; ++h) {
            const int n = n0 + c_lo + 32 * h;
            const bool ok = m < M && n < N;
            const float4* gp = reinterpret_cast<const float4*>(epi.gx + (size_t)m * 4 * epi.hp + n);
#pragma unroll
            for (int j = 0; j < 8; ++j) gx[h][j] = ok ? gp[j] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4* cq = reinterpret_cast<const float4*>(epi.cprev + (size_t)m * epi.hp + (n >> 2));
            cp[h][0] = ok && epi.cprev ? cq[0] : make_float4(0.f, 0.f, 0.f, 0.f);
            cp[h][1] = ok && epi.cprev ? cq[1] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          ptx::mbar_wait(accf + b, (lt >> 1) & 1);
          ptx::tc_fence_after();
          const uint32_t tq = tbase + b * BN + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll
          for (int h = 0; h < NCH; ++h) {
            const int c = c_lo + 32 * h;
            float v[32];
            ptx::tmem_ld16_nowait(tq + c, *reinterpret_cast<float(*)[16]>(v));
            ptx::tmem_ld16_nowait(tq + c + 16, *reinterpret_cast<float(*)[16]>(v + 16));
            ptx::tmem_wait_ld();
            if (m < M && n0 + c < N) lstm_fwd_chunk_reg(epi, m, n0 + c, v, gx[h], cp[h]);
          }
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) drained(b);
          continue;
        }
      }
      ptx::mbar_wait(accf + b, (lt >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tq = tbase + b * BN + (static_cast<uint32_t>(q * 32) << 16);
      if (epi.mode == EPI_LSTM_FWD) {
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += 32) {
          if (n0 + c >= N) break;
          float v[32];
          ptx::tmem_ld16_nowait(tq + c, *reinterpret_cast<float(*)[16]>(v));
          ptx::tmem_ld16_nowait(tq + c + 16, *reinterpret_cast<float(*)[16]>(v + 16));
          ptx::tmem_wait_ld();
          if (m < M) lstm_fwd_chunk(epi, m, n0 + c, v);
        }
      } else if (fast) {
        // 32 x 32 chunk through shared memory; every store instruction then writes
        // 4 whole rows (lane -> row i*4 + lane/8, 4 consecutive columns)
        float* o32 = epi.mode == EPI_SPLITK ? ws + (size_t)z * M * N : reinterpret_cast<float*>(epi.out);
        const long ldo = epi.mode == EPI_SPLITK ? N : epi.ldo;
        const bool vec = f16 ? ((ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(o16) & 7) == 0)
                             : ((ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(o32) & 15) == 0);
        const float bm = (post && epi.bias && epi.bias_on_m && m < M) ? bias_at(epi, m) : 0.f;
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += 32) {
          if (n0 + c >= N) break;
          float v[32];
          ptx::tmem_ld16_nowait(tq + c, *reinterpret_cast<float(*)[16]>(v));
          ptx::tmem_ld16_nowait(tq + c + 16, *reinterpret_cast<float(*)[16]>(v + 16));
          // column bias: one coalesced load per lane, broadcast by shuffles
          const float bl = (post && epi.bias && !epi.bias_on_m && n0 + c + lane < N) ? bias_at(epi, n0 + c + lane) : 0.f;
          ptx::tmem_wait_ld();
          if (post) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float x = v[j] + (epi.bias_on_m ? bm : __shfl_sync(0xffffffffu, bl, j));
              if (epi.relu) x = fmaxf(x, 0.f);
              v[j] = x;
            }
          }
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(st + lane * C::EPI_LD + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = i * 4 + (lane >> 3), cc = (lane & 7) * 4;
            const int mr = m0 + q * 32 + r, n = n0 + c + cc;
            if (mr < M && n < N) {
              const float4 qq = *reinterpret_cast<const float4*>(st + r * C::EPI_LD + cc);
              const float qv[4] = {qq.x, qq.y, qq.z, qq.w};
              if (f16) {
                __align__(8) uint16_t h[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  h[u] = cvt16(qv[u], epi.bf16);
                  if (n + u < N) nf += nonfinite16(h[u], epi.bf16);
                }
                uint16_t* dst = o16 + (size_t)mr * ldo + n;
                if (vec && n + 4 <= N) {
                  *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(h);
                } else {
                  for (int u = 0; u < 4; ++u)
                    if (n + u < N) dst[u] = h[u];
                }
              } else {
                float* dst = o32 + (size_t)mr * ldo + n;
                if (vec && n + 4 <= N) {
                  *reinterpret_cast<float4*>(dst) = qq;
                } else {
                  for (int u = 0; u < 4; ++u)
                    if (n + u < N) dst[u] = qv[u];
                }
              }
            }
          }
          __syncwarp();
        }
      } else {
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += 16) {
          float v[16];
          ptx::tmem_ld16(tq + c, v);
          if (n0 + c < N) epi_store16(epi, ws, M, N, m, n0 + c, v, nf);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) drained(b);
    }
    if (epi.mode == EPI_F16 && epi.nonfinite) {
      nf = __reduce_add_sync(0xffffffffu, nf);
      if (lane == 0 && nf) atomicAdd(epi.nonfinite, nf);
    }
  }
  ptx::tc_fence_before();
  __syncwarp();
  if constexpr (CL > 1) ptx::cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (CG > 1) ptx::tmem_dealloc2(tbase, 2 * BN);
    else ptx::tmem_dealloc(tbase, 2 * BN);
  }
}

// Deterministic split-K reduction + the requested epilogue.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N, Epilogue epi) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  const size_t total = (size_t)M * N;
  int nf = 0;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    float s = ws[idx];
    for (int z = 1; z < splits; ++z) s += ws[(size_t)z * total + idx];
    if (epi.mode == EPI_LSTM_BWD) {
      lstm_bwd_unit(epi, idx, s);
      continue;
    }
    const int m = (int)(idx / N), n = (int)(idx % N);
    if (epi.bias) s += epi.bias_on_m ? bias_at(epi, m) : bias_at(epi, n);
    if (epi.relu) s = fmaxf(s, 0.f);
    if (epi.mode == EPI_F32) {
      float* o = reinterpret_cast<float*>(epi.out) + (size_t)m * epi.ldo + n;
      *o = epi.accumulate ? *o + s : s;
    } else if (epi.mode == EPI_F32_T) {
      float* o = reinterpret_cast<float*>(epi.out) + (size_t)n * epi.ldo + m;
      *o = epi.accumulate ? *o + s : s;
    } else {
      const uint16_t h = cvt16(s, epi.bf16);
      nf += nonfinite16(h, epi.bf16);
      reinterpret_cast<uint16_t*>(epi.out)[(size_t)m * epi.ldo + n] = h;
    }
  }
  if (epi.mode == EPI_F16 && epi.nonfinite) {
    nf = __reduce_add_sync(0xffffffffu, nf);
    if ((threadIdx.x & 31) == 0 && nf) atomicAdd(epi.nonfinite, nf);
  }
}

// ---------------------------------------------------------------- fp32 SIMT GEMM
// 64x64 tile, 256 threads, 4x4 per thread, sequential k (deterministic).
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, long sam, long sak,
                                                       const float* __restrict__ B, long sbn, long sbk, int M,
                                                       int N, int K, Epilogue epi) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e / 64, r = e % 64;
      const int m = m0 + r, n = n0 + r, k = k0 + kk;
      As[kk][r] = (m < M && k < K) ? A[(size_t)m * sam + (size_t)k * sak] : 0.f;
      Bs[kk][r] = (n < N && k < K) ? B[(size_t)n * sbn + (size_t)k * sbk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m >= M || n >= N) continue;
      float s = acc[i][j];
      if (epi.bias) s += epi.bias_on_m ? bias_at(epi, m) : bias_at(epi, n);
      if (epi.relu) s = fmaxf(s, 0.f);
      float* o = reinterpret_cast<float*>(epi.out) + (epi.mode == EPI_F32_T ? (size_t)n * epi.ldo + m
                                                                            : (size_t)m * epi.ldo + n);
      *o = epi.accumulate ? *o + s : s;
    }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 2-D fp16 tensor map, inner dimension contiguous, SWIZZLE_128B, 64-element inner box.
int make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
              uint32_t box_outer) {
  if (!get_encode()) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "cuTensorMapEncodeTiled unavailable");
    return -2;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((row_stride_elems * 2) & 15)) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "TMA operand not 16-byte aligned (base %p, stride %llu elems)", base,
             (unsigned long long)row_stride_elems);
    return -1;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "cuTensorMapEncodeTiled failed (%d): inner %llu outer %llu stride %llu",
             (int)r, (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_stride_elems);
    return -2;
  }
  return 0;
}

}  // namespace

int encode_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                   uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
  if (!get_encode()) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "cuTensorMapEncodeTiled unavailable");
    return -2;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return -2;
  }
  return 0;
}

namespace {

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        n <= 0)
      n = 148;
  }
  return n;
}

// programmatic dependent launch of the GEMM / split-K kernels: opt-in (option "pdl"); measured
// on the C4 per-step chain it did not shorten the step (37.6 vs 37.3 ms), the prologue it
// overlaps is short next to the predecessor's drain + flush
bool use_pdl() { return opt(OPT_PDL) == 1; }

template <int BN, int AMN, int BMN, int CN = 1, int CG = 1, int CR = 1>
cudaError_t launch_tc(const GemmPlan& p, cudaStream_t s) {
  using C = TileCfg<BN, CG>;
  constexpr int CL = CN * CG * CR;
  const int groups = ((p.M + BM * CG - 1) / (BM * CG)) * ((((p.N + BN - 1) / BN) + CN - 1) / CN) * p.splits;
  Epilogue e = p.epi;
  if (CR == 1 && (p.splits > 1 || e.mode == EPI_LSTM_BWD)) e.mode = EPI_SPLITK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CR > 1 ? groups : std::min(groups, num_sms() / CL) * CL);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (CL > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = CL;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (use_pdl()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, AMN, BMN, CN, CG, CR>, p.ta, p.tb, p.M, p.N, p.K, p.kbps,
                            p.splits, e, p.ws);
}

template <int BN, int AMN, int BMN, int CN = 1, int CG = 1, int CR = 1>
cudaError_t set_attr() {
  return cudaFuncSetAttribute(gemm_tc_kernel<BN, AMN, BMN, CN, CG, CR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              TileCfg<BN, CG>::SMEM);
}
template <int BN>
cudaError_t set_attr_bn() {
  cudaError_t e;
  if ((e = set_attr<BN, 0, 0>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 1>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 1, 0>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 0, 2>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 1, 2>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 0, 4>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 1, 4>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 0, 8>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 1, 8>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 0, 1, 2>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 0, 1, 1, 2>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 1, 0, 1, 2>()) != cudaSuccess) return e;
  if ((e = set_attr<BN, 1, 1, 1, 2>()) != cudaSuccess) return e;
  return set_attr<BN, 1, 1>();
}

template <int BN>
cudaError_t launch_tc_bn(const GemmPlan& p, cudaStream_t s) {
  if constexpr (BN == 256)
    if (p.cr == 8) return launch_tc<256, 0, 1, 1, 1, 8>(p, s);
  if (p.amn == 0 && p.cg == 2) return p.bmn ? launch_tc<BN, 0, 1, 1, 2>(p, s) : launch_tc<BN, 0, 0, 1, 2>(p, s);
  if (p.amn == 1 && p.cg == 2) return p.bmn ? launch_tc<BN, 1, 1, 1, 2>(p, s) : launch_tc<BN, 1, 0, 1, 2>(p, s);
  if (p.amn == 0 && p.cn == 2) return p.bmn ? launch_tc<BN, 0, 1, 2>(p, s) : launch_tc<BN, 0, 0, 2>(p, s);
  if (p.amn == 0 && p.cn == 4) return p.bmn ? launch_tc<BN, 0, 1, 4>(p, s) : launch_tc<BN, 0, 0, 4>(p, s);
  if (p.amn == 0 && p.cn == 8) return p.bmn ? launch_tc<BN, 0, 1, 8>(p, s) : launch_tc<BN, 0, 0, 8>(p, s);
  if (p.amn == 0 && p.bmn == 0) return launch_tc<BN, 0, 0>(p, s);
  if (p.amn == 0 && p.bmn == 1) return launch_tc<BN, 0, 1>(p, s);
  if (p.amn == 1 && p.bmn == 0) return launch_tc<BN, 1, 0>(p, s);
  return launch_tc<BN, 1, 1>(p, s);
}

int choose_bn(int M, int N) {
  const int mt = (M + BM - 1) / BM;
  if (N <= 64) return 64;
  // latency-bound: more CTAs -- unless 128-wide tiles already cover most SMs
  // (C4 K2, 256 x 8192 x 2048: 128 tiles of 128 x 128 take 17 us, 256 of 128 x 64 27 us)
  if (mt * ((N + 127) / 128) < 100) return 64;
  if (mt * ((N + 255) / 256) >= 148) return 256;
  return 128;
}

}  // namespace

cudaError_t gemm_init() {
  cudaError_t e;
  if ((e = set_attr_bn<64>()) != cudaSuccess) return e;
  if ((e = set_attr_bn<128>()) != cudaSuccess) return e;
  if ((e = set_attr<256, 0, 1, 1, 1, 8>()) != cudaSuccess) return e;
  return set_attr_bn<256>();
}

size_t gemm_ws_floats(int M, int N, int K) {
  // automatic plans split K at most 16 ways
  (void)K;
  return (size_t)16 * M * N;
}

int gemm_plan_tc(GemmPlan* p, const __half* A, long lda, int a_mn, const __half* B, long ldb, int b_mn, int M,
                 int N, int K, const Epilogue& epi, float* ws, size_t ws_floats, int force_bn, int force_splits,
                 int force_cg) {
  *p = GemmPlan();
  p->tc = true;
  p->A = A;
  p->B = B;
  p->lda = lda;
  p->ldb = ldb;
  p->M = M;
  p->N = N;
  p->K = K;
  p->amn = a_mn;
  p->bmn = b_mn;
  p->epi = epi;
  p->ws = ws;
  if (M <= 0 || N <= 0 || K <= 0) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "empty GEMM %dx%dx%d", M, N, K);
    return -1;
  }
  int bn = force_bn ? force_bn : choose_bn(M, N);
  if (bn != 64 && bn != 128 && bn != 256) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "bad BN %d", bn);
    return -1;
  }
  p->bn = bn;
  const int kb = (K + BK - 1) / BK;
  int splits = 1;
  if (force_splits > 0) {
    splits = force_splits;
  } else {
    const int tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    if (tiles < 120 && kb >= 16) {
      splits = 148 / tiles;
      if (splits > kb / 8) splits = kb / 8;
      if (splits > 16) splits = 16;
      if (splits < 1) splits = 1;
    }
  }
  if (splits > kb) splits = kb;
  int kbps = (kb + splits - 1) / splits;
  splits = (kb + kbps - 1) / kbps;
  if (epi.mode == EPI_LSTM_FWD) {
    splits = 1;
    kbps = kb;
  }
  if (splits > 1 && (!ws || ws_floats < (size_t)splits * M * N)) {
    splits = 1;
    kbps = kb;
  }
  if (epi.mode == EPI_LSTM_FWD || epi.mode == EPI_LSTM_BWD) {
    if (epi.hp <= 0 || (epi.hp & 7) || N != (epi.mode == EPI_LSTM_FWD ? 4 * epi.hp : epi.hp)) {
      snprintf(g_gemm_err, sizeof g_gemm_err, "fused cell epilogue: N %d does not match hp %d", N, epi.hp);
      return -1;
    }
    if (epi.mode == EPI_LSTM_BWD && (!ws || ws_floats < (size_t)splits * M * N)) {
      snprintf(g_gemm_err, sizeof g_gemm_err, "fused cell backward needs %zu workspace floats",
               (size_t)splits * M * N);
      return -1;
    }
  }
  p->splits = splits;
  p->kbps = kbps;
  // A multicast across a cluster of CN CTAs sharing the M tile (K-major A only), opt-in via
  // the gemm_cluster_n option (2 or 4).  Measured on the C4 per-step shapes it does not pay (K2 256x8192x2048:
  // 16.7 / 17.6 / 18.4 us at CN = 1 / 2 / 4): those GEMMs are bound by the chip's L2 -> SM
  // operand throughput (~46 B/clk/SM, the same rate the 8192^3 GEMM streams at), which
  // unicast already reaches -- L2 de-duplicates the concurrent reads of the shared A tile
  int cn = 1;
  {
    cn = opt(OPT_GEMM_CLUSTER_N);
    if (cn != 2 && cn != 4 && cn != 8) cn = 1;
    if (a_mn != 0) cn = 1;
  }
  p->cn = cn;
  // CTA pairs (cta_group::2, 256-row tiles): force_cg 1 / 2 (or the gemm_cta_group option) forces; automatic
  // for the large GEMMs (K1, K8, K9): per SM half the B bytes of a 128 x 256 tile for the same
  // flops (8192^3: 1052 -> 1393 TFLOP/s; K1 at C4 961 -> 1105; K9 983 -> 1228).
  // The short-K per-step GEMMs (K2 / K7) measured slower with pairs and keep single CTAs.
  int cg = force_cg;
  {
    if (opt(OPT_GEMM_CTA_GROUP)) cg = opt(OPT_GEMM_CTA_GROUP);
    if (cg == 0) {
      const int pair_tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + bn - 1) / bn) * splits;
      cg = (bn == 256 && N >= 512 && pair_tiles >= 148) ? 2 : 1;
    }
    if (cg != 2 || cn != 1 || bn < 128) cg = 1;
  }
  p->cg = cg;
  // the fused cell backward at 8 K-splits of 256-wide tiles (C4's K7): the splits of a tile
  // reduce inside an 8-CTA cluster (option k7_cluster, off by default: B200 co-schedules at
  // most 15 such clusters of one-CTA-per-SM CTAs, tools/micro/cluster_occ.cu, and C4's K7
  // needs 16 -- the 16th runs as a second wave; C4 step 34.3 -> 59.0 ms with it on)
  {
    const int tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    if (epi.mode == EPI_LSTM_BWD && bn == 256 && splits == 8 && a_mn == 0 && b_mn == 1 && cg == 1 && cn == 1 &&
        tiles * splits <= num_sms() && opt(OPT_K7_CLUSTER))
      p->cr = 8;
  }
  int r;
  if (a_mn == 0)
    r = make_tmap(&p->ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, BM / cn);
  else
    r = make_tmap(&p->ta, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, BK);
  if (r) return r;
  if (b_mn == 0)
    r = make_tmap(&p->tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, (uint32_t)(bn / cg));
  else
    r = make_tmap(&p->tb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, BK);
  return r;
}

int gemm_plan_f32(GemmPlan* p, const float* A, long lda, int a_mn, const float* B, long ldb, int b_mn, int M,
                  int N, int K, const Epilogue& epi) {
  *p = GemmPlan();
  p->tc = false;
  p->A = A;
  p->B = B;
  p->lda = lda;
  p->ldb = ldb;
  p->M = M;
  p->N = N;
  p->K = K;
  p->amn = a_mn;
  p->bmn = b_mn;
  p->epi = epi;
  if (M <= 0 || N <= 0 || K <= 0) return -1;
  if (epi.mode == EPI_F16) {
    snprintf(g_gemm_err, sizeof g_gemm_err, "fp32 GEMM cannot write fp16");
    return -1;
  }
  return 0;
}

cudaError_t gemm_run(const GemmPlan& p, cudaStream_t s) {
  if (!p.tc) {
    const long sam = p.amn ? 1 : p.lda, sak = p.amn ? p.lda : 1;
    const long sbn = p.bmn ? 1 : p.ldb, sbk = p.bmn ? p.ldb : 1;
    dim3 grid((p.M + 63) / 64, (p.N + 63) / 64);
    gemm_f32_kernel<<<grid, 256, 0, s>>>(static_cast<const float*>(p.A), sam, sak, static_cast<const float*>(p.B),
                                         sbn, sbk, p.M, p.N, p.K, p.epi);
    return cudaGetLastError();
  }
  cudaError_t e;
  switch (p.bn) {
    case 64: e = launch_tc_bn<64>(p, s); break;
    case 128: e = launch_tc_bn<128>(p, s); break;
    default: e = launch_tc_bn<256>(p, s); break;
  }
  if (e != cudaSuccess || (p.splits <= 1 && p.epi.mode != EPI_LSTM_BWD) || p.cr > 1) return e;
  const size_t total = (size_t)p.M * p.N;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel, (const float*)p.ws, p.splits, p.M, p.N, p.epi);
}

}  // namespace hdp
