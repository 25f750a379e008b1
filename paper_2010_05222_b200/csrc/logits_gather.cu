// K5 + K6 fused (bf16 tensor-core path, global batch M <= 256): gather of the sampled fp32 W rows, their norms,
// the bf16 operand W_s and the logits contraction in one persistent kernel (Alg.1 L3; the sampled
// rows W_s of L3 are read once from HBM instead of gather -> W_s -> logits re-read).
//
// Per 128-class tile t (sampled positions n0 .. n0+127) and 64-wide K block kb:
//   warps 0-1   producers: TMA of the two X_hat halves (bf16, 128-byte swizzle) + 16-byte cp.async of the sampled
//               fp32 W row chunks (padded pitch) into the stage, all completing on one mbarrier
//   warp 2      tcgen05.mma issuer: C[256 x 128] (two M = 128 halves) += X_hat . bf16(w)^T into TMEM
//   warps 3-6   converters, one thread per class row: fp32 row chunk -> sum of squares (the row norm after the
//               last kb) and bf16, written in place as the K-major swizzled UMMA B tile
//   warp 7      TMA store of that bf16 tile into W_s (the K9 dX operand; rows past k_i are zero)
//   warps 8-15  epilogue: cos = acc / ||w|| (the norm folds in per column, R25), fp16 class-major store and the
//               per-(row, tile) max / sum partials exactly as the unfused logits kernel (gemm_tc.cu)
// W_s holds bf16(w) un-normalised; K8 folds 1/||w_j|| into G (so dX_hat = G' W_s), and the dW / SGD consumers
// take G' = G / ||w|| (R25).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <algorithm>
#include <cstdlib>

#include "pfc_internal.cuh"
#include "tc_common.cuh"

namespace pfc {
namespace {

constexpr int LG_BK = 64;
constexpr int LG_STAGES = 3;
constexpr int LG_ACC = 2;
#ifndef PFC_LG_PROD
#define PFC_LG_PROD 2
#endif
constexpr int LG_PROD = PFC_LG_PROD;                    // producer warps (128 / LG_PROD W rows each; 4: no faster)
constexpr int LG_PRW = 128 / LG_PROD;                   // rows per producer warp
constexpr int LG_MMA_WARP = LG_PROD;
constexpr int LG_CONV0 = LG_MMA_WARP + 1;
constexpr int LG_CONV = 4;                              // converter warps: thread = class row of the tile
constexpr int LG_EPI = 8;                               // epilogue warps: two sets of 4 (64 columns each)
constexpr int LG_STORE_WARP = LG_CONV0 + LG_CONV;
constexpr int LG_EPI_WARP0 = LG_STORE_WARP + 1;
constexpr int LG_THREADS = 32 * (LG_EPI_WARP0 + LG_EPI);
constexpr int LG_PITCH = 272;                           // fp32 chunk pitch: 256 B + 16 (conflict-free LDS.128)
constexpr int LG_A_BYTES = 2 * 128 * LG_BK * 2;         // X_hat, two M halves
constexpr int LG_W_BYTES = 35 * 1024;                   // 128 x 272 B rounded up to 1 KB
constexpr int LG_STAGE = LG_A_BYTES + LG_W_BYTES;
constexpr int LG_AUX = 256 /*barriers*/ + LG_ACC * 128 * 4 /*s_inv*/ + LG_ACC * 2 * 128 * 8 /*s_part*/;
constexpr int LG_SMEM = LG_STAGES * LG_STAGE + 1024 + LG_AUX;
static_assert(LG_SMEM <= 232448, "shared memory overflow");
static_assert(128 * LG_PITCH <= LG_W_BYTES, "W stage too small");
constexpr int LG_WS_OFF = 128 * LG_BK * 2;              // the bf16 W_s tile after the fp16 operand tile
static_assert(2 * LG_WS_OFF <= LG_W_BYTES, "W stage too small for both 16-bit tiles");

struct LgParams {
  int M, ldm, d;
  const SamplerState* st;
  const float* W;          // C_local x d fp32 shard
  const int32_t* idx;      // sampled local rows, ascending
  float* inv_norm;         // out: 1/||w_j|| per sampled position (0 past k_i)
  int* err;
  const int32_t* tcol;     // per row: sampled position of its target or -1
  float s_log2e, scale;
  __half* cosv;            // class-major [k_pad][ldm]
  float2* partials;        // M x n_ltiles
  int n_ltiles;
};

__device__ __forceinline__ uint32_t pack_f16(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// EF (E-form, DESIGN.md f1): store E = bf16(e^{s c}) (c the fp16-rounded cosine the partials use) instead of the
// fp16 cosine: the fused dW/dX kernel then consumes E directly (G = (s/M) e^{-LSE_n} E off the target entries), so
// the softmax-gradient pass over the cosines disappears.
template <bool EF, bool G4, bool WS>
__global__ void __launch_bounds__(LG_THREADS, 1)
    k_logits_gather(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmWs,
                    const __grid_constant__ CUtensorMap tmW, LgParams p) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* aux = smem + LG_STAGES * LG_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* conv = full + LG_STAGES;
  uint64_t* empty = conv + LG_STAGES;
  uint64_t* acc_full = empty + LG_STAGES;
  uint64_t* acc_empty = acc_full + LG_ACC;
  uint64_t* inv_full = acc_empty + LG_ACC;
  uint64_t* inv_empty = inv_full + LG_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(inv_empty + LG_ACC);
  float* s_inv = reinterpret_cast<float*>(aux + 256);                 // [ACC][128]
  float2* s_part = reinterpret_cast<float2*>(s_inv + LG_ACC * 128);   // [ACC][2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = p.st->k;
  const int nt = (k + 127) / 128;                 // class tiles holding sampled classes
  const int n_kb = p.d / LG_BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < LG_STAGES; ++i) {
      mbar_init(&full[i], G4 ? 1 : 1 + 32 * LG_PROD);   // TMA expect_tx (+ one cp.async arrive per producer lane)
      mbar_init(&conv[i], LG_CONV);
      mbar_init(&empty[i], 2);                    // MMA commit + W_s store read back
    }
    for (int i = 0; i < LG_ACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], LG_EPI);
      mbar_init(&inv_full[i], LG_CONV);
      mbar_init(&inv_empty[i], LG_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmWs); if (G4) tma_prefetch(&tmW); }
  if (warp == LG_MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (G4 && warp < LG_PROD) {
    // ---------------------------------------------------------------- producer (TMA gather4 variant)
    // lane l gathers rows 4l .. 4l + 3 of the tile: two 32-column boxes (128 B per row, 128-byte swizzle) per K
    // block, the two halves 16 KB apart; rows past k_i fetch row 0 (their converter threads write zeros)
    if (warp == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < nt; t += gridDim.x) {
        const int n0 = t * 128;
        int r4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = n0 + 4 * lane + i;
          r4[i] = r < k ? p.idx[r] : 0;
        }
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * LG_STAGE;
          uint8_t* sw = sa + LG_A_BYTES;
          if (lane == 0) {
            mbar_expect_tx(&full[stage], (uint32_t)(LG_A_BYTES + 128 * LG_BK * 4));
            tma_load_2d(sa, &tmA, &full[stage], kb * LG_BK, 0);
            tma_load_2d(sa + 128 * LG_BK * 2, &tmA, &full[stage], kb * LG_BK, 128);
          }
          __syncwarp();
#pragma unroll
          for (int h = 0; h < 2; ++h)
            tma_gather4(sw + h * 16384 + lane * 512, &tmW, &full[stage], kb * LG_BK + h * 32, r4[0], r4[1], r4[2], r4[3]);
          if (++stage == LG_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp < LG_PROD) {
    // ---------------------------------------------------------------- producers
    // W rows: 16-byte cp.async (LDGSTS); a warp instruction moves two rows x 256 B (coalesced); warp pw owns
    // rows LG_PRW pw .. LG_PRW (pw + 1) - 1 of the tile, their ids held in registers for the whole tile; completion is
    // tracked by the stage mbarrier (cp.async.mbarrier.arrive.noinc). X_hat by TMA. (One 256-byte
    // cp.async.bulk per row, a single producer warp reading row ids from smem, and TMA tile::gather4 of 128-byte row
    // boxes (PFC_LG_G4=1, the variant branch above) were measured slower.)
    int stage = 0;
    uint32_t phase = 0;
    const int half = lane >> 4, ch = lane & 15;
    const int rbase = warp * LG_PRW + half;
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      const int n0 = t * 128;
      int rid[LG_PRW / 2];
#pragma unroll
      for (int i = 0; i < LG_PRW / 2; ++i) {
        const int r = n0 + rbase + 2 * i;
        rid[i] = r < k ? p.idx[r] : -1;
      }
      for (int kb = 0; kb < n_kb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * LG_STAGE;
        uint8_t* sw = sa + LG_A_BYTES;
        if (warp == 0 && lane == 0) {
          mbar_expect_tx(&full[stage], (uint32_t)LG_A_BYTES);
          tma_load_2d(sa, &tmA, &full[stage], kb * LG_BK, 0);
          tma_load_2d(sa + 128 * LG_BK * 2, &tmA, &full[stage], kb * LG_BK, 128);
        }
        const uint32_t dst0 = smem_u32(sw) + rbase * LG_PITCH + ch * 16;
        const float* srcc = p.W + kb * LG_BK + ch * 4;
#pragma unroll
        for (int i = 0; i < LG_PRW / 2; ++i) {
          if (rid[i] >= 0)
            asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst0 + 2 * i * LG_PITCH),
                         "l"(srcc + (int64_t)rid[i] * p.d)
                         : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[stage])) : "memory");
        if (++stage == LG_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == LG_MMA_WARP) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC = make_idesc(128, 128, false, false, true);   // fp16 operands (R27)
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tacc = tmem_base + acc * 256;
      for (int kb = 0; kb < n_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&conv[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * LG_STAGE);
          const uint32_t sb = sa + LG_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < LG_BK / 16; ++kk) {
#pragma unroll
            for (int ms = 0; ms < 2; ++ms)
              tc_mma(tacc + ms * 128, make_desc(sa + ms * 128 * LG_BK * 2 + kk * 32, 16, 1024),
                     make_desc(sb + kk * 32, 16, 1024), IDESC, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == LG_STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tc_commit(&acc_full[acc]);
      __syncwarp();
      if (++acc == LG_ACC) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp < LG_STORE_WARP) {
    // ---------------------------------------------------------------- converters (thread = class row r)
    const int r = (warp - LG_CONV0) * 32 + lane;
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      const int n0 = t * 128;
      const bool valid = n0 + r < k;
      float ss = 0.f, amax = 0.f;
      for (int kb = 0; kb < n_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        uint8_t* sw = smem + stage * LG_STAGE + LG_A_BYTES;
        uint32_t pk[32], pb[32];
        constexpr bool wb = WS;
        if (valid) {
          const float4* src = reinterpret_cast<const float4*>(sw + r * LG_PITCH);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            // gather4 layout: half q / 8 (16 KB apart), row r at 128 B, 16-byte chunk (q % 8) ^ (r % 8)
            const float4 v = G4 ? *reinterpret_cast<const float4*>(sw + (q >> 3) * 16384 + r * 128 +
                                                                   (((q & 7) ^ (r & 7)) << 4))
                                  : src[q];
            ss = fmaf(v.x, v.x, ss); ss = fmaf(v.y, v.y, ss); ss = fmaf(v.z, v.z, ss); ss = fmaf(v.w, v.w, ss);
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
            pk[2 * q] = pack_f16(v.x, v.y);
            pk[2 * q + 1] = pack_f16(v.z, v.w);
            if (wb) {
              pb[2 * q] = pack_bf16(v.x, v.y);
              pb[2 * q + 1] = pack_bf16(v.z, v.w);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) pk[q] = pb[q] = 0u;
        }
        // every row read before the 16-bit tiles overwrite the head of the fp32 buffer
        asm volatile("bar.sync 5, %0;" ::"n"(32 * LG_CONV) : "memory");
        // K-major SW128: row r, 16-byte chunk c ^ (r % 8); the fp16 tile is the MMA operand (R27), the bf16 tile
        // (16 KB further) the W_s copy for the separate dX contraction
        uint4* dst = reinterpret_cast<uint4*>(sw + r * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) dst[c ^ (r & 7)] = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        if (wb) {
          uint4* dstb = reinterpret_cast<uint4*>(sw + LG_WS_OFF + r * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            dstb[c ^ (r & 7)] = make_uint4(pb[4 * c], pb[4 * c + 1], pb[4 * c + 2], pb[4 * c + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[stage]);
        if (++stage == LG_STAGES) { stage = 0; phase ^= 1; }
      }
      const float nrm = sqrtf(ss);
      const float inv = valid ? 1.f / fmaxf(nrm, kNormEps) : 0.f;
      p.inv_norm[n0 + r] = inv;
      if (valid && !(nrm > 0.f)) atomicOr(p.err, ERR_DEGENERATE);
      if (amax >= 65504.f) atomicOr(p.err, ERR_NUMERIC);   // an element outside the fp16 operand range (R27)
      mbar_wait(&inv_empty[acc], acc_phase ^ 1);
      s_inv[acc * 128 + r] = inv;
      __syncwarp();
      if (lane == 0) mbar_arrive(&inv_full[acc]);
      if (++acc == LG_ACC) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp == LG_STORE_WARP) {
    // ---------------------------------------------------------------- W_s store (bf16 tile -> global)
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      for (int kb = 0; kb < n_kb; ++kb) {
        mbar_wait(&conv[stage], phase);
        if (lane == 0) {
          if (WS) {
            tma_store_2d(&tmWs, smem + stage * LG_STAGE + LG_A_BYTES + LG_WS_OFF, kb * LG_BK, t * 128);
            bulk_commit();
            bulk_wait_read0();                      // smem read back: the stage may be refilled
          }
          mbar_arrive(&empty[stage]);
        }
        __syncwarp();
        if (++stage == LG_STAGES) { stage = 0; phase ^= 1; }
      }
    }
    if (lane == 0) bulk_wait0();
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - LG_EPI_WARP0;
    const int lg = warp & 3;                 // TMEM lane quarter of this warp
    const int row_in = lg * 32 + lane;
    const int eset = ew >> 2;                // two sets of 4 warps: columns 64*eset .. +63
    const float sl = p.s_log2e;
    int acc = 0;
    uint32_t acc_phase = 0;
    // the (max, sum) of this thread's rows over every class tile of this CTA, folded in the CTA's fixed tile order:
    // one partial per (row, CTA) at the end instead of k / 128 (row_combine reads gridDim.x slots per row)
    float racc_m[2] = {-INFINITY, -INFINITY}, racc_l[2] = {0.f, 0.f};
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      const int n0 = t * 128;
      mbar_wait(&inv_full[acc], acc_phase);
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(lg * 32) << 16) + acc * 256;
      const float* inv_t = s_inv + acc * 128;
      float pm[2], ps[2];
#pragma unroll
      for (int ms = 0; ms < 2; ++ms) {
        const int row = ms * 128 + row_in;
        const bool rv = row < p.M;
        const int tc = rv ? p.tcol[row] : -1;
        float mx = EF ? 0.f : -INFINITY, sum = 0.f;   // EF: unshifted sums (s + ln k < 80, api.cu)
#pragma unroll 1
        for (int c = eset * 2; c < eset * 2 + 2; ++c) {
          uint32_t v[32];
          tmem_ld32(tacc + ms * 128 + c * 32, v);
          const int col0 = n0 + c * 32;
          const float4* iv = reinterpret_cast<const float4*>(inv_t + c * 32);
          __half2 h2[16];
          float cf[32];
#pragma unroll
          if (EF) {   // E is formed from the fp32 cosine (no cosine is stored: no fp16 rounding to match, R26)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 s4 = iv[q];
              cf[4 * q] = __uint_as_float(v[4 * q]) * s4.x;
              cf[4 * q + 1] = __uint_as_float(v[4 * q + 1]) * s4.y;
              cf[4 * q + 2] = __uint_as_float(v[4 * q + 2]) * s4.z;
              cf[4 * q + 3] = __uint_as_float(v[4 * q + 3]) * s4.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {   // fp16 cosine stored; the partials use the fp32 value (R27)
              const float4 s4 = iv[q];
              cf[4 * q] = __uint_as_float(v[4 * q]) * s4.x;
              cf[4 * q + 1] = __uint_as_float(v[4 * q + 1]) * s4.y;
              cf[4 * q + 2] = __uint_as_float(v[4 * q + 2]) * s4.z;
              cf[4 * q + 3] = __uint_as_float(v[4 * q + 3]) * s4.w;
              h2[2 * q] = __floats2half2_rn(cf[4 * q], cf[4 * q + 1]);
              h2[2 * q + 1] = __floats2half2_rn(cf[4 * q + 2], cf[4 * q + 3]);
            }
          }
          if (col0 + 32 > k || (unsigned)(tc - col0) < 32u) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col0 + j >= k || col0 + j == tc) cf[j] = -INFINITY;
          }
          if (EF) {   // E_j = e^{s c_j} = 2^{c_j s log2 e} unshifted (0 at the target / padding columns: c = -inf)
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) cf[j] = ex2_ftz(cf[j] * sl);
#pragma unroll
            for (int j = 0; j < 32; j += 4) { s0 += cf[j]; s1 += cf[j + 1]; s2 += cf[j + 2]; s3 += cf[j + 3]; }
            sum += (s0 + s1) + (s2 + s3);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const __nv_bfloat162 b = __floats2bfloat162_rn(cf[2 * i], cf[2 * i + 1]);
              h2[i] = *reinterpret_cast<const __half2*>(&b);   // bit pattern carried through the store below
            }
          } else {
            float q0 = cf[0], q1 = cf[1], q2 = cf[2], q3 = cf[3];
#pragma unroll
            for (int j = 4; j < 32; j += 4) {
              q0 = fmaxf(q0, cf[j]); q1 = fmaxf(q1, cf[j + 1]); q2 = fmaxf(q2, cf[j + 2]); q3 = fmaxf(q3, cf[j + 3]);
            }
            const float nmx = fmaxf(mx, fmaxf(fmaxf(q0, q1), fmaxf(q2, q3)));
            if (nmx > -INFINITY) {
              const float nb = nmx * sl;
              float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                s0 += ex2_ftz(fmaf(cf[j], sl, -nb));
                s1 += ex2_ftz(fmaf(cf[j + 1], sl, -nb));
                s2 += ex2_ftz(fmaf(cf[j + 2], sl, -nb));
                s3 += ex2_ftz(fmaf(cf[j + 3], sl, -nb));
              }
              sum = (mx > -INFINITY ? sum * ex2_ftz((mx - nmx) * sl) : 0.f) + ((s0 + s1) + (s2 + s3));
              mx = nmx;
            }
          }
          // class-major store, lane pairs exchanging halves: each 32-bit store covers rows (n, n+1) of one class
          const bool odd = lane & 1;
          __half* cb = p.cosv + (row & ~1);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const __half send = odd ? __low2half(h2[i]) : __high2half(h2[i]);
            const unsigned short rcv = (unsigned short)__shfl_xor_sync(0xffffffffu, (int)__half_as_ushort(send), 1);
            const __half other = __ushort_as_half(rcv);
            const __half2 pr = odd ? __halves2half2(other, __high2half(h2[i])) : __halves2half2(__low2half(h2[i]), other);
            if (row < p.ldm) *reinterpret_cast<__half2*>(cb + (int64_t)(col0 + 2 * i + (odd ? 1 : 0)) * p.ldm) = pr;
          }
        }
        pm[ms] = mx;
        ps[ms] = sum;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) { mbar_arrive(&acc_empty[acc]); mbar_arrive(&inv_empty[acc]); }
      float2* sp = s_part + acc * 256;
      if (eset == 1) {
#pragma unroll
        for (int ms = 0; ms < 2; ++ms) sp[ms * 128 + row_in] = make_float2(pm[ms], ps[ms]);
      }
      asm volatile("bar.sync 4, %0;" ::"n"(32 * LG_EPI) : "memory");
      if (eset == 0) {
#pragma unroll
        for (int ms = 0; ms < 2; ++ms) {
          const int row = ms * 128 + row_in;
          const float2 o = sp[ms * 128 + row_in];
          const float m = fmaxf(pm[ms], o.x);
          float l = 0.f;
          if (m > -INFINITY)
            l = (pm[ms] > -INFINITY ? ps[ms] * ex2_ftz((pm[ms] - m) * sl) : 0.f) +
                (o.x > -INFINITY ? o.y * ex2_ftz((o.x - m) * sl) : 0.f);
          (void)row;
          const float nm = fmaxf(racc_m[ms], m);
          if (nm > -INFINITY) {
            racc_l[ms] = (racc_m[ms] > -INFINITY ? racc_l[ms] * ex2_ftz((racc_m[ms] - nm) * sl) : 0.f) +
                         (m > -INFINITY ? l * ex2_ftz((m - nm) * sl) : 0.f);
            racc_m[ms] = nm;
          }
        }
      }
      if (++acc == LG_ACC) { acc = 0; acc_phase ^= 1; }
    }
    if (eset == 0) {   // slot blockIdx.x of each row (written also when this CTA had no tile: -inf, 0)
#pragma unroll
      for (int ms = 0; ms < 2; ++ms) {
        const int row = ms * 128 + row_in;
        if (row < p.M)
          p.partials[(int64_t)row * p.n_ltiles + blockIdx.x] =
              make_float2(racc_m[ms] > -INFINITY ? racc_m[ms] * p.scale : -INFINITY, racc_l[ms]);
      }
    }
  }
  __syncthreads();
  if (warp == LG_MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

}  // namespace

bool logits_gather_supported(const Sizes& sz) {
  const int forced = env_int("PFC_FUSED_GATHER", 1);
  return forced != 0 && sz.M <= 256 && sz.d % LG_BK == 0 && sz.k_pad % 128 == 0;
}

int launch_logits_gather_tc(const Sizes& sz, const float* W, const int32_t* idx, const __half* Xh,
                            __nv_bfloat16* Ws, bool write_ws, float* inv_norm, const int32_t* tcol, const SamplerState* st,
                            MarginParams mp, __half* cosv, float2* partials, int* err, bool eform, int* nparts,
                            cudaStream_t s) {
  // WS: the bf16 W_s copy is stored (the separate dX GEMM needs it; the fused dW/dX kernel does not)
  using KernT = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, LgParams);
  static const KernT kerns[8] = {k_logits_gather<false, false, false>, k_logits_gather<false, false, true>,
                                 k_logits_gather<false, true, false>,  k_logits_gather<false, true, true>,
                                 k_logits_gather<true, false, false>,  k_logits_gather<true, false, true>,
                                 k_logits_gather<true, true, false>,   k_logits_gather<true, true, true>};
  static bool attr = false;
  if (!attr) {
    for (KernT k : kerns) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, LG_SMEM);
    attr = true;
  }
  const CUtensorMap a = make_map(Xh, sz.M_pad, sz.d, 64, 128);   // fp16 X_hat (R27)
  const CUtensorMap ws = make_map(Ws, sz.k_pad, sz.d, 64, 128);
  const int g4 = env_int("PFC_LG_G4", 0);
  const CUtensorMap wm = g4 ? make_map_typed(W, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)sz.C_local, sz.d, 32, 1)
                            : ws;
  TC_MAPS_OK();
  LgParams p{};
  p.M = sz.M; p.ldm = sz.M_pad; p.d = sz.d; p.st = st; p.W = W; p.idx = idx; p.inv_norm = inv_norm; p.err = err;
  p.tcol = tcol; p.s_log2e = mp.s * 1.4426950408889634f; p.scale = mp.s; p.cosv = cosv; p.partials = partials;
  p.n_ltiles = sz.n_ltiles;
  const int grid = (int)std::min<int64_t>(sz.k_pad / 128, num_sms());
  *nparts = grid;   // one folded LSE partial per (row, CTA)
  // G4 (PFC_LG_G4=1): the W rows by TMA tile::gather4 (128-byte swizzled 32-column boxes); parity holds, measured
  // 2x slower at C4 (1.07 vs 0.55 ms: ~19 cycles of TMA per 128-byte row)
  launch_pdl(kerns[(eform ? 4 : 0) + (g4 ? 2 : 0) + (write_ws ? 1 : 0)], dim3(grid), dim3(LG_THREADS), LG_SMEM, s, a, ws, wm, p);
  return 1;
}

}  // namespace pfc
