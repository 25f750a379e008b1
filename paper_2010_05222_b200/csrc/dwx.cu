// K9 + K11 + K12 fused (train step, bf16 tensor-core path, global batch M <= 256): one persistent kernel computes,
// per 128-class tile of the sampled shard,
//   dW_hat tile  D1[128 x 128] = G'^T X_hat            (Alg.1 L10, tcgen05.mma: A = G' K-major, B = X_hat MN-major)
//   the lazy momentum-SGD update of those W / V rows  (as K12 / the DWF kernel of gemm_tc.cu)
//   dX_hat partial D2[M x 128] += G' bf16(w_old)       (Alg.1 L12, A = G' MN-major, B = bf16(w) MN-major)
// The old W rows the update loads anyway are converted to bf16 in shared memory and fed to the dX contraction, so
// neither the bf16 copy W_s (written by the logits kernel otherwise) nor a separate dX GEMM pass over it is needed.
// G' = G / ||w_j|| (R25) makes bf16(w) un-normalised the right operand: dX_hat = sum_j G'_nj w_j.
//
// CTA b owns the 128-column d-tile b / gper and the class tiles g, g + gper, ... (g = b % gper); its dX_hat
// partial for that d-tile stays in TMEM for the whole kernel and is written once to the split workspace, reduced
// over g by k_splitk_reduce (deterministic order).
//   warp 0    TMA producer: the dW operands (G' and X_hat 64-batch chunks, 2-stage ring) and, a tile behind, a
//             second copy of the whole G' tile (an L2 hit) for the dX contraction
//   warp 1    MMA issuer: dW(t) into D1[t % 2], then dX(t - 1) into D2 once the epilogue has staged bf16 w_old(t - 1)
//   warps 2-9 epilogue per tile: D1 -> smem, coalesced W / V row updates (rows L2-prefetched a tile ahead) that
//             also stage the old w as the bf16 dX operand
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pfc_internal.cuh"
#include "tc_common.cuh"

namespace pfc {
namespace {

constexpr int DX_EPI = 8;
#ifndef PFC_DWX_DIAG
#define PFC_DWX_DIAG 0
#endif
// build-time diagnostics (PFC_BUILD_TAG=diag PFC_NVCC_EXTRA=-DPFC_DWX_DIAG=1): the per-tile epilogue trace
// (PFC_DWX_TRACE) and the prefetch-timing variants (PFC_DWX_PF = 0 / 2 / 3) of k_dwx_t; compiled out by default,
// where their checks cost the kernel 3-4% (measured)
constexpr bool kDiag = PFC_DWX_DIAG != 0;
#ifndef PFC_DX_DOTW
#define PFC_DX_DOTW 2
#endif
constexpr int DX_DOTW = PFC_DX_DOTW;        // E-form: warps forming the radial dot from the E chunks
constexpr int DX_THREADS = 64 + 32 * DX_EPI;
constexpr int DX_THREADS_EF = DX_THREADS + 32 * DX_DOTW;
constexpr int G_CHUNK = 128 * 64 * 2;       // 128 classes x 64 batch columns (bf16, 128-byte swizzle)
constexpr int G_BUF = 4 * G_CHUNK;          // M_pad <= 256
constexpr int X_CHUNK = 64 * 128 * 2;       // 64 batch rows x 128 columns (two 64-column swizzled halves)
constexpr int R_STAGES = 2;                 // dW operand ring: (G' chunk, X_hat chunk) per stage
constexpr int R_STAGE = G_CHUNK + X_CHUNK;
constexpr int WB_HALF = 128 * 128;          // 128 classes x 64 columns bf16
constexpr int OFF_R = 0;
constexpr int OFF_G = OFF_R + R_STAGES * R_STAGE;   // the dX operand: the whole G' tile, loaded a second time
constexpr int OFF_WB = OFF_G + G_BUF;
constexpr int OFF_ST = OFF_WB + 2 * WB_HALF;
constexpr int OFF_AUX = OFF_ST + 128 * 128 * 4;
constexpr int DX_SMEM = OFF_AUX + 256 + 3 * 128 * 4 + 1024;
static_assert(DX_SMEM <= 232448, "shared memory overflow");

struct DwxParams {
  int M, d, nkb;        // nkb = M_pad / 64
  int gper;             // CTAs per d-tile
  const SamplerState* st;
  SgdArgs sgd;
  float* ws;            // [gper][M][d] dX_hat partials
  // E-form (DESIGN.md f1): the G operand is E (bf16 e^{s c}, target entries G_t / f_n), the dW operand X~ = f X_hat
  const float* f;       // [M] f_n = (s/M) e^{-LSE_n}
  const int32_t* tcol;  // [M] sampled position of row n's target or -1
  const float* dcorr;   // [k_pad] sum of G_t c_t over the target entries of each sampled class
  float* xch;           // [nct][n_dt][128] per-d-tile partial radial dots
  int* cnt;             // [nct] partials published per class tile (zeroed each step)
  int* err;
  float s;              // logit scale
  int pfnow;            // prefetch the current tile's W / V rows at its start (as well as the next tile's)
  int pf;               // PFC_DWX_PF: 1 (default) the next tile's W / V rows into L2 during this tile's update; 0 none;
                        // 2 two tiles ahead; 3 the next tile's at this tile's start (k_dwx_t: diagnostic builds)
  uint64_t* trace;      // PFC_DWX_TRACE=1 (eager launches): per-tile epilogue timestamps, [cta][tile][8]
  int trace_tiles;
};

__device__ __forceinline__ uint64_t gtimer_dx() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <bool HINT, bool EF>
__global__ void __launch_bounds__(EF ? DX_THREADS_EF : DX_THREADS, 1)
    k_dwx_t(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmX, DwxParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sR = smem + OFF_R;
  uint8_t* sG = smem + OFF_G;
  uint8_t* sWb = smem + OFF_WB;
  float4* s_tile = reinterpret_cast<float4*>(smem + OFF_ST);     // [128 rows][32 float4], XOR-swizzled
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_AUX);
  uint64_t* g_full = bars;            // dX copy of the G' tile
  uint64_t* g_empty = bars + 1;
  uint64_t* x_full = bars + 2;        // [R_STAGES] dW operand ring
  uint64_t* x_empty = bars + 6;       // [R_STAGES]
  uint64_t* d1_full = bars + 10;      // [2]
  uint64_t* d1_empty = bars + 12;     // [2]
  uint64_t* wb_full = bars + 14;
  uint64_t* wb_empty = bars + 15;
  uint64_t* d2_full = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  int32_t* s_rowj = reinterpret_cast<int32_t*>(smem + OFF_AUX + 256);
  float* s_inv = reinterpret_cast<float*>(s_rowj + 128);
  float* s_rad = s_inv + 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = p.st->k;
  const int nct = (k + 127) / 128;
  const int g = blockIdx.x % p.gper;
  const int n0 = (blockIdx.x / p.gper) * 128;               // this CTA's d-tile
  const int ntl = g < nct ? (nct - g + p.gper - 1) / p.gper : 0;
  const int nkb = p.nkb, nh = p.nkb / 2 > 0 ? p.nkb / 2 : 1;   // dX M-halves of 128 batch rows

  if (threadIdx.x == 0) {
    mbar_init(g_full, 1); mbar_init(g_empty, 1);
    for (int i = 0; i < R_STAGES; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], EF ? 1 + DX_DOTW : 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&d1_full[i], 1); mbar_init(&d1_empty[i], DX_EPI); }
    mbar_init(wb_full, DX_EPI);
    mbar_init(wb_empty, 1);
    mbar_init(d2_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmG); tma_prefetch(&tmX); }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;     // cols [0, 256): D1 x 2; [256, 512): D2 halves

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      int xs = 0;
      uint32_t xph = 0;
      auto load_gdx = [&](int i) {     // the dX operand copy of tile i's G' (an L2 hit: read for dW(i) before)
        mbar_wait(g_empty, (uint32_t)((i & 1) ^ 1));       // dX(i - 1) has read the previous copy
        mbar_expect_tx(g_full, (uint32_t)(nkb * G_CHUNK));
        for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sG + kb * G_CHUNK, &tmG, g_full, kb * 64, (g + i * p.gper) * 128);
      };
      for (int i = 0; i < ntl; ++i) {
        const int ct = g + i * p.gper;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&x_empty[xs], xph ^ 1);
          mbar_expect_tx(&x_full[xs], (uint32_t)R_STAGE);
          uint8_t* st = sR + xs * R_STAGE;
          tma_load_2d(st, &tmG, &x_full[xs], kb * 64, ct * 128);
          tma_load_2d(st + G_CHUNK, &tmX, &x_full[xs], n0, kb * 64);
          tma_load_2d(st + G_CHUNK + X_CHUNK / 2, &tmX, &x_full[xs], n0 + 64, kb * 64);
          if (++xs == R_STAGES) { xs = 0; xph ^= 1; }
        }
        if (i > 0) load_gdx(i - 1);
      }
      if (ntl > 0) load_gdx(ntl - 1);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC_DW = make_idesc(128, 128, false, true);
    constexpr uint32_t IDESC_DX = make_idesc(128, 128, true, true);
    int xs = 0, acc = 0;
    uint32_t xph = 0, aph = 0;
    auto dx = [&](int i) {      // D2 += G'(tile i) bf16(w_old(tile i)), then release both operands
      mbar_wait(wb_full, (uint32_t)(i & 1));
      mbar_wait(g_full, (uint32_t)(i & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint32_t ga = smem_u32(sG), wa = smem_u32(sWb);
        for (int h = 0; h < nh; ++h)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma(tmem_base + 256 + h * 128, make_desc(ga + 2 * h * G_CHUNK + ks * 2048, G_CHUNK, 1024),
                   make_desc(wa + ks * 2048, WB_HALF, 1024), IDESC_DX, (i > 0 || ks > 0) ? 1u : 0u);
        tc_commit(g_empty);
        tc_commit(wb_empty);
      }
      __syncwarp();
    };
    for (int i = 0; i < ntl; ++i) {
      mbar_wait(&d1_empty[acc], aph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&x_full[xs], xph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ga = smem_u32(sR + xs * R_STAGE), xa = ga + G_CHUNK;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma(tmem_base + acc * 128, make_desc(ga + kk * 32, 16, 1024), make_desc(xa + kk * 2048, X_CHUNK / 2, 1024),
                   IDESC_DW, (kb > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&x_empty[xs]);
        }
        __syncwarp();
        if (++xs == R_STAGES) { xs = 0; xph ^= 1; }
      }
      if (lane == 0) tc_commit(&d1_full[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; aph ^= 1; }
      if (i > 0) dx(i - 1);     // bf16 w_old(t - 1) is staged by the epilogue's update of tile t - 1
    }
    if (ntl > 0) dx(ntl - 1);
    if (lane == 0) {
      if (ntl > 0) tc_commit(d2_full);
      else mbar_arrive(d2_full);
    }
    __syncwarp();
  } else if (warp >= 2 + DX_EPI) {
    // ---------------------------------------------------------------- E-form radial dot (2 warps)
    // dotw_j = sum_n G_nj c_nj (the w-normalisation backprop, Eq.6): off the target entries G = f_n E and
    // c = ln(E)/s, so each E chunk of the dW ring contributes (ln2/s) sum_n f_n E lg2(E); the target entries
    // (E' = G_t/f_n < 0, clamped away) contribute G_t c_t through dcorr (k_eform_prep). This CTA covers the batch
    // chunks kb = dt mod n_dt of its class tiles and publishes its partial per class row; the epilogues of the
    // n_dt d-tile CTAs sum them.
    if (EF) {
      constexpr int RPT = 128 / (32 * DX_DOTW);        // tile rows per thread: t, t + 32 DX_DOTW, ...
      const int t = threadIdx.x - 32 * (2 + DX_EPI);
      const int n_dt = p.d / 128, dt = blockIdx.x / p.gper;
      const float kc = 0.69314718f / p.s;
      int xs = 0;
      uint32_t xph = 0;
      for (int i = 0; i < ntl; ++i) {
        const int ct = g + i * p.gper;
        float B[RPT];   // sum_n f_n E lg2(E) over this CTA's chunks
#pragma unroll
        for (int q = 0; q < RPT; ++q) B[q] = 0.f;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&x_full[xs], xph);
          if (kb % n_dt == dt) {
            const uint8_t* ga = sR + xs * R_STAGE;
            const float4* f4 = reinterpret_cast<const float4*>(p.f + kb * 64);
#pragma unroll 2
            for (int u = 0; u < 8; ++u) {
              const float4 fa = __ldg(f4 + 2 * u), fb = __ldg(f4 + 2 * u + 1);
              const float fv[8] = {fa.x, fa.y, fa.z, fa.w, fb.x, fb.y, fb.z, fb.w};
#pragma unroll
              for (int q = 0; q < RPT; ++q) {
                const int row = t + q * 32 * DX_DOTW;
                const uint4 qv = *reinterpret_cast<const uint4*>(ga + row * 128 + ((u ^ (row & 7)) << 4));
                const uint32_t r[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                  const float el = fmaxf(__uint_as_float(r[e2] << 16), 1e-37f);
                  const float eh = fmaxf(__uint_as_float(r[e2] & 0xFFFF0000u), 1e-37f);
                  float ll, lh;
                  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(ll) : "f"(el));
                  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lh) : "f"(eh));
                  B[q] = fmaf(el * fv[2 * e2], ll, fmaf(eh * fv[2 * e2 + 1], lh, B[q]));
                }
              }
            }
          }
          __syncwarp();
          if ((t & 31) == 0) mbar_arrive(&x_empty[xs]);
          if (++xs == R_STAGES) { xs = 0; xph ^= 1; }
        }
        float* dst = p.xch + ((int64_t)ct * n_dt + dt) * 128;
#pragma unroll
        for (int q = 0; q < RPT; ++q) dst[t + q * 32 * DX_DOTW] = kc * B[q];
        if (DX_DOTW > 1) asm volatile("bar.sync 5, %0;" ::"n"(32 * DX_DOTW) : "memory");
        else __syncwarp();
        if (kDiag && t == 0 && p.trace && i < p.trace_tiles) p.trace[((int64_t)blockIdx.x * p.trace_tiles + i) * 8 + 7] = gtimer_dx();
        if (t == 0) {
          // release (cumulative over the barrier above): the partials are visible at gpu scope before the count
          // (the epilogues poll it with acquire loads)
          asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.cnt + ct) : "memory");
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int lg = warp & 3;
    const int row_in = lg * 32 + lane;
    const int eset = ew >> 2;
    const float lr = *p.sgd.lr;
    const uint64_t pol = HINT ? policy_evict_first() : 0;
    int32_t nx_j = -1;
    float nx_inv = 0.f, nx_rad = 0.f;
    if (eset == 0 && ntl > 0) {
      const int prow = g * 128 + row_in;
      if (prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; nx_rad = EF ? 0.f : p.sgd.dotw[prow]; }
    }
    int acc = 0;
    uint32_t aph = 0;
    const int col = n0 + lane * 4;           // row-update mapping: one 512-byte row segment per warp instruction
    for (int i = 0; i < ntl; ++i) {
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DX_EPI) : "memory");   // previous tile fully consumed
      uint64_t* tr = (kDiag && p.trace && threadIdx.x == 64 && i < p.trace_tiles)
                         ? p.trace + ((int64_t)blockIdx.x * p.trace_tiles + i) * 8 : nullptr;
      if (tr) tr[0] = gtimer_dx();
      if (eset == 0) {
        s_rowj[row_in] = nx_j; s_inv[row_in] = nx_inv; s_rad[row_in] = nx_rad;
        if (kDiag && p.pfnow && nx_j >= 0) {   // this tile's W / V row segments into L2 (PFC_DWX_PFNOW=1, diag)
          const float* wp = p.sgd.W + (int64_t)nx_j * p.d + n0;
          const float* vp = p.sgd.V + (int64_t)nx_j * p.d + n0;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
          }
        }
        nx_j = -1; nx_inv = 0.f; nx_rad = 0.f;
        if (i + 1 < ntl) {
          const int prow = (g + (i + 1) * p.gper) * 128 + row_in;
          if (prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; nx_rad = EF ? 0.f : p.sgd.dotw[prow]; }
        }
        if (kDiag && p.pf == 3 && nx_j >= 0) {   // the next tile's rows into L2 now, a whole tile ahead
          const float* wp = p.sgd.W + (int64_t)nx_j * p.d + n0;
          const float* vp = p.sgd.V + (int64_t)nx_j * p.d + n0;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
          }
        }
      }
      // (2) D1 -> smem staging (XOR-swizzled float4 rows), TMEM released
      mbar_wait(&d1_full[acc], aph);
      tc_fence_after();
      if (tr) tr[1] = gtimer_dx();
      float rad16 = 0.f;   // E-form: lane l < 16 forms the radial dot of row ew * 16 + l
      float radp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (EF) {
        // the radial dots of this warp's 16 rows: the n_dt d-tile CTAs' partials (all CTAs are resident: one per
        // SM; their dotw warps finish this tile with its dW operands), loads in flight during the staging
        const int ct = g + i * p.gper, n_dt = p.d / 128;
        if (lane == 0) {
          const int* c = p.cnt + ct;
          int v, spins = 0;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
          } while (v < n_dt && ++spins < (1 << 26));
          if (v < n_dt) atomicOr(p.err, ERR_INTERNAL);   // never expected: bounded instead of a hang
        }
        __syncwarp();
        if (tr) tr[2] = gtimer_dx();
        if (lane < 16) {   // loads only: summed after the staging
          const int row = ew * 16 + lane;
          rad16 = __ldcg(p.dcorr + ct * 128 + row);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < n_dt) radp[q] = __ldcg(p.xch + ((int64_t)ct * n_dt + q) * 128 + row);
        }
      }
      {
        const uint32_t tacc = tmem_base + ((uint32_t)(lg * 32) << 16) + acc * 128;
#pragma unroll 1
        for (int c = eset * 2; c < eset * 2 + 2; ++c) {
          uint32_t v[32];
          tmem_ld32(tacc + c * 32, v);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            s_tile[row_in * 32 + ((c * 8 + q) ^ (row_in & 31))] =
                make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                            __uint_as_float(v[4 * q + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d1_empty[acc]);
      if (++acc == 2) { acc = 0; aph ^= 1; }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DX_EPI) : "memory");
      if (tr) tr[3] = gtimer_dx();
      // (3) momentum-SGD row updates (rows L2-prefetched a tile ahead), 8 rows in flight per lane; the old w
      // also goes to the bf16 dX operand tile, once dX(t - 1) has read the previous one
      mbar_wait(wb_empty, (uint32_t)((i & 1) ^ 1));
      if (tr) tr[4] = gtimer_dx();
      if (EF) {   // into the per-row slot the update loop reads (a shuffle there serialises the row updates)
#pragma unroll
        for (int q = 0; q < 8; ++q) rad16 += radp[q];
        if (lane < 16) s_rad[ew * 16 + lane] = rad16;
        __syncwarp();
      }
#pragma unroll 1
      for (int r0 = 0; r0 < 16; r0 += 8) {
        float4 wv[8], mv[8];
        int32_t jr[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          jr[r] = s_rowj[ew * 16 + r0 + r];
          PFC_DCHECK(jr[r] < p.sgd.rows);
          if (jr[r] >= 0) {
            if (HINT) {
              wv[r] = ld_hint4(p.sgd.W + (int64_t)jr[r] * p.d + col, pol);
              mv[r] = ld_hint4(p.sgd.V + (int64_t)jr[r] * p.d + col, pol);
            } else {
              wv[r] = *reinterpret_cast<const float4*>(p.sgd.W + (int64_t)jr[r] * p.d + col);
              mv[r] = *reinterpret_cast<const float4*>(p.sgd.V + (int64_t)jr[r] * p.d + col);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int rr = ew * 16 + r0 + r;
          {
            const float ws = EF ? s_inv[rr] : 1.f;    // E-form: the dX operand is w_hat (G' carries no 1/||w||)
            const uint2 wb = jr[r] >= 0 ? make_uint2(pack_bf16x2(wv[r].x * ws, wv[r].y * ws),
                                                     pack_bf16x2(wv[r].z * ws, wv[r].w * ws))
                                        : make_uint2(0u, 0u);
            const int hc = lane >> 4, cq = lane & 15;   // MN-major swizzled B tile: half hc, row rr, 8 bytes
            *reinterpret_cast<uint2*>(sWb + hc * WB_HALF + rr * 128 + ((((cq >> 1) ^ (rr & 7)) << 4) | ((cq & 1) << 3))) = wb;
          }
          if (jr[r] >= 0) {
            const float inv = s_inv[rr];
            const float rad = s_rad[rr] * inv;
            const float4 g4 = s_tile[rr * 32 + (lane ^ (rr & 31))];
            float4 w = wv[r], m = mv[r];
            const float oi = p.sgd.gsc ? 1.f : inv;
            m.x = p.sgd.mu * m.x + (g4.x - w.x * rad) * oi + p.sgd.lambda * w.x;
            m.y = p.sgd.mu * m.y + (g4.y - w.y * rad) * oi + p.sgd.lambda * w.y;
            m.z = p.sgd.mu * m.z + (g4.z - w.z * rad) * oi + p.sgd.lambda * w.z;
            m.w = p.sgd.mu * m.w + (g4.w - w.w * rad) * oi + p.sgd.lambda * w.w;
            w.x -= lr * m.x; w.y -= lr * m.y; w.z -= lr * m.z; w.w -= lr * m.w;
            if (HINT) {
              st_hint4(p.sgd.V + (int64_t)jr[r] * p.d + col, m, pol);
              st_hint4(p.sgd.W + (int64_t)jr[r] * p.d + col, w, pol);
            } else {
              *reinterpret_cast<float4*>(p.sgd.V + (int64_t)jr[r] * p.d + col) = m;
              *reinterpret_cast<float4*>(p.sgd.W + (int64_t)jr[r] * p.d + col) = w;
            }
          }
        }
        if (tr) tr[5 + r0 / 8] = gtimer_dx();
        int32_t pj = (!kDiag || p.pf == 1) ? nx_j : -1;
        if (kDiag && p.pf == 2 && r0 == 0 && eset == 0 && i + 2 < ntl) {   // two tiles ahead
          const int prow = (g + (i + 2) * p.gper) * 128 + row_in;
          if (prow < k) pj = p.sgd.idx[prow];
        }
        if (r0 == 0 && eset == 0 && pj >= 0) {   // the next tile's W / V row segments into L2
          const float* wp = p.sgd.W + (int64_t)pj * p.d + n0;
          const float* vp = p.sgd.V + (int64_t)pj * p.d + n0;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(wb_full);
    }
    // dX_hat partial of this CTA (zeros when it had no class tile) -> split workspace
    mbar_wait(d2_full, 0);
    tc_fence_after();
    if (eset < nh) {
      const int row = eset * 128 + row_in;
      float* dst = p.ws + ((int64_t)g * p.M + row) * p.d + n0;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(lg * 32) << 16) + 256 + eset * 128 + c * 32, v);
        if (ntl == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0u;
        }
        if (row < p.M) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            reinterpret_cast<uint4*>(dst + c * 32)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// ------------------------------------------------------------------------------------------------------------------
// k_dwx_ring (PFC_DWX_RING=1): the same per-tile work as k_dwx_t with the W / V row stream decoupled from the tile
// pipeline. Two loader warps copy the 512-byte W and V segments of the tile's classes into a 64 KB shared ring
// (16-byte cp.async, 8 classes per slot, up to 64 classes ahead, across tile boundaries), so the HBM reads stay in
// flight while the epilogue waits for accumulators and radial dots. dW is computed transposed,
//   D1^T[128 d-columns x 128 classes] = X~^T G'   (A = X~ chunk MN-major, B = G' chunk K-major),
// so a TMEM lane is a d-column: each epilogue thread updates one column of 4 classes per slot straight from
// tcgen05.ld (no fp32 staging tile) with 128-byte coalesced W / V stores per warp instruction.
//   warp 0 TMA producer, warp 1 MMA issuer (as k_dwx_t), warps 2-9 epilogue, warps 10-11 ring loaders,
//   warps 12-13 (E-form) radial-dot partials (as k_dwx_t)
constexpr int RG_SLOTS = 8;
constexpr int RG_SLOT = 8 * 1024;                   // 8 classes x (W 512 B + V 512 B)
constexpr int RG_OFF_RING = OFF_WB + 2 * WB_HALF;
constexpr int RG_OFF_AUX = RG_OFF_RING + RG_SLOTS * RG_SLOT;
constexpr int RG_SMEM = RG_OFF_AUX + 256 + 3 * 128 * 4 + 1024;
static_assert(RG_SMEM <= 232448, "shared memory overflow");
constexpr int RG_LOAD_WARP0 = 2 + DX_EPI;
constexpr int RG_DOT_WARP0 = RG_LOAD_WARP0 + 2;
constexpr int RG_THREADS = 32 * RG_DOT_WARP0;
constexpr int RG_THREADS_EF = RG_THREADS + 32 * DX_DOTW;

__device__ __forceinline__ void st_hint1(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}

template <bool HINT, bool EF>
__global__ void __launch_bounds__(EF ? RG_THREADS_EF : RG_THREADS, 1)
    k_dwx_ring(const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmX, DwxParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sR = smem + OFF_R;
  uint8_t* sG = smem + OFF_G;
  uint8_t* sWb = smem + OFF_WB;
  float* ring = reinterpret_cast<float*>(smem + RG_OFF_RING);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RG_OFF_AUX);
  uint64_t* g_full = bars;
  uint64_t* g_empty = bars + 1;
  uint64_t* x_full = bars + 2;        // [R_STAGES]
  uint64_t* x_empty = bars + 4;       // [R_STAGES]
  uint64_t* d1_full = bars + 6;       // [2]
  uint64_t* d1_empty = bars + 8;      // [2]
  uint64_t* wb_full = bars + 10;
  uint64_t* wb_empty = bars + 11;
  uint64_t* d2_full = bars + 12;
  uint64_t* r_full = bars + 13;       // [RG_SLOTS]
  uint64_t* r_empty = bars + 13 + RG_SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13 + 2 * RG_SLOTS);
  int32_t* s_rowj = reinterpret_cast<int32_t*>(smem + RG_OFF_AUX + 256);
  float* s_inv = reinterpret_cast<float*>(s_rowj + 128);
  float* s_rad = s_inv + 128;
  static_assert(R_STAGES == 2, "barrier layout");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = p.st->k;
  const int nct = (k + 127) / 128;
  const int g = blockIdx.x % p.gper;
  const int n0 = (blockIdx.x / p.gper) * 128;
  const int ntl = g < nct ? (nct - g + p.gper - 1) / p.gper : 0;
  const int nkb = p.nkb, nh = p.nkb / 2 > 0 ? p.nkb / 2 : 1;

  if (threadIdx.x == 0) {
    mbar_init(g_full, 1); mbar_init(g_empty, 1);
    for (int i = 0; i < R_STAGES; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], EF ? 1 + DX_DOTW : 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&d1_full[i], 1); mbar_init(&d1_empty[i], DX_EPI); }
    mbar_init(wb_full, DX_EPI);
    mbar_init(wb_empty, 1);
    mbar_init(d2_full, 1);
    for (int i = 0; i < RG_SLOTS; ++i) { mbar_init(&r_full[i], 64); mbar_init(&r_empty[i], DX_EPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmG); tma_prefetch(&tmX); }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;     // cols [0, 256): D1^T x 2; [256, 512): D2 halves

  if (warp == 0) {
    // ---------------------------------------------------------------- producer (as k_dwx_t)
    if (lane == 0) {
      int xs = 0;
      uint32_t xph = 0;
      auto load_gdx = [&](int i) {
        mbar_wait(g_empty, (uint32_t)((i & 1) ^ 1));
        mbar_expect_tx(g_full, (uint32_t)(nkb * G_CHUNK));
        for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sG + kb * G_CHUNK, &tmG, g_full, kb * 64, (g + i * p.gper) * 128);
      };
      for (int i = 0; i < ntl; ++i) {
        const int ct = g + i * p.gper;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&x_empty[xs], xph ^ 1);
          mbar_expect_tx(&x_full[xs], (uint32_t)R_STAGE);
          uint8_t* st = sR + xs * R_STAGE;
          tma_load_2d(st, &tmG, &x_full[xs], kb * 64, ct * 128);
          tma_load_2d(st + G_CHUNK, &tmX, &x_full[xs], n0, kb * 64);
          tma_load_2d(st + G_CHUNK + X_CHUNK / 2, &tmX, &x_full[xs], n0 + 64, kb * 64);
          if (++xs == R_STAGES) { xs = 0; xph ^= 1; }
        }
        if (i > 0) load_gdx(i - 1);
      }
      if (ntl > 0) load_gdx(ntl - 1);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t IDESC_DWT = make_idesc(128, 128, true, false);   // A = X~ (MN-major), B = G' (K-major)
    constexpr uint32_t IDESC_DX = make_idesc(128, 128, true, true);
    int xs = 0, acc = 0;
    uint32_t xph = 0, aph = 0;
    auto dx = [&](int i) {
      mbar_wait(wb_full, (uint32_t)(i & 1));
      mbar_wait(g_full, (uint32_t)(i & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint32_t ga = smem_u32(sG), wa = smem_u32(sWb);
        for (int h = 0; h < nh; ++h)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            tc_mma(tmem_base + 256 + h * 128, make_desc(ga + 2 * h * G_CHUNK + ks * 2048, G_CHUNK, 1024),
                   make_desc(wa + ks * 2048, WB_HALF, 1024), IDESC_DX, (i > 0 || ks > 0) ? 1u : 0u);
        tc_commit(g_empty);
        tc_commit(wb_empty);
      }
      __syncwarp();
    };
    for (int i = 0; i < ntl; ++i) {
      mbar_wait(&d1_empty[acc], aph ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&x_full[xs], xph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t ga = smem_u32(sR + xs * R_STAGE), xa = ga + G_CHUNK;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma(tmem_base + acc * 128, make_desc(xa + kk * 2048, X_CHUNK / 2, 1024), make_desc(ga + kk * 32, 16, 1024),
                   IDESC_DWT, (kb > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&x_empty[xs]);
        }
        __syncwarp();
        if (++xs == R_STAGES) { xs = 0; xph ^= 1; }
      }
      if (lane == 0) tc_commit(&d1_full[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; aph ^= 1; }
      if (i > 0) dx(i - 1);
    }
    if (ntl > 0) dx(ntl - 1);
    if (lane == 0) {
      if (ntl > 0) tc_commit(d2_full);
      else mbar_arrive(d2_full);
    }
    __syncwarp();
  } else if (warp >= RG_DOT_WARP0) {
    // ---------------------------------------------------------------- E-form radial-dot partials (as k_dwx_t)
    if (EF) {
      constexpr int RPT = 128 / (32 * DX_DOTW);
      const int t = threadIdx.x - 32 * RG_DOT_WARP0;
      const int n_dt = p.d / 128, dt = blockIdx.x / p.gper;
      const float kc = 0.69314718f / p.s;
      int xs = 0;
      uint32_t xph = 0;
      for (int i = 0; i < ntl; ++i) {
        const int ct = g + i * p.gper;
        float B[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) B[q] = 0.f;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&x_full[xs], xph);
          if (kb % n_dt == dt) {
            const uint8_t* ga = sR + xs * R_STAGE;
            const float4* f4 = reinterpret_cast<const float4*>(p.f + kb * 64);
#pragma unroll 2
            for (int u = 0; u < 8; ++u) {
              const float4 fa = __ldg(f4 + 2 * u), fb = __ldg(f4 + 2 * u + 1);
              const float fv[8] = {fa.x, fa.y, fa.z, fa.w, fb.x, fb.y, fb.z, fb.w};
#pragma unroll
              for (int q = 0; q < RPT; ++q) {
                const int row = t + q * 32 * DX_DOTW;
                const uint4 qv = *reinterpret_cast<const uint4*>(ga + row * 128 + ((u ^ (row & 7)) << 4));
                const uint32_t r[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                  const float el = fmaxf(__uint_as_float(r[e2] << 16), 1e-37f);
                  const float eh = fmaxf(__uint_as_float(r[e2] & 0xFFFF0000u), 1e-37f);
                  float ll, lh;
                  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(ll) : "f"(el));
                  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lh) : "f"(eh));
                  B[q] = fmaf(el * fv[2 * e2], ll, fmaf(eh * fv[2 * e2 + 1], lh, B[q]));
                }
              }
            }
          }
          __syncwarp();
          if ((t & 31) == 0) mbar_arrive(&x_empty[xs]);
          if (++xs == R_STAGES) { xs = 0; xph ^= 1; }
        }
        float* dst = p.xch + ((int64_t)ct * n_dt + dt) * 128;
#pragma unroll
        for (int q = 0; q < RPT; ++q) dst[t + q * 32 * DX_DOTW] = kc * B[q];
        if (DX_DOTW > 1) asm volatile("bar.sync 5, %0;" ::"n"(32 * DX_DOTW) : "memory");
        else __syncwarp();
        if (t == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p.cnt + ct) : "memory");
      }
    }
  } else if (warp >= RG_LOAD_WARP0) {
    // ---------------------------------------------------------------- ring loaders (64 threads)
    // thread t copies 16-byte chunk t of each class's 1 KB (W segment: t < 32, V segment: t >= 32), 8 classes per
    // slot; the row ids come from idx (8 broadcast loads per slot); rows past k_i are not copied
    const int t = threadIdx.x - 32 * RG_LOAD_WARP0;
    (void)k;
    const float* base = t < 32 ? p.sgd.W : p.sgd.V;
    const int coff = 4 * (t & 31);
    const uint32_t doff = (uint32_t)((t < 32 ? 0 : 512) + 16 * (t & 31));
    const uint64_t pol = HINT ? policy_evict_first() : 0;
    int rs = 0;
    uint32_t rph = 0;
    // the tile's 128 row ids in registers (lane l: classes l, l + 32, l + 64, l + 96), the next tile's loaded a
    // tile ahead; each slot's 8 ids are shuffled out of them
    auto ids = [&](int i, int32_t (&r)[4]) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int prow = (g + i * p.gper) * 128 + 32 * q + lane;
        r[q] = (i < ntl && prow < k) ? __ldg(p.sgd.idx + prow) : -1;
      }
    };
    int32_t cur[4], nxt[4];
    ids(0, nxt);
    for (int i = 0; i < ntl; ++i) {
#pragma unroll
      for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
      ids(i + 1, nxt);
      for (int grp = 0; grp < 16; ++grp) {
        // slot grp holds classes 4 grp .. 4 grp + 3 (positions 0-3) and 64 + 4 grp .. (positions 4-7): each
        // epilogue class set walks 64 contiguous TMEM columns
        const int32_t lo = (grp >> 3) == 0 ? cur[0] : cur[1];
        const int32_t hi = (grp >> 3) == 0 ? cur[2] : cur[3];
        int32_t jj[8];
#pragma unroll
        for (int cl = 0; cl < 8; ++cl) jj[cl] = __shfl_sync(0xffffffffu, cl < 4 ? lo : hi, ((grp & 7) << 2) + (cl & 3));
        mbar_wait(&r_empty[rs], rph ^ 1);
        const uint32_t dst = smem_u32(ring) + rs * RG_SLOT + doff;
#pragma unroll
        for (int cl = 0; cl < 8; ++cl)
          if (jj[cl] >= 0) {
            const float* src = base + (int64_t)jj[cl] * p.d + n0 + coff;
            if (HINT)
              asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst + cl * 1024),
                           "l"(src), "l"(pol)
                           : "memory");
            else
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + cl * 1024), "l"(src) : "memory");
          }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&r_full[rs])) : "memory");
        if (++rs == RG_SLOTS) { rs = 0; rph ^= 1; }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    // ---------------------------------------------------------------- epilogue (thread = d-column of a quarter)
    const int ew = warp - 2;
    const int lg = warp & 3;
    const int row_in = lg * 32 + lane;       // this thread's d-column in the tile (its TMEM lane); also a class row
                                             // for the per-tile scalars
    const int eset = ew >> 2;                // classes 4 eset .. 4 eset + 3 of every 8-class slot
    const float lr = *p.sgd.lr;
    const uint64_t pol = HINT ? policy_evict_first() : 0;
    int32_t nx_j = -1;
    float nx_inv = 0.f, nx_rad = 0.f;
    if (eset == 0 && ntl > 0) {
      const int prow = g * 128 + row_in;
      if (prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; nx_rad = EF ? 0.f : p.sgd.dotw[prow]; }
    }
    int acc = 0, rs = 0;
    uint32_t aph = 0, rph = 0;
    const int half = row_in >> 6, xi = row_in & 63;
    for (int i = 0; i < ntl; ++i) {
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DX_EPI) : "memory");   // previous tile's scalars consumed
      uint64_t* tr = (kDiag && p.trace && threadIdx.x == 64 && i < p.trace_tiles)
                         ? p.trace + ((int64_t)blockIdx.x * p.trace_tiles + i) * 8 : nullptr;
      if (tr) tr[0] = gtimer_dx();
      if (eset == 0) {
        s_rowj[row_in] = nx_j; s_inv[row_in] = nx_inv; s_rad[row_in] = nx_rad;
        nx_j = -1; nx_inv = 0.f; nx_rad = 0.f;
        if (i + 1 < ntl) {
          const int prow = (g + (i + 1) * p.gper) * 128 + row_in;
          if (prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; nx_rad = EF ? 0.f : p.sgd.dotw[prow]; }
        }
      }
      float rad16 = 0.f;
      float radp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (EF) {   // radial dots of classes ew * 16 + l (l < 16): dcorr + the n_dt d-tile partials
        const int ct = g + i * p.gper, n_dt = p.d / 128;
        if (lane == 0) {
          const int* c = p.cnt + ct;
          int v, spins = 0;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
          } while (v < n_dt && ++spins < (1 << 26));
          if (v < n_dt) atomicOr(p.err, ERR_INTERNAL);
        }
        __syncwarp();
        if (lane < 16) {
          const int row = ew * 16 + lane;
          rad16 = __ldcg(p.dcorr + ct * 128 + row);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < n_dt) radp[q] = __ldcg(p.xch + ((int64_t)ct * n_dt + q) * 128 + row);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) rad16 += radp[q];
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DX_EPI) : "memory");   // s_rowj / s_inv / s_rad of this tile
      if (EF) {
        if (lane < 16) s_rad[ew * 16 + lane] = rad16;
        asm volatile("bar.sync 3, %0;" ::"n"(32 * DX_EPI) : "memory");
      }
      if (tr) tr[1] = gtimer_dx();
      mbar_wait(&d1_full[acc], aph);
      tc_fence_after();
      if (tr) tr[2] = gtimer_dx();
      mbar_wait(wb_empty, (uint32_t)((i & 1) ^ 1));   // dX(t - 1) has read the previous bf16 w_old tile
      if (tr) tr[3] = gtimer_dx();
      const uint32_t tacc = tmem_base + ((uint32_t)(lg * 32) << 16) + acc * 128 + 64 * eset;
      uint64_t rwait = 0;
#pragma unroll 1
      for (int gh = 0; gh < 2; ++gh) {
      uint32_t dv[32];   // dW^T of this thread's column for classes 64 eset + 32 gh + 0..31
      tmem_ld32(tacc + 32 * gh, dv);
#pragma unroll
      for (int g8 = 0; g8 < 8; ++g8) {
        const int grp = gh * 8 + g8;
        const uint64_t tw0 = tr ? gtimer_dx() : 0;
        mbar_wait(&r_full[rs], rph);
        if (tr) rwait += gtimer_dx() - tw0;
        float* sl = ring + rs * (RG_SLOT / 4);
        // (a) column-wise update of this warp's 4 classes, written back into the slot in place
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int cl = 4 * eset + u, c = 64 * eset + 4 * grp + u;
          const int32_t j = s_rowj[c];
          const float wo = sl[cl * 256 + row_in];
          const float mo = sl[cl * 256 + 128 + row_in];
          const float ws = EF ? s_inv[c] : 1.f;
          const __nv_bfloat16 wb = __float2bfloat16_rn(j >= 0 ? wo * ws : 0.f);
          *reinterpret_cast<__nv_bfloat16*>(sWb + half * WB_HALF + c * 128 + ((((xi >> 3) ^ (c & 7)) << 4) | ((xi & 7) << 1))) = wb;
          if (j >= 0) {
            const float inv = s_inv[c];
            const float rad = s_rad[c] * inv;
            const float oi = p.sgd.gsc ? 1.f : inv;
            const float m = p.sgd.mu * mo + (__uint_as_float(dv[4 * g8 + u]) - wo * rad) * oi + p.sgd.lambda * wo;
            sl[cl * 256 + row_in] = wo - lr * m;
            sl[cl * 256 + 128 + row_in] = m;
          }
        }
        // (b) the 4 warps of this class set (one per column quarter) done: warp lg stores class 4 eset + lg's W and V
        // segments row-wise (512-byte coalesced float4 stores)
        asm volatile("bar.sync %0, 128;" ::"r"(6 + eset) : "memory");
        {
          const int cl = 4 * eset + lg, c = 64 * eset + 4 * grp + lg;
          const int32_t j = s_rowj[c];
          if (j >= 0) {
            const float4 w4 = reinterpret_cast<const float4*>(sl + cl * 256)[lane];
            const float4 m4 = reinterpret_cast<const float4*>(sl + cl * 256 + 128)[lane];
            float* wp = p.sgd.W + (int64_t)j * p.d + n0 + 4 * lane;
            float* vp = p.sgd.V + (int64_t)j * p.d + n0 + 4 * lane;
            if (HINT) { st_hint4(vp, m4, pol); st_hint4(wp, w4, pol); }
            else { *reinterpret_cast<float4*>(vp) = m4; *reinterpret_cast<float4*>(wp) = w4; }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&r_empty[rs]);
        if (++rs == RG_SLOTS) { rs = 0; rph ^= 1; }
        if (tr && grp == 7) tr[4] = gtimer_dx();
        if (grp == 0 && eset == 0 && nx_j >= 0 && p.pf) {   // the next tile's rows into L2 (the ring reads them)
          const float* wp = p.sgd.W + (int64_t)nx_j * p.d + n0;
          const float* vp = p.sgd.V + (int64_t)nx_j * p.d + n0;
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
          }
        }
      }
      }
      if (tr) { tr[5] = gtimer_dx(); tr[6] = tr[5] - rwait; }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d1_empty[acc]);
      if (++acc == 2) { acc = 0; aph ^= 1; }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(wb_full);
    }
    // dX_hat partial of this CTA -> split workspace (as k_dwx_t)
    mbar_wait(d2_full, 0);
    tc_fence_after();
    if (eset < nh) {
      const int row = eset * 128 + row_in;
      float* dst = p.ws + ((int64_t)g * p.M + row) * p.d + n0;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(lg * 32) << 16) + 256 + eset * 128 + c * 32, v);
        if (ntl == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0u;
        }
        if (row < p.M) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            reinterpret_cast<uint4*>(dst + c * 32)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// dX_hat = sum of the split partials (fixed order); E-form: times f_n per batch row (dX_hat_n = f_n sum_j E'_nj w_hat_j)
// P.n > 0 (fused reduce-scatter): each row goes straight into its owner's xdx slot `rank`
__global__ void k_ws_reduce(int64_t n, int nsplit, int64_t stride, int d, const float* __restrict__ ws,
                            const float* __restrict__ f, float* __restrict__ out, Peers P, int B) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  float4 acc = *reinterpret_cast<const float4*>(ws + i);
#pragma unroll 4
  for (int s = 1; s < nsplit; ++s) {
    const float4 v = *reinterpret_cast<const float4*>(ws + s * stride + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (f) {
    const float fn = f[i / d];
    acc.x *= fn; acc.y *= fn; acc.z *= fn; acc.w *= fn;
  }
  *reinterpret_cast<float4*>(dx_dst(P, out, i, d, B)) = acc;
}

int dwx_gper(const Sizes& sz) { return std::max(1, num_sms() / (sz.d / 128)); }

}  // namespace

bool dwx_supported(const Sizes& sz) {
  const int forced = env_int("PFC_DWX", 1);
  return forced != 0 && sz.M <= 256 && sz.d % 128 == 0;
}

int64_t dwx_ws_floats(const Sizes& sz) { return (int64_t)dwx_gper(sz) * sz.M * sz.d; }

int launch_dwx_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                  const SgdArgs& sa, float* ws, float* dXh, const EformArgs* ef, const Peers* P, cudaStream_t s) {
  // W / V streamed with an L2 evict-first policy so that the G' tile re-read for dX stays resident (-0.1 to -0.2 GB
  // of DRAM reads per step at C4); PFC_DWX_HINT=0 disables
  const bool hint = env_int("PFC_DWX_HINT", 1) != 0;
  const bool ringk = env_int("PFC_DWX_RING", 0) != 0;
  auto kern = ringk ? (ef ? (hint ? k_dwx_ring<true, true> : k_dwx_ring<false, true>)
                          : (hint ? k_dwx_ring<true, false> : k_dwx_ring<false, false>))
                    : (ef ? (hint ? k_dwx_t<true, true> : k_dwx_t<false, true>)
                          : (hint ? k_dwx_t<true, false> : k_dwx_t<false, false>));
  const int nthreads = ringk ? (ef ? RG_THREADS_EF : RG_THREADS) : (ef ? DX_THREADS_EF : DX_THREADS);
  const int smem_bytes = ringk ? RG_SMEM : DX_SMEM;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dwx_ring<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, RG_SMEM);
    cudaFuncSetAttribute(k_dwx_ring<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, RG_SMEM);
    cudaFuncSetAttribute(k_dwx_ring<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, RG_SMEM);
    cudaFuncSetAttribute(k_dwx_ring<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, RG_SMEM);
    cudaFuncSetAttribute(k_dwx_t<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, DX_SMEM);
    cudaFuncSetAttribute(k_dwx_t<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, DX_SMEM);
    cudaFuncSetAttribute(k_dwx_t<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, DX_SMEM);
    cudaFuncSetAttribute(k_dwx_t<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, DX_SMEM);
    attr = true;
  }
  const CUtensorMap tg = make_map(G, sz.k_pad, sz.M_pad, 64, 128);   // G' (or E') class-major: 128 classes x 64 batch
  const CUtensorMap tx = make_map(Xb, sz.M_pad, sz.d, 64, 64);       // X_hat (or X~): 64 batch rows x 64 columns
  TC_MAPS_OK();
  DwxParams p{};
  p.M = sz.M; p.d = sz.d; p.nkb = (int)(sz.M_pad / 64); p.gper = dwx_gper(sz); p.st = st; p.sgd = sa; p.ws = ws;
  p.pfnow = env_int("PFC_DWX_PFNOW", 0);
  p.pf = env_int("PFC_DWX_PF", 1);
  if (ef) {
    p.f = ef->f; p.tcol = ef->tcol; p.dcorr = ef->dcorr; p.xch = ef->xch; p.cnt = ef->cnt; p.err = ef->err;
    p.s = ef->s;
    cudaMemsetAsync(ef->cnt, 0, (size_t)(sz.k_pad / 128) * sizeof(int), s);
  }
  const int grid = p.gper * (sz.d / 128);
  static uint64_t* trace = nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  const int ttiles = (int)((sz.k_pad / 128 + p.gper - 1) / p.gper);
  if (kDiag && env_int("PFC_DWX_TRACE", 0) && cs == cudaStreamCaptureStatusNone) {
    static size_t cap = 0;
    const size_t need = (size_t)grid * ttiles * 8 * sizeof(uint64_t);
    if (need > cap) { if (trace) cudaFree(trace); cudaMalloc(&trace, need); cap = need; }
    cudaMemsetAsync(trace, 0, need, s);
    p.trace = trace;
    p.trace_tiles = ttiles;
  }
  if (ef) {
    // the E-form epilogue waits on radial-dot partials published by the other d-tile CTAs of its class tile: a
    // cooperative launch guarantees that the whole grid (<= one CTA per SM) is co-resident, or fails loudly
    // (cudaErrorCooperativeLaunchTooLarge, reported by the step) instead of spinning on a CTA that never runs
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(nthreads);
    lc.dynamicSmemBytes = smem_bytes;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, kern, tg, tx, p);
  } else {
    kern<<<grid, nthreads, smem_bytes, s>>>(tg, tx, p);
  }
  if (p.trace) {
    std::vector<uint64_t> h((size_t)grid * ttiles * 8);
    cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const char* fn = std::getenv("PFC_DWX_TRACE_FILE");
    if (FILE* f = std::fopen(fn ? fn : "dwx_trace.csv", "w")) {
      std::fprintf(f, "cta,tile,start,d1_full,cnt_ok,staged,wb_empty,batch0,update_done,dot_published\n");
      for (int c = 0; c < grid; ++c)
        for (int i = 0; i < ttiles; ++i) {
          const uint64_t* r = h.data() + ((size_t)c * ttiles + i) * 8;
          if (!r[0]) continue;
          std::fprintf(f, "%d,%d", c, i);
          for (int q = 0; q < 8; ++q) std::fprintf(f, ",%llu", (unsigned long long)r[q]);
          std::fprintf(f, "\n");
        }
      std::fclose(f);
    }
  }
  const int64_t n = (int64_t)sz.M * sz.d;
  Peers q{};
  if (P) q = *P;
  launch_pdl(k_ws_reduce, dim3((unsigned)((n / 4 + 255) / 256)), dim3(256), 0, s, n, p.gper, n, sz.d, ws, ef ? ef->f : nullptr, dXh, q,
                                                              sz.B);
  return 2;
}

}  // namespace pfc
