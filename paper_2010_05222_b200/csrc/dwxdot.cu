// K11 + radial dot + K12 on CTA pairs, the radial dot exchanged between the pairs of a class tile's column halves
// (train step, bf16 tensor-core path, M > 256, d = 512; no separate radial-dot pass over E).
//
// As k_dw_sgd_pair (dwpair.cu): a cluster of two CTAs computes the dW_hat unit of 256 sampled classes x 256 columns
// = E'^T X~ (Alg.1 L10, tcgen05.mma.cta_group::2, K = the global batch) and applies the lazy momentum-SGD update of
// those W / V rows in its epilogue. Units u = 2t + h (class tile t, column half h) go to pairs
// pair + i * npairs, so the two halves of a tile are computed at the same time by the neighbouring pairs 2m, 2m + 1.
// The w-normalisation backprop needs w_hat_j . dW_hat_j over all 512 columns (R14); each CTA forms its half of that
// dot from its own accumulator (R29: sum_c w_jc acc_jc over its 256 columns), publishes it, and takes the partner
// CTA's half (same classes, other column half) — sum in the fixed order h0 + h1 on both sides. All CTAs are
// co-resident (cooperative launch; one CTA per SM), so the short wait for the partner cannot deadlock.
// Per unit the epilogue stages the whole 128 x 256 accumulator to shared memory and releases TMEM at once (the
// next unit's MMAs start while the dot, the exchange and the update run).
//   warp 0    TMA producer (its halves, onto the leader's mbarrier)
//   warp 1    TMEM allocation (cta_group::2); MMA issue (leader), commits multicast to both CTAs
//   warps 2-9 epilogue (this CTA's 128 classes)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pfc_internal.cuh"
#include "tc_common.cuh"

namespace pfc {
namespace {

#ifndef PFC_DWX_DIAG
#define PFC_DWX_DIAG 0
#endif
// build-time diagnostics (PFC_BUILD_TAG=diag PFC_NVCC_EXTRA=-DPFC_DWX_DIAG=1): the per-unit trace (PFC_DW_TRACE) and
// the non-default prefetch / hoist / E-hint variants; compiled out by default (runtime checks in the epilogue cost)
constexpr bool kXDiag = PFC_DWX_DIAG != 0;
constexpr int XP_BK = 64;
constexpr int XP_STAGES = 3;
constexpr int XP_ACC = 2;
// epilogue warps: 8 (2 per TMEM lane quadrant, 16 rows each). Per-unit trace (PFC_DW_TRACE) at the per-rank C4 shape:
// dot pass 3.8 us, partner wait 5.3 us, update 16.9 us per unit against ~12 us of MMAs. PFC_XP_EPI=16 at build time
// (4 per quadrant, twice the loads in flight) measured slower: update 19.5 us, kernel 0.484 vs 0.41 ms.
#ifndef PFC_XP_EPI
#define PFC_XP_EPI 8
#endif
constexpr int XP_EPI = PFC_XP_EPI;
constexpr int XP_RPW = 128 / XP_EPI;                  // rows per warp (16 or 8)
constexpr int XP_NSET = XP_EPI / 4;                   // column sets per TMEM lane quadrant
static_assert(XP_RPW == 8 || XP_RPW == 16, "epilogue layout");
constexpr int XP_DB = XP_RPW == 16 ? 8 : 4;           // rows per batch of the dot pass (register budget)
constexpr int XP_THREADS = 32 * (2 + XP_EPI);
constexpr int XP_HALF = 128 * XP_BK * 2;              // 16 KB
constexpr int XP_STAGE = 2 * XP_HALF;                 // A (128 classes x 64 batch) + B (64 batch x 128 columns)
constexpr int XP_ST = 128 * 256 * 4;                  // fp32 staging of the 128 x 256 accumulator
constexpr int XP_SMEM = XP_STAGES * XP_STAGE + XP_ST + 1024 + 256 + 3 * 128 * 4;
static_assert(XP_SMEM <= 232448, "shared memory overflow");

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct XpParams {
  int M, d;
  const SamplerState* st;
  SgdArgs sgd;
  float* xdot;      // [n_units][128 * 2] this unit's half-dots, by CTA rank and row
  int* flag;        // [n_units][2] published (zeroed before the launch)
  int* err;
  int ehint;   // E' loads: 0 default L2 policy, 1 evict-last, 2 evict-first
  int pfnow;
  int hoist;   // the update's first W / V loads issued before the partner wait   // prefetch this unit's W / V rows into L2 when its scalars are known (else the next unit's, a unit ahead)
  uint64_t* trace;   // PFC_DW_TRACE=1 (eager launches only): per CTA and unit, globaltimer at 6 epilogue points
  int trace_units;
};

// staging index of float4 q (0..63) of row r (XOR swizzle inside each 32-float4 half)
__device__ __forceinline__ int xidx(int r, int q) { return r * 64 + (q & 32) + ((q & 31) ^ (r & 31)); }

template <bool HINT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(XP_THREADS, 1)
    k_dw_sgd_pairx(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, XpParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float4* s_st = reinterpret_cast<float4*>(smem + XP_STAGES * XP_STAGE);       // [128 rows][64 float4]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + XP_STAGES * XP_STAGE + XP_ST);   // leader: both CTAs
  uint64_t* empty = full + XP_STAGES;                                          // each CTA
  uint64_t* acc_full = empty + XP_STAGES;                                      // each CTA
  uint64_t* acc_empty = acc_full + XP_ACC;                                     // leader: both CTAs' epilogues
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + XP_ACC);
  int32_t* s_rowj = reinterpret_cast<int32_t*>(smem + XP_STAGES * XP_STAGE + XP_ST + 256);
  float* s_inv = reinterpret_cast<float*>(s_rowj + 128);
  float* s_dot = s_inv + 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pr = (int)cluster_rank();
  const bool leader = pr == 0;
  const int k = p.st->k;
  const int nct = (k + 255) / 256;
  const int n_units = nct * 2, n_kb = (p.M + XP_BK - 1) / XP_BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < XP_STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < XP_ACC; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 2 * XP_EPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer (this CTA's halves)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // PFC_DW_EHINT=1: E' loads with an L2 evict-last policy (read by the two partner pairs of a tile at the same
      // time) — measured no better (c4rank 1.015 vs 1.008 ms), off by default
      const uint64_t epol = p.ehint == 2 ? policy_evict_first() : policy_evict_last();
      for (int u = pair; u < n_units; u += npairs) {
        const int c0 = (u >> 1) * 256 + 128 * pr, d0 = (u & 1) * 256 + 128 * pr;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], (uint32_t)(4 * XP_HALF));
          uint8_t* sa = smem + stage * XP_STAGE;
          if (kXDiag && p.ehint) tma_load_2d_pair_hint(sa, &tmA, &full[stage], kb * XP_BK, c0, epol);  // E' rows: its classes
          else tma_load_2d_pair(sa, &tmA, &full[stage], kb * XP_BK, c0);
          tma_load_2d_pair(sa + XP_HALF, &tmB, &full[stage], d0, kb * XP_BK);             // X~: its columns
          tma_load_2d_pair(sa + XP_HALF + XP_HALF / 2, &tmB, &full[stage], d0 + 64, kb * XP_BK);
          if (++stage == XP_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader)
    if (leader) {
      constexpr uint32_t IDESC = make_idesc(256, 256, false, true);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = pair; u < n_units; u += npairs) {
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tacc = tmem_base + acc * 256;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + stage * XP_STAGE), sb = sa + XP_HALF;
#pragma unroll
            for (int kk = 0; kk < XP_BK / 16; ++kk)
              tc_mma_pair(tacc, make_desc(sa + kk * 32, 16, 1024), make_desc(sb + kk * 2048, XP_HALF / 2, 1024), IDESC,
                          (kb > 0 || kk > 0) ? 1u : 0u);
            tc_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == XP_STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) tc_commit_pair(&acc_full[acc]);
        __syncwarp();
        if (++acc == XP_ACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (this CTA's 128 classes)
    const int ew = warp - 2;
    const int lg = warp & 3;
    const int row_in = lg * 32 + lane;
    const int eset = ew >> 2;
    const float lr = *p.sgd.lr;
    const float mu = p.sgd.mu, lam = p.sgd.lambda;
    const uint64_t pol = HINT ? policy_evict_first() : 0;
    const uint32_t acce_leader = leader_addr(&acc_empty[0]);
    const int d = p.d;
    int32_t nx_j = -1;
    float nx_inv = 0.f;
    auto scalars = [&](int u) {
      const int prow = (u >> 1) * 256 + 128 * pr + row_in;
      nx_j = -1; nx_inv = 0.f;
      if (u < n_units && prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; }
    };
    if (eset == 0) scalars(pair);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < n_units; u += npairs) {
      const int h = u & 1, dcol0 = h * 256;
      asm volatile("bar.sync 3, %0;" ::"n"(32 * XP_EPI) : "memory");   // previous unit consumed
      int32_t pf_j = -1;
      if (eset == 0) {
        s_rowj[row_in] = nx_j; s_inv[row_in] = nx_inv;
        const int pfnow = kXDiag ? p.pfnow : 1;
        if (pfnow && nx_j >= 0) {   // this unit's W / V row segments into L2 now (used ~10 us later)
          const float* wp = p.sgd.W + (int64_t)nx_j * d + h * 256;
          const float* vp = p.sgd.V + (int64_t)nx_j * d + h * 256;
#pragma unroll
          for (int l = 0; l < 8; ++l) {
            if (pfnow == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
          }
        }
        scalars(u + npairs);
        pf_j = pfnow == 1 ? -1 : nx_j;
      }
      const int ui = (u - pair) / npairs;
      uint64_t* tr = (kXDiag && p.trace && threadIdx.x == 64 && ui < p.trace_units) ? p.trace + ((int64_t)blockIdx.x * p.trace_units + ui) * 6 : nullptr;
      if (tr) tr[0] = gtimer();
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      if (tr) tr[1] = gtimer();
      {   // the whole 128 x 256 accumulator -> staging (thread = row), TMEM released at once
        const uint32_t tacc = tmem_base + ((uint32_t)(lg * 32) << 16) + acc * 256;
#pragma unroll 1
        for (int c = 0; c < 16 / XP_NSET; ++c) {
          uint32_t v[16];
          tmem_ld16(tacc + eset * (256 / XP_NSET) + c * 16, v);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            s_st[xidx(row_in, eset * (64 / XP_NSET) + c * 4 + q)] =
                make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                            __uint_as_float(v[4 * q + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&acc_empty[acc]);
        else mbar_arrive_cluster(acce_leader + acc * 8);
      }
      if (++acc == XP_ACC) { acc = 0; acc_phase ^= 1; }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * XP_EPI) : "memory");   // staging and scalars complete
      if (tr) tr[2] = gtimer();
      // this half's dots: warp per row, lanes along the 256 columns (W segments read coalesced; they stay in L2 for
      // the update below)
#pragma unroll 1
      for (int r8 = 0; r8 < XP_RPW; r8 += XP_DB) {
        float4 wa[XP_DB], wb[XP_DB];
        int32_t j8[XP_DB];
#pragma unroll
        for (int r = 0; r < XP_DB; ++r) {
          j8[r] = s_rowj[ew * XP_RPW + r8 + r];
          if (j8[r] >= 0) {
            const float* wp = p.sgd.W + (int64_t)j8[r] * d + dcol0 + lane * 4;
            wa[r] = *reinterpret_cast<const float4*>(wp);
            wb[r] = *reinterpret_cast<const float4*>(wp + 128);
          } else {
            wa[r] = wb[r] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int r = 0; r < XP_DB; ++r) {
          const int rr = ew * XP_RPW + r8 + r;
          const float4 ga = s_st[xidx(rr, lane)], gb = s_st[xidx(rr, 32 + lane)];
          float v = wa[r].x * ga.x + wa[r].y * ga.y + wa[r].z * ga.z + wa[r].w * ga.w;
          v += wb[r].x * gb.x + wb[r].y * gb.y + wb[r].z * gb.z + wb[r].w * gb.w;
          v = warp_sum(v);
          if (lane == 0) p.xdot[((int64_t)u * 2 + pr) * 128 + rr] = v;
        }
      }
      if (tr) tr[3] = gtimer();
      // publish this CTA's half-dots, then take the partner CTA's (unit u ^ 1, same classes, same rank); the first
      // W / V loads of the update are issued before the wait (they need the rows, not the dot)
      asm volatile("bar.sync 3, %0;" ::"n"(32 * XP_EPI) : "memory");
      if (ew == 0 && lane == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.flag + (u * 2 + pr)), "r"(1) : "memory");
      }
      float4 wv[2][4], mv[2][4];
      int32_t jr[2][4];
      auto load = [&](int sh, int b, int slot) {
        const int col = dcol0 + sh * 128 + lane * 4;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int rr = ew * XP_RPW + 4 * b + r;
          jr[slot][r] = s_rowj[rr];
          PFC_DCHECK(jr[slot][r] < p.sgd.rows);
          if (jr[slot][r] >= 0) {
            wv[slot][r] = *reinterpret_cast<const float4*>(p.sgd.W + (int64_t)jr[slot][r] * d + col);
            mv[slot][r] = HINT ? ld_hint4(p.sgd.V + (int64_t)jr[slot][r] * d + col, pol)
                               : *reinterpret_cast<const float4*>(p.sgd.V + (int64_t)jr[slot][r] * d + col);
          }
        }
      };
      // momentum-SGD update of 4 rows over 128 columns (the staging holds dW_hat of this unit)
      auto upd = [&](int sh, int b, int slot) {
        const int col = dcol0 + sh * 128 + lane * 4;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int rr = ew * XP_RPW + 4 * b + r;
          if (jr[slot][r] >= 0) {
            const float inv = s_inv[rr];
            const float rad = s_dot[rr] * inv * inv;        // (w_hat . dW_hat) / ||w||
            const float4 g = s_st[xidx(rr, sh * 32 + lane)];
            float4 w = wv[slot][r], m = mv[slot][r];
            m.x = mu * m.x + (g.x - w.x * rad) * inv + lam * w.x;
            m.y = mu * m.y + (g.y - w.y * rad) * inv + lam * w.y;
            m.z = mu * m.z + (g.z - w.z * rad) * inv + lam * w.z;
            m.w = mu * m.w + (g.w - w.w * rad) * inv + lam * w.w;
            w.x -= lr * m.x; w.y -= lr * m.y; w.z -= lr * m.z; w.w -= lr * m.w;
            float* wp = p.sgd.W + (int64_t)jr[slot][r] * d + col;
            float* vp = p.sgd.V + (int64_t)jr[slot][r] * d + col;
            if (HINT) { st_hint4(vp, m, pol); st_hint4(wp, w, pol); }
            else { *reinterpret_cast<float4*>(vp) = m; *reinterpret_cast<float4*>(wp) = w; }
          }
        }
      };
      const bool hoist = !kXDiag || p.hoist;
      if (hoist) {
        load(0, 0, 0);
        load(0, 1, 1);
      }
      if (ew == 0 && lane == 0) {
        PFC_DCHECK((u ^ 1) < n_units);
        const int* f = p.flag + ((u ^ 1) * 2 + pr);
        int v = 0, spins = 0;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        } while (!v && ++spins < (1 << 26));
        if (!v) atomicOr(p.err, ERR_INTERNAL);
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * XP_EPI) : "memory");
      if (eset == 0) {   // w . dW_hat over all 512 columns, summed h0 + h1 on both sides (R29)
        const float d0 = __ldcg(p.xdot + ((int64_t)(u & ~1) * 2 + pr) * 128 + row_in);
        const float d1 = __ldcg(p.xdot + ((int64_t)(u | 1) * 2 + pr) * 128 + row_in);
        s_dot[row_in] = d0 + d1;
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * XP_EPI) : "memory");
      if (tr) tr[4] = gtimer();
      if (pf_j >= 0) {   // the next unit's W (and, without PFC_DW_PFNOW, V) row segments (256 columns) into L2
        const int ndc = ((u + npairs) & 1) * 256;
        const float* wp = p.sgd.W + (int64_t)pf_j * d + ndc;
        const float* vp = p.sgd.V + (int64_t)pf_j * d + ndc;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
          if (kXDiag && !p.pfnow) asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
        }
      }
      // the update, 4-row batches per 128-column quarter, the next batch's W / V loads in flight
#pragma unroll
      for (int sh = 0; sh < 2; ++sh) {
        if (sh == 1 || !hoist) {
          load(sh, 0, 0);
          load(sh, 1, 1);
        }
        upd(sh, 0, 0);
        if constexpr (XP_RPW == 16) {
          load(sh, 2, 0);
          upd(sh, 1, 1);
          load(sh, 3, 1);
          upd(sh, 2, 0);
          upd(sh, 3, 1);
        } else {
          upd(sh, 1, 1);
        }
      }
      if (tr) tr[5] = gtimer();
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

}  // namespace

bool dw_sgd_pairx_enabled(const Sizes& sz, int gsc) {
  const int forced = env_int("PFC_DW_XDOT", 1);
  return forced != 0 && gsc == 0 && sz.M >= 2048 && sz.d == 512 && sz.k_pad % 256 == 0;
}

int64_t dw_sgd_pairx_ws_floats(const Sizes& sz) { return (sz.k_pad / 256) * 2 * 256 + (sz.k_pad / 256) * 4; }

int launch_dw_sgd_pairx_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                           const SgdArgs& sa, float* ws, int* err, cudaStream_t s) {
  const bool hint = env_int("PFC_DW_HINT", 1) != 0;
  auto kern = hint ? k_dw_sgd_pairx<true> : k_dw_sgd_pairx<false>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dw_sgd_pairx<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, XP_SMEM);
    cudaFuncSetAttribute(k_dw_sgd_pairx<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, XP_SMEM);
    attr = true;
  }
  const CUtensorMap a = make_map(G, sz.k_pad, sz.M_pad, 64, 128);    // E' / G class-major: 128 classes x 64 batch
  const CUtensorMap b = make_map(Xb, sz.M_pad, sz.d, 64, 64);        // X~ / X_hat: 64 batch rows x 64 columns
  TC_MAPS_OK();
  const int64_t units = (sz.k_pad / 256) * 2;
  XpParams p{};
  p.M = sz.M; p.d = sz.d; p.st = st; p.sgd = sa; p.err = err;
  p.xdot = ws;
  const int ehint = env_int("PFC_DW_EHINT", 0);
  p.ehint = ehint;
  p.pfnow = env_int("PFC_DW_PFNOW", 1);
  p.hoist = env_int("PFC_DW_HOIST", 1);
  p.flag = reinterpret_cast<int*>(ws + units * 256);
  cudaMemsetAsync(p.flag, 0, (size_t)units * 2 * sizeof(int), s);
  // every pair of the grid is co-resident (one CTA per SM, units in lock-step): the partner waits cannot deadlock.
  // A cooperative launch makes that a guarantee (or fails loudly).
  const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(units, (num_sms() / 2) & ~1));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(2 * pairs);
  lc.blockDim = dim3(XP_THREADS);
  lc.dynamicSmemBytes = XP_SMEM;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  // PFC_DW_TRACE=1: per-unit epilogue timestamps of one eager launch, written to $PFC_DW_TRACE_FILE (diagnostic)
  static uint64_t* trace = nullptr;
  const bool tracing = kXDiag && env_int("PFC_DW_TRACE", 0) != 0;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  const int tunits = (int)((units + pairs - 1) / pairs);
  if (tracing && cs == cudaStreamCaptureStatusNone) {
    if (!trace) cudaMalloc(&trace, (size_t)2 * pairs * tunits * 6 * sizeof(uint64_t));
    cudaMemsetAsync(trace, 0, (size_t)2 * pairs * tunits * 6 * sizeof(uint64_t), s);
    p.trace = trace;
    p.trace_units = tunits;
  }
  cudaLaunchKernelEx(&lc, kern, a, b, p);
  if (p.trace) {
    std::vector<uint64_t> h((size_t)2 * pairs * tunits * 6);
    cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const char* fn = std::getenv("PFC_DW_TRACE_FILE");
    if (FILE* f = std::fopen(fn ? fn : "dw_trace.csv", "w")) {
      std::fprintf(f, "cta,unit,wait_start,acc_full,staged,dot_done,xchg_done,update_done\n");
      for (int c = 0; c < 2 * pairs; ++c)
        for (int i = 0; i < tunits; ++i) {
          const uint64_t* r = h.data() + ((size_t)c * tunits + i) * 6;
          if (!r[0]) continue;
          std::fprintf(f, "%d,%d,%llu,%llu,%llu,%llu,%llu,%llu\n", c, i, (unsigned long long)r[0],
                       (unsigned long long)r[1], (unsigned long long)r[2], (unsigned long long)r[3],
                       (unsigned long long)r[4], (unsigned long long)r[5]);
        }
      std::fclose(f);
    }
  }
  return 2;
}

}  // namespace pfc
