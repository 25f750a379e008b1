// K11 + K12 fused on CTA pairs (train step, bf16 tensor-core path, M >= 2048, d % 256 == 0): the dW_hat tile of
// 256 sampled classes x 256 columns = G^T X_hat (Alg.1 L10) with tcgen05.mma.cta_group::2 (M = 256 classes split
// across the pair, N = 256 columns split across the pair), and the lazy momentum-SGD update of those W / V rows
// in each CTA's epilogue. CTA r stages per 64-batch K block its 128 classes of G (K-major A) and its
// 128 columns of X_hat (MN-major B), 32 KB, instead of the 48 KB per 256 x 128 tile of the single-CTA kernel
// (gemm_tc.cu DWF2); its TMEM accumulates its 128 classes x all 256 columns.
//   warp 0    TMA producer (its halves, onto the leader's mbarrier)
//   warp 1    TMEM allocation (cta_group::2); MMA issue (leader), commits multicast to both CTAs
//   warps 2-9 epilogue: per 128-column half, TMEM -> XOR-swizzled smem, then 8 warps update 16 rows each with
//             512-byte coalesced W / V segments; per-row scalars and the next tile's rows prefetched a tile ahead;
//             TMEM release signalled to the leader (remote arrive for the peer)
#include <algorithm>
#include <cstdlib>

#include "pfc_internal.cuh"
#include "tc_common.cuh"

namespace pfc {
namespace {

constexpr int DP_BK = 64;
constexpr int DP_STAGES = 4;
constexpr int DP_ACC = 2;
// epilogue warps: 8 (2 per TMEM lane quadrant, 16 rows each); PFC_DP_EPI=16 (4 per quadrant, 8 rows each, twice
// the warps in flight) measured no faster: 0.352 vs 0.345 ms at the per-rank C4 shape, the kernel is DRAM-bound)
#ifndef PFC_DP_EPI
#define PFC_DP_EPI 8
#endif
constexpr int DP_EPI = PFC_DP_EPI;
constexpr int DP_NSET = DP_EPI / 4;                   // warps per TMEM lane quadrant (column sets of the staging)
constexpr int DP_RPW = 128 / DP_EPI;                  // rows per warp in the update
static_assert(DP_RPW == 8 || DP_RPW == 16, "epilogue layout");
constexpr int DP_THREADS = 32 * (2 + DP_EPI);
constexpr int DP_HALF = 128 * DP_BK * 2;              // 16 KB
constexpr int DP_STAGE = 2 * DP_HALF;                 // A (128 classes x 64 batch) + B (64 batch x 128 columns)
constexpr int DP_ST = 128 * 128 * 4;                  // fp32 staging of a 128 x 128 half tile
constexpr int DP_SMEM = DP_STAGES * DP_STAGE + DP_ST + 1024 + 256 + 3 * 128 * 4;
static_assert(DP_SMEM <= 232448, "shared memory overflow");

struct DpParams {
  int M, d;
  int tile_major;
  const SamplerState* st;
  SgdArgs sgd;
};

template <bool HINT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(DP_THREADS, 1)
    k_dw_sgd_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, DpParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float4* s_tile = reinterpret_cast<float4*>(smem + DP_STAGES * DP_STAGE);    // [128 rows][32 float4]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DP_STAGES * DP_STAGE + DP_ST);   // leader: both CTAs
  uint64_t* empty = full + DP_STAGES;                                          // each CTA
  uint64_t* acc_full = empty + DP_STAGES;                                      // each CTA
  uint64_t* acc_empty = acc_full + DP_ACC;                                     // leader: both CTAs' epilogues
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + DP_ACC);
  int32_t* s_rowj = reinterpret_cast<int32_t*>(smem + DP_STAGES * DP_STAGE + DP_ST + 256);
  float* s_inv = reinterpret_cast<float*>(s_rowj + 128);
  float* s_rad = s_inv + 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pr = (int)rank;
  const bool leader = pr == 0;
  const int k = p.st->k;
  const int ndq = p.d / 256, nct = (k + 255) / 256;    // units: (class tile, 256-column d tile)
  const int n_units = nct * ndq, n_kb = (p.M + DP_BK - 1) / DP_BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  auto dtile = [&](int u) { return (u % ndq) * 256; };
  // unit order: unit u = pair + i * npairs (the two column halves of a tile go to neighbouring pairs at the same
  // time); PFC_DW_ORDER=1: pair p takes the class tiles p, p + npairs, ... and, for each, its column halves back to
  // back (the tile's E' block re-read right after the first half) — measured slower (0.40 vs 0.346 ms, c4rank)
  const bool tile_major = p.tile_major;
  const int u_first = tile_major ? pair * ndq : pair;
  auto u_next = [&](int u) {
    if (!tile_major) return u + npairs;
    return (u % ndq + 1 < ndq) ? u + 1 : (u / ndq + npairs) * ndq;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < DP_STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < DP_ACC; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 2 * DP_EPI); }
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
      for (int u = u_first; u < n_units; u = u_next(u)) {
        const int c0 = (u / ndq) * 256 + 128 * pr, d0 = dtile(u) + 128 * pr;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], (uint32_t)(4 * DP_HALF));
          uint8_t* sa = smem + stage * DP_STAGE;
          tma_load_2d_pair(sa, &tmA, &full[stage], kb * DP_BK, c0);                       // G rows: its classes
          tma_load_2d_pair(sa + DP_HALF, &tmB, &full[stage], d0, kb * DP_BK);             // X_hat: its columns
          tma_load_2d_pair(sa + DP_HALF + DP_HALF / 2, &tmB, &full[stage], d0 + 64, kb * DP_BK);
          if (++stage == DP_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader)
    if (leader) {
      constexpr uint32_t IDESC = make_idesc(256, 256, false, true);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = u_first; u < n_units; u = u_next(u)) {
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tacc = tmem_base + acc * 256;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + stage * DP_STAGE), sb = sa + DP_HALF;
#pragma unroll
            for (int kk = 0; kk < DP_BK / 16; ++kk)
              tc_mma_pair(tacc, make_desc(sa + kk * 32, 16, 1024), make_desc(sb + kk * 2048, DP_HALF / 2, 1024), IDESC,
                          (kb > 0 || kk > 0) ? 1u : 0u);
            tc_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == DP_STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) tc_commit_pair(&acc_full[acc]);
        __syncwarp();
        if (++acc == DP_ACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (this CTA's 128 classes)
    const int ew = warp - 2;
    const int lg = warp & 3;
    const int row_in = lg * 32 + lane;
    const int eset = ew >> 2;                  // 0 .. DP_NSET-1
    const float lr = *p.sgd.lr;
    const uint64_t pol = HINT ? policy_evict_first() : 0;
    const uint32_t acce_leader = leader_addr(&acc_empty[0]);
    int32_t nx_j = -1;
    float nx_inv = 0.f, nx_rad = 0.f;
    auto scalars = [&](int u) {
      const int prow = (u / ndq) * 256 + 128 * pr + row_in;
      nx_j = -1; nx_inv = 0.f; nx_rad = 0.f;
      if (u < n_units && prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; nx_rad = p.sgd.dotw[prow]; }
    };
    if (eset == 0) scalars(u_first);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = u_first; u < n_units; u = u_next(u)) {
      const int dcol0 = dtile(u);
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DP_EPI) : "memory");   // previous tile consumed
      int32_t pf_j = -1;
      if (eset == 0) {
        s_rowj[row_in] = nx_j; s_inv[row_in] = nx_inv; s_rad[row_in] = nx_rad;
        scalars(u_next(u));
        pf_j = nx_j;
      }
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(lg * 32) << 16) + acc * 256;
      const int ew16 = ew * DP_RPW;
      // W / V rows of 4-row batch b (rows ew16 + 4b .. +3) of column half h into registers
      auto load = [&](int h, int b, float4 (&wv)[4], float4 (&mv)[4], int32_t (&jr)[4]) {
        const int col = dcol0 + h * 128 + lane * 4;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          jr[r] = s_rowj[ew16 + 4 * b + r];
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
      };
      auto update = [&](int h, int b, float4 (&wv)[4], float4 (&mv)[4], const int32_t (&jr)[4]) {
        const int col = dcol0 + h * 128 + lane * 4;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int rr = ew16 + 4 * b + r;
          if (jr[r] >= 0) {
            const float inv = s_inv[rr], rad = s_rad[rr] * inv;
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
      };
      auto stage = [&](int h) {
#pragma unroll 1
        for (int c = eset * (8 / DP_NSET); c < (eset + 1) * (8 / DP_NSET); ++c) {
          uint32_t v[16];
          tmem_ld16(tacc + h * 128 + c * 16, v);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            s_tile[row_in * 32 + ((c * 4 + q) ^ (row_in & 31))] =
                make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                            __uint_as_float(v[4 * q + 3]));
        }
      };
      // software pipeline: the W / V loads of the next batch are in flight while the current batch (or the TMEM
      // staging of the next column half) runs
      float4 wa[4], ma[4], wb[4], mb[4];
      int32_t ja[4], jb[4];
      load(0, 0, wa, ma, ja);
      stage(0);
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DP_EPI) : "memory");
      load(0, 1, wb, mb, jb);
      update(0, 0, wa, ma, ja);
      if (pf_j >= 0) {   // the next tile's W / V row segments (256 columns) into L2
        const int ndc = dtile(u_next(u));
        const float* wp = p.sgd.W + (int64_t)pf_j * p.d + ndc;
        const float* vp = p.sgd.V + (int64_t)pf_j * p.d + ndc;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
        }
      }
      if constexpr (DP_RPW == 16) {
        load(0, 2, wa, ma, ja);
        update(0, 1, wb, mb, jb);
        load(0, 3, wb, mb, jb);
        update(0, 2, wa, ma, ja);
        load(1, 0, wa, ma, ja);
        update(0, 3, wb, mb, jb);
      } else {
        load(1, 0, wa, ma, ja);
        update(0, 1, wb, mb, jb);
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DP_EPI) : "memory");   // staging free
      stage(1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&acc_empty[acc]);
        else mbar_arrive_cluster(acce_leader + acc * 8);
      }
      if (++acc == DP_ACC) { acc = 0; acc_phase ^= 1; }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DP_EPI) : "memory");
      load(1, 1, wb, mb, jb);
      update(1, 0, wa, ma, ja);
      if constexpr (DP_RPW == 16) {
        load(1, 2, wa, ma, ja);
        update(1, 1, wb, mb, jb);
        load(1, 3, wb, mb, jb);
        update(1, 2, wa, ma, ja);
        update(1, 3, wb, mb, jb);
      } else {
        update(1, 1, wb, mb, jb);
      }
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

bool dw_sgd_pair_enabled(const Sizes& sz) {
  const int forced = env_int("PFC_DW_PAIR", 1);
  return forced != 0 && sz.M >= 2048 && sz.d % 256 == 0 && sz.k_pad % 256 == 0;   // M = 1024: DWF2 is as fast
}

int launch_dw_sgd_pair_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                          const SgdArgs& sa, cudaStream_t s) {
  // W / V streamed with an L2 evict-first policy (the G tile shared by the pairs of both d-halves stays resident);
  // PFC_DW_HINT=0 disables
  const bool hint = env_int("PFC_DW_HINT", 1) != 0;
  auto kern = hint ? k_dw_sgd_pair<true> : k_dw_sgd_pair<false>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dw_sgd_pair<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, DP_SMEM);
    cudaFuncSetAttribute(k_dw_sgd_pair<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, DP_SMEM);
    attr = true;
  }
  const CUtensorMap a = make_map(G, sz.k_pad, sz.M_pad, 64, 128);    // G class-major: 128 classes x 64 batch
  const CUtensorMap b = make_map(Xb, sz.M_pad, sz.d, 64, 64);        // X_hat: 64 batch rows x 64 columns
  TC_MAPS_OK();
  // tile-major order measured slower at the per-rank C4 shape (0.40 vs 0.346 ms): the interleaved order is the default
  const int order = env_int("PFC_DW_ORDER", 0);
  DpParams p{};
  p.M = sz.M; p.d = sz.d; p.st = st; p.sgd = sa; p.tile_major = order;
  const int64_t units = (sz.k_pad / 256) * (sz.d / 256);
  const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(units, num_sms() / 2));   // 74 co-resident
  kern<<<2 * pairs, DP_THREADS, DP_SMEM, s>>>(a, b, p);
  return 1;
}

}  // namespace pfc
