// K11 + radial dot + K12 on CTA pairs over ALL d columns of a 256-class tile (train step, bf16 tensor-core path,
// M > 256, d in {256, 512}): dW_hat = E'^T X~ (E-form, R26) or G^T X_hat (Alg.1 L10) with
// tcgen05.mma.cta_group::2 (M = 256 classes split across the pair, N = 256 columns per half, K = the global batch),
// the radial dot w_hat . dW_hat of each class formed from the accumulator itself, and the lazy momentum-SGD update
// of the tile's W / V rows (R14 backprop through ||w||; R15 optimiser) in each CTA's epilogue.
//
// One pair owns whole class tiles, so the tile's E' (or G) block is read from HBM once (its second half-pass hits
// L2 right after the first) and no separate radial-dot pass over E is needed (the k_eform_dotw pass of the
// k_dw_sgd_pair path). Per tile and CTA (128 classes x d columns), TMEM holds two 256-column accumulators:
//   buffer 0 = columns [0, 256) (h0), buffer 1 = columns [256, 512) (h1) when d = 512; when d = 256 the tiles
//   alternate buffers.
// Epilogue order (d = 512): h0 accumulator -> fp32 staging in shared memory, TMEM released (the next tile's h0
// MMAs start); partial dots over h0 (W rows read coalesced; the h1 W segments prefetched into L2); h1 partial
// dots straight from TMEM (thread = row); update of h0 from the staging (W from L2, V from HBM); h1 accumulator ->
// staging, TMEM released; update of h1. The full-row dot is ((h0 + eset0) + eset1): a fixed summation order.
//   warp 0    TMA producer (its halves, onto the leader's mbarrier)
//   warp 1    TMEM allocation (cta_group::2, 512 columns); MMA issue (leader), commits multicast to both CTAs
//   warps 2-9 epilogue (this CTA's 128 classes)
#include <algorithm>
#include <cstdlib>

#include "pfc_internal.cuh"
#include "tc_common.cuh"

namespace pfc {
namespace {

constexpr int DF_BK = 64;
constexpr int DF_STAGES = 3;
constexpr int DF_EPI = 8;
constexpr int DF_THREADS = 32 * (2 + DF_EPI);
constexpr int DF_HALF = 128 * DF_BK * 2;              // 16 KB
constexpr int DF_STAGE = 2 * DF_HALF;                 // A (128 classes x 64 batch) + B (64 batch x 128 columns)
constexpr int DF_ST = 128 * 256 * 4;                  // fp32 staging of 128 rows x 256 columns
constexpr int DF_SMEM = DF_STAGES * DF_STAGE + DF_ST + 1024 + 256 + 3 * 128 * 4;
static_assert(DF_SMEM <= 232448, "shared memory overflow");

struct DfParams {
  int M, d;
  const SamplerState* st;
  SgdArgs sgd;
};

// staging index of float4 q (0..63) of row r: XOR swizzle inside each 32-float4 half so that both the thread-per-row
// writes (TMEM -> smem) and the lane-per-column reads of the update are bank-conflict free
__device__ __forceinline__ int sidx(int r, int q) { return r * 64 + (q & 32) + ((q & 31) ^ (r & 31)); }

__device__ __forceinline__ void ld8(const float* a, float (&v)[8]) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(a));
}

template <bool HINT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(DF_THREADS, 1)
    k_dw_sgd_full(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, DfParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float4* s_st = reinterpret_cast<float4*>(smem + DF_STAGES * DF_STAGE);        // [128 rows][64 float4]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DF_STAGES * DF_STAGE + DF_ST);   // leader: both CTAs
  uint64_t* empty = full + DF_STAGES;                                          // each CTA
  uint64_t* acc_full = empty + DF_STAGES;                                      // each CTA
  uint64_t* acc_empty = acc_full + 2;                                          // leader: both CTAs' epilogues
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int32_t* s_rowj = reinterpret_cast<int32_t*>(smem + DF_STAGES * DF_STAGE + DF_ST + 256);
  float* s_inv = reinterpret_cast<float*>(s_rowj + 128);
  float* s_dot = s_inv + 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pr = (int)cluster_rank();
  const bool leader = pr == 0;
  const int k = p.st->k;
  const int nh = p.d / 256, nct = (k + 255) / 256;
  const int n_kb = (p.M + DF_BK - 1) / DF_BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < DF_STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 2 * DF_EPI); }
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
      for (int t = pair; t < nct; t += npairs)
        for (int h = 0; h < nh; ++h) {
          const int c0 = t * 256 + 128 * pr, d0 = h * 256 + 128 * pr;
          for (int kb = 0; kb < n_kb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (leader) mbar_expect_tx(&full[stage], (uint32_t)(4 * DF_HALF));
            uint8_t* sa = smem + stage * DF_STAGE;
            tma_load_2d_pair(sa, &tmA, &full[stage], kb * DF_BK, c0);                     // E' rows: its classes
            tma_load_2d_pair(sa + DF_HALF, &tmB, &full[stage], d0, kb * DF_BK);           // X~: its columns
            tma_load_2d_pair(sa + DF_HALF + DF_HALF / 2, &tmB, &full[stage], d0 + 64, kb * DF_BK);
            if (++stage == DF_STAGES) { stage = 0; phase ^= 1; }
          }
        }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader)
    if (leader) {
      constexpr uint32_t IDESC = make_idesc(256, 256, false, true);
      int stage = 0, it = 0;
      uint32_t phase = 0, eph0 = 0, eph1 = 0;
      for (int t = pair; t < nct; t += npairs, ++it)
        for (int h = 0; h < nh; ++h) {
          const int buf = nh == 2 ? h : (it & 1);
          mbar_wait(&acc_empty[buf], (buf ? eph1 : eph0) ^ 1);
          if (buf) eph1 ^= 1; else eph0 ^= 1;
          tc_fence_after();
          const uint32_t tacc = tmem_base + buf * 256;
          for (int kb = 0; kb < n_kb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t sa = smem_u32(smem + stage * DF_STAGE), sb = sa + DF_HALF;
#pragma unroll
              for (int kk = 0; kk < DF_BK / 16; ++kk)
                tc_mma_pair(tacc, make_desc(sa + kk * 32, 16, 1024), make_desc(sb + kk * 2048, DF_HALF / 2, 1024),
                            IDESC, (kb > 0 || kk > 0) ? 1u : 0u);
              tc_commit_pair(&empty[stage]);
            }
            __syncwarp();
            if (++stage == DF_STAGES) { stage = 0; phase ^= 1; }
          }
          if (lane == 0) tc_commit_pair(&acc_full[buf]);
          __syncwarp();
        }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (this CTA's 128 classes)
    const int ew = warp - 2;            // 0..7: rows ew*16 .. ew*16+15 in the lane-per-column passes
    const int lg = warp & 3;            // TMEM lane quadrant
    const int row_in = lg * 32 + lane;  // thread-per-row passes
    const int eset = ew >> 2;           // column half (128 of the 256) in the thread-per-row passes
    const float lr = *p.sgd.lr;
    const float mu = p.sgd.mu, lam = p.sgd.lambda;
    const uint64_t pol = HINT ? policy_evict_first() : 0;
    const uint32_t acce_leader = leader_addr(&acc_empty[0]);
    const uint32_t tl = tmem_base + ((uint32_t)(lg * 32) << 16);
    const int d = p.d;
    int32_t nx_j = -1;
    float nx_inv = 0.f;
    auto scalars = [&](int t) {
      const int prow = t * 256 + 128 * pr + row_in;
      nx_j = -1; nx_inv = 0.f;
      if (t < nct && prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; }
    };
    if (eset == 0) scalars(pair);
    // TMEM buffer -> fp32 staging (thread = row, this eset's 128 columns)
    auto stage_acc = [&](int buf) {
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t v[16];
        tmem_ld16(tl + buf * 256 + eset * 128 + c * 16, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          s_st[sidx(row_in, eset * 32 + c * 4 + q)] =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                          __uint_as_float(v[4 * q + 3]));
      }
    };
    auto release = [&](int buf) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&acc_empty[buf]);
        else mbar_arrive_cluster(acce_leader + buf * 8);
      }
    };
    // the 16 rows of this warp: momentum-SGD update of the 256 columns [h*256, h*256 + 256) from the staging, in two
    // 128-column sub-halves of 4-row batches; the W / V loads of the next batch in flight during the current one
    auto update_half = [&](int h) {
#pragma unroll 1
      for (int sh = 0; sh < 2; ++sh) {
        const int col = h * 256 + sh * 128 + lane * 4;
        float4 wv[2][4], mv[2][4];
        int32_t jr[2][4];
        auto load = [&](int b, int slot) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int rr = ew * 16 + 4 * b + r;
            jr[slot][r] = s_rowj[rr];
            if (jr[slot][r] >= 0) {
              const float* wp = p.sgd.W + (int64_t)jr[slot][r] * d + col;
              const float* vp = p.sgd.V + (int64_t)jr[slot][r] * d + col;
              wv[slot][r] = *reinterpret_cast<const float4*>(wp);      // second touch: an L2 hit
              mv[slot][r] = HINT ? ld_hint4(vp, pol) : *reinterpret_cast<const float4*>(vp);
            }
          }
        };
        auto upd = [&](int b, int slot) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int rr = ew * 16 + 4 * b + r;
            if (jr[slot][r] >= 0) {
              const float inv = s_inv[rr];
              const float rad = s_dot[rr] * inv * inv;        // (w_hat . dW_hat) / ||w||
              const float4 g = s_st[sidx(rr, sh * 32 + lane)];
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
        load(0, 0);
        load(1, 1);
        upd(0, 0);
        load(2, 0);
        upd(1, 1);
        load(3, 1);
        upd(2, 0);
        upd(3, 1);
      }
    };

    uint32_t fph0 = 0, fph1 = 0;
    int it = 0;
    for (int t = pair; t < nct; t += npairs, ++it) {
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // previous tile fully consumed
      if (eset == 0) {
        s_rowj[row_in] = nx_j; s_inv[row_in] = nx_inv;
        scalars(t + npairs);
      }
      const int b0 = nh == 2 ? 0 : (it & 1);
      mbar_wait(&acc_full[b0], b0 ? fph1 : fph0);
      if (b0) fph1 ^= 1; else fph0 ^= 1;
      tc_fence_after();
      stage_acc(b0);
      release(b0);                                                     // the next h0 MMAs may start
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // staging and scalars complete
      // partial radial dots over h0: warp per row, lanes along the columns (the first, DRAM touch of the W rows)
#pragma unroll 1
      for (int r8 = 0; r8 < 16; r8 += 8) {
        float4 wa[8], wb[8];
        int32_t j8[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int rr = ew * 16 + r8 + r;
          j8[r] = s_rowj[rr];
          if (j8[r] >= 0) {
            const float* wp = p.sgd.W + (int64_t)j8[r] * d + lane * 4;
            wa[r] = *reinterpret_cast<const float4*>(wp);
            wb[r] = *reinterpret_cast<const float4*>(wp + 128);
            if (nh == 2 && lane < 8)   // the row's h1 segment (8 lines of 128 B) into L2 for the h1 dot pass
              asm volatile("prefetch.global.L2 [%0];" ::"l"(p.sgd.W + (int64_t)j8[r] * d + 256 + lane * 32));
          } else {
            wa[r] = wb[r] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int rr = ew * 16 + r8 + r;
          const float4 ga = s_st[sidx(rr, lane)], gb = s_st[sidx(rr, 32 + lane)];
          float v = wa[r].x * ga.x + wa[r].y * ga.y + wa[r].z * ga.z + wa[r].w * ga.w;
          v += wb[r].x * gb.x + wb[r].y * gb.y + wb[r].z * gb.z + wb[r].w * gb.w;
          v = warp_sum(v);
          if (lane == 0) s_dot[rr] = v;
        }
      }
      if (nh == 2) {
        // partial dots over h1 straight from TMEM: thread = row, this eset's 128 columns in 4 chunks of 32
        mbar_wait(&acc_full[1], fph1);
        fph1 ^= 1;
        tc_fence_after();
        const int32_t j = s_rowj[row_in];
        const float* wp = p.sgd.W + (int64_t)(j >= 0 ? j : 0) * d + 256 + eset * 128;
        float pd = 0.f;
        // tcgen05.ld is warp-collective (.sync.aligned): every lane issues it, rows past k_i included; only the W
        // loads and the products are predicated
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float w8[4][8];
          if (j >= 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ld8(wp + c * 32 + q * 8, w8[q]);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int e = 0; e < 8; ++e) w8[q][e] = 0.f;
          }
          uint32_t v[32];
          tmem_ld32(tl + 256 + eset * 128 + c * 32, v);
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int e = 0; e < 8; ++e) pd += w8[q][e] * __uint_as_float(v[q * 8 + e]);
        }
        asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // h0 partials written
        if (eset == 0) s_dot[row_in] += pd;
        asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");
        if (eset == 1) s_dot[row_in] += pd;
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");     // full-row dots complete
      update_half(0);
      if (nh == 2) {
        asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // staging free
        stage_acc(1);
        release(1);
        asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");
        update_half(1);
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

bool dw_sgd_full_enabled(const Sizes& sz, int gsc) {
  static const int forced = [] { const char* e = std::getenv("PFC_DWFULL"); return e ? std::atoi(e) : 0; }();
  return forced != 0 && gsc == 0 && sz.M > 256 && (sz.d == 256 || sz.d == 512) && sz.k_pad % 256 == 0;
}

int launch_dw_sgd_full_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                          const SgdArgs& sa, cudaStream_t s) {
  // V streamed with an L2 evict-first policy; W's first touch (the dot pass) keeps the default policy so that the
  // update's second read hits L2; PFC_DW_HINT=0 disables the hints
  static const bool hint = [] { const char* e = std::getenv("PFC_DW_HINT"); return !e || std::atoi(e) != 0; }();
  auto kern = hint ? k_dw_sgd_full<true> : k_dw_sgd_full<false>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dw_sgd_full<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, DF_SMEM);
    cudaFuncSetAttribute(k_dw_sgd_full<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, DF_SMEM);
    attr = true;
  }
  const CUtensorMap a = make_map(G, sz.k_pad, sz.M_pad, 64, 128);    // E' / G class-major: 128 classes x 64 batch
  const CUtensorMap b = make_map(Xb, sz.M_pad, sz.d, 64, 64);        // X~ / X_hat: 64 batch rows x 64 columns
  TC_MAPS_OK();
  DfParams p{};
  p.M = sz.M; p.d = sz.d; p.st = st; p.sgd = sa;
  const int64_t tiles = sz.k_pad / 256;
  const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms() / 2));
  kern<<<2 * pairs, DF_THREADS, DF_SMEM, s>>>(a, b, p);
  return 1;
}

}  // namespace pfc
