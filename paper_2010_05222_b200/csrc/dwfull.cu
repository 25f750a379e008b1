// K11 + radial dot + K12 on CTA pairs over ALL d columns of a 256-class tile (train step, bf16 tensor-core path,
// M > 256, d = 512): dW_hat = E'^T X~ (E-form, R26) or G^T X_hat (Alg.1 L10) with
// tcgen05.mma.cta_group::2 (M = 256 classes split across the pair, two N = 256 column halves, K = the global batch),
// the radial dot w_hat . dW_hat of each class formed from the accumulator itself (R29), and the lazy momentum-SGD
// update of the tile's W / V rows (R14 backprop through ||w||; R15 optimiser) in each CTA's epilogue.
//
// One pair owns whole class tiles and both column halves, so the tile's E' (or G) block is read from HBM exactly once
// (each K block's A stage feeds the MMAs of both halves) and no separate radial-dot pass over E is needed.
// TMEM holds the whole 128-class x 512-column accumulator of a tile; to let the next tile's MMAs start at once the
// epilogue evacuates it right away: columns [0, 256) into a 128 KB fp32 staging tile in shared memory, columns
// [256, 512) into registers (thread = row, 128 per thread), then releases TMEM. From there:
//   partial dots: h1 from the registers (thread = row, W row segment by 32-byte loads), h0 from the staging
//   (warp = row, coalesced W segments); full dot = ((h0 + eset0) + eset1), a fixed order (R29)
//   update of h1 from the registers (thread = row, 32-byte W / V pieces), then of h0 from the staging (warp = row,
//   coalesced 512-byte W / V segments).
// The tile's W and V rows are prefetched into L2 when its scalars are known (while its MMAs still run).
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
constexpr int DF_STAGES = 2;
constexpr int DF_EPI = 8;
constexpr int DF_THREADS = 32 * (2 + DF_EPI);
constexpr int DF_HALF = 128 * DF_BK * 2;              // 16 KB
constexpr int DF_STAGE = 3 * DF_HALF;                 // A (128 classes x 64 batch) + B (64 batch x 128 cols) x 2
constexpr int DF_ST = 128 * 256 * 4;                  // fp32 staging of 128 rows x 256 columns
constexpr int DF_SMEM = DF_STAGES * DF_STAGE + DF_ST + 1024 + 256 + 3 * 128 * 4;
static_assert(DF_SMEM <= 232448, "shared memory overflow");

struct DfParams {
  int M, d;
  const SamplerState* st;
  SgdArgs sgd;
};

// staging index of float4 q (0..63) of row r: XOR swizzle inside each 32-float4 half so that both the thread-per-row
// writes and the lane-per-column reads are bank-conflict free
__device__ __forceinline__ int sidx(int r, int q) { return r * 64 + (q & 32) + ((q & 31) ^ (r & 31)); }

template <bool HINT>
__device__ __forceinline__ void st8h(float* a, const float (&v)[8], uint64_t pol) {
  if (HINT)
    asm volatile("st.global.L2::cache_hint.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(a), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "l"(pol)
                 : "memory");
  else
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

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
  uint64_t* acc_empty = acc_full + 1;                                          // leader: both CTAs' epilogues
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  int32_t* s_rowj = reinterpret_cast<int32_t*>(smem + DF_STAGES * DF_STAGE + DF_ST + 256);
  float* s_inv = reinterpret_cast<float*>(s_rowj + 128);
  float* s_dot = s_inv + 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pr = (int)cluster_rank();
  const bool leader = pr == 0;
  const int k = p.st->k;
  const int nct = (k + 255) / 256;
  const int n_kb = (p.M + DF_BK - 1) / DF_BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < DF_STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 2 * DF_EPI);
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
      for (int t = pair; t < nct; t += npairs) {
        const int c0 = t * 256 + 128 * pr, d0 = 128 * pr;
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], (uint32_t)(6 * DF_HALF));
          uint8_t* sa = smem + stage * DF_STAGE;
          tma_load_2d_pair(sa, &tmA, &full[stage], kb * DF_BK, c0);                       // E' rows: its classes
#pragma unroll
          for (int h = 0; h < 2; ++h) {                                                   // X~: its columns of h
            uint8_t* sb = sa + DF_HALF * (1 + h);
            tma_load_2d_pair(sb, &tmB, &full[stage], 256 * h + d0, kb * DF_BK);
            tma_load_2d_pair(sb + DF_HALF / 2, &tmB, &full[stage], 256 * h + d0 + 64, kb * DF_BK);
          }
          if (++stage == DF_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader)
    if (leader) {
      constexpr uint32_t IDESC = make_idesc(256, 256, false, true);
      int stage = 0;
      uint32_t phase = 0, eph = 0;
      for (int t = pair; t < nct; t += npairs) {
        mbar_wait(acc_empty, eph ^ 1);
        eph ^= 1;
        tc_fence_after();
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + stage * DF_STAGE);
#pragma unroll
            for (int kk = 0; kk < DF_BK / 16; ++kk)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                tc_mma_pair(tmem_base + 256 * h, make_desc(sa + kk * 32, 16, 1024),
                            make_desc(sa + DF_HALF * (1 + h) + kk * 2048, DF_HALF / 2, 1024), IDESC,
                            (kb > 0 || kk > 0) ? 1u : 0u);
            tc_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == DF_STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) tc_commit_pair(acc_full);
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (this CTA's 128 classes)
    const int ew = warp - 2;            // 0..7: rows ew*16 .. ew*16+15 in the lane-per-column passes
    const int lg = warp & 3;            // TMEM lane quadrant
    const int row_in = lg * 32 + lane;  // thread-per-row passes
    const int eset = ew >> 2;           // column half (128 of 256) in the thread-per-row passes
    const float lr = *p.sgd.lr;
    const float mu = p.sgd.mu, lam = p.sgd.lambda;
    const uint64_t pol = HINT ? policy_evict_first() : 0;
    const uint32_t acce_leader = leader_addr(acc_empty);
    const uint32_t tl = tmem_base + ((uint32_t)(lg * 32) << 16);
    const int d = p.d;
    auto st8 = [&](float* a, const float (&v)[8], uint64_t pl) { st8h<HINT>(a, v, pl); };
    int32_t nx_j = -1;
    float nx_inv = 0.f;
    auto scalars = [&](int t) {
      const int prow = t * 256 + 128 * pr + row_in;
      nx_j = -1; nx_inv = 0.f;
      if (t < nct && prow < k) { nx_j = p.sgd.idx[prow]; nx_inv = p.sgd.inv_norm[prow]; }
    };
    if (eset == 0) scalars(pair);
    // momentum-SGD update of the 16 rows of this warp over the 256 columns [h*256, h*256 + 256) from the staging,
    // two 128-column sub-halves of 4-row batches, the W / V loads of the next batch in flight (W, V rows L2-resident:
    // prefetched at the start of the tile)
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
              wv[slot][r] = *reinterpret_cast<const float4*>(p.sgd.W + (int64_t)jr[slot][r] * d + col);
              mv[slot][r] = *reinterpret_cast<const float4*>(p.sgd.V + (int64_t)jr[slot][r] * d + col);
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

    uint32_t fph = 0;
    for (int t = pair; t < nct; t += npairs) {
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // previous tile fully consumed
      if (eset == 0) {
        s_rowj[row_in] = nx_j; s_inv[row_in] = nx_inv;
        if (nx_j >= 0) {   // this row's W and V (2 x 2 KB) into L2 while the tile's MMAs run
          const float* wr = p.sgd.W + (int64_t)nx_j * d;
          const float* vr = p.sgd.V + (int64_t)nx_j * d;
#pragma unroll
          for (int l = 0; l < 16; ++l) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(wr + 32 * l));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vr + 32 * l));
          }
        }
        scalars(t + npairs);
      }
      mbar_wait(acc_full, fph);
      fph ^= 1;
      tc_fence_after();
      // evacuate TMEM: h0 -> staging (fp32), h1 -> registers (this eset's 128 columns of row row_in)
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t v[16];
        tmem_ld16(tl + eset * 128 + c * 16, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          s_st[sidx(row_in, eset * 32 + c * 4 + q)] =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                          __uint_as_float(v[4 * q + 3]));
      }
      uint32_t hr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tl + 256 + eset * 128 + c * 32, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) hr[c * 32 + e] = v[e];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {   // TMEM free: the next tile's MMAs may start
        if (leader) mbar_arrive(acc_empty);
        else mbar_arrive_cluster(acce_leader);
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // staging and scalars complete
      // partial dot over h1 (thread = row) from the registers
      const int32_t jme = s_rowj[row_in];
      float pd = 0.f;
      if (jme >= 0) {
        const float* wp = p.sgd.W + (int64_t)jme * d + 256 + eset * 128;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float w8[8];
          ld8(wp + c * 8, w8);
#pragma unroll
          for (int e = 0; e < 8; ++e) pd = fmaf(w8[e], __uint_as_float(hr[c * 8 + e]), pd);
        }
      }
      // partial dots over h0: warp per row, lanes along the columns, from the staging
#pragma unroll 1
      for (int r4 = 0; r4 < 16; r4 += 4) {
        float4 wa[4], wb[4];
        int32_t j4[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          j4[r] = s_rowj[ew * 16 + r4 + r];
          if (j4[r] >= 0) {
            const float* wp = p.sgd.W + (int64_t)j4[r] * d + lane * 4;
            wa[r] = *reinterpret_cast<const float4*>(wp);
            wb[r] = *reinterpret_cast<const float4*>(wp + 128);
          } else {
            wa[r] = wb[r] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int rr = ew * 16 + r4 + r;
          const float4 ga = s_st[sidx(rr, lane)], gb = s_st[sidx(rr, 32 + lane)];
          float v = wa[r].x * ga.x + wa[r].y * ga.y + wa[r].z * ga.z + wa[r].w * ga.w;
          v += wb[r].x * gb.x + wb[r].y * gb.y + wb[r].z * gb.z + wb[r].w * gb.w;
          v = warp_sum(v);
          if (lane == 0) s_dot[rr] = v;
        }
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // h0 partials written
      if (eset == 0) s_dot[row_in] += pd;
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");
      if (eset == 1) s_dot[row_in] += pd;
      asm volatile("bar.sync 3, %0;" ::"n"(32 * DF_EPI) : "memory");   // full-row dots complete
      // update of h1 straight from the registers: thread = row, 32-byte W / V pieces (L2 hits after the prefetch)
      if (jme >= 0) {
        const float inv = s_inv[row_in];
        const float rad = s_dot[row_in] * inv * inv;          // (w_hat . dW_hat) / ||w||
        float* wp = p.sgd.W + (int64_t)jme * d + 256 + eset * 128;
        float* vp = p.sgd.V + (int64_t)jme * d + 256 + eset * 128;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float w8[8], m8[8];
          ld8(wp + c * 8, w8);
          ld8(vp + c * 8, m8);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            m8[e] = mu * m8[e] + (__uint_as_float(hr[c * 8 + e]) - w8[e] * rad) * inv + lam * w8[e];
            w8[e] -= lr * m8[e];
          }
          st8(vp + c * 8, m8, pol);
          st8(wp + c * 8, w8, pol);
        }
      }
      update_half(0);
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
  const int forced = env_int("PFC_DWFULL", 0);
  return forced != 0 && gsc == 0 && sz.M > 256 && sz.d == 512 && sz.k_pad % 256 == 0;
}

int launch_dw_sgd_full_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                          const SgdArgs& sa, cudaStream_t s) {
  // W / V stores carry an L2 evict-first policy (PFC_DW_HINT=0 disables); their loads are L2 hits after the prefetch
  const bool hint = env_int("PFC_DW_HINT", 1) != 0;
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
