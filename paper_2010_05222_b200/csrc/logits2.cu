// K6 logits for global batches M > 256 on CTA pairs (tcgen05 cta_group::2): C[M x k] = X_hat . W_s^T with the same
// fused epilogue as the single-CTA kernel of gemm_tc.cu (Alg.1 L3-5; fp16 class-major cosines,
// per-(row, 128-column tile) max / sum partials with the target column excluded, R22).
//
// A cluster of two CTAs computes a 256 (batch rows) x 256 (classes) tile: CTA r stages batch rows 128 r .. +127
// of X_hat and class rows 128 r .. +127 of W_s per 64-wide K block (TMA, 128-byte swizzle, both landing on the
// leader CTA's mbarrier), and the leader's single MMA thread issues tcgen05.mma.cta_group::2 (M = 256, N = 256),
// which reads A from both CTAs' shared memory along M and B along N and accumulates into each CTA's TMEM its own
// 128 rows x 256 columns. Per K block and SM that is 32 KB of operands for 4.2 MFLOP instead of 48 KB for the
// single-CTA 256 x 128 tile: the contraction is less bound by the L2 -> SM operand stream at large M.
//   warp 0     TMA producer (each CTA its halves)
//   warp 1     TMEM allocation (both CTAs, cta_group::2); MMA issue (leader CTA only); commits multicast to both
//   warps 2-17 epilogue (each CTA its 128 rows): four sets of 4 warps, 64 columns each; the two sets of a
//              128-column logits tile combine their (max, sum) through shared memory; TMEM release is signalled
//              to the leader's barrier (remote arrive for the peer CTA)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pfc_internal.cuh"
#include "tc_common.cuh"

namespace pfc {
namespace {

constexpr int L2_BK = 64;
constexpr int L2_STAGES = 6;
constexpr int L2_ACC = 2;
constexpr int L2_EPI = 16;
constexpr int L2_THREADS = 32 * (2 + L2_EPI);
constexpr int L2_HALF = 128 * L2_BK * 2;                // 16 KB: 128 rows x 64 K (bf16)
constexpr int L2_STAGE = 2 * L2_HALF;                   // A half + B half
constexpr int L2_PART = L2_ACC * 2 * 128 * 8;           // s_part: [acc][ltile pair][row] float2
constexpr int L2_SMEM = L2_STAGES * L2_STAGE + 1024 + 256 + L2_PART;
// ARES (A resident, d <= 512): this CTA's 128 rows of X_hat stay in shared memory for the whole kernel (each pair
// keeps one 256-row M tile and walks class tiles), only the W_s tiles stream: half the operand traffic from L2
constexpr int L2R_KB = 8;                               // d / 64 <= 8
constexpr int L2R_A = L2R_KB * L2_HALF;                 // 128 KB
#ifndef PFC_L2R_STAGES
#define PFC_L2R_STAGES 6
#endif
constexpr int L2R_STAGES = PFC_L2R_STAGES;              // B ring: 16 KB stages (no s_part: ARES folds per thread)
constexpr int L2R_SMEM = L2R_A + L2R_STAGES * L2_HALF + 1024 + 256;
static_assert(L2_SMEM <= 232448 && L2R_SMEM <= 232448, "shared memory overflow");
static_assert(L2_SMEM <= 232448, "shared memory overflow");
struct L2Params {
  int M, ldm, d;
  const SamplerState* st;
  const int32_t* tcol;
  float s_log2e, scale;
  __half* cosv;
  float2* partials;
  int n_ltiles;
  unsigned long long* trace;   // diagnostic build (PFC_DWX_DIAG) with PFC_LP_TRACE=1: per CTA, summed wait times
};
#ifndef PFC_DWX_DIAG
#define PFC_DWX_DIAG 0
#endif
constexpr bool kLpDiag = PFC_DWX_DIAG != 0;
__device__ __forceinline__ unsigned long long lp_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// EF (E-form train step, DESIGN.md f1): store E = bf16(e^{s c}) of the fp16-rounded cosine the partials use (0 at
// the target and padding columns) instead of the cosine; the softmax-gradient pass then disappears (dX / dW
// contract E directly, see k_eform_prep / k_eform_dotw)
template <bool EF, bool ARES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(L2_THREADS, 1)
    k_logits_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, L2Params p) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int NST = ARES ? L2R_STAGES : L2_STAGES;               // ring stages
  constexpr int STB = ARES ? L2_HALF : L2_STAGE;                   // ring stage bytes (ARES: B only)
  constexpr int RING0 = ARES ? L2R_A : 0;                          // ring offset (ARES: after the resident A)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING0 + NST * STB);   // leader: both CTAs' bytes
  uint64_t* empty = full + NST;                                                 // each CTA: MMA done with stage
  uint64_t* acc_full = empty + NST;                                             // each CTA
  uint64_t* acc_empty = acc_full + L2_ACC;                                      // leader: both CTAs' epilogues
  uint64_t* a_full = acc_empty + L2_ACC;                                        // ARES: the resident A landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 1);
  float2* s_part = reinterpret_cast<float2*>(smem + RING0 + NST * STB + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int k = p.st->k;
  const int mt = (p.M + 255) / 256, nt = (k + 255) / 256;
  const int n_kb = p.d / L2_BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // units: M fastest, so concurrent pairs share the W_s tile in L2. ARES: pair p keeps M tile p % mt and takes
  // the class tiles g, g + G, ... of its group g = p / mt (npairs = G mt); the pairs of a group run the same class
  // tile at the same time
  const int G = ARES ? npairs / mt : 1;
  const int n_units = ARES ? (pair / mt < G ? (nt - pair / mt + G - 1) / G : 0) : mt * nt;
  auto unit = [&](int i, int& m0, int& n0) {
    if (ARES) { m0 = (pair % mt) * 256; n0 = (pair / mt + i * G) * 256; }
    else { const int u = pair + i * npairs; m0 = (u % mt) * 256; n0 = (u / mt) * 256; }
  };
  const int n_iter = ARES ? n_units : (pair < n_units ? (n_units - pair + npairs - 1) / npairs : 0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < L2_ACC; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 2 * L2_EPI); }
    mbar_init(a_full, 1);
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
  cluster_sync();            // barriers initialised and TMEM allocated in both CTAs before any remote traffic
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const unsigned long long tk0 = (kLpDiag && p.trace) ? lp_clock() : 0ull;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer (this CTA's halves)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      if (ARES && n_iter > 0) {   // this CTA's 128 rows of X_hat, all K blocks, once
        int m0, n0;
        unit(0, m0, n0);
        if (leader) mbar_expect_tx(a_full, (uint32_t)(2 * n_kb * L2_HALF));
        for (int kb = 0; kb < n_kb; ++kb)
          tma_load_2d_pair(smem + kb * L2_HALF, &tmA, a_full, kb * L2_BK, m0 + 128 * (int)rank);
      }
      for (int it = 0; it < n_iter; ++it) {
        int m0, n0;
        unit(it, m0, n0);
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + RING0 + stage * STB;
          if (ARES) {
            if (leader) mbar_expect_tx(&full[stage], (uint32_t)(2 * L2_HALF));
            tma_load_2d_pair(sa, &tmB, &full[stage], kb * L2_BK, n0 + 128 * (int)rank);
          } else {
            if (leader) mbar_expect_tx(&full[stage], (uint32_t)(4 * L2_HALF));
            tma_load_2d_pair(sa, &tmA, &full[stage], kb * L2_BK, m0 + 128 * (int)rank);
            tma_load_2d_pair(sa + L2_HALF, &tmB, &full[stage], kb * L2_BK, n0 + 128 * (int)rank);
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    if (leader) {
      constexpr uint32_t IDESC = make_idesc(256, 256, false, false, true);   // fp16 operands (R27)
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      if (ARES && n_iter > 0) {
        mbar_wait(a_full, 0);
        tc_fence_after();
      }
      for (int it = 0; it < n_iter; ++it) {
        const unsigned long long t0 = (kLpDiag && p.trace) ? lp_clock() : 0ull;
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        if (kLpDiag && p.trace && lane == 0) atomicAdd(p.trace + blockIdx.x * 4 + 0, lp_clock() - t0);
        tc_fence_after();
        const uint32_t tacc = tmem_base + acc * 256;
        for (int kb = 0; kb < n_kb; ++kb) {
          const unsigned long long t1 = (kLpDiag && p.trace) ? lp_clock() : 0ull;
          mbar_wait(&full[stage], phase);
          if (kLpDiag && p.trace && lane == 0) atomicAdd(p.trace + blockIdx.x * 4 + 1, lp_clock() - t1);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sst = smem_u32(smem + RING0 + stage * STB);
            const uint32_t sa = ARES ? smem_u32(smem + kb * L2_HALF) : sst, sb = ARES ? sst : sst + L2_HALF;
#pragma unroll
            for (int kk = 0; kk < L2_BK / 16; ++kk)
              tc_mma_pair(tacc, make_desc(sa + kk * 32, 16, 1024), make_desc(sb + kk * 32, 16, 1024), IDESC,
                          (kb > 0 || kk > 0) ? 1u : 0u);
            tc_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) tc_commit_pair(&acc_full[acc]);
        __syncwarp();
        if (++acc == L2_ACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (this CTA's 128 rows)
    const int ew = warp - 2;
    const int lg = warp & 3;
    const int row_in = lg * 32 + lane;
    const int eset = ew >> 2;                 // 64 columns each; sets (0, 1) and (2, 3) form 128-column tiles
    const float sl = p.s_log2e;
    const uint32_t acc_empty_leader = leader_addr(&acc_empty[0]);
    int acc = 0;
    uint32_t acc_phase = 0;
    // ARES: this thread's row is fixed for the whole kernel, so the (max, sum) of its 128-column half of every class
    // tile the pair takes are folded here, in the pair's fixed tile order, and one partial per (row, group, half)
    // is stored at the end: 2 G partials per row instead of k / 128 scattered 8-byte stores (which cost a DRAM
    // read-modify-write per store once the partials outgrow L2, 2.3 GB per launch at the 12.5M-class shard)
    float racc_m = -INFINITY, racc_l = 0.f;   // ARES: this thread's 64-column set of every tile, folded
    for (int it = 0; it < n_iter; ++it) {
      int m0, n0;
      unit(it, m0, n0);
      const int row = m0 + 128 * (int)rank + row_in;
      const bool rv = row < p.M;
      const int tc = rv ? p.tcol[row] : -1;
      const unsigned long long t2 = (kLpDiag && p.trace) ? lp_clock() : 0ull;
      mbar_wait(&acc_full[acc], acc_phase);
      if (kLpDiag && p.trace && threadIdx.x == 64) atomicAdd(p.trace + blockIdx.x * 4 + 2, lp_clock() - t2);
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(lg * 32) << 16) + acc * 256;
      float mx = EF ? 0.f : -INFINITY, sum = 0.f;   // EF: unshifted sums (s + ln k < 80, api.cu)
#pragma unroll 1
      for (int c = eset * 2; c < eset * 2 + 2; ++c) {
        uint32_t v[32];
        tmem_ld32(tacc + c * 32, v);
        const int col0 = n0 + c * 32;
        __half2 h2[16];
        float cf[32];
        if (EF) {   // E is formed from the fp32 cosine (no cosine is stored: no fp16 rounding to match, R26)
#pragma unroll
          for (int j = 0; j < 32; ++j) cf[j] = __uint_as_float(v[j]);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {   // fp16 cosine stored; the partials use the fp32 value (R27)
            cf[2 * i] = __uint_as_float(v[2 * i]);
            cf[2 * i + 1] = __uint_as_float(v[2 * i + 1]);
            h2[i] = __floats2half2_rn(cf[2 * i], cf[2 * i + 1]);
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
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {                              // TMEM buffer consumed (the leader's barrier counts both CTAs)
        if (leader) mbar_arrive(&acc_empty[acc]);
        else mbar_arrive_cluster(acc_empty_leader + acc * 8);
      }
      if (ARES) {   // fold this thread's (max, sum) of its 64 columns; no exchange between the column sets
        const float nm = fmaxf(racc_m, mx);
        if (nm > -INFINITY) {
          racc_l = (racc_m > -INFINITY ? racc_l * ex2_ftz((racc_m - nm) * sl) : 0.f) +
                   (mx > -INFINITY ? sum * ex2_ftz((mx - nm) * sl) : 0.f);
          racc_m = nm;
        }
      }
      float2* sp = s_part + acc * 256;
      if (!ARES && (eset & 1)) sp[(eset >> 1) * 128 + row_in] = make_float2(mx, sum);
      if (!ARES) asm volatile("bar.sync 4, %0;" ::"n"(32 * L2_EPI) : "memory");
      if (!ARES && !(eset & 1)) {
        const float2 o = sp[(eset >> 1) * 128 + row_in];
        const float m = fmaxf(mx, o.x);
        float l = 0.f;
        if (m > -INFINITY)
          l = (mx > -INFINITY ? sum * ex2_ftz((mx - m) * sl) : 0.f) + (o.x > -INFINITY ? o.y * ex2_ftz((o.x - m) * sl) : 0.f);
        if (rv) {
          p.partials[(int64_t)row * p.n_ltiles + n0 / 128 + (eset >> 1)] =
              make_float2(m > -INFINITY ? m * p.scale : -INFINITY, l);
        }
      }
      if (++acc == L2_ACC) { acc = 0; acc_phase ^= 1; }
    }
    if (ARES) {   // slot 4 g + column set of this row (every group has at least one class tile)
      const int row = (pair % mt) * 256 + 128 * (int)rank + row_in;
      if (row < p.M)
        p.partials[(int64_t)row * p.n_ltiles + 4 * (pair / mt) + eset] =
            make_float2(racc_m > -INFINITY ? racc_m * p.scale : -INFINITY, racc_l);
    }
  }
  if (kLpDiag && p.trace && threadIdx.x == 64) p.trace[blockIdx.x * 4 + 3] = lp_clock() - tk0;
  tc_fence_before();
  cluster_sync();            // no CTA leaves while its pair may still read its shared memory or signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

}  // namespace

bool logits_pair_enabled(const Sizes& sz) {
  const int forced = env_int("PFC_LOGITS_PAIR", 1);
  return forced != 0 && sz.M > 256 && sz.k_pad % 256 == 0;
}

int launch_logits_pair_tc(const Sizes& sz, const __half* Xh, const __half* Ws, const int32_t* tcol,
                          const SamplerState* st, MarginParams mp, __half* cosv, float2* partials, bool eform,
                          int* nparts, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_logits_pair<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, L2_SMEM);
    cudaFuncSetAttribute(k_logits_pair<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, L2_SMEM);
    cudaFuncSetAttribute(k_logits_pair<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, L2R_SMEM);
    cudaFuncSetAttribute(k_logits_pair<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, L2R_SMEM);
    attr = true;
  }
  const CUtensorMap a = make_map(Xh, sz.M_pad, sz.d, 64, 128);   // fp16 operands (R27)
  const CUtensorMap b = make_map(Ws, sz.k_pad, sz.d, 64, 128);
  TC_MAPS_OK();
  L2Params p{};
  p.M = sz.M; p.ldm = (int)sz.M_pad; p.d = sz.d; p.st = st; p.tcol = tcol;
  p.s_log2e = mp.s * 1.4426950408889634f; p.scale = mp.s; p.cosv = cosv; p.partials = partials;
  p.n_ltiles = sz.n_ltiles;
  static unsigned long long* trace = nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  const bool tracing = kLpDiag && env_int("PFC_LP_TRACE", 0) != 0 && cs == cudaStreamCaptureStatusNone;
  if (tracing) {
    if (!trace) cudaMalloc(&trace, 4 * 1024 * sizeof(unsigned long long));
    cudaMemsetAsync(trace, 0, 4 * 1024 * sizeof(unsigned long long), s);
    p.trace = trace;
  }
  const int mt = (int)((sz.M + 255) / 256);
  const int max_pairs = num_sms() / 2;
  const bool ares_on = env_int("PFC_LOGITS_ARES", 1) != 0;
  const int64_t nt_all = sz.k_pad / 256;
  const int groups = (int)std::max<int64_t>(1, std::min<int64_t>(max_pairs / std::max(1, mt), nt_all));
  if (ares_on && sz.d <= 64 * L2R_KB && mt <= max_pairs && 4 * groups <= sz.n_ltiles) {
    const int pairs = groups * mt;
    *nparts = 4 * groups;   // per-row partials folded per group and 64-column set (ARES epilogue)
    if (eform) launch_pdl(k_logits_pair<true, true>, dim3(2 * pairs), dim3(L2_THREADS), L2R_SMEM, s, a, b, p);
    else launch_pdl(k_logits_pair<false, true>, dim3(2 * pairs), dim3(L2_THREADS), L2R_SMEM, s, a, b, p);
  } else {
    *nparts = 0;            // one partial per 128-column tile
    const int64_t units = (int64_t)mt * (sz.k_pad / 256);
    const int pairs = (int)std::max<int64_t>(1, std::min<int64_t>(units, max_pairs));
    if (eform) launch_pdl(k_logits_pair<true, false>, dim3(2 * pairs), dim3(L2_THREADS), L2_SMEM, s, a, b, p);
    else launch_pdl(k_logits_pair<false, false>, dim3(2 * pairs), dim3(L2_THREADS), L2_SMEM, s, a, b, p);
  }
  if (tracing) {   // medians over the CTAs: MMA waits for a free accumulator / for W_s stages, epilogue waits, total
    std::vector<unsigned long long> h(4 * 1024);
    cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::vector<double> v[4];
    for (int b = 0; b < 1024; ++b)
      if (h[b * 4 + 3])
        for (int q = 0; q < 4; ++q)
          if (q >= 2 || (b & 1) == 0) v[q].push_back(h[b * 4 + q] / 1e3);   // MMA waits: leader CTAs only
    for (auto& x : v) std::sort(x.begin(), x.end());
    if (!v[3].empty())
      std::fprintf(stderr, "logits_pair (us, median over %zu CTAs, leader-only for the MMA waits): acc_empty %.1f  "
                           "full %.1f  epilogue acc_full %.1f  total %.1f\n", v[3].size(), v[0][v[0].size() / 2],
                   v[1][v[1].size() / 2], v[2][v[2].size() / 2], v[3][v[3].size() / 2]);
  }
  return 1;
}

}  // namespace pfc
