// tcgen05 / TMEM / TMA bf16 contractions of the Partial FC step (sm_100a).
//
//   K6  logits  C[M x k]  = X_hat[M x d] . W_s[k x d]^T     A K-major, B K-major   (Alg.1 L3)
//       epilogue: fp16 cosine store, margin-free scaled logits z = s c, per-(row, 128-column tile) max and
//       sum of e^{z - max} excluding the row's target column (finalize adds it exactly; rows.cu)
//   K9  dX      dX[M x d] = Gc[M x k] . W_s[k x d]          A MN-major, B MN-major (Alg.1 L12)
//       split-K over the sampled classes, fp32 partial per split, deterministic reduction kernel
//   K11 dW      dW[k x d] = Gc^T[k x M] . X_hat[M x d]      A K-major, B MN-major  (Alg.1 L10)
// cos and Gc are stored class-major ([k_pad][M_pad]): per sampled class the batch entries are contiguous.
//
// One kernel template: a persistent, warp-specialised CTA (warp 0: TMA producer, warp 1: TMEM allocator and
// single-thread MMA issuer, warps 2-5: epilogue reading the fp32 accumulator from TMEM with tcgen05.ld).
// Operands are staged by TMA (cp.async.bulk.tensor, 128-byte swizzle) into a STAGES-deep smem ring guarded by
// mbarriers; tcgen05.mma (kind::f16, bf16 x bf16 -> fp32, cta_group::1, M = 128 per instruction) accumulates
// into TMEM; tcgen05.commit releases smem stages and signals the epilogue; the accumulator is double-buffered
// in TMEM when it fits so that the epilogue of tile t overlaps the MMAs of tile t + 1.
#include <cuda.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "pfc_internal.cuh"
#include "tc_common.cuh"

namespace pfc {
namespace {

// ------------------------------------------------------------------------------------------------ kernel
// *128: d-tile 128 (d % 256 != 0); DWF: dW with the momentum-SGD update fused into the epilogue
// DWF2: the same with 256-class tiles (two M = 128 halves share each X_hat tile: half the operand re-reads)
enum Kind { LOGITS = 0, DX = 1, DW = 2, DX128 = 3, DW128 = 4, DWF = 5, DWF2 = 6 };
__host__ __device__ constexpr int base_kind(int k) {
  return k == DX128 ? DX : (k == DW128 || k == DWF || k == DWF2) ? DW : k;
}
__host__ __device__ constexpr bool is_fused(int k) { return k == DWF || k == DWF2; }

constexpr int BK = 64;          // K elements per stage (128 B of bf16: one swizzle row)

template <int KIND>
struct Cfg;
template <>
struct Cfg<LOGITS> {  // tile 256 x 128 (two M = 128 halves sharing the B tile), K = d
  static constexpr int MSUB = 2, NMMA = 1, UMMA_N = 128, STAGES = 4, ACC = 2, EPI_WARPS = 16;
  static constexpr bool A_MN = false, B_MN = false;
};
template <>
struct Cfg<DX> {      // tile 256 x 256 (M halves x d half), K = a split of the sampled classes
  static constexpr int MSUB = 2, NMMA = 1, UMMA_N = 256, STAGES = 3, ACC = 1, EPI_WARPS = 4;
  static constexpr bool A_MN = true, B_MN = true;     // A = G class-major: batch rows contiguous
};
template <>
struct Cfg<DW> {      // tile 128 classes x 256 dims, K = M (the global batch)
  static constexpr int MSUB = 1, NMMA = 1, UMMA_N = 256, STAGES = 4, ACC = 2, EPI_WARPS = 4;
  static constexpr bool A_MN = false, B_MN = true;    // A = G class-major read as G^T: K (batch) contiguous
};
template <>
struct Cfg<DX128> : Cfg<DX> { static constexpr int UMMA_N = 128, STAGES = 4; };
template <>
struct Cfg<DW128> : Cfg<DW> { static constexpr int UMMA_N = 128; };
template <>
struct Cfg<DWF> : Cfg<DW> { static constexpr int UMMA_N = 128, STAGES = 3, ACC = 2, EPI_WARPS = 8; };
template <>
struct Cfg<DWF2> : Cfg<DW> { static constexpr int MSUB = 2, UMMA_N = 128, STAGES = 3, ACC = 2, EPI_WARPS = 8; };

template <int KIND>
struct Smem {
  using C = Cfg<KIND>;
  static constexpr int A_BYTES = C::MSUB * 128 * BK * 2;            // per stage
  static constexpr int B_BYTES = C::NMMA * C::UMMA_N * BK * 2;      // per stage
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = C::MSUB * C::NMMA * C::UMMA_N * C::ACC;
  static constexpr int EPI_BYTES =
      is_fused(KIND) ? 128 * 128 * 4 + C::MSUB * 128 * 16 : KIND == LOGITS ? (C::EPI_WARPS / 4 - 1) * C::ACC * C::MSUB * 128 * 8 : 0;
  static constexpr int THREADS = 64 + 32 * C::EPI_WARPS;
  static constexpr int TOTAL = C::STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_BYTES;
  static_assert(TMEM_COLS <= 512, "TMEM overflow");
  static_assert(C::STAGES * STAGE_BYTES + 1024 + 256 + (is_fused(KIND) ? 128 * 128 * 4 + C::MSUB * 128 * 16 : 4096) <=
                    232448,
                "shared memory overflow (227 KB per CTA)");
};

struct TcParams {
  int M;                 // global batch rows
  int ldm;               // M rounded up to 128: leading dimension of the class-major cos / Gc
  int d;
  int64_t k_pad;
  const SamplerState* st;
  // logits epilogue
  const int32_t* tcol;
  float s_log2e;         // s * log2(e)
  float scale;           // s
  __half* cosv;          // M x k_pad
  float2* partials;      // M x n_ltiles
  int n_ltiles;
  // dx epilogue
  float* split_ws;       // nsplit x M x d
  int nsplit;
  int kb_per_split;
  // dw epilogue
  float* dWh;            // k_pad x d (unfused)
  SgdArgs sgd;           // fused momentum SGD (sgd.W != nullptr)
};

// Work decomposition shared by all roles (identical sequence on every warp of the CTA).
template <int KIND_>
struct Work {
  static constexpr int KIND = base_kind(KIND_);
  static constexpr int NT = Cfg<KIND_>::UMMA_N;
  int n_units, n_kb;
  int mt, nt;  // tiles along M / N (or units for DX)
  __device__ Work(const TcParams& p, int k) {
    using C = Cfg<KIND_>;
    if (KIND == LOGITS) {
      mt = (p.M + 255) / 256;
      nt = (k + 127) / 128;
      n_units = mt * nt;
      n_kb = p.d / BK;
    } else if (KIND == DX) {
      mt = (p.M + 255) / 256;
      nt = p.d / NT;
      n_units = mt * nt * p.nsplit;
      n_kb = (k + BK - 1) / BK;  // total k-blocks over the sampled classes
    } else {
      mt = (k + 128 * C::MSUB - 1) / (128 * C::MSUB);   // class tiles
      nt = p.d / NT;
      n_units = mt * nt;
      n_kb = (p.M + BK - 1) / BK;
    }
    (void)C::MSUB;
  }
  // unit -> (m0, n0, kb_begin, kb_end)
  __device__ void decode(const TcParams& p, int u, int& m0, int& n0, int& kb0, int& kb1) const {
    if (KIND == LOGITS) {
      const int nb = u / mt, mb = u % mt;  // M fastest: concurrent CTAs share the B (W_s) tile in L2
      m0 = mb * 256; n0 = nb * 128; kb0 = 0; kb1 = n_kb;
    } else if (KIND == DX) {
      const int sp = u / (mt * nt), r = u % (mt * nt);
      const int nb = r / mt, mb = r % mt;
      m0 = mb * 256; n0 = nb * NT;
      kb0 = sp * p.kb_per_split;
      kb1 = min(n_kb, kb0 + p.kb_per_split);
    } else {
      const int cb = u / nt, nb = u % nt;  // the d-tiles of a class tile adjacent: A (G) slice hits L2
      m0 = cb * 128 * Cfg<KIND_>::MSUB; n0 = nb * NT; kb0 = 0; kb1 = n_kb;
    }
  }
};

template <int KIND_>
__global__ void __launch_bounds__(Smem<KIND_>::THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  constexpr int KIND = base_kind(KIND_);
  using C = Cfg<KIND_>;
  using S = Smem<KIND_>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * S::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;
  uint64_t* acc_empty = acc_full + C::ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C::ACC);
  // fused-SGD staging (DWF only): the 128 x 128 fp32 dW_hat tile (float4-XOR-swizzled rows) + per-row
  // (row id, 1/||w||, radial factor)
  float4* s_tile = reinterpret_cast<float4*>(smem + C::STAGES * S::STAGE_BYTES + 256);
  int32_t* s_rowj = reinterpret_cast<int32_t*>(s_tile + 128 * 32);
  float* s_inv = reinterpret_cast<float*>(s_rowj + 128 * C::MSUB);
  float* s_rad = s_inv + 128 * C::MSUB;
  // logits: per-row (max cos, sum) of the second warp set, per accumulator buffer and M-half
  float2* s_part = reinterpret_cast<float2*>(smem + C::STAGES * S::STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = p.st->k;
  const Work<KIND_> w(p, k);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < C::ACC; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], C::EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(S::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer (lane 0 issues)
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < w.n_units; u += gridDim.x) {
        int m0, n0, kb0, kb1;
        w.decode(p, u, m0, n0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (lane == 0) {
          mbar_expect_tx(&full[stage], S::STAGE_BYTES);
          uint8_t* sa = smem + stage * S::STAGE_BYTES;
          uint8_t* sb = sa + S::A_BYTES;
          if (KIND == LOGITS) {
            tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
            tma_load_2d(sa + 128 * BK * 2, &tmA, &full[stage], kb * BK, m0 + 128);
            tma_load_2d(sb, &tmB, &full[stage], kb * BK, n0);
          } else if (KIND == DX) {
#pragma unroll
            for (int c = 0; c < 4; ++c) tma_load_2d(sa + c * BK * 128, &tmA, &full[stage], m0 + c * 64, kb * BK);
#pragma unroll
            for (int c = 0; c < C::UMMA_N / 64; ++c)
              tma_load_2d(sb + c * BK * 128, &tmB, &full[stage], n0 + c * 64, kb * BK);
          } else {
#pragma unroll
            for (int ms = 0; ms < C::MSUB; ++ms)
              tma_load_2d(sa + ms * 128 * BK * 2, &tmA, &full[stage], kb * BK, m0 + ms * 128);
#pragma unroll
            for (int c = 0; c < C::UMMA_N / 64; ++c)
              tma_load_2d(sb + c * BK * 128, &tmB, &full[stage], n0 + c * 64, kb * BK);
          }
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (one thread)
    constexpr uint32_t IDESC = make_idesc(128, C::UMMA_N, C::A_MN, C::B_MN, KIND == LOGITS);   // logits: fp16 (R27)
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int u = blockIdx.x; u < w.n_units; u += gridDim.x) {
      int m0, n0, kb0, kb1;
      w.decode(p, u, m0, n0, kb0, kb1);
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tacc = tmem_base + acc * (C::MSUB * C::NMMA * C::UMMA_N);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * S::STAGE_BYTES);
          const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
#pragma unroll
            for (int ms = 0; ms < C::MSUB; ++ms) {
              uint64_t ad, bd;
              if (C::A_MN) ad = make_desc(sa + ms * 128 * BK * 2 + kk * 16 * 128, BK * 128, 1024);
              else ad = make_desc(sa + ms * 128 * BK * 2 + kk * 32, 16, 1024);
              if (C::B_MN) bd = make_desc(sb + kk * 16 * 128, BK * 128, 1024);
              else bd = make_desc(sb + kk * 32, 16, 1024);
              tc_mma(tacc + ms * C::UMMA_N, ad, bd, IDESC, (kb > kb0 || kk > 0) ? 1u : 0u);
            }
          }
          tc_commit(&empty[stage]);     // frees the smem stage once these MMAs have read it
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tc_commit(&acc_full[acc]);   // accumulator complete
      __syncwarp();
      if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2 .. 2 + EPI_WARPS)
    const int lg = warp & 3;                 // TMEM lane group this warp may access
    const int row_in = lg * 32 + lane;       // accumulator row (TMEM lane) of this thread
    const int eset = (warp - 2) >> 2;        // with 8 epilogue warps: two sets splitting the 32-column chunks
    constexpr int NSET = C::EPI_WARPS / 4;
    int32_t nx_j[C::MSUB];                   // fused SGD: per-row scalars of the next tile (prefetched)
    float nx_inv[C::MSUB], nx_rad[C::MSUB];
#pragma unroll
    for (int h = 0; h < C::MSUB; ++h) { nx_j[h] = -1; nx_inv[h] = 0.f; nx_rad[h] = 0.f; }
    if (is_fused(KIND_) && eset == 0 && (int)blockIdx.x < w.n_units) {
      int m1, n1, k0_, k1_;
      w.decode(p, blockIdx.x, m1, n1, k0_, k1_);
#pragma unroll
      for (int h = 0; h < C::MSUB; ++h) {
        const int prow = m1 + h * 128 + row_in;
        if (prow < k) { nx_j[h] = p.sgd.idx[prow]; nx_inv[h] = p.sgd.inv_norm[prow]; nx_rad[h] = p.sgd.dotw[prow]; }
      }
    }
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < w.n_units; u += gridDim.x) {
      int m0, n0, kb0, kb1;
      w.decode(p, u, m0, n0, kb0, kb1);
      const uint32_t tacc = tmem_base + ((uint32_t)(lg * 32) << 16) + acc * (C::MSUB * C::NMMA * C::UMMA_N);
      if constexpr (!is_fused(KIND_)) {
        mbar_wait(&acc_full[acc], acc_phase);
        tc_fence_after();
      }
      if constexpr (is_fused(KIND_)) {
        // Fused lazy momentum SGD of 128*MSUB sampled classes x 128 dims (rows.cu K12 is the unfused
        // form), one 128-class half at a time: (1) two warp sets copy two 32-column chunks each of the accumulator
        // half TMEM -> XOR-swizzled smem (TMEM released after the last half); (2) each of the 8 warps updates 16
        // rows, one 512-byte coalesced W and V segment per row and instruction, 16 loads per lane in flight. The
        // per-row scalars of tile u + gridDim are prefetched into registers during tile u.
        asm volatile("bar.sync 3, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");  // previous tile consumed
        int nx_n0 = 0;                                           // d-offset of the next tile (W/V L2 prefetch)
        if (eset == 0) {
#pragma unroll
          for (int h = 0; h < C::MSUB; ++h) {
            s_rowj[h * 128 + row_in] = nx_j[h];
            s_inv[h * 128 + row_in] = nx_inv[h];
            s_rad[h * 128 + row_in] = nx_rad[h];
          }
          // per-row scalars of the next tile: issued now, consumed a whole tile later
          const int un = u + gridDim.x;
#pragma unroll
          for (int hh = 0; hh < C::MSUB; ++hh) { nx_j[hh] = -1; nx_inv[hh] = 0.f; nx_rad[hh] = 0.f; }
          if (un < w.n_units) {
            int m1, k0_, k1_;
            w.decode(p, un, m1, nx_n0, k0_, k1_);
#pragma unroll
            for (int hh = 0; hh < C::MSUB; ++hh) {
              const int prow = m1 + hh * 128 + row_in;
              if (prow < k) {
                nx_j[hh] = p.sgd.idx[prow];
                nx_inv[hh] = p.sgd.inv_norm[prow];
                nx_rad[hh] = p.sgd.dotw[prow];
              }
            }
          }
        }
        mbar_wait(&acc_full[acc], acc_phase);
        tc_fence_after();
        const int ew = warp - 2;                                 // rows ew*16 .. ew*16+15 of each half
        const int col = n0 + lane * 4;
        const float lr = *p.sgd.lr;                              // device scalar (CUDA-graph replayable)
#pragma unroll 1
        for (int h = 0; h < C::MSUB; ++h) {
          if (h > 0) asm volatile("bar.sync 3, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");  // staging free
#pragma unroll 1
          for (int c = eset * 2; c < eset * 2 + 2; ++c) {
            uint32_t v[32];
            tmem_ld32(tacc + h * C::UMMA_N + c * 32, v);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              s_tile[row_in * 32 + ((c * 8 + q) ^ (row_in & 31))] =
                  make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                              __uint_as_float(v[4 * q + 3]));
          }
          if (h == C::MSUB - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);         // TMEM free: next tile's MMAs may start
            if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
          }
          asm volatile("bar.sync 3, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
#pragma unroll 1
          for (int r0 = 0; r0 < 16; r0 += 8) {
            float4 wv[8], mv[8];
            int32_t jr[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              jr[r] = s_rowj[h * 128 + ew * 16 + r0 + r];
              if (jr[r] >= 0) {
                wv[r] = *reinterpret_cast<const float4*>(p.sgd.W + (int64_t)jr[r] * p.d + col);
                mv[r] = *reinterpret_cast<const float4*>(p.sgd.V + (int64_t)jr[r] * p.d + col);
              }
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const int rr = ew * 16 + r0 + r;                   // row within the half
              if (jr[r] >= 0) {
                const float inv = s_inv[h * 128 + rr], rad = s_rad[h * 128 + rr] * inv;  // w*rad = w_hat (w_hat.dw_hat)
                const float4 g4 = s_tile[rr * 32 + (lane ^ (rr & 31))];
                float4 w = wv[r], m = mv[r];
                const float oi = p.sgd.gsc ? 1.f : inv;          // R25: G' already carries 1/||w||
                m.x = p.sgd.mu * m.x + (g4.x - w.x * rad) * oi + p.sgd.lambda * w.x;
                m.y = p.sgd.mu * m.y + (g4.y - w.y * rad) * oi + p.sgd.lambda * w.y;
                m.z = p.sgd.mu * m.z + (g4.z - w.z * rad) * oi + p.sgd.lambda * w.z;
                m.w = p.sgd.mu * m.w + (g4.w - w.w * rad) * oi + p.sgd.lambda * w.w;
                w.x -= lr * m.x; w.y -= lr * m.y; w.z -= lr * m.z; w.w -= lr * m.w;
                *reinterpret_cast<float4*>(p.sgd.V + (int64_t)jr[r] * p.d + col) = m;
                *reinterpret_cast<float4*>(p.sgd.W + (int64_t)jr[r] * p.d + col) = w;
              }
            }
            if (r0 == 0 && h == C::MSUB - 1 && eset == 0) {
              // the next tile's W / V row segments into L2 while this tile's second batch is in flight
#pragma unroll
              for (int hh = 0; hh < C::MSUB; ++hh) {
                if (nx_j[hh] >= 0) {
                  const float* wp = p.sgd.W + (int64_t)nx_j[hh] * p.d + nx_n0;
                  const float* vp = p.sgd.V + (int64_t)nx_j[hh] * p.d + nx_n0;
#pragma unroll
                  for (int l = 0; l < C::UMMA_N / 32; ++l) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(wp + 32 * l));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(vp + 32 * l));
                  }
                }
              }
            }
          }
        }
        continue;
      }
      if constexpr (KIND_ == LOGITS) {
        // Two warp sets split the 128 columns (64 each). Per row and set: fp16-round the cosines (the rounded
        // value is what K7/K8 see), store them class-major, and accumulate max c and sum 2^{(c - max) s log2 e}
        // over the columns that are sampled (< k_i) and not the row's target (R22); set 1 hands its pair to
        // set 0 through shared memory, set 0 writes the (row, tile) partial in natural units (max z = s max c).
        const float sl = p.s_log2e;
        float pm[C::MSUB], ps[C::MSUB];
#pragma unroll
        for (int ms = 0; ms < C::MSUB; ++ms) {
          const int row = m0 + ms * 128 + row_in;
          const bool rv = row < p.M;
          const int tc = rv ? p.tcol[row] : -1;
          float mx = -INFINITY, sum = 0.f;
#pragma unroll 1
          for (int c = eset * (4 / NSET); c < (eset + 1) * (4 / NSET); ++c) {
            uint32_t v[32];
            tmem_ld32(tacc + ms * C::UMMA_N + c * 32, v);
            const int col0 = n0 + c * 32;
            __half2 h2[16];
            float cf[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {   // fp16 cosine stored; the partials use the fp32 value (R27)
              cf[2 * i] = __uint_as_float(v[2 * i]);
              cf[2 * i + 1] = __uint_as_float(v[2 * i + 1]);
              h2[i] = __floats2half2_rn(cf[2 * i], cf[2 * i + 1]);
            }
            if (col0 + 32 > k || (unsigned)(tc - col0) < 32u) {     // rare: mask columns >= k_i and the target
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (col0 + j >= k || col0 + j == tc) cf[j] = -INFINITY;
            }
            // four independent accumulators: short dependency chains (the epilogue is latency-bound)
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
            // class-major store: lane pairs swap halves so that every 32-bit store covers rows (n, n+1) of one
            // class; a warp instruction writes two 64-byte runs
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
        if (lane == 0) mbar_arrive(&acc_empty[acc]);             // accumulator consumed
        // sets 1 .. NSET-1 hand their (max, sum) pairs to set 0 (slot per set, accumulator buffer and row)
        float2* sp = s_part + acc * (C::MSUB * 128);
        constexpr int SET_STRIDE = C::ACC * C::MSUB * 128;
        if (eset > 0) {
#pragma unroll
          for (int ms = 0; ms < C::MSUB; ++ms) sp[(eset - 1) * SET_STRIDE + ms * 128 + row_in] = make_float2(pm[ms], ps[ms]);
        }
        asm volatile("bar.sync 4, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
        if (eset == 0) {
#pragma unroll
          for (int ms = 0; ms < C::MSUB; ++ms) {
            const int row = m0 + ms * 128 + row_in;
            float m = pm[ms];
            float2 o[NSET - 1];
#pragma unroll
            for (int e = 0; e < NSET - 1; ++e) {
              o[e] = sp[e * SET_STRIDE + ms * 128 + row_in];
              m = fmaxf(m, o[e].x);
            }
            float l = 0.f;
            if (m > -INFINITY) {
              l = pm[ms] > -INFINITY ? ps[ms] * ex2_ftz((pm[ms] - m) * sl) : 0.f;
#pragma unroll
              for (int e = 0; e < NSET - 1; ++e) l += o[e].x > -INFINITY ? o[e].y * ex2_ftz((o[e].x - m) * sl) : 0.f;
            }
            if (row < p.M)
              p.partials[(int64_t)row * p.n_ltiles + n0 / 128] = make_float2(m > -INFINITY ? m * p.scale : -INFINITY, l);
          }
        }
        if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
        continue;
      }
#pragma unroll 1
      for (int ms = 0; ms < C::MSUB; ++ms) {
        const int row = m0 + ms * 128 + row_in;
        if (false) {
        } else if (KIND == DX) {
          const int sp = u / (w.mt * w.nt);
          const bool rv = row < p.M;
          const bool none = kb1 <= kb0;  // split past k_i: the accumulator was not written
          float* dst = p.split_ws + ((int64_t)sp * p.M + row) * p.d + n0;
#pragma unroll 1
          for (int c = 0; c < C::UMMA_N / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(tacc + ms * C::UMMA_N + c * 32, v);
            if (none) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = 0u;
            }
            if (rv) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                reinterpret_cast<uint4*>(dst + c * 32)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
          }
        } else if (p.sgd.W == nullptr) {
          const bool rv = row < k;
          float* dst = p.dWh + (int64_t)row * p.d + n0;
#pragma unroll 1
          for (int c = eset; c < C::UMMA_N / 32; c += NSET) {
            uint32_t v[32];
            tmem_ld32(tacc + c * 32, v);
            if (rv) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                reinterpret_cast<uint4*>(dst + c * 32)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(S::TMEM_COLS));
  }
}

// Deterministic split-K reduction: dX[r][c] = sum_s ws[s][r][c] (fixed split order).
// P.n > 0 (fused reduce-scatter): each row goes straight into its owner's xdx slot `rank`
__global__ void k_splitk_reduce(int64_t n, int nsplit, int64_t stride, int d, const float* __restrict__ ws,
                                const float* __restrict__ rowscale, float* __restrict__ out, Peers P, int B) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i >= n) return;
  float4 acc = *reinterpret_cast<const float4*>(ws + i);
  for (int s = 1; s < nsplit; ++s) {
    float4 v = *reinterpret_cast<const float4*>(ws + s * stride + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (rowscale) {   // E-form: dX_hat_n = f_n sum_j E'_nj w_hat_j
    const float r = rowscale[i / d];
    acc.x *= r; acc.y *= r; acc.z *= r; acc.w *= r;
  }
  *reinterpret_cast<float4*>(dx_dst(P, out, i, d, B)) = acc;
}

template <int KIND>
void launch(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p, int grid, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tc_gemm<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<KIND>::TOTAL);
    attr = true;
  }
  launch_pdl(k_tc_gemm<KIND>, dim3(grid), dim3(Smem<KIND>::THREADS), Smem<KIND>::TOTAL, s, a, b, p);
}

}  // namespace

int& tmap_error() {
  static thread_local int e = 0;
  return e;
}

bool tc_available() {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0 && encode_fn() != nullptr;
}

int launch_logits_tc(const Sizes& sz, const __half* Xh, const __half* Ws, const int32_t* tcol,
                     const float* ct, const SamplerState* st, MarginParams mp, __half* cosv, float2* partials,
                     cudaStream_t s) {
  (void)ct;
  CUtensorMap a = make_map(Xh, sz.M_pad, sz.d, 64, 128);   // fp16 operands (R27)
  CUtensorMap b = make_map(Ws, sz.k_pad, sz.d, 64, 128);
  TC_MAPS_OK();
  TcParams p{};
  p.M = sz.M; p.ldm = sz.M_pad; p.d = sz.d; p.k_pad = sz.k_pad; p.st = st; p.tcol = tcol;
  p.s_log2e = mp.s * 1.4426950408889634f; p.scale = mp.s; p.cosv = cosv; p.partials = partials; p.n_ltiles = sz.n_ltiles;
  const int64_t units = ((sz.M + 255) / 256) * ((sz.k_pad + 127) / 128);
  launch<LOGITS>(a, b, p, (int)std::min<int64_t>(units, num_sms()), s);
  return 1;
}

static int dtile(const Sizes& sz) { return sz.d % 256 == 0 ? 256 : 128; }

static void dx_split(const Sizes& sz, int& nsplit, int& kb_per_split) {
  const int tiles = ((sz.M + 255) / 256) * (sz.d / dtile(sz));
  const int64_t n_kb = sz.k_pad / 64;
  nsplit = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)num_sms() / tiles, n_kb, (int64_t)kMaxSplits}));
  kb_per_split = (int)((n_kb + nsplit - 1) / nsplit);
  nsplit = (int)((n_kb + kb_per_split - 1) / kb_per_split);
}

int64_t dx_split_ws_floats(const Sizes& sz) {
  int ns, kbs;
  dx_split(sz, ns, kbs);
  return (int64_t)ns * sz.M * sz.d;
}

int launch_dx_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Ws, const SamplerState* st, float* dXh,
                 float* split_ws, const float* rowscale, const Peers* P, cudaStream_t s) {
  CUtensorMap a = make_map(G, sz.k_pad, sz.M_pad, 64, 64);      // Gc class-major, MN-major A
  CUtensorMap b = make_map(Ws, sz.k_pad, sz.d, 64, 64);
  TC_MAPS_OK();
  TcParams p{};
  p.M = sz.M; p.ldm = sz.M_pad; p.d = sz.d; p.k_pad = sz.k_pad; p.st = st; p.split_ws = split_ws;
  const int tiles = ((sz.M + 255) / 256) * (sz.d / dtile(sz));
  int nsplit;
  dx_split(sz, nsplit, p.kb_per_split);
  p.nsplit = nsplit;
  if (dtile(sz) == 256) launch<DX>(a, b, p, std::min(tiles * nsplit, num_sms()), s);
  else launch<DX128>(a, b, p, std::min(tiles * nsplit, num_sms()), s);
  const int64_t n = (int64_t)sz.M * sz.d;
  Peers q{};
  if (P) q = *P;
  launch_pdl(k_splitk_reduce, dim3((unsigned)((n / 4 + 255) / 256)), dim3(256), 0, s, n, nsplit, n, sz.d, split_ws, rowscale, dXh, q,
                                                                  sz.B);
  return 2;
}

int launch_dw_sgd_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                     const SgdArgs& sa, cudaStream_t s) {
  if (dw_sgd_full_enabled(sz, sa.gsc)) return launch_dw_sgd_full_tc(sz, G, Xb, st, sa, s);   // dwfull.cu
  if (sa.xws && dw_sgd_pairx_enabled(sz, sa.gsc))                                              // dwxdot.cu
    return launch_dw_sgd_pairx_tc(sz, G, Xb, st, sa, sa.xws, sa.err, s);
  if (dw_sgd_pair_enabled(sz)) return launch_dw_sgd_pair_tc(sz, G, Xb, st, sa, s);   // dwpair.cu (CTA pairs)
  CUtensorMap a = make_map(G, sz.k_pad, sz.M_pad, 64, 128);     // Gc class-major, K-major A (= Gc^T)
  CUtensorMap b = make_map(Xb, sz.M_pad, sz.d, 64, 64);
  TC_MAPS_OK();
  TcParams p{};
  p.M = sz.M; p.ldm = sz.M_pad; p.d = sz.d; p.k_pad = sz.k_pad; p.st = st; p.sgd = sa;
  // 256-class tiles pay off when the contraction is long (K = M >= 1024: operand-bandwidth bound); at small M
  // the update is HBM-bound and holding TMEM across the two halves only serialises it (PFC_DWF=1|2 overrides)
  const int forced = env_int("PFC_DWF", 0);
  const int variant = forced ? forced : (sz.M >= 1024 ? 2 : 1);
  if (variant == 1) {
    const int64_t units = (sz.k_pad / 128) * (sz.d / 128);
    launch<DWF>(a, b, p, (int)std::min<int64_t>(units, num_sms()), s);
  } else {
    const int64_t units = ((sz.k_pad + 255) / 256) * (sz.d / 128);
    launch<DWF2>(a, b, p, (int)std::min<int64_t>(units, num_sms()), s);
  }
  return 1;
}

int launch_dw_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st, float* dWh,
                 cudaStream_t s) {
  CUtensorMap a = make_map(G, sz.k_pad, sz.M_pad, 64, 128);
  CUtensorMap b = make_map(Xb, sz.M_pad, sz.d, 64, 64);
  TC_MAPS_OK();
  TcParams p{};
  p.M = sz.M; p.ldm = sz.M_pad; p.d = sz.d; p.k_pad = sz.k_pad; p.st = st; p.dWh = dWh;
  const int64_t units = (sz.k_pad / 128) * (sz.d / dtile(sz));
  if (dtile(sz) == 256) launch<DW>(a, b, p, (int)std::min<int64_t>(units, num_sms()), s);
  else launch<DW128>(a, b, p, (int)std::min<int64_t>(units, num_sms()), s);
  return 1;
}

}  // namespace pfc
