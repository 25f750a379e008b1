// Internal declarations of the B200 Partial FC library (not part of the C-ABI).
// Kernel numbering K1..K12 follows SURVEY.md §2.2 / DESIGN.md §Kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <nccl.h>
#include <stdint.h>
#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/pfc.h"

namespace pfc {

// Device-side bounds checks of the row / slot indices the kernels address (compute-sanitizer is closed on the GPU
// pool): compiled in with -DPFC_DEBUG_CHECKS (PFC_BUILD_TAG=checks python -m paper_2010_05222_b200.build builds
// _lib/libpfc-checks.so; PFC_LIB selects it), where a violated check is a device assert (cudaErrorAssert, loud).
#ifdef PFC_DEBUG_CHECKS
#include <cassert>
#define PFC_DCHECK(cond) assert(cond)
#else
#define PFC_DCHECK(cond) ((void)0)
#endif

// Kernel-selection knobs (PFC_* environment variables, for A/B timing): read at every call, not cached, so that a
// process (the test suite) can switch them between contexts.
inline int env_int(const char* name, int def) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : def;
}

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may be scheduled while its stream
// predecessor is still running; its first statement is pdl_wait(), which returns once the predecessor grid has
// completed and its memory is visible (transitively every earlier kernel), and pdl_trigger() lets the kernel's own
// dependents be scheduled as its CTAs retire. Both are no-ops for a normally launched kernel. PFC_PDL=0 launches
// everything without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = env_int("PFC_PDL", 1) != 0 ? 1 : 0;
  return cudaLaunchKernelEx(&lc, kern, std::forward<Args>(args)...);
}

// Sticky device error bits (reported as pfc_status by the next synchronising call).
enum : int { ERR_DATA = 1, ERR_DEGENERATE = 2, ERR_NUMERIC = 4, ERR_INTERNAL = 8 };

constexpr float kNormEps = 1e-12f;   // DESIGN.md R8
constexpr float kArcDerivEps = 1e-6f;  // DESIGN.md R10

// Device-resident state of the sampler for one step.
struct SamplerState {
  int npos;          // |P_i|
  int k;             // k_i (R1 / R23 / R24)
  int n_neg;         // n_i = k_i - |P_i|
  int none;          // n_i == 0: no negative selected
  uint32_t prefix1;  // radix select: top 11 bits of the threshold key (pass 1)
  int rem1;          //   rank of the threshold inside that bucket (1-based)
  uint32_t prefix2;  //   top 22 bits (pass 2)
  int rem2;
  uint32_t T;        // threshold key
  int t;             // number of tied (key == T) negatives to take, smallest ids first
  int total;         // number of selected rows written by the compaction (== k)
  int pad[5];
};

// Margin parameters used by the epilogues (R9-R11).
struct MarginParams {
  int type;          // pfc_margin
  float s;           // scale
  float m;           // margin
  float cos_m, sin_m, th, mm;  // ArcFace: cos m, sin m, cos(pi - m), m sin m
};

__device__ __forceinline__ float margin_phi(const MarginParams& mp, float c) {
  if (mp.type == PFC_MARGIN_COSFACE) return c - mp.m;
  if (mp.type == PFC_MARGIN_ARCFACE) {
    float cc = fminf(1.f, fmaxf(-1.f, c));
    if (cc > mp.th) {
      float sn = sqrtf(fmaxf(0.f, 1.f - cc * cc));
      return cc * mp.cos_m - sn * mp.sin_m;        // cos(theta + m)
    }
    return c - mp.mm;                               // theta + m >= pi (R9)
  }
  return c;
}

__device__ __forceinline__ float margin_dphi(const MarginParams& mp, float c) {
  if (mp.type == PFC_MARGIN_ARCFACE) {
    float cc = fminf(1.f, fmaxf(-1.f, c));
    if (cc > mp.th) {
      float sn = fmaxf(sqrtf(fmaxf(0.f, 1.f - cc * cc)), kArcDerivEps);
      return mp.cos_m + cc * mp.sin_m / sn;        // d/dc cos(acos c + m)
    }
  }
  return 1.f;
}

// Philox4x32-10 (Random123 constants), first output word: the sampler key of global class j
// (R2): ctr = {j lo, j hi, step, 0}, key = {seed lo, seed hi}.
__device__ __forceinline__ uint32_t philox_class_key(uint64_t j, uint32_t step, uint64_t seed) {
  uint32_t c0 = (uint32_t)j, c1 = (uint32_t)(j >> 32), c2 = step, c3 = 0u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return c0;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------------------------
// Launchers (host side). Each returns the number of kernels it launched.
// ---------------------------------------------------------------------------------------------
struct Sizes {
  int64_t C, C_local, a;   // classes, shard rows, shard start
  int d, B, M, M_pad;      // dim, per-rank batch, global batch, M rounded up to 128
  int rank, world;
  int64_t budget;          // ceil(r C_local)
  double rate;             // r
  int sample_mode;         // pfc_sample_mode
  int64_t k_max, k_pad;    // workspace bound and its padding to the tile width
  int ltile;               // columns per logits partial tile (64 SIMT, 128 tcgen05)
  int n_ltiles;            // number of logits column tiles (k_pad / ltile)
  int ntiles_sel;          // sampler compaction tiles
};

constexpr int kMaxLoopback = 16;
// Collectives fused into the kernels (PFC_COMM_NCCL_FUSED / PFC_COMM_LOOPBACK_FUSED): every
// rank owns one "exchange region" laid out identically on all ranks (an NCCL symmetric window, or a plain
// allocation of each loopback context), and the producing kernels store straight into the peers' regions:
//   x32  [M_pad][d] f32   all-gathered x_hat: rank r writes rows [rB, rB + B) of every peer   (Alg.1 L2)
//   y    [M] i64          all-gathered labels, likewise
//   xmax [world][M] f32   slot r = rank r's row maxima                                          (Alg.1 L6-7)
//   xred [world][3M+1]    slot r = rank r's rescaled sums / target logits / CA_pcc numerator
//   xdx  [world][B][d]    slot r = rank r's dX_hat partial of this owner's rows                  (Alg.1 L12-13)
// The consumers reduce the slots in rank order (deterministic). Peers.n == 0: plain (non-fused) kernels.
struct SymLayout {
  int64_t x32, y, xmax, xred, xdx, bytes;
};
struct Peers {
  char* base[kMaxLoopback];   // every rank's exchange region, indexed by rank (base[rank] = this rank's)
  int n, rank;
  SymLayout lay;
  __host__ __device__ float* f32(int q, int64_t off) const { return reinterpret_cast<float*>(base[q] + off); }
};
SymLayout sym_layout(const Sizes& sz);

constexpr int kSelTile = 8192;   // sampler compaction tile (256 threads x 32)
constexpr int kKPad = 256;       // k_pad granularity (multiple of every GEMM tile width)

// sampler.cu
int launch_sampler(const Sizes& sz, const int64_t* Y, uint64_t seed, const uint64_t* step_dev, uint32_t* bits,
                   uint32_t* keys, int* hist, int* tile_cnt, SamplerState* st, int32_t* idx, int32_t* tcol,
                   int* err, cudaStream_t s);

// rows.cu
// ignore != 0: label -1 marks an ignored row (f3, R28) instead of a DATA error
int launch_normalize_x(const Sizes& sz, const float* x, const int64_t* labels, float* xh_local, float* xnorm,
                       float* X32, int64_t* Y, int* err, const Peers* P, int ignore, cudaStream_t s);
// X_hat -> bf16 Xb (dW / dX operand) and, when Xh16 != NULL, fp16 Xh16 (the logits operand, R27)
int launch_x_to_bf16(const Sizes& sz, const float* X32, __nv_bfloat16* Xb, __half* Xh16, cudaStream_t s);
// K5: normalised sampled rows -> W_s (bf16, or fp32 in fp32 mode) and, when Ws16 != NULL, an fp16 copy (R27)
int launch_gather_w(const Sizes& sz, bool bf16, const float* W, const int32_t* idx, const SamplerState* st,
                    void* Ws, __half* Ws16, float* inv_norm, int* err, cudaStream_t s);
int launch_target_cos(const Sizes& sz, const float* X32, const float* W, const int64_t* Y, const int32_t* idx,
                      const SamplerState* st, const int* tile_cnt /* sampler K4 tile offsets */, int32_t* tcol,
                      float* ct, cudaStream_t s);
// nparts > 0: the logits kernel folded its per-row partials into the first nparts slots of each row (else one
// partial per 128-column tile up to k_i)
int launch_row_combine(const Sizes& sz, const float2* partials, int nparts, const int64_t* Y, const float* ct,
                       const SamplerState* st, MarginParams mp, float* rowmax, float* rowsum, float* zt, const Peers* P,
                       cudaStream_t s);
// fused (P): gmax is computed here from the peers' xmax slots (max in rank order) and written
int launch_prep_sum(const Sizes& sz, const float* rowmax, float* gmax, const float* rowsum, const float* zt,
                    const int32_t* tcol, const int64_t* Y, const float* ct, float* red, const Peers* P, cudaStream_t s);
// metrics[0] = loss, [1] = CA_pcc, [2] = M_valid (rows not ignored, >= 1): the mean's and gradients' divisor
int launch_finalize(const Sizes& sz, const float* gmax, const float* red, float* lse, float* gt, float* loss_out,
                    float* metrics, int* err, const Peers* P, const int64_t* Y, int ignore, cudaStream_t s);
int launch_softmax_grad(const Sizes& sz, bool bf16, const void* cosv, const float* lse, const float* gt,
                        const int32_t* tcol, const float* ct, const SamplerState* st, MarginParams mp, void* G,
                        float* dotw /* per-class w_hat . dW_hat, or NULL */,
                        const float* gsc /* R25: per-class 1/||w|| folded into G, or NULL */,
                        const float* mvalid /* device: rows not ignored (finalize) */, cudaStream_t s);
// fused (P): dxh is ignored, the owner's xdx slots are summed in rank order
int launch_xnorm_backward(const Sizes& sz, const float* dxh, const float* xh_local, const float* xnorm,
                          float* grad_x, const Peers* P, cudaStream_t s);
// fused fallback for the SIMT (fp32) dX: push the local dX_hat rows of every owner into its xdx slot
int launch_push_dx(const Sizes& sz, const float* dXh, const Peers& P, cudaStream_t s);
int launch_sgd(const Sizes& sz, float* W, float* V, const float* dWh, const int32_t* idx, const float* inv_norm,
               const SamplerState* st, const float* lr_dev, float mu, float lambda, int gsc, cudaStream_t s);
int launch_set_scalar(float* dst, float v, cudaStream_t s);
// f4 staging: sampled rows W[idx_p], V[idx_p] <-> Wst[p], Vst[p] (p < k_i)
int launch_stage_rows(const Sizes& sz, float* W, float* V, const int32_t* idx, const SamplerState* st, float* Wst,
                      float* Vst, bool to_host, cudaStream_t s);
int launch_iota(int32_t* out, int64_t n, int32_t base);   // out[i] = base + i (legacy stream)
int launch_advance_step(uint64_t* step_dev, const int* err_dev, int* err_host_mapped, cudaStream_t s);
int launch_raw_grad(const Sizes& sz, const float* W, const float* dWh, const int32_t* idx, const float* inv_norm,
                    const SamplerState* st, float* out, int gsc, cudaStream_t s);

// loopback collectives: dst[r][i] = op_{q ascending} src[q][src_off + i] for r < ndst (op 0 = sum, 1 = max)

struct PtrPack { float* p[kMaxLoopback]; };
int launch_group_reduce(int64_t n, const PtrPack& src, int64_t src_off, const PtrPack& dst, int nranks, int ndst,
                        int op, cudaStream_t s);
int launch_idx_to_global(int64_t k_max, const int32_t* idx, const SamplerState* st, int64_t a, int64_t* out,
                         cudaStream_t s);

// gemm_simt.cu — fp32 (and bf16-operand) FFMA contractions
int launch_logits_simt(const Sizes& sz, bool bf16, const void* X, const void* Ws, const int32_t* tcol,
                       const float* ct, const SamplerState* st, MarginParams mp, void* cosv, float2* partials,
                       cudaStream_t s);
int launch_dx_simt(const Sizes& sz, bool bf16, const void* G, const void* Ws, const SamplerState* st, float* dXh,
                   cudaStream_t s);
int launch_dw_simt(const Sizes& sz, bool bf16, const void* G, const void* X, const SamplerState* st, float* dWh,
                   cudaStream_t s);

// gemm_tc.cu — tcgen05 / TMEM / TMA bf16 contractions (sm_100a)
constexpr int kMaxSplits = 64;   // split-K bound of the dx contraction
bool tc_available();
int& tmap_error();   // tc_common.cuh: status of the last failed tensor-map encode (per host thread)
int64_t dx_split_ws_floats(const Sizes& sz);
int launch_logits_tc(const Sizes& sz, const __half* Xh, const __half* Ws16, const int32_t* tcol,
                     const float* ct, const SamplerState* st, MarginParams mp, __half* cosv, float2* partials,
                     cudaStream_t s);
// logits_gather.cu — K5 + K6 fused (M <= 256): sampled fp32 W rows -> norms, bf16 W_s (un-normalised), logits
bool logits_gather_supported(const Sizes& sz);
int launch_logits_gather_tc(const Sizes& sz, const float* W, const int32_t* idx, const __half* Xh16,
                            __nv_bfloat16* Ws, bool write_ws, float* inv_norm, const int32_t* tcol, const SamplerState* st,
                            MarginParams mp, __half* cosv, float2* partials, int* err, bool eform, int* nparts,
                            cudaStream_t s);
// logits2.cu — K6 on CTA pairs (tcgen05 cta_group::2, 256 x 256 tiles) for M > 256
bool logits_pair_enabled(const Sizes& sz);
int launch_logits_pair_tc(const Sizes& sz, const __half* Xh16, const __half* Ws16, const int32_t* tcol,
                          const SamplerState* st, MarginParams mp, __half* cosv, float2* partials, bool eform,
                          int* nparts, cudaStream_t s);
// dX_hat = G W_s (split-K + fixed-order reduction); rowscale (E-form f_n, or NULL) multiplies each output row
// P: the split-K reduction stores each owner's rows straight into its xdx slot (fused reduce-scatter)
int launch_dx_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Ws, const SamplerState* st,
                 float* dXh, float* split_ws, const float* rowscale, const Peers* P, cudaStream_t s);
int launch_dw_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                 float* dWh, cudaStream_t s);
// Fused K11 + K12: dW_hat tile in TMEM -> g = (dw_hat - w_hat dot)/||w||,
// v <- mu v + g + lambda w, w <- w - lr v, written straight into the W and V shard rows.
struct SgdArgs {
  float* W; float* V; const int32_t* idx; const float* inv_norm; const float* dotw; const float* lr; float mu, lambda;
  int gsc;   // R25: G carries 1/||w|| (dW_hat tile is already scaled)
  float* xws = nullptr;   // dwxdot.cu: the partner pairs' half-dots and flags (dw_sgd_pairx_ws_floats)
  int* err = nullptr;
  int64_t rows = INT64_MAX;   // shard rows addressable through idx (PFC_DCHECK bounds)
};
int launch_dw_sgd_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                     const SgdArgs& a, cudaStream_t s);
// dwpair.cu — K11 + K12 on CTA pairs (M >= 2048, d % 256 == 0; PFC_DW_PAIR=0 disables)
bool dw_sgd_pair_enabled(const Sizes& sz);
int launch_dw_sgd_pair_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                          const SgdArgs& sa, cudaStream_t s);
// dwfull.cu — K11 + radial dot + K12 on CTA pairs over all d columns of 256-class tiles (M > 256, d in {256, 512},
// normalised W_s operand); the radial dots come from the accumulator, sa.dotw is not read (PFC_DWFULL=0 disables)
bool dw_sgd_full_enabled(const Sizes& sz, int gsc);
int launch_dw_sgd_full_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                          const SgdArgs& sa, cudaStream_t s);
// dwxdot.cu — K11 + radial dot + K12 on CTA pairs, the dot's two column halves exchanged between partner pairs
// (M >= 2048, d = 512, normalised W_s; PFC_DW_XDOT=0 disables): no radial-dot pass over E
bool dw_sgd_pairx_enabled(const Sizes& sz, int gsc);
int64_t dw_sgd_pairx_ws_floats(const Sizes& sz);
int launch_dw_sgd_pairx_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                           const SgdArgs& sa, float* ws, int* err, cudaStream_t s);
// dwx.cu — K9 + K11 + K12 fused for the train step (M <= 256, R25 scaling): dW + SGD update + dX_hat partials
bool dwx_supported(const Sizes& sz);
int64_t dwx_ws_floats(const Sizes& sz);
// E-form (DESIGN.md f1): the logits kernel stored E = e^{s c}; no softmax-gradient pass
struct EformArgs {
  const float* f; const int32_t* tcol; const float* dcorr; float* xch; int* cnt; int* err; float s;
};
int launch_dwx_tc(const Sizes& sz, const __nv_bfloat16* G, const __nv_bfloat16* Xb, const SamplerState* st,
                  const SgdArgs& sa, float* ws, float* dXh, const EformArgs* ef, const Peers* P, cudaStream_t s);
// fused_comm.cu — NCCL device-API exchange (PFC_COMM_NCCL_FUSED): symmetric window, LSA barrier
struct FusedNccl;
pfc_status fused_nccl_create(ncclComm_t comm, const Sizes& sz, FusedNccl** out, char** local_region, Peers* P,
                             std::string* err);
void fused_nccl_destroy(ncclComm_t comm, FusedNccl* f);
int launch_lsa_barrier(const FusedNccl* f, cudaStream_t s);
// the fused dX_hat push shared by the split-K reductions: row i of the M x d result goes to owner i / B, slot rank
__device__ __forceinline__ float* dx_dst(const Peers& P, float* local, int64_t i, int d, int B) {
  if (P.n == 0) return local + i;
  const int64_t row = i / d, col = i % d;
  const int q = (int)(row / B);
  PFC_DCHECK(q < P.n && P.lay.xdx + ((int64_t)P.rank * B + (row % B) + 1) * d * 4 <= P.lay.bytes);
  return P.f32(q, P.lay.xdx) + ((int64_t)P.rank * B + (row % B)) * d + col;
}
// eform.cu — E-form preparation (f_n, X~, target entries of E) and the radial dots for the unfused-dX path
int launch_eform_prep(const Sizes& sz, const float* X32, const float* lse, const float* gt, const int32_t* tcol,
                      const float* ct, MarginParams mp, float* f, __nv_bfloat16* Xt, __nv_bfloat16* E, float* dcorr,
                      const float* mvalid /* device: rows not ignored (finalize) */, cudaStream_t s);
int launch_eform_dotw(const Sizes& sz, const __nv_bfloat16* E, const float* f, const float* dcorr,
                      const SamplerState* st, MarginParams mp, float* dotw, cudaStream_t s);

}  // namespace pfc
