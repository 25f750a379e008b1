// E-form helpers of the train step (DESIGN.md f1): the logits kernels stored E_nj = bf16(e^{s c_nj}) (class-major,
// 0 at each row's target column) instead of the cosine, so no softmax-gradient pass is needed:
//   off the target, G_nj = (s/M)(p_nj - 0) = f_n E_nj with f_n = (s/M) e^{-LSE_n}   (Eq.5 with Alg.1 L8-9)
//   dW_hat = G^T X_hat = E'^T X~ with X~_n = f_n x_hat_n, dX_hat_n = f_n sum_j E'_nj w_hat_j      (Alg.1 L10-12)
// where E' is E with the target entries replaced by G_t / f_n. The w-normalisation backprop needs
// w_hat_j . dW_hat_j = sum_n G_nj c_nj (Eq.6), formed from E by c = ln(E) / s.
#include <cuda_bf16.h>
#include <algorithm>

#include "pfc_internal.cuh"

namespace pfc {
namespace {

// E-form preparation, after the global LSE (Alg.1 L8-9 in this representation): f_n = (s/M) e^{-LSE_n};
// X~ = bf16(f_n x_hat_n) (the dW operand); the target entry E'[t_n][n] = G_t / f_n with
// G_t = (s/M)(p_t - 1) phi'(c_t) (the cancellation-free p_t - 1 of finalize), and dcorr[t_n] += G_t c_t for the
// radial dot (several rows may share a class; dcorr zeroed before).
__global__ void k_eform_prep(int M, int ldm, int d, const float* __restrict__ X32, const float* __restrict__ lse,
                             const float* __restrict__ gt, const int32_t* __restrict__ tcol,
                             const float* __restrict__ ct, MarginParams mp, float* __restrict__ f,
                             __nv_bfloat16* __restrict__ Xt, __nv_bfloat16* __restrict__ E, float* __restrict__ dcorr,
                             const float* __restrict__ mvalid) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  const int n = blockIdx.x;
  if (n >= M) return;
  const float gs = mp.s / *mvalid;   // the mean runs over the rows not ignored (finalize; = M without ignore_index)
  const float fn = gs * expf(-lse[n]);
  for (int c = threadIdx.x * 2; c < d; c += blockDim.x * 2) {
    const float2 v = *reinterpret_cast<const float2*>(X32 + (int64_t)n * d + c);
    *reinterpret_cast<__nv_bfloat162*>(Xt + (int64_t)n * d + c) = __floats2bfloat162_rn(fn * v.x, fn * v.y);
  }
  if (threadIdx.x == 0) {
    f[n] = fn;
    const int j = tcol[n];
    PFC_DCHECK(n < ldm);
    if (j >= 0) {
      const float c_t = ct[n];
      const float g_t = gs * gt[n] * margin_dphi(mp, c_t);
      E[(int64_t)j * ldm + n] = __float2bfloat16_rn(g_t / fn);
      atomicAdd(dcorr + j, g_t * c_t);
    }
  }
}

// dotw_j = sum_n G_nj c_nj over the non-target entries, (ln 2 / s) sum_n f_n E_nj lg2(E_nj), plus dcorr_j (the
// target entries' G_t c_t, from k_eform_prep; the E' entries there are negative and clamp to a zero term). One
// warp streams a class row (M_pad contiguous bf16) at a time; f is held transposed in shared memory.
constexpr int EU = 4;   // 256-entry chunks of a class row in flight per warp
__global__ void __launch_bounds__(256) k_eform_dotw(int64_t k_pad, int ldm, float kc, const __nv_bfloat16* __restrict__ E,
                                                    const float* __restrict__ f, const float* __restrict__ dcorr,
                                                    const SamplerState* st, float* __restrict__ dotw) {
  extern __shared__ float s_f[];              // pos(n) = (n % 8) * (ldm / 8) + n / 8: conflict-free per-lane reads
  const int l8 = ldm >> 3;
  for (int n = threadIdx.x; n < ldm; n += blockDim.x) s_f[(n & 7) * l8 + (n >> 3)] = f[n];
  __syncthreads();
  const int64_t k = st->k;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int nit = (ldm + 255) / 256;
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < k_pad; j += nw) {
    float acc = 0.f;
    if (j < k) {
      for (int it = 0; it < nit; it += EU) {
        uint4 q[EU];
#pragma unroll
        for (int u = 0; u < EU; ++u) {
          const int n0 = (it + u) * 256 + lane * 8;
          q[u] = (it + u < nit && n0 < ldm) ? __ldcs(reinterpret_cast<const uint4*>(E + j * ldm + n0))
                                            : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < EU; ++u) {
          const int n0 = (it + u) * 256 + lane * 8;
          if (it + u >= nit || n0 >= ldm) break;
          const uint32_t r[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float el = fmaxf(__uint_as_float(r[e] << 16), 1e-37f);
            const float eh = fmaxf(__uint_as_float(r[e] & 0xFFFF0000u), 1e-37f);
            float ll, lh;
            asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(ll) : "f"(el));
            asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lh) : "f"(eh));
            const int pl = (2 * e) * l8 + lane + 32 * (it + u), ph = (2 * e + 1) * l8 + lane + 32 * (it + u);
            acc = fmaf(el * s_f[pl], ll, fmaf(eh * s_f[ph], lh, acc));
          }
        }
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) dotw[j] = j < k ? kc * acc + dcorr[j] : 0.f;
  }
}

}  // namespace

int launch_eform_prep(const Sizes& sz, const float* X32, const float* lse, const float* gt, const int32_t* tcol,
                      const float* ct, MarginParams mp, float* f, __nv_bfloat16* Xt, __nv_bfloat16* E, float* dcorr,
                      const float* mvalid, cudaStream_t s) {
  cudaMemsetAsync(dcorr, 0, (size_t)sz.k_pad * sizeof(float), s);
  launch_pdl(k_eform_prep, dim3(sz.M), dim3(128), 0, s, sz.M, (int)sz.M_pad, sz.d, X32, lse, gt, tcol, ct, mp, f, Xt, E, dcorr, mvalid);
  return 1;
}

int launch_eform_dotw(const Sizes& sz, const __nv_bfloat16* E, const float* f, const float* dcorr,
                      const SamplerState* st, MarginParams mp, float* dotw, cudaStream_t s) {
  static int grid = 0;
  static size_t grid_smem = 0;
  const size_t smem = (size_t)sz.M_pad * sizeof(float);
  if (!grid || grid_smem != smem) {
    grid_smem = smem;
    cudaFuncSetAttribute(k_eform_dotw, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eform_dotw, 256, smem);
    grid = std::max(1, per_sm) * sms;   // persistent: the resident blocks, a whole number of waves
  }
  const int64_t need = (sz.k_pad + 7) / 8;
  k_eform_dotw<<<(unsigned)std::min<int64_t>(grid, need), 256, smem, s>>>(sz.k_pad, (int)sz.M_pad,
                                                                          0.69314718f / mp.s, E, f, dcorr, st, dotw);
  return 1;
}

}  // namespace pfc
