// FFMA (CUDA-core) contractions for the fp32 mode (tf32 is too coarse for the
// 1e-4 bar, so the fp32 mode multiplies in fp32). 64x64 output tile, K step 16, 256 threads, 4x4 per
// thread with a 16-stride so that each row's 16 threads are 16 consecutive lanes (row reductions of the
// logits epilogue are half-warp shuffles).
//   logits (K6f): cos[n][p] = X_hat[n] . W_s[p], fused margin / scale / per-tile (max, sum-exp)
//   dx     (K9f): dX_hat = Gc W_s, split-K over the sampled classes, fp32 atomics
//   dw     (K11f): dW_hat = Gc^T X_hat
#include <algorithm>
#include "pfc_internal.cuh"

namespace pfc {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;
enum { MODE_LOGITS = 0, MODE_ATOMIC = 1, MODE_STORE = 2 };

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

struct Epi {
  // logits (cos stored class-major: cosv[p * ldm + n])
  const int32_t* tcol; const float* ct; MarginParams mp; void* cosv; float2* partials; int ntiles; int bf16; int ldm;
  // generic output
  float* C; int64_t ldc;
  int rows_valid;  // M for logits / dx; k for dw (read from st when < 0)
};

// C[m][n] = sum_k A(m,k) B(k,n); A(m,k) = AK ? A[m*lda+k] : A[k*lda+m]; B(k,n) = BK ? B[n*ldb+k] : B[k*ldb+n]
template <typename T, bool AK, bool BKM, int MODE>
__global__ void __launch_bounds__(256) k_gemm(int Mdim, int64_t Ndim, int64_t Kdim, const T* __restrict__ A, int64_t lda,
                                              const T* __restrict__ B, int64_t ldb, const SamplerState* st,
                                              int64_t k_chunk, Epi e) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int k_sampled = st->k;
  const int64_t m_base = (int64_t)blockIdx.y * BM;
  const int64_t n_base = (int64_t)blockIdx.x * BN;
  // data-dependent bounds: logits cols < k; dw rows < k; dx K-range < k
  int64_t Mlim = Mdim, Nlim = Ndim, Klo = 0, Khi = Kdim;
  if (MODE == MODE_LOGITS) { Nlim = k_sampled; Mlim = e.ldm; }   // padding rows [M, M_pad) are stored as 0
  if (MODE == MODE_STORE) Mlim = k_sampled;
  if (MODE == MODE_ATOMIC) { Klo = (int64_t)blockIdx.z * k_chunk; Khi = min(Klo + k_chunk, (int64_t)k_sampled); }
  if (m_base >= Mlim || n_base >= Nlim || Klo >= Khi) return;

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = Klo; k0 < Khi; k0 += BK) {
    // A tile -> As[k][m]
    if (AK) {
      const int mm = tid >> 2, kq = (tid & 3) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t gm = m_base + mm, gk = k0 + kq + q;
        As[kq + q][mm] = (gm < Mdim && gk < Khi) ? to_f(A[gm * lda + gk]) : 0.f;
      }
    } else {
      const int kk = tid >> 4, mq = (tid & 15) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t gm = m_base + mq + q, gk = k0 + kk;
        As[kk][mq + q] = (gm < Mdim && gk < Khi) ? to_f(A[gk * lda + gm]) : 0.f;
      }
    }
    if (BKM) {
      const int nn = tid >> 2, kq = (tid & 3) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t gn = n_base + nn, gk = k0 + kq + q;
        Bs[kq + q][nn] = (gn < Ndim && gk < Khi) ? to_f(B[gn * ldb + gk]) : 0.f;
      }
    } else {
      const int kk = tid >> 4, nq = (tid & 15) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int64_t gn = n_base + nq + q, gk = k0 + kk;
        Bs[kk][nq + q] = (gn < Ndim && gk < Khi) ? to_f(B[gk * ldb + gn]) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  if (MODE == MODE_LOGITS) {
    const MarginParams mp = e.mp;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t n = m_base + ty + 16 * i;
      const bool rv = n < Mdim;
      const int tc = rv ? e.tcol[n] : -1;
      float z[4];
      float zmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t p = n_base + tx + 16 * j;
        float c = acc[i][j];
        const bool in = n < e.ldm && p < Ndim;     // rows [M, M_pad) get 0: K8 reads every stored cosine
        if (e.bf16) {
          __half h = __float2half_rn(rv ? c : 0.f);
          c = __half2float(h);
          if (in) ((__half*)e.cosv)[p * e.ldm + n] = h;
        } else {
          if (in) ((float*)e.cosv)[p * e.ldm + n] = rv ? c : 0.f;
        }
        // the target column is excluded from the partials (finalize adds it exactly, see rows.cu)
        z[j] = (p < Nlim && p != tc) ? mp.s * c : -INFINITY;
        zmax = fmaxf(zmax, z[j]);
      }
#pragma unroll
      for (int o = 8; o; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) l += (z[j] > -INFINITY) ? __expf(z[j] - zmax) : 0.f;  // zmax finite here
#pragma unroll
      for (int o = 8; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      if (rv && tx == 0) e.partials[n * e.ntiles + blockIdx.x] = make_float2(zmax, zmax > -INFINITY ? l : 0.f);
    }
  } else if (MODE == MODE_ATOMIC) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t m = m_base + ty + 16 * i;
      if (m >= Mdim) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t n = n_base + tx + 16 * j;
        if (n < Ndim) atomicAdd(&e.C[m * e.ldc + n], acc[i][j]);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t m = m_base + ty + 16 * i;
      if (m >= Mlim) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t n = n_base + tx + 16 * j;
        if (n < Ndim) e.C[m * e.ldc + n] = acc[i][j];
      }
    }
  }
}

}  // namespace

int launch_logits_simt(const Sizes& sz, bool bf16, const void* X, const void* Ws, const int32_t* tcol, const float* ct,
                       const SamplerState* st, MarginParams mp, void* cosv, float2* partials, cudaStream_t s) {
  Epi e{};
  e.tcol = tcol; e.ct = ct; e.mp = mp; e.cosv = cosv; e.partials = partials; e.ntiles = sz.n_ltiles; e.bf16 = bf16;
  e.ldm = sz.M_pad;
  dim3 grid((unsigned)(sz.k_pad / BN), (unsigned)(sz.M_pad / BM));
  if (bf16)
    k_gemm<__nv_bfloat16, true, true, MODE_LOGITS><<<grid, 256, 0, s>>>(
        sz.M, sz.k_pad, sz.d, (const __nv_bfloat16*)X, sz.d, (const __nv_bfloat16*)Ws, sz.d, st, 0, e);
  else
    k_gemm<float, true, true, MODE_LOGITS><<<grid, 256, 0, s>>>(sz.M, sz.k_pad, sz.d, (const float*)X, sz.d,
                                                                (const float*)Ws, sz.d, st, 0, e);
  return 1;
}

int launch_dx_simt(const Sizes& sz, bool bf16, const void* G, const void* Ws, const SamplerState* st, float* dXh,
                   cudaStream_t s) {
  cudaMemsetAsync(dXh, 0, (size_t)sz.M * sz.d * sizeof(float), s);
  Epi e{};
  e.C = dXh; e.ldc = sz.d;
  // split K = k_pad into chunks so that the grid fills the 148 SMs several times
  const int tiles = (int)(((sz.M + BM - 1) / BM) * (sz.d / BN));
  int64_t nsplit = std::max<int64_t>(1, std::min<int64_t>(sz.k_pad / 256, (148 * 8 + tiles - 1) / tiles));
  int64_t chunk = ((sz.k_pad + nsplit - 1) / nsplit + BK - 1) / BK * BK;
  nsplit = (sz.k_pad + chunk - 1) / chunk;
  dim3 grid((unsigned)(sz.d / BN), (unsigned)((sz.M + BM - 1) / BM), (unsigned)nsplit);
  if (bf16)
    k_gemm<__nv_bfloat16, false, false, MODE_ATOMIC><<<grid, 256, 0, s>>>(
        sz.M, sz.d, sz.k_pad, (const __nv_bfloat16*)G, sz.M_pad, (const __nv_bfloat16*)Ws, sz.d, st, chunk, e);
  else
    k_gemm<float, false, false, MODE_ATOMIC><<<grid, 256, 0, s>>>(sz.M, sz.d, sz.k_pad, (const float*)G, sz.M_pad,
                                                                  (const float*)Ws, sz.d, st, chunk, e);
  return 2;
}

int launch_dw_simt(const Sizes& sz, bool bf16, const void* G, const void* X, const SamplerState* st, float* dWh,
                   cudaStream_t s) {
  Epi e{};
  e.C = dWh; e.ldc = sz.d;
  dim3 grid((unsigned)(sz.d / BN), (unsigned)(sz.k_pad / BM));
  if (bf16)
    k_gemm<__nv_bfloat16, true, false, MODE_STORE><<<grid, 256, 0, s>>>(
        (int)sz.k_pad, sz.d, sz.M, (const __nv_bfloat16*)G, sz.M_pad, (const __nv_bfloat16*)X, sz.d, st, 0, e);
  else
    k_gemm<float, true, false, MODE_STORE><<<grid, 256, 0, s>>>((int)sz.k_pad, sz.d, sz.M, (const float*)G, sz.M_pad,
                                                                (const float*)X, sz.d, st, 0, e);
  return 1;
}

}  // namespace pfc
