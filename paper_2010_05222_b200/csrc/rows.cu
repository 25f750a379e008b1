// Row-wise and streaming kernels of the Partial FC step (everything that is not a contraction).
//   K1  normalize_x      x_hat = x / max(||x||, eps) (Eq.6) into the all-gather slot
//   K5  gather_w         W_s[p] = W[idx_p] / ||W[idx_p]|| (bf16 or fp32), inv_norm[p]
//   K5b target_cos       c_t[n] = x_hat_n . w_hat_{y_n} in fp32
//   K7  row_combine      per-row (max, sum-exp) over the logits tiles (Alg.1 L5 den_i)
//       prep_sum/finalize global LSE after the all-reduces (Alg.1 L6-7), loss (Eq.5)
//   K8  softmax_grad     Gc = (s/M)(p - onehot) phi'(c_t) (Alg.1 L8-9)
//   K10 xnorm_backward   dx = (dx_hat - x_hat (x_hat . dx_hat)) / ||x||
//   K12 sgd              lazy momentum SGD of the sampled rows
#include <algorithm>
#include <climits>
#include "pfc_internal.cuh"

namespace pfc {
namespace {

// ---------------------------------------------------------------- K1
// Fused (P.n > 0): the all-gather of Alg.1 L2 is these stores — row rB + n of x_hat and its
// label go straight into every rank's exchange region (NVLink peer stores in PFC_COMM_NCCL_FUSED).
__global__ void k_normalize_x(int B, int d, int rank, int64_t C, const float* __restrict__ x,
                              const int64_t* __restrict__ labels, float* __restrict__ xh_local,
                              float* __restrict__ xnorm, float* __restrict__ X32, int64_t* __restrict__ Y, int* err,
                              Peers P, int ignore) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B) return;
  const float* xr = x + (int64_t)warp * d;
  float ss = 0.f;
  for (int c = lane; c < d; c += 32) { float v = xr[c]; ss += v * v; }
  ss = warp_sum(ss);
  const float nrm = sqrtf(ss);
  const float inv = 1.f / fmaxf(nrm, kNormEps);
  float* out_l = xh_local + (int64_t)warp * d;
  float* out_g = X32 + ((int64_t)rank * B + warp) * d;
  const int64_t grow = (int64_t)rank * B + warp;
  for (int c = lane; c < d; c += 32) {
    float v = xr[c] * inv;
    out_l[c] = v;
    if (P.n == 0) out_g[c] = v;
    for (int q = 0; q < P.n; ++q) P.f32(q, P.lay.x32)[grow * d + c] = v;
  }
  if (lane == 0) {
    xnorm[warp] = nrm;
    int64_t y = labels[warp];
    if (P.n == 0) Y[grow] = y;
    for (int q = 0; q < P.n; ++q) reinterpret_cast<int64_t*>(P.base[q] + P.lay.y)[grow] = y;
    if ((y < 0 || y >= C) && !(ignore && y == -1)) atomicOr(err, ERR_DATA);
    if (!(nrm > 0.f)) atomicOr(err, ERR_DEGENERATE);
  }
}

// X_hat operands: bf16 for the dW / dX contractions, fp16 for the logits contraction (R27: the normalised features
// sit in [-1, 1], where fp16's 11-bit significand is 8x finer than bf16's)
__global__ void k_x_to_bf16(int64_t n, const float* __restrict__ X32, __nv_bfloat16* __restrict__ Xb,
                            __half* __restrict__ Xh16) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const float v = X32[i];
    Xb[i] = __float2bfloat16_rn(v);
    if (Xh16) Xh16[i] = __float2half_rn(v);
  }
}

// ---------------------------------------------------------------- K5: one warp per sampled row
template <bool BF16>
__global__ void k_gather_w(int64_t k_pad, int d, const float* __restrict__ W, const int32_t* __restrict__ idx,
                           const SamplerState* st, void* __restrict__ Ws, __half* __restrict__ Ws16,
                           float* __restrict__ inv_norm, int* err) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= k_pad) return;
  const int k = st->k;
  if (p >= k) {  // padding rows: zero so that the K = k contraction sees exact zeros
    for (int c = lane * 4; c < d; c += 128) {
      if (BF16) {
        __nv_bfloat162 z = __floats2bfloat162_rn(0.f, 0.f);
        __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>((__nv_bfloat16*)Ws + p * d + c);
        o[0] = z; o[1] = z;
        if (Ws16) *reinterpret_cast<uint2*>(Ws16 + p * d + c) = make_uint2(0u, 0u);
      } else {
        *reinterpret_cast<float4*>((float*)Ws + p * d + c) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (lane == 0) inv_norm[p] = 0.f;
    return;
  }
  const float* wr = W + (int64_t)idx[p] * d;
  float4 v[4];
  const int nv = d / 128;  // d % 128 == 0 checked at init for the vector path
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nv) {
      v[i] = __ldg(reinterpret_cast<const float4*>(wr + i * 128 + lane * 4));
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
  }
  for (int c = 512 + lane * 4; c < d; c += 128) {  // d > 512
    float4 u = __ldg(reinterpret_cast<const float4*>(wr + c));
    ss += u.x * u.x + u.y * u.y + u.z * u.z + u.w * u.w;
  }
  ss = warp_sum(ss);
  const float nrm = sqrtf(ss);
  const float inv = 1.f / fmaxf(nrm, kNormEps);
  if (lane == 0) {
    inv_norm[p] = inv;
    if (!(nrm > 0.f)) atomicOr(err, ERR_DEGENERATE);
  }
  auto store = [&](int c, float4 u) {
    if (BF16) {
      __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>((__nv_bfloat16*)Ws + p * d + c);
      o[0] = __floats2bfloat162_rn(u.x * inv, u.y * inv);
      o[1] = __floats2bfloat162_rn(u.z * inv, u.w * inv);
      if (Ws16) {   // the fp16 copy: B operand of the logits contraction (R27)
        __half2* h = reinterpret_cast<__half2*>(Ws16 + p * d + c);
        h[0] = __floats2half2_rn(u.x * inv, u.y * inv);
        h[1] = __floats2half2_rn(u.z * inv, u.w * inv);
      }
    } else {
      *reinterpret_cast<float4*>((float*)Ws + p * d + c) = make_float4(u.x * inv, u.y * inv, u.z * inv, u.w * inv);
    }
  };
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < nv) store(i * 128 + lane * 4, v[i]);
  for (int c = 512 + lane * 4; c < d; c += 128) store(c, __ldg(reinterpret_cast<const float4*>(wr + c)));
}

// ---------------------------------------------------------------- K5b: one warp per batch row
// c_t[n] = x_hat_n . W[y_n] / ||W[y_n]|| in fp32 for every row whose class is on this shard (sampled or not:
// fully random sampling may leave the positive out, R24); 0 elsewhere. Used for the target logit, CA_pcc (Eq.7)
// and the ArcFace derivative.
// Also tcol[n] = position of y_n in the sampled set idx (binary search; -1 when not sampled on this rank).
__global__ void k_target_cos(int M, int d, int64_t a, int64_t C_local, const float* __restrict__ X32,
                             const float* __restrict__ W, const int64_t* __restrict__ Y,
                             const int32_t* __restrict__ idx, const SamplerState* st,
                             const int* __restrict__ sel_off, int ntiles, int32_t* __restrict__ tcol,
                             float* __restrict__ ct) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (n >= M) return;
  const int64_t j = Y[n] - a;
  if (j < 0 || j >= C_local) {
    if (lane == 0) { ct[n] = 0.f; tcol[n] = -1; }
    return;
  }
  const float* xr = X32 + (int64_t)n * d;
  const float* wr = W + j * d;
  // the row's loads first (in flight during the search)
  float acc = 0.f, ss = 0.f;
  if ((d & 127) == 0 && d <= 512) {
    float4 xv[4], wv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q * 128 < d) {
        xv[q] = __ldg(reinterpret_cast<const float4*>(xr + q * 128 + lane * 4));
        wv[q] = __ldg(reinterpret_cast<const float4*>(wr + q * 128 + lane * 4));
      }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q * 128 < d) {
        acc += xv[q].x * wv[q].x + xv[q].y * wv[q].y + xv[q].z * wv[q].z + xv[q].w * wv[q].w;
        ss += wv[q].x * wv[q].x + wv[q].y * wv[q].y + wv[q].z * wv[q].z + wv[q].w * wv[q].w;
      }
  } else {
    for (int c = lane; c < d; c += 32) { const float w = wr[c]; acc += xr[c] * w; ss += w * w; }
  }
  // tcol: search only the positions of j's compaction tile, [sel_off[t], sel_off[t + 1]) (K4b exclusive scan),
  // 32-ary with the warp (ascending ids: the lanes whose probe is <= j form a prefix)
  {
    const int t = (int)(j / kSelTile);
    int lo = sel_off[t], hi = (t + 1 < ntiles ? sel_off[t + 1] : st->k) - 1, res = -1;
    while (hi - lo + 1 > 32) {
      const int step = (hi - lo + 1 + 31) / 32;
      const int pos = lo + lane * step;
      const int v = pos <= hi ? __ldg(idx + pos) : INT_MAX;
      const unsigned le = __ballot_sync(0xffffffffu, v <= (int)j);
      if (!le) { hi = lo - 1; break; }                 // j below the segment: not sampled
      const int nlo = lo + (31 - __clz(le)) * step;
      hi = min(hi, nlo + step - 1);
      lo = nlo;
    }
    if (lo <= hi) {
      const int pos = lo + lane;
      const unsigned eq = __ballot_sync(0xffffffffu, pos <= hi && __ldg(idx + pos) == (int)j);
      if (eq) res = lo + __ffs(eq) - 1;
    }
    if (lane == 0) tcol[n] = res;
  }
  acc = warp_sum(acc);
  ss = warp_sum(ss);
  if (lane == 0) ct[n] = acc / fmaxf(sqrtf(ss), kNormEps);
}

// ---------------------------------------------------------------- K7: one 256-thread block per batch row
// (the row's ~k/128 tile partials are spread over the block; two-level max then rescaled sum)
__global__ void __launch_bounds__(256) k_row_combine(int M, int ntiles, int ltile, int nparts, int64_t a,
                                                     int64_t C_local, const float2* __restrict__ partials,
                                                     const int64_t* __restrict__ Y, const float* __restrict__ ct,
                                                     const SamplerState* st, MarginParams mp,
                                                     float* __restrict__ rowmax, float* __restrict__ rowsum,
                                                     float* __restrict__ zt, Peers P) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  __shared__ float sm[8], ss[8];
  const int n = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float2* pr = partials + (int64_t)n * ntiles;
  // tiles past k_i are never written; nparts > 0: the logits kernel folded each row into its first nparts slots
  const int nvalid = nparts > 0 ? min(ntiles, nparts) : min(ntiles, (st->k + ltile - 1) / ltile);
  // online (max, sum) per thread, four independent accumulators (loads in flight together)
  float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, lq[4] = {0.f, 0.f, 0.f, 0.f};
  for (int t0 = threadIdx.x; t0 < nvalid; t0 += 4 * blockDim.x) {
    float2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = t0 + q * (int)blockDim.x < nvalid ? pr[t0 + q * blockDim.x] : make_float2(-INFINITY, 0.f);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (v[q].x > mq[q]) { lq[q] = lq[q] * __expf(mq[q] - v[q].x) + v[q].y; mq[q] = v[q].x; }
      else if (v[q].x > -INFINITY) lq[q] += v[q].y * __expf(v[q].x - mq[q]);
    }
  }
  float m = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])), l = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) l += mq[q] > -INFINITY ? lq[q] * __expf(mq[q] - m) : 0.f;
  const float wm = warp_max(m);
  l = (m > -INFINITY) ? l * __expf(m - wm) : 0.f;
  l = warp_sum(l);
  if (lane == 0) { sm[w] = wm; ss[w] = l; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M_ = -INFINITY;
    for (int i = 0; i < 8; ++i) M_ = fmaxf(M_, sm[i]);
    float L = 0.f;
    if (M_ > -INFINITY)
      for (int i = 0; i < 8; ++i) L += sm[i] > -INFINITY ? ss[i] * __expf(sm[i] - M_) : 0.f;
    rowmax[n] = M_;
    rowsum[n] = L;
    for (int q = 0; q < P.n; ++q) P.f32(q, P.lay.xmax)[(int64_t)P.rank * M + n] = M_;   // fused MAX all-reduce: push
    const int64_t j = Y[n] - a;
    zt[n] = (j >= 0 && j < C_local) ? mp.s * margin_phi(mp, ct[n]) : 0.f;   // owner rank of the positive
  }
}

// The per-tile partials exclude each row's target column (its logit z_t = s phi(c_t) is known exactly
// from K5b), so that the loss and the target gradient can be formed without cancellation when p_t -> 1:
//   q_n = sum_{j != t} e^{z_j - z_t},  loss_n = log1p(q_n),  p_t - 1 = -q_n / (1 + q_n)          (R22)
// Layout of the SUM all-reduce buffer (3M + 1 floats):
//   red[n]      = l_n e^{m_n - gm_n}  (sum over the sampled non-target columns, relative to the global max)
//   red[M + n]  = z_t of row n on the rank owning its class (0 elsewhere)
//   red[2M + n] = 1 if the rank sampled row n's class (the sum is 1 iff the positive is in S; R24)
//   red[3M]     = sum of c_t over the rows whose class is on this rank (CA_pcc numerator, Eq.7)
// Fused (P.n > 0): gm_n = max over the peers' xmax slots (the MAX all-reduce, read in rank order) is formed here and
// stored to gmax; the 3M + 1 values are pushed into slot `rank` of every peer's xred (the SUM all-reduce's send).
__global__ void __launch_bounds__(1024) k_prep_sum(int M, int64_t a, int64_t C_local, const float* __restrict__ rowmax,
                                                   float* __restrict__ gmax, const float* __restrict__ rowsum,
                                                   const float* __restrict__ zt, const int32_t* __restrict__ tcol,
                                                   const int64_t* __restrict__ Y, const float* __restrict__ ct,
                                                   float* __restrict__ red, Peers P) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  __shared__ float sh[32];
  float acc = 0.f;
  const int64_t ld = 3 * (int64_t)M + 1;
  auto put = [&](int64_t i, float v) {
    if (P.n == 0) red[i] = v;
    for (int q = 0; q < P.n; ++q) P.f32(q, P.lay.xred)[(int64_t)P.rank * ld + i] = v;
  };
  for (int n = threadIdx.x; n < M; n += blockDim.x) {
    const float rm = rowmax[n];
    float gm;
    if (P.n) {
      const float* xm = P.f32(P.rank, P.lay.xmax);
      gm = xm[n];
      for (int q = 1; q < P.n; ++q) gm = fmaxf(gm, xm[(int64_t)q * M + n]);
      gmax[n] = gm;
    } else {
      gm = gmax[n];
    }
    put(n, rm > -INFINITY ? rowsum[n] * __expf(rm - gm) : 0.f);
    put(M + n, zt[n]);
    put(2 * M + n, tcol[n] >= 0 ? 1.f : 0.f);
    const int64_t j = Y[n] - a;
    if (j >= 0 && j < C_local) acc += ct[n];
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) put(3 * M, v);
  }
}

// Global LSE_n, loss (Eq.5 over the global batch, R13), g_t[n] = p_t - 1 for K8, CA_pcc (Eq.7).
// Fused (P.n > 0): the SUM all-reduce is completed here — each value is the rank-ordered sum of the xred slots.
__global__ void __launch_bounds__(1024) k_finalize(int M, const float* __restrict__ gmax, const float* __restrict__ red,
                                                   float* __restrict__ lse, float* __restrict__ gt,
                                                   float* __restrict__ loss_out, float* __restrict__ metrics, int* err,
                                                   Peers P, const int64_t* __restrict__ Y, int ignore) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  __shared__ float sh[32];
  __shared__ int shn[32];
  float acc = 0.f;
  int nvalid = 0;
  const int64_t ld = 3 * (int64_t)M + 1;
  auto R = [&](int64_t i) {
    if (P.n == 0) return red[i];
    const float* xr = P.f32(P.rank, P.lay.xred);
    float v = xr[i];
    for (int q = 1; q < P.n; ++q) v += xr[(int64_t)q * ld + i];
    return v;
  };
  for (int n = threadIdx.x; n < M; n += blockDim.x) {
    const float gm = gmax[n], S = R(n), z = R(M + n);
    const bool sampled = R(2 * M + n) > 0.5f;
    float L, g, ls;
    if (ignore && Y[n] == -1) {                   // ignored row (f3, R28): no loss term, no gradient (p = 0)
      lse[n] = INFINITY;
      gt[n] = 0.f;
      continue;
    }
    ++nvalid;
    if (!sampled) {                               // positive not in S (fully random): Eq.9 over S, no pull
      ls = (gm > -INFINITY && S > 0.f) ? gm + __logf(S) : -INFINITY;
      L = ls - z;
      g = 0.f;
    } else if (!(gm > -INFINITY) || S == 0.f) {   // no negative in the sampled set: p_t = 1
      ls = z; L = 0.f; g = 0.f;
    } else {
      // lS = log of the non-target sum; whichever side dominates, the exponent is <= 0 (no overflow) and
      // neither p_t - 1 nor the loss is formed by cancellation (R22). Holds for any shift gm (the E-form
      // logits kernels report unshifted sums, gm = 0).
      const float lS = gm + __logf(S);
      if (z >= lS) {
        const float q = __expf(lS - z);
        L = log1pf(q);
        ls = z + L;
        g = -q / (1.f + q);
      } else {
        const float r = __expf(z - lS);
        ls = lS + log1pf(r);
        L = ls - z;
        g = -1.f / (1.f + r);
      }
    }
    lse[n] = ls;
    gt[n] = g;
    acc += L;
  }
  acc = warp_sum(acc);
  for (int o = 16; o; o >>= 1) nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
  if ((threadIdx.x & 31) == 0) { sh[threadIdx.x >> 5] = acc; shn[threadIdx.x >> 5] = nvalid; }
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
    int nv = threadIdx.x < (blockDim.x >> 5) ? shn[threadIdx.x] : 0;
    v = warp_sum(v);
    for (int o = 16; o; o >>= 1) nv += __shfl_xor_sync(0xffffffffu, nv, o);
    if (threadIdx.x == 0) {
      const float Mv = (float)max(nv, 1);          // every row ignored: loss 0, no gradient
      const float Lm = v / Mv;
      if (loss_out) *loss_out = Lm;
      metrics[0] = Lm;
      metrics[1] = R(3 * M) / Mv;
      metrics[2] = Mv;
      if (!isfinite(Lm)) atomicOr(err, ERR_NUMERIC);
    }
  }
}

template <bool BF16>
__device__ __forceinline__ void load8(const void* cosv, int64_t base, float (&c)[8]) {
  if (BF16) {
    uint4 raw = __ldcs(reinterpret_cast<const uint4*>((const __half*)cosv + base));
    const __half2* h = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) { float2 f = __half22float2(h[i]); c[2 * i] = f.x; c[2 * i + 1] = f.y; }
  } else {
    float4 a = __ldcs(reinterpret_cast<const float4*>((const float*)cosv + base));
    float4 b = __ldcs(reinterpret_cast<const float4*>((const float*)cosv + base + 4));
    c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w; c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
  }
}

template <bool BF16>
__device__ __forceinline__ void store8(void* G, int64_t base, const float (&g)[8]) {
  if (BF16) {
    uint4 o;
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) ob[i] = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
    *reinterpret_cast<uint4*>((__nv_bfloat16*)G + base) = o;
  } else {
    *reinterpret_cast<float4*>((float*)G + base) = make_float4(g[0], g[1], g[2], g[3]);
    *reinterpret_cast<float4*>((float*)G + base + 4) = make_float4(g[4], g[5], g[6], g[7]);
  }
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Every element as a non-target: Gc[j][n] = 2^min(c sl - off'_n, log2(s/M)) with off'_n = LSE_n log2 e -
// log2(s/M) (the s/M factor folded into the exponent); padding rows have off' = +inf (their stored cosine is 0).
// The target entries (one per row) are then rewritten by k_softmax_grad_targets.
#ifndef PFC_K8_U
#define PFC_K8_U 2
#endif
template <bool BF16, bool DOT>
__global__ void __launch_bounds__(256) k_softmax_grad(int64_t k_pad, int M, int ldm, const void* __restrict__ cosv,
                                                      const float* __restrict__ lse, const SamplerState* st,
                                                      MarginParams mp, void* __restrict__ G,
                                                      float* __restrict__ dotw, const float* __restrict__ gsc,
                                                      const float* __restrict__ mvalid) {
  extern __shared__ float s_off[];            // transposed: pos(n) = (n % 8) * (ldm / 8) + n / 8
  const float L2E = 1.4426950408889634f;
  const float lgs = log2f(mp.s / *mvalid);    // (s / M_valid): the mean over the rows not ignored
  const int l8 = ldm >> 3;
  for (int n = threadIdx.x; n < ldm; n += blockDim.x) s_off[(n & 7) * l8 + (n >> 3)] = n < M ? lse[n] * L2E - lgs : INFINITY;
  __syncthreads();
  const int k = st->k;
  const float sl = mp.s * L2E;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  constexpr int U = PFC_K8_U;
  const int nit = (ldm + 255) / 256;
  if (nit == 1) {
    // one 8-row chunk per lane: its offsets stay in registers for the whole class loop, U classes in flight
    const int n0 = lane * 8;
    const bool act = n0 < ldm;
    float off[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) off[i] = act ? s_off[i * l8 + lane] : INFINITY;
    for (int64_t jb = w0; jb < k_pad; jb += U * nw) {
      float c[U][8], sc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = jb + u * nw;
        sc[u] = 1.f;                             // R25: G' = G / ||w_j|| when W_s holds un-normalised rows
        if (gsc && j < k) sc[u] = __ldg(gsc + j);
        if (act && j < k) load8<BF16>(cosv, j * ldm + n0, c[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = jb + u * nw;
        if (j >= k_pad) break;
        float g[8];
        float d = 0.f;
        if (act && j < k) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            // p <= 1 for every non-target entry (LSE >= z_j); the clamp only bounds the provisional value at
            // the target column (margin not applied there), which k_softmax_grad_targets replaces exactly
            g[i] = ex2_ftz(fminf(fmaf(c[u][i], sl, -off[i]), lgs)) * sc[u];
            if (DOT) d = fmaf(g[i], c[u][i], d);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) g[i] = 0.f;
        }
        if (act) store8<BF16>(G, j * ldm + n0, g);
        if (DOT) {
          d = warp_sum(d);
          if (lane == 0) dotw[j] = d;
        }
      }
    }
  } else {
    // M > 256: a warp streams one whole class row (ldm entries, contiguous) at a time, two 256-row chunks in
    // flight; the row offsets come from the transposed (conflict-free) shared array
    for (int64_t j = w0; j < k_pad; j += nw) {
      const bool valid = j < k;
      const float sc = gsc && valid ? gsc[j] : 1.f;
      float d = 0.f;
      for (int it = 0; it < nit; it += U) {
        float c[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int n0 = (it + u) * 256 + lane * 8;
          if (valid && it + u < nit && n0 < ldm) load8<BF16>(cosv, j * ldm + n0, c[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int n0 = (it + u) * 256 + lane * 8;
          if (it + u >= nit || n0 >= ldm) break;
          float g[8];
          if (valid) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              g[i] = ex2_ftz(fminf(fmaf(c[u][i], sl, -s_off[i * l8 + lane + 32 * (it + u)]), lgs)) * sc;
              if (DOT) d = fmaf(g[i], c[u][i], d);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) g[i] = 0.f;
          }
          store8<BF16>(G, j * ldm + n0, g);
        }
      }
      if (DOT) {
        d = warp_sum(d);
        if (lane == 0) dotw[j] = d;
      }
    }
  }
}

// Target entries: Gc[t_n][n] = (s/M)(p_t - 1) phi'(c_t) with the cancellation-free p_t - 1 of finalize, and the
// radial dot corrected by (new - old) g c of that entry (several rows may share a class: atomics).
template <bool BF16, bool DOT>
__global__ void k_softmax_grad_targets(int M, int ldm, const void* __restrict__ cosv, const float* __restrict__ lse,
                                       const float* __restrict__ gt, const int32_t* __restrict__ tcol,
                                       const float* __restrict__ ct, MarginParams mp, void* __restrict__ G,
                                       float* __restrict__ dotw, const float* __restrict__ gsc,
                                       const float* __restrict__ mvalid) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= M) return;
  const int j = tcol[n];
  if (j < 0) return;
  const float L2E = 1.4426950408889634f;
  const float gs = mp.s / *mvalid;
  const int64_t e = (int64_t)j * ldm + n;
  const float cst = BF16 ? __half2float(((const __half*)cosv)[e]) : ((const float*)cosv)[e];
  const float lgs = log2f(gs);
  const float sc = gsc ? gsc[j] : 1.f;
  const float g_old = ex2_ftz(fminf(fmaf(cst, mp.s * L2E, -(lse[n] * L2E - lgs)), lgs)) * sc;   // as k_softmax_grad
  const float c_t = ct[n];
  const float g_new = gs * gt[n] * margin_dphi(mp, c_t) * sc;
  if (BF16) ((__nv_bfloat16*)G)[e] = __float2bfloat16_rn(g_new);
  else ((float*)G)[e] = g_new;
  if (DOT) atomicAdd(&dotw[j], g_new * c_t - g_old * cst);
}

// ---------------------------------------------------------------- K10
// Fused (P.n > 0): dX_hat row n of this owner = the rank-ordered sum of its xdx slots (the reduce-scatter's
// reduction, Alg.1 L12-13).
__global__ void k_xnorm_backward(int B, int d, const float* __restrict__ dxh, const float* __restrict__ xh,
                                 const float* __restrict__ xnorm, float* __restrict__ gx, Peers P) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (n >= B) return;
  const float* xr = xh + (int64_t)n * d;
  const float* xd = P.n ? P.f32(P.rank, P.lay.xdx) : nullptr;
  auto G = [&](int c) {
    if (P.n == 0) return dxh[(int64_t)n * d + c];
    float v = xd[(int64_t)n * d + c];
    for (int q = 1; q < P.n; ++q) v += xd[((int64_t)q * B + n) * d + c];
    return v;
  };
  float dot = 0.f;
  for (int c = lane; c < d; c += 32) dot += xr[c] * G(c);
  dot = warp_sum(dot);
  const float inv = 1.f / fmaxf(xnorm[n], kNormEps);
  for (int c = lane; c < d; c += 32) gx[(int64_t)n * d + c] = (G(c) - xr[c] * dot) * inv;
}

__global__ void k_push_dx(int64_t n, int d, int B, const float* __restrict__ dXh, Peers P) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  PFC_DCHECK(i >= n || (int)(i / d / B) < P.n);
  if (i < n) *dx_dst(P, nullptr, i, d, B) = dXh[i];
}

// ---------------------------------------------------------------- K12 (+ raw-gradient introspection)
template <bool UPDATE>
__global__ void k_sgd(int64_t k_pad, int d, float* __restrict__ W, float* __restrict__ V, const float* __restrict__ dWh,
                      const int32_t* __restrict__ idx, const float* __restrict__ inv_norm, const SamplerState* st,
                      const float* __restrict__ lr_dev, float mu, float lambda, float* __restrict__ out, int gsc) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const float lr = UPDATE ? *lr_dev : 0.f;
  const int lane = threadIdx.x & 31;
  if (p >= st->k) return;
  const int64_t j = idx[p];
  float* wr = W + j * d;
  const float* gr = dWh + p * d;
  const float inv = inv_norm[p];
  float dot = 0.f;
  for (int c = lane * 4; c < d; c += 128) {
    float4 w = *reinterpret_cast<const float4*>(wr + c);
    float4 g = *reinterpret_cast<const float4*>(gr + c);
    dot += (w.x * g.x + w.y * g.y + w.z * g.z + w.w * g.w);
  }
  dot = warp_sum(dot) * inv;  // w_hat . dw_hat
  const float oi = gsc ? 1.f : inv;   // R25: dWh = G'^T X_hat already carries 1/||w||
  for (int c = lane * 4; c < d; c += 128) {
    float4 w = *reinterpret_cast<const float4*>(wr + c);
    float4 g = *reinterpret_cast<const float4*>(gr + c);
    float4 gg;
    gg.x = (g.x - w.x * inv * dot) * oi;
    gg.y = (g.y - w.y * inv * dot) * oi;
    gg.z = (g.z - w.z * inv * dot) * oi;
    gg.w = (g.w - w.w * inv * dot) * oi;
    if (UPDATE) {
      float* vr = V + j * d;
      float4 v = *reinterpret_cast<const float4*>(vr + c);
      v.x = mu * v.x + gg.x + lambda * w.x;
      v.y = mu * v.y + gg.y + lambda * w.y;
      v.z = mu * v.z + gg.z + lambda * w.z;
      v.w = mu * v.w + gg.w + lambda * w.w;
      w.x -= lr * v.x; w.y -= lr * v.y; w.z -= lr * v.z; w.w -= lr * v.w;
      *reinterpret_cast<float4*>(vr + c) = v;
      *reinterpret_cast<float4*>(wr + c) = w;
    } else {
      *reinterpret_cast<float4*>(out + p * d + c) = gg;
    }
  }
}

}  // namespace

static Peers none_or(const Peers* P) {
  Peers q{};
  if (P) q = *P;
  return q;
}

SymLayout sym_layout(const Sizes& sz) {
  auto up = [](int64_t v) { return (v + 255) / 256 * 256; };
  SymLayout L{};
  L.x32 = 0;
  L.y = up((int64_t)sz.M_pad * sz.d * 4);
  L.xmax = L.y + up((int64_t)sz.M * 8);
  L.xred = L.xmax + up((int64_t)sz.world * sz.M * 4);
  L.xdx = L.xred + up((int64_t)sz.world * (3 * (int64_t)sz.M + 1) * 4);
  L.bytes = L.xdx + up((int64_t)sz.world * sz.B * sz.d * 4);
  return L;
}

int launch_normalize_x(const Sizes& sz, const float* x, const int64_t* labels, float* xh_local, float* xnorm,
                       float* X32, int64_t* Y, int* err, const Peers* P, int ignore, cudaStream_t s) {
  launch_pdl(k_normalize_x, dim3((sz.B * 32 + 255) / 256), dim3(256), 0, s, sz.B, sz.d, sz.rank, sz.C, x, labels, xh_local, xnorm, X32, Y,
                                                        err, none_or(P), ignore);
  return 1;
}

int launch_x_to_bf16(const Sizes& sz, const float* X32, __nv_bfloat16* Xb, __half* Xh16, cudaStream_t s) {
  int64_t n = (int64_t)sz.M * sz.d;
  launch_pdl(k_x_to_bf16, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, n, X32, Xb, Xh16);
  return 1;
}

int launch_gather_w(const Sizes& sz, bool bf16, const float* W, const int32_t* idx, const SamplerState* st, void* Ws,
                    __half* Ws16, float* inv_norm, int* err, cudaStream_t s) {
  unsigned grid = (unsigned)((sz.k_pad * 32 + 255) / 256);
  if (bf16) launch_pdl(k_gather_w<true>, dim3(grid), dim3(256), 0, s, sz.k_pad, sz.d, W, idx, st, Ws, Ws16, inv_norm, err);
  else launch_pdl(k_gather_w<false>, dim3(grid), dim3(256), 0, s, sz.k_pad, sz.d, W, idx, st, Ws, nullptr, inv_norm, err);
  return 1;
}

int launch_target_cos(const Sizes& sz, const float* X32, const float* W, const int64_t* Y, const int32_t* idx,
                      const SamplerState* st, const int* tile_cnt, int32_t* tcol, float* ct, cudaStream_t s) {
  launch_pdl(k_target_cos, dim3((sz.M * 32 + 255) / 256), dim3(256), 0, s, sz.M, sz.d, sz.a, sz.C_local, X32, W, Y, idx, st,
                                                       tile_cnt + 3 * sz.ntiles_sel, sz.ntiles_sel, tcol, ct);
  return 1;
}

int launch_row_combine(const Sizes& sz, const float2* partials, int nparts, const int64_t* Y, const float* ct,
                       const SamplerState* st, MarginParams mp, float* rowmax, float* rowsum, float* zt, const Peers* P,
                       cudaStream_t s) {
  launch_pdl(k_row_combine, dim3(sz.M), dim3(256), 0, s, sz.M, sz.n_ltiles, sz.ltile, nparts, sz.a, sz.C_local, partials, Y, ct, st, mp, rowmax,
                                     rowsum, zt, none_or(P));
  return 1;
}

int launch_prep_sum(const Sizes& sz, const float* rowmax, float* gmax, const float* rowsum, const float* zt,
                    const int32_t* tcol, const int64_t* Y, const float* ct, float* red, const Peers* P, cudaStream_t s) {
  launch_pdl(k_prep_sum, dim3(1), dim3(1024), 0, s, sz.M, sz.a, sz.C_local, rowmax, gmax, rowsum, zt, tcol, Y, ct, red, none_or(P));
  return 1;
}

int launch_finalize(const Sizes& sz, const float* gmax, const float* red, float* lse, float* gt, float* loss_out,
                    float* metrics, int* err, const Peers* P, const int64_t* Y, int ignore, cudaStream_t s) {
  launch_pdl(k_finalize, dim3(1), dim3(1024), 0, s, sz.M, gmax, red, lse, gt, loss_out, metrics, err, none_or(P), Y, ignore);
  return 1;
}

int launch_softmax_grad(const Sizes& sz, bool bf16, const void* cosv, const float* lse, const float* gt,
                        const int32_t* tcol, const float* ct, const SamplerState* st, MarginParams mp, void* G,
                        float* dotw, const float* gsc, const float* mvalid, cudaStream_t s) {
  const size_t smem = (size_t)sz.M_pad * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_softmax_grad<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_softmax_grad<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_softmax_grad<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(k_softmax_grad<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr = true;
  }
  // persistent grid: exactly the resident blocks (a whole number of waves over the SMs)
  static int per_sm[4] = {0, 0, 0, 0}, sms = 0;
  const int ti = (bf16 ? 2 : 0) + (dotw ? 1 : 0);
  if (!per_sm[ti]) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const void* f = bf16 ? (dotw ? (const void*)k_softmax_grad<true, true> : (const void*)k_softmax_grad<true, false>)
                         : (dotw ? (const void*)k_softmax_grad<false, true> : (const void*)k_softmax_grad<false, false>);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[ti], f, 256, 2048 * sizeof(float));
    if (per_sm[ti] < 1) per_sm[ti] = 1;
  }
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(sz.k_pad / 8, (int64_t)per_sm[ti] * sms));
  const int ldm = sz.M_pad;
  const unsigned tg = (unsigned)((sz.M + 255) / 256);
  if (bf16) {
    if (dotw) {
      k_softmax_grad<true, true><<<grid, 256, smem, s>>>(sz.k_pad, sz.M, ldm, cosv, lse, st, mp, G, dotw, gsc, mvalid);
      k_softmax_grad_targets<true, true><<<tg, 256, 0, s>>>(sz.M, ldm, cosv, lse, gt, tcol, ct, mp, G, dotw, gsc, mvalid);
    } else {
      k_softmax_grad<true, false><<<grid, 256, smem, s>>>(sz.k_pad, sz.M, ldm, cosv, lse, st, mp, G, dotw, gsc, mvalid);
      k_softmax_grad_targets<true, false><<<tg, 256, 0, s>>>(sz.M, ldm, cosv, lse, gt, tcol, ct, mp, G, dotw, gsc, mvalid);
    }
  } else {
    if (dotw) {
      k_softmax_grad<false, true><<<grid, 256, smem, s>>>(sz.k_pad, sz.M, ldm, cosv, lse, st, mp, G, dotw, gsc, mvalid);
      k_softmax_grad_targets<false, true><<<tg, 256, 0, s>>>(sz.M, ldm, cosv, lse, gt, tcol, ct, mp, G, dotw, gsc, mvalid);
    } else {
      k_softmax_grad<false, false><<<grid, 256, smem, s>>>(sz.k_pad, sz.M, ldm, cosv, lse, st, mp, G, dotw, gsc, mvalid);
      k_softmax_grad_targets<false, false><<<tg, 256, 0, s>>>(sz.M, ldm, cosv, lse, gt, tcol, ct, mp, G, dotw, gsc, mvalid);
    }
  }
  return 2;
}

int launch_xnorm_backward(const Sizes& sz, const float* dxh, const float* xh_local, const float* xnorm, float* grad_x,
                          const Peers* P, cudaStream_t s) {
  launch_pdl(k_xnorm_backward, dim3((sz.B * 32 + 255) / 256), dim3(256), 0, s, sz.B, sz.d, dxh, xh_local, xnorm, grad_x, none_or(P));
  return 1;
}

int launch_push_dx(const Sizes& sz, const float* dXh, const Peers& P, cudaStream_t s) {
  const int64_t n = (int64_t)sz.M * sz.d;
  k_push_dx<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, sz.d, sz.B, dXh, P);
  return 1;
}

int launch_sgd(const Sizes& sz, float* W, float* V, const float* dWh, const int32_t* idx, const float* inv_norm,
               const SamplerState* st, const float* lr_dev, float mu, float lambda, int gsc, cudaStream_t s) {
  unsigned grid = (unsigned)((sz.k_pad * 32 + 255) / 256);
  k_sgd<true><<<grid, 256, 0, s>>>(sz.k_pad, sz.d, W, V, dWh, idx, inv_norm, st, lr_dev, mu, lambda, nullptr, gsc);
  return 1;
}

namespace {
// f4 staging: one warp per sampled position p moves the d-float rows
// W[idx_p], V[idx_p] of the (host-mapped) shard to / from the compact HBM rows Wst[p], Vst[p]. Many rows in
// flight per SM so that the PCIe / C2C reads stream.
template <bool TO_HOST>
__global__ void k_stage_rows(int64_t k_pad, int d, float* __restrict__ W, float* __restrict__ V,
                             const int32_t* __restrict__ idx, const SamplerState* st, float* __restrict__ Wst,
                             float* __restrict__ Vst) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= st->k) return;
  const int64_t j = idx[p];
  PFC_DCHECK(j >= 0 && p < k_pad);
  for (int c = lane * 4; c < d; c += 128) {
    if (TO_HOST) {
      *reinterpret_cast<float4*>(W + j * d + c) = *reinterpret_cast<const float4*>(Wst + p * d + c);
      *reinterpret_cast<float4*>(V + j * d + c) = *reinterpret_cast<const float4*>(Vst + p * d + c);
    } else {
      const float4 w = *reinterpret_cast<const float4*>(W + j * d + c);
      const float4 v = *reinterpret_cast<const float4*>(V + j * d + c);
      *reinterpret_cast<float4*>(Wst + p * d + c) = w;
      *reinterpret_cast<float4*>(Vst + p * d + c) = v;
    }
  }
}
__global__ void k_iota(int32_t* out, int64_t n, int32_t base) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = base + (int32_t)i;
}
__global__ void k_set_f32(float* dst, float v) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  pdl_trigger(); *dst = v; }
// end of a step: advance the device step counter and publish the sticky device error word to the host-mapped word
// (plain store into page-locked memory; the host reads it at the next hot-path call without synchronising)
__global__ void k_end_step(uint64_t* dst, uint64_t v, const int* err, volatile int* err_host) {
  pdl_wait();      // programmatic dependent launch: the predecessor kernel has completed
  // (no early trigger: the dependents launch as this grid completes)
  *dst += v;
  if (err_host) *err_host = *err;
}
}  // namespace

int launch_stage_rows(const Sizes& sz, float* W, float* V, const int32_t* idx, const SamplerState* st, float* Wst,
                      float* Vst, bool to_host, cudaStream_t s) {
  const unsigned grid = (unsigned)((sz.k_pad * 32 + 255) / 256);
  if (to_host) k_stage_rows<true><<<grid, 256, 0, s>>>(sz.k_pad, sz.d, W, V, idx, st, Wst, Vst);
  else k_stage_rows<false><<<grid, 256, 0, s>>>(sz.k_pad, sz.d, W, V, idx, st, Wst, Vst);
  return 1;
}

int launch_iota(int32_t* out, int64_t n, int32_t base) {
  k_iota<<<(unsigned)((n + 255) / 256), 256>>>(out, n, base);
  return 1;
}

int launch_set_scalar(float* dst, float v, cudaStream_t s) {
  launch_pdl(k_set_f32, dim3(1), dim3(1), 0, s, dst, v);
  return 1;
}

int launch_advance_step(uint64_t* step_dev, const int* err_dev, int* err_host_mapped, cudaStream_t s) {
  launch_pdl(k_end_step, dim3(1), dim3(1), 0, s, step_dev, 1, err_dev, err_host_mapped);
  return 1;
}

int launch_raw_grad(const Sizes& sz, const float* W, const float* dWh, const int32_t* idx, const float* inv_norm,
                    const SamplerState* st, float* out, int gsc, cudaStream_t s) {
  unsigned grid = (unsigned)((sz.k_pad * 32 + 255) / 256);
  k_sgd<false><<<grid, 256, 0, s>>>(sz.k_pad, sz.d, const_cast<float*>(W), nullptr, dWh, idx, inv_norm, st, nullptr,
                                    0.f, 0.f, out, gsc);
  return 1;
}

}  // namespace pfc

// ---------------------------------------------------------------- loopback collectives (one process, k ranks)
namespace pfc {
namespace {
__global__ void k_group_reduce(int64_t n, PtrPack src, int64_t src_off, PtrPack dst, int nranks, int nd, int op) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = src.p[0][src_off + i];
  for (int r = 1; r < nranks; ++r) {  // rank-ascending
    float v = src.p[r][src_off + i];
    acc = op == 0 ? acc + v : fmaxf(acc, v);
  }
  for (int r = 0; r < nd; ++r) dst.p[r][i] = acc;
}
}  // namespace

int launch_group_reduce(int64_t n, const PtrPack& src, int64_t src_off, const PtrPack& dst, int nranks, int ndst,
                        int op, cudaStream_t s) {
  k_group_reduce<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, src, src_off, dst, nranks, ndst, op);
  return 1;
}

namespace {
__global__ void k_idx_to_global(const int32_t* __restrict__ idx, const SamplerState* st, int64_t a,
                                int64_t* __restrict__ out) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < st->k) out[p] = a + idx[p];
}
}  // namespace

int launch_idx_to_global(int64_t k_max, const int32_t* idx, const SamplerState* st, int64_t a, int64_t* out,
                         cudaStream_t s) {
  k_idx_to_global<<<(unsigned)((k_max + 255) / 256), 256, 0, s>>>(idx, st, a, out);
  return 1;
}
}  // namespace pfc
