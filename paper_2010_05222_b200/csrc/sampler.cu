// PPRN sampler on one shard (steps 1-3 and Eq.10), bit-exact selection recipe of
// DESIGN.md §Sampler:
//   K2  mark_positives : bitmap of labels in [a, a + C_local) and |P_i| (step 1, dedup R5)
//   K3  keys + radix select : h_j = Philox key of every non-positive class (R2); three histogram passes
//       (11/11/10 bits) find the threshold key T of the n_i-th smallest (h, j) and t, the number of
//       tied (h == T) negatives to take, smallest ids first (R3)
//   K4  compaction : idx_i = ascending ids of (positive or selected) via tile counts + scan + write (R4);
//       tcol[n] = position of y_n in idx_i (binary search) or -1 when y_n is not in this shard.
// Everything is device-resident (k_i is data-dependent); no host synchronisation.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include "pfc_internal.cuh"

namespace pfc {
namespace {

constexpr int kThreads = 256;

int num_sms_host() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

__global__ void k_mark_positives(const int64_t* __restrict__ Y, int M, int64_t a, int64_t C_local,
                                 uint32_t* __restrict__ bits, SamplerState* st, int mode) {
  int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= M || mode == PFC_SAMPLE_RANDOM) return;   // fully random: labels ignored (R24)
  int64_t y = Y[n] - a;
  if (y >= 0 && y < C_local) {
    uint32_t mask = 1u << (y & 31);
    uint32_t old = atomicOr(&bits[y >> 5], mask);
    if (!(old & mask)) atomicAdd(&st->npos, 1);
  }
}

__device__ __forceinline__ bool is_pos(const uint32_t* bits, int64_t j) {
  return (__ldg(&bits[j >> 5]) >> (j & 31)) & 1u;
}

// Pass 1: compute and store every key, histogram of the top 11 bits over non-positive classes.
__global__ void __launch_bounds__(kThreads) k_keys_hist(int64_t a, int64_t C_local, uint64_t seed,
                                                        const uint64_t* __restrict__ step_dev,
                                                        const uint32_t* __restrict__ bits, uint32_t* __restrict__ keys,
                                                        int* __restrict__ hist) {
  const uint32_t step = (uint32_t)*step_dev;   // device-resident step counter (CUDA-graph replayable)
  __shared__ int sh[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  // two independent Philox chains per thread and iteration (the 10 dependent rounds of one key leave the
  // integer-multiply pipe idle otherwise)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; j + stride < C_local; j += 2 * stride) {
    const uint32_t h0 = philox_class_key((uint64_t)(a + j), step, seed);
    const uint32_t h1 = philox_class_key((uint64_t)(a + j + stride), step, seed);
    keys[j] = h0;
    keys[j + stride] = h1;
    if (!is_pos(bits, j)) atomicAdd(&sh[h0 >> 21], 1);
    if (!is_pos(bits, j + stride)) atomicAdd(&sh[h1 >> 21], 1);
  }
  if (j < C_local) {
    const uint32_t h = philox_class_key((uint64_t)(a + j), step, seed);
    keys[j] = h;
    if (!is_pos(bits, j)) atomicAdd(&sh[h >> 21], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Locate, with a 256-thread block, the bucket b of `hist` (nbins) holding the `need`-th smallest key:
// cum(b) < need <= cum(b) + hist[b]. Returns b and need - cum(b) (1-based rank inside the bucket).
__device__ void block_select(const int* __restrict__ hist, int nbins, int need, int& bucket, int& rem) {
  __shared__ int wsum[kThreads / 32];
  __shared__ int res[2];
  const int per = nbins / kThreads;            // 8 (2048 bins) or 4 (1024 bins)
  const int b0 = threadIdx.x * per;
  int local = 0;
  for (int b = 0; b < per; ++b) local += hist[b0 + b];
  // block exclusive scan of `local`
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int before = incl - local;
  for (int i = 0; i < w; ++i) before += wsum[i];
  if (before < need && need <= before + local) {
    int cum = before;
    for (int b = 0; b < per; ++b) {
      const int h = hist[b0 + b];
      if (cum < need && need <= cum + h) { res[0] = b0 + b; res[1] = need - cum; break; }
      cum += h;
    }
  }
  __syncthreads();
  bucket = res[0];
  rem = res[1];
}

// k_i and n_i from |P_i| (R1, R23, R24)
__device__ __forceinline__ int budget_k(int npos, int64_t budget, int64_t C_local, double rate, int mode) {
  if (mode == PFC_SAMPLE_PPRN_PAPER) {   // R23: |P_i| + round_half_up((C_local - |P_i|) r)
    const int64_t rest = C_local - npos;
    int64_t n = (int64_t)floor((double)rest * rate + 0.5);
    n = n < 0 ? 0 : (n > rest ? rest : n);
    return npos + (int)n;
  }
  if (mode == PFC_SAMPLE_RANDOM) return (int)budget;
  return (int)max(budget, (int64_t)npos);   // R1
}

// Pass 2: every block selects the 11-bit bucket of pass 1 from hist0 (block 0 records it), then histograms the
// next 11 bits of the keys inside it.
__global__ void __launch_bounds__(kThreads) k_hist_pass2(int64_t C_local, int64_t budget, double rate, int mode,
                                                         const uint32_t* __restrict__ bits,
                                                         const uint32_t* __restrict__ keys, const int* __restrict__ hist0,
                                                         SamplerState* st, int* __restrict__ hist1) {
  __shared__ int sh[2048];
  const int npos = st->npos;
  const int k = budget_k(npos, budget, C_local, rate, mode);
  const int n_neg = k - npos;
  if (n_neg == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { st->k = k; st->n_neg = 0; st->none = 1; }
    return;
  }
  int b1, rem1;
  block_select(hist0, 2048, n_neg, b1, rem1);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->k = k; st->n_neg = n_neg; st->none = 0; st->prefix1 = (uint32_t)b1; st->rem1 = rem1;
  }
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  // 4 consecutive keys per thread and iteration (the key array is padded to whole tiles), two in flight
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
#pragma unroll 2
  for (int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; j0 < C_local; j0 += stride) {
    const uint4 h4 = *reinterpret_cast<const uint4*>(keys + j0);
    const uint32_t pw = __ldg(&bits[j0 >> 5]) >> (j0 & 31);
    const uint32_t hh[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if ((hh[i] >> 21) == (uint32_t)b1 && !((pw >> i) & 1u) && j0 + i < C_local) atomicAdd(&sh[(hh[i] >> 10) & 0x7FF], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist1[i], sh[i]);
}

// Pass 3: select the second digit from hist1, histogram the last 10 bits.
__global__ void __launch_bounds__(kThreads) k_hist_pass3(int64_t C_local, const uint32_t* __restrict__ bits,
                                                         const uint32_t* __restrict__ keys, const int* __restrict__ hist1,
                                                         SamplerState* st, int* __restrict__ hist2) {
  __shared__ int sh[1024];
  if (st->none) return;
  int b2, rem2;
  block_select(hist1, 2048, st->rem1, b2, rem2);
  const uint32_t pre = (st->prefix1 << 11) | (uint32_t)b2;
  if (blockIdx.x == 0 && threadIdx.x == 0) { st->prefix2 = pre; st->rem2 = rem2; }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
#pragma unroll 2
  for (int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; j0 < C_local; j0 += stride) {
    const uint4 h4 = *reinterpret_cast<const uint4*>(keys + j0);
    const uint32_t pw = __ldg(&bits[j0 >> 5]) >> (j0 & 31);
    const uint32_t hh[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if ((hh[i] >> 10) == pre && !((pw >> i) & 1u) && j0 + i < C_local) atomicAdd(&sh[hh[i] & 0x3FF], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist2[i], sh[i]);
}

// Flags of the 32 consecutive classes j0 .. j0+31 (j0 % 32 == 0) of one thread as bit masks: definitely selected
// (positive, or key < T) and tied (key == T, non-positive); classes >= C_local have neither.
__device__ __forceinline__ void flags32(int64_t j0, int64_t C_local, const uint32_t* bits, const uint32_t* keys,
                                        bool none, uint32_t T, uint32_t& def, uint32_t& tie) {
  def = 0u; tie = 0u;
  if (j0 >= C_local) return;
  const uint32_t pw = __ldg(&bits[j0 >> 5]);
  const uint32_t valid = C_local - j0 >= 32 ? 0xFFFFFFFFu : ((1u << (C_local - j0)) - 1u);
  uint32_t lt = 0u, eq = 0u;
  if (!none) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 h = *reinterpret_cast<const uint4*>(keys + j0 + 4 * q);
      lt |= (uint32_t)(h.x < T) << (4 * q) | (uint32_t)(h.y < T) << (4 * q + 1) | (uint32_t)(h.z < T) << (4 * q + 2) |
            (uint32_t)(h.w < T) << (4 * q + 3);
      eq |= (uint32_t)(h.x == T) << (4 * q) | (uint32_t)(h.y == T) << (4 * q + 1) | (uint32_t)(h.z == T) << (4 * q + 2) |
            (uint32_t)(h.w == T) << (4 * q + 3);
    }
  }
  def = (pw | lt) & valid;
  tie = eq & ~pw & valid;
}

// Block-wide exclusive scan of small per-thread counts (256 threads); returns the prefix, sets the total.
__device__ __forceinline__ int block_count_scan(int v, int* wsum, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int pre = incl - v, tot = 0;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) {
    const int x = wsum[i];
    pre += i < w ? x : 0;
    tot += x;
  }
  __syncthreads();
  total = tot;
  return pre;
}

// K4a: select the threshold key T (and t, the number of tied keys to take) from hist2 (block 0 records them),
// then count definitely-selected and tied classes per 8192-class tile.
__global__ void __launch_bounds__(kThreads) k_tile_counts(int64_t C_local, const uint32_t* __restrict__ bits,
                                                          const uint32_t* __restrict__ keys, const int* __restrict__ hist2,
                                                          SamplerState* st, int* __restrict__ tile_cnt, int ntiles) {
  __shared__ int sdef, stie;
  const bool none = st->none;
  uint32_t T = 0;
  if (!none) {
    int b3, rem3;
    block_select(hist2, 1024, st->rem2, b3, rem3);
    T = (st->prefix2 << 10) | (uint32_t)b3;
    if (blockIdx.x == 0 && threadIdx.x == 0) { st->T = T; st->t = rem3; }
  }
  const int64_t base = (int64_t)blockIdx.x * kSelTile;
  uint32_t dm, tm;
  flags32(base + 32 * threadIdx.x, C_local, bits, keys, none, T, dm, tm);
  int ndef = __popc(dm), ntie = __popc(tm);
  if (threadIdx.x == 0) { sdef = 0; stie = 0; }
  __syncthreads();
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ndef += __shfl_xor_sync(0xffffffffu, ndef, o);
    ntie += __shfl_xor_sync(0xffffffffu, ntie, o);
  }
  if ((threadIdx.x & 31) == 0) { atomicAdd(&sdef, ndef); atomicAdd(&stie, ntie); }
  __syncthreads();
  if (threadIdx.x == 0) {
    tile_cnt[blockIdx.x] = sdef;
    tile_cnt[ntiles + blockIdx.x] = stie;
  }
}

// K4b: single block. Exclusive scans: tie offsets, then selected counts (definite + ties ranked < t); warp-shuffle
// block scans over 1024 tiles at a time.
__global__ void __launch_bounds__(1024) k_tile_scan(int* __restrict__ tile_cnt, int ntiles, SamplerState* st,
                                                    int* err) {
  __shared__ int wsum[32];
  const SamplerState s = *st;
  int* def = tile_cnt;
  int* tie = tile_cnt + ntiles;
  int* tie_off = tile_cnt + 2 * ntiles;
  int* sel_off = tile_cnt + 3 * ntiles;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    int carry = 0;
    for (int base = 0; base < ntiles; base += 1024) {
      const int i = base + threadIdx.x;
      int v = 0;
      if (i < ntiles) {
        if (pass == 0) v = tie[i];
        else v = def[i] + (s.none ? 0 : max(0, min(s.t - tie_off[i], tie[i])));
      }
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) wsum[w] = incl;
      __syncthreads();
      if (w == 0) {
        int x = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += u;
        }
        wsum[lane] = x;
      }
      __syncthreads();
      if (i < ntiles) (pass == 0 ? tie_off : sel_off)[i] = carry + (w ? wsum[w - 1] : 0) + incl - v;
      carry += wsum[31];
      __syncthreads();
    }
    if (pass == 1 && threadIdx.x == 0) {
      st->total = carry;
      if (carry != s.k) atomicOr(err, ERR_INTERNAL);
    }
  }
}

// K4c: order-preserving write of the selected local ids, 4 consecutive classes per thread per iteration.
__global__ void __launch_bounds__(kThreads) k_tile_write(int64_t C_local, const uint32_t* __restrict__ bits,
                                                         const uint32_t* __restrict__ keys, const SamplerState* st,
                                                         const int* __restrict__ tile_cnt, int ntiles,
                                                         int32_t* __restrict__ idx) {
  __shared__ int wsum[kThreads / 32];
  const bool none = st->none;
  const uint32_t T = st->T;
  const int tsel = st->t;
  const int64_t base = (int64_t)blockIdx.x * kSelTile;
  const int64_t j0 = base + 32 * threadIdx.x;     // this thread's 32 consecutive classes, in id order
  uint32_t dm, tm;
  flags32(j0, C_local, bits, keys, none, T, dm, tm);
  int ttot;
  int trank = tile_cnt[2 * ntiles + blockIdx.x] + block_count_scan(__popc(tm), wsum, ttot);
  uint32_t sel = dm;
  while (tm) {                                    // ties are taken smallest id first (R3): rank < t
    const int i = __ffs(tm) - 1;
    tm &= tm - 1;
    if (trank < tsel) sel |= 1u << i;
    ++trank;
  }
  int stot;
  int pos = tile_cnt[3 * ntiles + blockIdx.x] + block_count_scan(__popc(sel), wsum, stot);
  while (sel) {
    const int i = __ffs(sel) - 1;
    sel &= sel - 1;
    idx[pos++] = (int32_t)(j0 + i);
  }
}

// All of K2-K4 in ONE cooperative kernel (the default; PFC_SAMPLER_FUSED=0: the seven kernels above): the same
// phases and arithmetic — so the same bit-exact selection — separated by grid-wide barriers instead of kernel
// boundaries; the 40 MB key array stays L2-resident between the phases, and the launch gaps and tails of seven
// kernels (plus three memsets) become six grid barriers. Each phase walks the classes (or 8192-class tiles) with a
// grid stride; per-block selection from the histograms is computed redundantly by every block, as before.
__global__ void __launch_bounds__(kThreads) k_sampler_fused(const int64_t* __restrict__ Y, int M, int64_t a,
                                                            int64_t C_local, uint64_t seed,
                                                            const uint64_t* __restrict__ step_dev, int64_t budget,
                                                            double rate, int mode, uint32_t* __restrict__ bits,
                                                            uint32_t* __restrict__ keys, int* __restrict__ hist,
                                                            int* __restrict__ tile_cnt, int ntiles, SamplerState* st,
                                                            int32_t* __restrict__ idx, int* err,
                                                            unsigned long long* trace) {
  namespace cg = cooperative_groups;
  int tp = 0;
  auto mark = [&]() {   // PFC_SAMPLER_TRACE=1: globaltimer at every phase boundary (block 0)
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[tp] = t;
    }
    ++tp;
  };
  mark();
  cg::grid_group grid = cg::this_grid();
  __shared__ int sh[2048];
  __shared__ int wsum[kThreads / 32];
  __shared__ int sdef, stie;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t nwords = (C_local + 31) / 32;
  // phase 0: zero the bitmap, the histograms and the state
  for (int64_t i = gtid; i < nwords; i += gthreads) bits[i] = 0u;
  for (int64_t i = gtid; i < 2048 + 2048 + 1024; i += gthreads) hist[i] = 0;
  if (gtid < (int64_t)(sizeof(SamplerState) / sizeof(int))) reinterpret_cast<int*>(st)[gtid] = 0;
  grid.sync();
  mark();
  // phase 1 (K2): positives
  if (mode != PFC_SAMPLE_RANDOM)
    for (int64_t n = gtid; n < M; n += gthreads) {
      const int64_t y = Y[n] - a;
      if (y >= 0 && y < C_local) {
        const uint32_t mask = 1u << (y & 31);
        const uint32_t old = atomicOr(&bits[y >> 5], mask);
        if (!(old & mask)) atomicAdd(&st->npos, 1);
      }
    }
  grid.sync();
  mark();
  // phase 2 (K3 pass 1): keys and the top-11-bit histogram of the non-positive classes
  {
    const uint32_t step = (uint32_t)*step_dev;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    int64_t j = gtid;
    for (; j + gthreads < C_local; j += 2 * gthreads) {
      const uint32_t h0 = philox_class_key((uint64_t)(a + j), step, seed);
      const uint32_t h1 = philox_class_key((uint64_t)(a + j + gthreads), step, seed);
      keys[j] = h0;
      keys[j + gthreads] = h1;
      if (!is_pos(bits, j)) atomicAdd(&sh[h0 >> 21], 1);
      if (!is_pos(bits, j + gthreads)) atomicAdd(&sh[h1 >> 21], 1);
    }
    if (j < C_local) {
      const uint32_t h = philox_class_key((uint64_t)(a + j), step, seed);
      keys[j] = h;
      if (!is_pos(bits, j)) atomicAdd(&sh[h >> 21], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
      if (sh[i]) atomicAdd(&hist[i], sh[i]);
  }
  grid.sync();
  mark();
  // phase 3 (K3 pass 2): k_i, n_i; the first digit; histogram of the second inside its bucket
  const int npos = st->npos;
  const int kk = budget_k(npos, budget, C_local, rate, mode);
  const int n_neg = kk - npos;
  const bool none = n_neg == 0;
  int b1 = 0, rem1 = 0;
  if (!none) {
    block_select(hist, 2048, n_neg, b1, rem1);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    // four coalesced 16-byte key loads in flight per thread (the L2-resident key array, padded to whole tiles)
    const int64_t s4 = gthreads * 4;
    for (int64_t base = gtid * 4; base < C_local; base += 4 * s4) {
      uint4 h4[4];
      uint32_t pw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j0 = base + u * s4;
        if (j0 < C_local) {
          h4[u] = *reinterpret_cast<const uint4*>(keys + j0);
          pw[u] = __ldg(&bits[j0 >> 5]) >> (j0 & 31);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j0 = base + u * s4;
        if (j0 >= C_local) break;
        const uint32_t hh[4] = {h4[u].x, h4[u].y, h4[u].z, h4[u].w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if ((hh[i] >> 21) == (uint32_t)b1 && !((pw[u] >> i) & 1u) && j0 + i < C_local)
            atomicAdd(&sh[(hh[i] >> 10) & 0x7FF], 1);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
      if (sh[i]) atomicAdd(&hist[2048 + i], sh[i]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->k = kk; st->n_neg = n_neg; st->none = none ? 1 : 0; st->prefix1 = (uint32_t)b1; st->rem1 = rem1;
  }
  grid.sync();
  mark();
  // phase 4 (K3 pass 3): the second digit; histogram of the last 10 bits
  uint32_t pre = 0;
  int rem2 = 0;
  if (!none) {
    int b2;
    block_select(hist + 2048, 2048, rem1, b2, rem2);
    pre = ((uint32_t)b1 << 11) | (uint32_t)b2;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t s4 = gthreads * 4;
    for (int64_t base = gtid * 4; base < C_local; base += 4 * s4) {
      uint4 h4[4];
      uint32_t pw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j0 = base + u * s4;
        if (j0 < C_local) {
          h4[u] = *reinterpret_cast<const uint4*>(keys + j0);
          pw[u] = __ldg(&bits[j0 >> 5]) >> (j0 & 31);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j0 = base + u * s4;
        if (j0 >= C_local) break;
        const uint32_t hh[4] = {h4[u].x, h4[u].y, h4[u].z, h4[u].w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if ((hh[i] >> 10) == pre && !((pw[u] >> i) & 1u) && j0 + i < C_local) atomicAdd(&sh[hh[i] & 0x3FF], 1);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += blockDim.x)
      if (sh[i]) atomicAdd(&hist[4096 + i], sh[i]);
    if (blockIdx.x == 0 && threadIdx.x == 0) { st->prefix2 = pre; st->rem2 = rem2; }
  }
  grid.sync();
  mark();
  // phase 5 (K4a): the threshold key T and t; definite / tied counts per 8192-class tile
  uint32_t T = 0;
  int tsel = 0;
  if (!none) {
    int b3;
    block_select(hist + 4096, 1024, rem2, b3, tsel);
    T = (pre << 10) | (uint32_t)b3;
    if (blockIdx.x == 0 && threadIdx.x == 0) { st->T = T; st->t = tsel; }
  }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    uint32_t dm, tm;
    flags32((int64_t)tile * kSelTile + 32 * threadIdx.x, C_local, bits, keys, none, T, dm, tm);
    int ndef = __popc(dm), ntie = __popc(tm);
    if (threadIdx.x == 0) { sdef = 0; stie = 0; }
    __syncthreads();
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      ndef += __shfl_xor_sync(0xffffffffu, ndef, o);
      ntie += __shfl_xor_sync(0xffffffffu, ntie, o);
    }
    if ((threadIdx.x & 31) == 0) { atomicAdd(&sdef, ndef); atomicAdd(&stie, ntie); }
    __syncthreads();
    if (threadIdx.x == 0) {
      tile_cnt[tile] = sdef;
      tile_cnt[ntiles + tile] = stie;
    }
    __syncthreads();
  }
  grid.sync();
  mark();
  // phase 6 (K4b): exclusive scans of the tile counts (block 0)
  if (blockIdx.x == 0) {
    int* def = tile_cnt;
    int* tie = tile_cnt + ntiles;
    int* tie_off = tile_cnt + 2 * ntiles;
    int* sel_off = tile_cnt + 3 * ntiles;
    // thread t scans the contiguous tiles [t cpt, (t + 1) cpt) serially around ONE block scan per pass
    const int cpt = (ntiles + kThreads - 1) / kThreads;
    const int i0 = min(ntiles, threadIdx.x * cpt), i1 = min(ntiles, i0 + cpt);
    for (int pass = 0; pass < 2; ++pass) {
      auto val = [&](int i) {
        return pass == 0 ? tie[i] : def[i] + (none ? 0 : max(0, min(tsel - tie_off[i], tie[i])));
      };
      int local = 0;
      for (int i = i0; i < i1; ++i) local += val(i);
      int tot;
      int run = block_count_scan(local, wsum, tot);
      for (int i = i0; i < i1; ++i) {
        const int v = val(i);
        (pass == 0 ? tie_off : sel_off)[i] = run;
        run += v;
      }
      if (pass == 1 && threadIdx.x == 0) {
        st->total = tot;
        if (tot != kk) atomicOr(err, ERR_INTERNAL);
      }
      __syncthreads();
    }
  }
  grid.sync();
  mark();
  // phase 7 (K4c): order-preserving write of the selected local ids
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t j0 = (int64_t)tile * kSelTile + 32 * threadIdx.x;
    uint32_t dm, tm;
    flags32(j0, C_local, bits, keys, none, T, dm, tm);
    int ttot;
    int trank = tile_cnt[2 * ntiles + tile] + block_count_scan(__popc(tm), wsum, ttot);
    uint32_t sel = dm;
    while (tm) {                                    // ties are taken smallest id first (R3): rank < t
      const int i = __ffs(tm) - 1;
      tm &= tm - 1;
      if (trank < tsel) sel |= 1u << i;
      ++trank;
    }
    int stot;
    int pos = tile_cnt[3 * ntiles + tile] + block_count_scan(__popc(sel), wsum, stot);
    while (sel) {
      const int i = __ffs(sel) - 1;
      sel &= sel - 1;
      idx[pos++] = (int32_t)(j0 + i);
    }
    __syncthreads();
  }
  grid.sync();
  mark();
}

}  // namespace

int launch_sampler(const Sizes& sz, const int64_t* Y, uint64_t seed, const uint64_t* step, uint32_t* bits, uint32_t* keys,
                   int* hist, int* tile_cnt, SamplerState* st, int32_t* idx, int32_t* tcol, int* err,
                   cudaStream_t s) {
  const bool fused = env_int("PFC_SAMPLER_FUSED", 1) != 0;
  if (fused) {
    static int per_sm = 0;
    if (!per_sm) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sampler_fused, kThreads, 0);
      per_sm = std::max(1, std::min(per_sm, 4));
    }
    // all blocks co-resident (cooperative launch: a guarantee, or a loud launch failure)
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((sz.C_local + kThreads - 1) / kThreads,
                                                                 (int64_t)per_sm * num_sms_host()));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kThreads);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    static unsigned long long* trace = nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    const bool tracing = env_int("PFC_SAMPLER_TRACE", 0) != 0 && cs == cudaStreamCaptureStatusNone;
    if (tracing && !trace) cudaMalloc(&trace, 64 * sizeof(unsigned long long));
    cudaLaunchKernelEx(&lc, k_sampler_fused, Y, sz.M, sz.a, sz.C_local, seed, step, sz.budget, sz.rate,
                       sz.sample_mode, bits, keys, hist, tile_cnt, sz.ntiles_sel, st, idx, err,
                       tracing ? trace : (unsigned long long*)nullptr);
    if (tracing) {
      unsigned long long h[16] = {0};
      cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      std::fprintf(stderr, "sampler phases (us):");
      for (int i = 1; i < 10 && h[i]; ++i) std::fprintf(stderr, " %.1f", (h[i] - h[i - 1]) / 1e3);
      std::fprintf(stderr, "  grid=%d\n", grid);
    }
    (void)tcol;
    return 1;
  }
  const int64_t nwords = (sz.C_local + 31) / 32;
  cudaMemsetAsync(bits, 0, nwords * sizeof(uint32_t), s);
  cudaMemsetAsync(hist, 0, (2048 + 2048 + 1024) * sizeof(int), s);
  cudaMemsetAsync(st, 0, sizeof(SamplerState), s);
  k_mark_positives<<<(sz.M + 255) / 256, 256, 0, s>>>(Y, sz.M, sz.a, sz.C_local, bits, st, sz.sample_mode);
  int grid = (int)std::min<int64_t>((sz.C_local + kThreads - 1) / kThreads, 148 * 8);
  k_keys_hist<<<grid, kThreads, 0, s>>>(sz.a, sz.C_local, seed, step, bits, keys, hist);
  k_hist_pass2<<<grid, kThreads, 0, s>>>(sz.C_local, sz.budget, sz.rate, sz.sample_mode, bits, keys, hist, st,
                                         hist + 2048);
  k_hist_pass3<<<grid, kThreads, 0, s>>>(sz.C_local, bits, keys, hist + 2048, st, hist + 4096);
  k_tile_counts<<<sz.ntiles_sel, kThreads, 0, s>>>(sz.C_local, bits, keys, hist + 4096, st, tile_cnt, sz.ntiles_sel);
  k_tile_scan<<<1, 1024, 0, s>>>(tile_cnt, sz.ntiles_sel, st, err);
  k_tile_write<<<sz.ntiles_sel, kThreads, 0, s>>>(sz.C_local, bits, keys, st, tile_cnt, sz.ntiles_sel, idx);
  (void)tcol;   // tcol is filled by the target-cosine kernel (binary search in idx)
  return 7;
}

}  // namespace pfc
