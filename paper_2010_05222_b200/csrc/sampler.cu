// PPRN sampler on one shard (steps 1-3 and Eq.10), bit-exact selection recipe of
// DESIGN.md §Sampler:
//   K2  mark_positives : bitmap of labels in [a, a + C_local) and |P_i| (step 1, dedup R5)
//   K3  keys + radix select : h_j = Philox key of every non-positive class (R2); three histogram passes
//       (11/11/10 bits) find the threshold key T of the n_i-th smallest (h, j) and t, the number of
//       tied (h == T) negatives to take, smallest ids first (R3)
//   K4  compaction : idx_i = ascending ids of (positive or selected) via tile counts + scan + write (R4);
//       tcol[n] = position of y_n in idx_i (binary search) or -1 when y_n is not in this shard.
// Everything is device-resident (k_i is data-dependent); no host synchronisation.
#include <algorithm>
#include "pfc_internal.cuh"

namespace pfc {
namespace {

constexpr int kThreads = 256;

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
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < C_local; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = philox_class_key((uint64_t)(a + j), step, seed);
    keys[j] = h;
    if (!is_pos(bits, j)) atomicAdd(&sh[h >> 21], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Passes 2 and 3: histogram of the next digit among keys whose higher digits equal the prefix.
__global__ void __launch_bounds__(kThreads) k_hist_pass(int64_t C_local, const uint32_t* __restrict__ bits,
                                                        const uint32_t* __restrict__ keys, const SamplerState* st,
                                                        int hi_shift, int lo_shift, uint32_t lo_mask,
                                                        int* __restrict__ hist) {
  __shared__ int sh[2048];
  if (st->none) return;
  const uint32_t prefix = st->prefix;
  for (int i = threadIdx.x; i <= (int)lo_mask; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < C_local; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = keys[j];
    if ((h >> hi_shift) == prefix && !is_pos(bits, j)) atomicAdd(&sh[(h >> lo_shift) & lo_mask], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= (int)lo_mask; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// Single block: locate the bucket holding the `remaining`-th smallest key of this pass.
// pass 0 also computes k_i and n_i from |P_i| (R1).
__global__ void __launch_bounds__(1024) k_select_bucket(const int* __restrict__ hist, int nbins, int pass,
                                                        int64_t budget, int64_t C_local, double rate, int mode,
                                                        SamplerState* st) {
  __shared__ int scan[1024];
  __shared__ int found;
  if (pass == 0) {
    if (threadIdx.x == 0) {
      int k;
      if (mode == PFC_SAMPLE_PPRN_PAPER) {   // R23: |P_i| + round_half_up((C_local - |P_i|) r)
        const int64_t rest = C_local - st->npos;
        int64_t n = (int64_t)floor((double)rest * rate + 0.5);
        n = n < 0 ? 0 : (n > rest ? rest : n);
        k = st->npos + (int)n;
      } else if (mode == PFC_SAMPLE_RANDOM) {
        k = (int)budget;
      } else {
        k = (int)max(budget, (int64_t)st->npos);   // R1
      }
      st->k = k;
      st->n_neg = k - st->npos;
      st->none = (st->n_neg == 0);
      st->remaining = st->n_neg;
      st->prefix = 0;
    }
    __syncthreads();
  }
  if (st->none) return;
  const int need = st->remaining;
  // each thread owns a contiguous chunk of bins
  const int per = (nbins + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  int local = 0;
  for (int b = b0; b < min(nbins, b0 + per); ++b) local += hist[b];
  scan[threadIdx.x] = local;
  if (threadIdx.x == 0) found = 0;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // inclusive Hillis-Steele scan
    int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  int before = scan[threadIdx.x] - local;
  if (before < need && need <= scan[threadIdx.x]) {
    int cum = before;
    for (int b = b0; b < min(nbins, b0 + per); ++b) {
      int h = hist[b];
      if (cum < need && need <= cum + h) {
        const int bits_of_pass = (pass == 2) ? 10 : 11;
        st->prefix = (st->prefix << bits_of_pass) | (uint32_t)b;
        st->remaining = need - cum;
        found = 1;
        break;
      }
      cum += h;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (pass == 2) {
      st->T = st->prefix;
      st->t = st->remaining;
    }
  }
}

// Block-wide exclusive scan of a 0/1 flag over 256 threads (8 warps); returns the prefix and the total.
__device__ __forceinline__ int block_flag_scan(bool f, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(0xffffffffu, f);
  const int wpre = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[w] = __popc(bal);
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) {
    int v = warp_tot[i];
    pre += (i < w) ? v : 0;
    tot += v;
  }
  __syncthreads();
  total = tot;
  return pre + wpre;
}

__device__ __forceinline__ void flags_of(int64_t j, int64_t C_local, const uint32_t* bits, const uint32_t* keys,
                                         const SamplerState& s, bool& def, bool& tie) {
  def = false; tie = false;
  if (j >= C_local) return;
  if (is_pos(bits, j)) { def = true; return; }
  if (s.none) return;
  uint32_t h = keys[j];
  def = h < s.T;
  tie = h == s.T;
}

// K4a: per-tile counts of definitely-selected and tied classes.
__global__ void __launch_bounds__(kThreads) k_tile_counts(int64_t C_local, const uint32_t* __restrict__ bits,
                                                          const uint32_t* __restrict__ keys, const SamplerState* st,
                                                          int* __restrict__ tile_cnt, int ntiles) {
  const SamplerState s = *st;
  const int64_t base = (int64_t)blockIdx.x * kSelTile;
  int ndef = 0, ntie = 0;
  for (int i = 0; i < kSelTile / kThreads; ++i) {
    bool d, t;
    flags_of(base + i * kThreads + threadIdx.x, C_local, bits, keys, s, d, t);
    ndef += d; ntie += t;
  }
  __shared__ int sdef, stie;
  if (threadIdx.x == 0) { sdef = 0; stie = 0; }
  __syncthreads();
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

// K4b: single block. Exclusive scans: tie offsets, then selected counts (definite + ties ranked < t).
__global__ void __launch_bounds__(1024) k_tile_scan(int* __restrict__ tile_cnt, int ntiles, SamplerState* st,
                                                    int* err) {
  __shared__ int scan[1024];
  __shared__ int carry;
  const SamplerState s = *st;
  int* def = tile_cnt;
  int* tie = tile_cnt + ntiles;
  int* tie_off = tile_cnt + 2 * ntiles;
  int* sel_off = tile_cnt + 3 * ntiles;
  for (int pass = 0; pass < 2; ++pass) {
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < ntiles; base += blockDim.x) {
      int i = base + threadIdx.x;
      int v = 0;
      if (i < ntiles) {
        if (pass == 0) v = tie[i];
        else v = def[i] + (s.none ? 0 : max(0, min(s.t - tie_off[i], tie[i])));
      }
      scan[threadIdx.x] = v;
      __syncthreads();
      for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        int u = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
        __syncthreads();
        scan[threadIdx.x] += u;
        __syncthreads();
      }
      if (i < ntiles) (pass == 0 ? tie_off : sel_off)[i] = carry + scan[threadIdx.x] - v;
      __syncthreads();
      if (threadIdx.x == blockDim.x - 1) carry += scan[threadIdx.x];
      __syncthreads();
    }
    if (pass == 1 && threadIdx.x == 0) {
      st->total = carry;
      if (carry != s.k) atomicOr(err, ERR_INTERNAL);
    }
    __syncthreads();
  }
}

// K4c: order-preserving write of the selected local ids.
__global__ void __launch_bounds__(kThreads) k_tile_write(int64_t C_local, const uint32_t* __restrict__ bits,
                                                         const uint32_t* __restrict__ keys, const SamplerState* st,
                                                         const int* __restrict__ tile_cnt, int ntiles,
                                                         int32_t* __restrict__ idx) {
  __shared__ int wt[kThreads / 32];
  const SamplerState s = *st;
  const int64_t base = (int64_t)blockIdx.x * kSelTile;
  int tie_run = tile_cnt[2 * ntiles + blockIdx.x];
  int out_run = tile_cnt[3 * ntiles + blockIdx.x];
  for (int i = 0; i < kSelTile / kThreads; ++i) {
    const int64_t j = base + i * kThreads + threadIdx.x;
    bool d, t;
    flags_of(j, C_local, bits, keys, s, d, t);
    int ntie;
    int tie_rank = tie_run + block_flag_scan(t, wt, ntie);
    bool sel = d || (t && tie_rank < s.t);
    int nsel;
    int pos = out_run + block_flag_scan(sel, wt, nsel);
    if (sel) idx[pos] = (int32_t)j;
    tie_run += ntie;
    out_run += nsel;
  }
}

__global__ void k_tcol(const int64_t* __restrict__ Y, int M, int64_t a, int64_t C_local,
                       const int32_t* __restrict__ idx, const SamplerState* st, int32_t* __restrict__ tcol) {
  int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= M) return;
  int64_t y = Y[n] - a;
  int res = -1;
  if (y >= 0 && y < C_local) {
    int lo = 0, hi = st->k - 1;
    while (lo <= hi) {
      int mid = (lo + hi) >> 1;
      int v = idx[mid];
      if (v == y) { res = mid; break; }
      if (v < y) lo = mid + 1; else hi = mid - 1;
    }
  }
  tcol[n] = res;
}

}  // namespace

int launch_sampler(const Sizes& sz, const int64_t* Y, uint64_t seed, const uint64_t* step, uint32_t* bits, uint32_t* keys,
                   int* hist, int* tile_cnt, SamplerState* st, int32_t* idx, int32_t* tcol, int* err,
                   cudaStream_t s) {
  const int64_t nwords = (sz.C_local + 31) / 32;
  cudaMemsetAsync(bits, 0, nwords * sizeof(uint32_t), s);
  cudaMemsetAsync(hist, 0, (2048 + 2048 + 1024) * sizeof(int), s);
  cudaMemsetAsync(st, 0, sizeof(SamplerState), s);
  k_mark_positives<<<(sz.M + 255) / 256, 256, 0, s>>>(Y, sz.M, sz.a, sz.C_local, bits, st, sz.sample_mode);
  int grid = (int)std::min<int64_t>((sz.C_local + kThreads - 1) / kThreads, 148 * 8);
  k_keys_hist<<<grid, kThreads, 0, s>>>(sz.a, sz.C_local, seed, step, bits, keys, hist);
  k_select_bucket<<<1, 1024, 0, s>>>(hist, 2048, 0, sz.budget, sz.C_local, sz.rate, sz.sample_mode, st);
  k_hist_pass<<<grid, kThreads, 0, s>>>(sz.C_local, bits, keys, st, 21, 10, 0x7FFu, hist + 2048);
  k_select_bucket<<<1, 1024, 0, s>>>(hist + 2048, 2048, 1, sz.budget, sz.C_local, sz.rate, sz.sample_mode, st);
  k_hist_pass<<<grid, kThreads, 0, s>>>(sz.C_local, bits, keys, st, 10, 0, 0x3FFu, hist + 4096);
  k_select_bucket<<<1, 1024, 0, s>>>(hist + 4096, 1024, 2, sz.budget, sz.C_local, sz.rate, sz.sample_mode, st);
  k_tile_counts<<<sz.ntiles_sel, kThreads, 0, s>>>(sz.C_local, bits, keys, st, tile_cnt, sz.ntiles_sel);
  k_tile_scan<<<1, 1024, 0, s>>>(tile_cnt, sz.ntiles_sel, st, err);
  k_tile_write<<<sz.ntiles_sel, kThreads, 0, s>>>(sz.C_local, bits, keys, st, tile_cnt, sz.ntiles_sel, idx);
  k_tcol<<<(sz.M + 255) / 256, 256, 0, s>>>(Y, sz.M, sz.a, sz.C_local, idx, st, tcol);
  return 11;
}

}  // namespace pfc
