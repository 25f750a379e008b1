// HBM probe for the access pattern of the lazy momentum-SGD update: read-modify-write of the W and V
// rows (fp32, d = 512) of a sorted 10% sample of C = 10M classes, against the same RMW over contiguous rows and a
// plain copy. Answers "what does HBM deliver for THIS pattern" — the ceiling k_dwx_t's update stream can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rmw_probe scripts/rmw_probe.cu && ./rmw_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1); } } while (0)

constexpr int D = 512;

// one warp per (row, seg) unit; seg = 128 columns (512 B) or the whole row (2 KB); ROWS rows in flight per warp
template <int SEG, int ROWS>
__global__ void __launch_bounds__(256) k_rmw(float* __restrict__ W, float* __restrict__ V, const int32_t* __restrict__ idx,
                                             int64_t k, float lr, float mu, float lam) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int NSEG = D / SEG;
  constexpr int V4 = SEG / 128;        // float4 per lane per row
  const int64_t units = k * NSEG;      // (row, seg), the seg index fastest: the segments of a row in adjacent warps
  for (int64_t u0 = warp * ROWS; u0 < units; u0 += nwarps * ROWS) {
    float4 w[ROWS][V4], m[ROWS][V4];
    int64_t off[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const int64_t u = u0 + r;
      off[r] = -1;
      if (u < units) off[r] = (int64_t)idx[u / NSEG] * D + (u % NSEG) * SEG + lane * 4;
#pragma unroll
      for (int q = 0; q < V4; ++q)
        if (off[r] >= 0) {
          w[r][q] = *reinterpret_cast<const float4*>(W + off[r] + q * 128);
          m[r][q] = *reinterpret_cast<const float4*>(V + off[r] + q * 128);
        }
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
      for (int q = 0; q < V4; ++q)
        if (off[r] >= 0) {
          float4 a = w[r][q], b = m[r][q];
          b.x = mu * b.x + 0.01f * a.x + lam * a.x; b.y = mu * b.y + 0.01f * a.y + lam * a.y;
          b.z = mu * b.z + 0.01f * a.z + lam * a.z; b.w = mu * b.w + 0.01f * a.w + lam * a.w;
          a.x -= lr * b.x; a.y -= lr * b.y; a.z -= lr * b.z; a.w -= lr * b.w;
          *reinterpret_cast<float4*>(W + off[r] + q * 128) = a;
          *reinterpret_cast<float4*>(V + off[r] + q * 128) = b;
        }
  }
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <class F>
float time_ms(F f, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  return best;
}

int main() {
  const int64_t C = 10000000, k = 1000000;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *W, *V;
  CK(cudaMalloc(&W, C * D * sizeof(float)));
  CK(cudaMalloc(&V, C * D * sizeof(float)));
  CK(cudaMemset(W, 0, C * D * sizeof(float)));
  CK(cudaMemset(V, 0, C * D * sizeof(float)));
  // sorted 10% sample (each row kept with probability k / C, topped up to exactly k), and the contiguous rows 0..k-1
  std::vector<int32_t> hs, hc(k);
  srand(7);
  for (int64_t j = 0; j < C && (int64_t)hs.size() < k; ++j)
    if ((rand() % 10) == 0 || C - j <= k - (int64_t)hs.size()) hs.push_back((int32_t)j);
  for (int64_t j = 0; j < k; ++j) hc[j] = (int32_t)j;
  int32_t *is, *ic;
  CK(cudaMalloc(&is, k * 4));
  CK(cudaMalloc(&ic, k * 4));
  CK(cudaMemcpy(is, hs.data(), k * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ic, hc.data(), k * 4, cudaMemcpyHostToDevice));
  const double bytes = (double)k * D * 16;   // W and V read + written
  const int grid = sms * 8;
  auto report = [&](const char* name, float ms) {
    std::printf("%-44s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  report("sampled rows, 512 B segments, 4 rows/warp", time_ms([&] { k_rmw<128, 4><<<grid, 256>>>(W, V, is, k, 0.1f, 0.9f, 5e-4f); }));
  report("sampled rows, 512 B segments, 8 rows/warp", time_ms([&] { k_rmw<128, 8><<<grid, 256>>>(W, V, is, k, 0.1f, 0.9f, 5e-4f); }));
  report("sampled rows, 2 KB rows, 2 rows/warp", time_ms([&] { k_rmw<512, 2><<<grid, 256>>>(W, V, is, k, 0.1f, 0.9f, 5e-4f); }));
  report("sampled rows, 2 KB rows, 4 rows/warp", time_ms([&] { k_rmw<512, 4><<<grid, 256>>>(W, V, is, k, 0.1f, 0.9f, 5e-4f); }));
  report("contiguous rows, 512 B segments, 8 rows/warp", time_ms([&] { k_rmw<128, 8><<<grid, 256>>>(W, V, ic, k, 0.1f, 0.9f, 5e-4f); }));
  report("contiguous rows, 2 KB rows, 4 rows/warp", time_ms([&] { k_rmw<512, 4><<<grid, 256>>>(W, V, ic, k, 0.1f, 0.9f, 5e-4f); }));
  // in-flight scaling at the dwx_t shape: one 256-thread CTA (8 warps) per SM, R rows of 512 B in flight per warp
  for (int bps : {1, 2, 4}) {
    char name[96];
    std::snprintf(name, sizeof(name), "sampled 512 B, %d CTA/SM, 8 rows/warp", bps);
    report(name, time_ms([&] { k_rmw<128, 8><<<sms * bps, 256>>>(W, V, is, k, 0.1f, 0.9f, 5e-4f); }));
    std::snprintf(name, sizeof(name), "sampled 512 B, %d CTA/SM, 16 rows/warp", bps);
    report(name, time_ms([&] { k_rmw<128, 16><<<sms * bps, 256>>>(W, V, is, k, 0.1f, 0.9f, 5e-4f); }));
  }
  // plain copy of the same byte count (8 GB moved: 4 GB read + 4 GB written)
  const int64_t n4 = (int64_t)(bytes / 2 / 16);
  const float ms = time_ms([&] { k_copy<<<grid, 256>>>(reinterpret_cast<const float4*>(W), reinterpret_cast<float4*>(V), n4); });
  report("copy (same bytes)", ms);
  return 0;
}
