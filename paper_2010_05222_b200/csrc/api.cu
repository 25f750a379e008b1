// C-ABI (include/pfc.h) and the stream-ordered step orchestrator.
//
// Per pfc_forward_backward on rank i (all on the caller's stream, no host sync):
//   K1 normalize_x -> [NCCL all-gather X_hat, Y] -> K1b X_hat->bf16 -> K2..K4 sampler -> K5 gather W_s
//   -> K5b target cos -> K6 logits GEMM (+margin, scale, per-tile max/sum-exp) -> K7 row combine
//   -> [NCCL all-reduce MAX] -> prep -> [NCCL all-reduce SUM] -> finalize (LSE, loss)
//   -> K8 softmax grad -> K9 dX GEMM -> [NCCL reduce-scatter] -> K10 x-norm backward -> K11 dW GEMM
// pfc_step: K12 lazy momentum SGD on the sampled rows.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <array>
#include <chrono>
#include <thread>
#include <vector>

#include "pfc_internal.cuh"

using namespace pfc;

static thread_local std::string g_init_error;

struct pfc_ctx {
  pfc_config cfg{};
  Sizes sz{};
  MarginParams mp{};
  bool bf16 = false;
  bool use_tc = false;
  bool fused_gather = false;   // K5 + K6 in one kernel (M <= 256); G carries 1/||w|| (R25)
  bool use_dwx = false;        // train step: K9 + K11 + K12 in one kernel (dwx.cu), no W_s copy
  bool sync_check = false;
  std::string err;
  ncclComm_t comm = nullptr;
  cudaStream_t side = nullptr;                    // multi-rank: dX exchange overlapping the dW kernel
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool nccl_solo = false;      // PFC_NCCL_SOLO=1 at world size 1: run the NCCL collectives on a 1-rank communicator
  // collectives fused into the kernels: PFC_COMM_NCCL_FUSED (NCCL device-API symmetric window,
  // LSA barriers) or PFC_COMM_LOOPBACK_FUSED (the loopback group's contexts writing into each other's regions)
  bool fused_nccl = false;
  FusedNccl* fnccl = nullptr;
  char* sym = nullptr;         // this rank's exchange region (pfc_internal.cuh SymLayout); X32 and Y live in it
  Peers peers{};
  const Peers* P() const { return peers.n ? &peers : nullptr; }
  uint64_t step = 0;
  bool fb_done = false;      // a forward_backward happened and its gradient was not yet applied
  cudaStream_t last_stream = nullptr;
  int64_t launches = 0;
  std::vector<void*> allocs;
  std::vector<void*> host_allocs;   // PFC_PARAMS_HOST: page-locked, device-mapped W and V
  float* W_host = nullptr;          // host addresses of W / V in that mode (c->W / c->V are the device mapping)
  // PFC_PARAMS_HOST with staging (default; PFC_HOST_STAGE=0: zero-copy in every kernel): the
  // sampled rows are gathered once into HBM (Wst / Vst, k_pad x d, by position), every kernel works on them with
  // the identity index idx_id, and the updated rows are scattered back into the host shard at the end of the step
  bool stage = false;
  float* Wst = nullptr;
  float* Vst = nullptr;
  int32_t* idx_id = nullptr;
  // what the W / V consumers address: (W, V, idx) in HBM mode, (Wst, Vst, idx_id) when staging
  float* Wk() const { return stage ? Wst : W; }
  float* Vk() const { return stage ? Vst : V; }
  const int32_t* idxk() const { return stage ? idx_id : idx; }
  float* V_host = nullptr;

  // parameters
  float* W = nullptr;
  float* V = nullptr;
  // features / labels
  float* xh_local = nullptr;   // B x d
  float* xnorm = nullptr;      // B
  float* X32 = nullptr;        // M_pad x d (all-gathered x_hat)
  int64_t* Y = nullptr;        // M
  __nv_bfloat16* Xb = nullptr; // M_pad x d
  __half* Xh16 = nullptr;      // M_pad x d fp16: the logits operand (bf16 mode, R27)
  // sampler
  uint32_t* bits = nullptr;
  uint32_t* keys = nullptr;
  int* hist = nullptr;
  int* tile_cnt = nullptr;
  SamplerState* st = nullptr;
  int32_t* idx = nullptr;      // k_pad
  int32_t* tcol = nullptr;     // M
  // sampled centres
  void* Ws = nullptr;          // k_pad x d (bf16 or fp32)
  __half* Ws16 = nullptr;      // k_pad x d fp16 copy: the logits operand of the unfused-gather tcgen05 paths (R27)
  float* inv_norm = nullptr;   // k_pad
  float* ct = nullptr;         // M
  // logits and softmax
  void* cosv = nullptr;        // M x k_pad (fp16 or fp32)
  float2* partials = nullptr;  // M x n_ltiles
  float* rowmax = nullptr;     // M
  float* gmax = nullptr;       // M
  float* rowsum = nullptr;     // M
  float* zt = nullptr;         // M
  float* red = nullptr;        // M + 1
  float* lse = nullptr;        // M
  float* gt = nullptr;         // M, p_t - 1 per row
  float* metrics = nullptr;    // {loss, CA_pcc} of the last step
  float* loss_dev = nullptr;   // 1 (scratch when the caller passes NULL)
  void* G = nullptr;           // M x k_pad (bf16 or fp32)
  // gradients
  float* dXh = nullptr;        // M x d
  float* dxh_local = nullptr;  // B x d (reduce-scatter output)
  float* split_ws = nullptr;   // split-K partials of the dx GEMM
  float* dWh = nullptr;        // k_pad x d
  float* dotw = nullptr;       // k_pad: w_hat . dW_hat per sampled class (fused SGD)
  // E-form train step (DESIGN.md f1; use_dwx): cosv holds E = e^{s c} (bf16), no softmax-gradient pass
  bool eform = false;                // M <= 256: inside the fused dW + SGD + dX kernel
  bool eform_pair = false;           // M > 256: CTA-pair logits store E, radial dots by k_eform_dotw, dX / dW on E
  float* ef_f = nullptr;             // M_pad: f_n = (s/M) e^{-LSE_n}
  __nv_bfloat16* Xt = nullptr;       // M_pad x d: bf16(f_n x_hat_n)
  float* dcorr = nullptr;            // k_pad: sum of G_t c_t over each class's target entries
  float* xch = nullptr;              // k_pad x (d/128): radial-dot partials
  float* xws = nullptr;              // dwxdot.cu: half-dots + flags of the partner pairs (M >= 2048, d = 512)
  int* cnt = nullptr;                // k_pad/128
  int* err_dev = nullptr;
  int* err_host = nullptr;           // page-locked mirror of err_dev written by the step's last kernel
  int* err_host_dev = nullptr;       // its device mapping
  // host-buffer entry point
  float* x_in = nullptr;
  int64_t* y_in = nullptr;
  float* gx_out = nullptr;
  // device-resident step counter and learning rate (the step is CUDA-graph replayable)
  uint64_t* step_dev = nullptr;
  float* lr_dev = nullptr;
  bool graph_on = true;
  int graph_warm = 0;
  int64_t graph_launches = 0;     // kernels inside one captured step
  struct GraphEntry {
    const void *x, *y, *gx, *loss;
    cudaStream_t s;
    bool fused;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  // per-kernel event timing (pfc_profile_*)
  bool prof = false;
  std::vector<std::array<cudaEvent_t, PFC_PROF_SECTIONS + 1>> prof_ev;
  std::vector<std::array<bool, PFC_PROF_SECTIONS + 1>> prof_set;
  size_t prof_used = 0;
  std::array<cudaEvent_t, PFC_PROF_SECTIONS + 1>* prof_cur = nullptr;
  std::array<bool, PFC_PROF_SECTIONS + 1>* prof_cur_set = nullptr;
};

namespace {

pfc_status set_err(pfc_ctx* c, pfc_status s, const std::string& msg) {
  if (c) c->err = msg; else g_init_error = msg;
  return s;
}

#define CUDA_TRY(ctx, expr)                                                                          \
  do {                                                                                               \
    cudaError_t e_ = (expr);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      return set_err(ctx, e_ == cudaErrorMemoryAllocation ? PFC_ERR_OOM : PFC_ERR_CUDA,              \
                     std::string(#expr) + ": " + cudaGetErrorString(e_));                            \
  } while (0)

#define NCCL_TRY(ctx, expr)                                                                          \
  do {                                                                                               \
    ncclResult_t r_ = (expr);                                                                        \
    if (r_ != ncclSuccess) return set_err(ctx, PFC_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

template <typename T>
pfc_status dalloc(pfc_ctx* c, T** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(bytes, 16));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(c, PFC_ERR_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
  }
  c->allocs.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return PFC_OK;
}

pfc_status decode_error(pfc_ctx* c, int h) {
  if (h & ERR_DATA) return set_err(c, PFC_ERR_DATA, "a label is outside [0, num_classes)");
  if (h & ERR_DEGENERATE) return set_err(c, PFC_ERR_DEGENERATE, "a feature or class-centre row has zero norm");
  if (h & ERR_NUMERIC) return set_err(c, PFC_ERR_NUMERIC, "non-finite loss");
  return set_err(c, PFC_ERR_CUDA, "internal consistency check failed (sampler count != k_i, or a radial-dot exchange timed out)");
}

// NCCL: a failed or hung peer surfaces as an asynchronous communicator error; poll it while waiting for the stream
// and abort the communicator on error or after PFC_NCCL_TIMEOUT_S seconds (default 600), so that no call blocks
// forever on a dead rank (SURVEY.md §5 failure detection).
pfc_status wait_stream(pfc_ctx* c, cudaStream_t s) {
  if (!c->comm) {
    CUDA_TRY(c, cudaStreamSynchronize(s));
    return PFC_OK;
  }
  static const double timeout_s = [] { const char* e = std::getenv("PFC_NCCL_TIMEOUT_S"); return e ? std::atof(e) : 600.0; }();
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) CUDA_TRY(c, q);
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(c->comm, &ar);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ar != ncclSuccess && ar != ncclInProgress) || el > timeout_s) {
      std::string m = ar != ncclSuccess ? std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar)
                                        : "collective did not complete within PFC_NCCL_TIMEOUT_S";
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      return set_err(c, PFC_ERR_NCCL, m + " (communicator aborted)");
    }
    if (el > 2e-3) std::this_thread::sleep_for(std::chrono::microseconds(50));   // spin for the first 2 ms
  }
  ncclResult_t ar = ncclSuccess;
  ncclCommGetAsyncError(c->comm, &ar);
  if (ar != ncclSuccess && ar != ncclInProgress) return set_err(c, PFC_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
  return PFC_OK;
}

pfc_status device_error(pfc_ctx* c) {
  int h = 0;
  CUDA_TRY(c, cudaMemcpy(&h, c->err_dev, sizeof(int), cudaMemcpyDeviceToHost));
  if (c->err_host) *(volatile int*)c->err_host = 0;
  if (!h) return PFC_OK;
  CUDA_TRY(c, cudaMemset(c->err_dev, 0, sizeof(int)));
  return decode_error(c, h);
}

// cheap check at the start of every hot-path call: the error word of an earlier, completed step, as published to
// host memory by that step's last kernel (no synchronisation; include/pfc.h "device-detected errors")
pfc_status pending_error(pfc_ctx* c) {
  if (!c->err_host || !*(volatile int*)c->err_host) return PFC_OK;
  CUDA_TRY(c, cudaDeviceSynchronize());
  return device_error(c);
}

pfc_status validate(const pfc_config* c) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "cfg is NULL");
  if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size)
    return set_err(nullptr, PFC_ERR_CONFIG, "need 0 <= rank < world_size");
  if (c->num_classes < c->world_size) return set_err(nullptr, PFC_ERR_CONFIG, "need num_classes >= world_size");
  if (c->num_classes >= (int64_t(1) << 31) * c->world_size)
    return set_err(nullptr, PFC_ERR_CONFIG, "shard larger than 2^31 rows");
  if (c->dim < 128 || c->dim % 128 != 0 || c->dim > 1024)
    return set_err(nullptr, PFC_ERR_CONFIG, "dim must be a multiple of 128 in [128, 1024]");
  if (c->batch < 1) return set_err(nullptr, PFC_ERR_CONFIG, "batch must be >= 1");
  if (!(c->sample_rate > 0.0 && c->sample_rate <= 1.0)) return set_err(nullptr, PFC_ERR_CONFIG, "sample_rate must be in (0, 1]");
  if (!(c->scale > 0.f)) return set_err(nullptr, PFC_ERR_CONFIG, "scale must be > 0");
  if (c->margin_type == PFC_MARGIN_ARCFACE && !(c->margin >= 0.f && c->margin < 1.5707963f))
    return set_err(nullptr, PFC_ERR_CONFIG, "ArcFace margin must be in [0, pi/2)");
  if (c->margin_type == PFC_MARGIN_COSFACE && !(c->margin >= 0.f && c->margin < 1.f))
    return set_err(nullptr, PFC_ERR_CONFIG, "CosFace margin must be in [0, 1)");
  if (c->margin_type < 0 || c->margin_type > 2) return set_err(nullptr, PFC_ERR_CONFIG, "unknown margin_type");
  if (c->precision != PFC_FP32 && c->precision != PFC_BF16) return set_err(nullptr, PFC_ERR_CONFIG, "unknown precision");
  if (!(c->momentum >= 0.f && c->momentum < 1.f)) return set_err(nullptr, PFC_ERR_CONFIG, "momentum must be in [0, 1)");
  if (!(c->weight_decay >= 0.f)) return set_err(nullptr, PFC_ERR_CONFIG, "weight_decay must be >= 0");
  if (c->sample_mode < PFC_SAMPLE_PPRN || c->sample_mode > PFC_SAMPLE_RANDOM)
    return set_err(nullptr, PFC_ERR_CONFIG, "unknown sample_mode");
  if (c->ignore_index != 0 && c->ignore_index != 1) return set_err(nullptr, PFC_ERR_CONFIG, "ignore_index must be 0 or 1");
  if (c->param_location != PFC_PARAMS_DEVICE && c->param_location != PFC_PARAMS_HOST)
    return set_err(nullptr, PFC_ERR_CONFIG, "unknown param_location");
  if (c->comm_mode < PFC_COMM_NCCL || c->comm_mode > PFC_COMM_LOOPBACK_FUSED)
    return set_err(nullptr, PFC_ERR_CONFIG, "unknown comm_mode");
  if (c->comm_mode != PFC_COMM_NCCL && c->world_size > kMaxLoopback)
    return set_err(nullptr, PFC_ERR_CONFIG, "loopback groups and fused collectives support at most 16 ranks");
  if (c->world_size > 1 && (c->comm_mode == PFC_COMM_NCCL || c->comm_mode == PFC_COMM_NCCL_FUSED) &&
      !c->nccl_unique_id)
    return set_err(nullptr, PFC_ERR_CONFIG, "world_size > 1 needs nccl_unique_id");
  if ((int64_t)c->world_size * c->batch > (1 << 24)) return set_err(nullptr, PFC_ERR_CONFIG, "global batch too large");
  return PFC_OK;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

}  // namespace

extern "C" {

const char* pfc_version(void) { return "pfc-b200 0.1 (sm_100a)"; }

const char* pfc_last_error(const pfc_ctx* ctx) {
  if (!ctx) return g_init_error.c_str();
  return ctx->err.c_str();
}

pfc_status pfc_get_unique_id(void* id_out) {
  if (!id_out) return set_err(nullptr, PFC_ERR_CONTRACT, "id_out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_err(nullptr, PFC_ERR_NCCL, ncclGetErrorString(r));
  std::memcpy(id_out, &id, sizeof(id));
  return PFC_OK;
}

pfc_status pfc_init(const pfc_config* cfg, pfc_ctx** out) {
  if (!out) return set_err(nullptr, PFC_ERR_CONTRACT, "out is NULL");
  *out = nullptr;
  pfc_status v = validate(cfg);
  if (v != PFC_OK) return v;
  pfc_ctx* c = new pfc_ctx();
  c->cfg = *cfg;
  c->cfg.nccl_unique_id = nullptr;
  c->bf16 = cfg->precision == PFC_BF16;
  const char* sc = std::getenv("PFC_SYNC_CHECK");
  c->sync_check = sc && sc[0] == '1';
  const char* gb = std::getenv("PFC_GEMM");
  c->use_tc = c->bf16 && tc_available() && !(gb && std::string(gb) == "simt");

  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) {
    delete c;
    return set_err(nullptr, PFC_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }

  Sizes& sz = c->sz;
  const int64_t C = cfg->num_classes;
  const int k = cfg->world_size, i = cfg->rank;
  sz.C = C;
  sz.world = k;
  sz.rank = i;
  sz.C_local = C / k + (i < C % k ? 1 : 0);                 // R6
  sz.a = (int64_t)i * (C / k) + std::min<int64_t>(i, C % k);
  sz.d = cfg->dim;
  sz.B = cfg->batch;
  sz.M = k * cfg->batch;
  sz.M_pad = (int)round_up(sz.M, 128);
  sz.budget = (int64_t)std::ceil((double)cfg->sample_rate * (double)sz.C_local);  // R1 (IEEE double)
  sz.rate = cfg->sample_rate;
  sz.sample_mode = cfg->sample_mode;
  if (cfg->sample_mode == PFC_SAMPLE_PPRN_PAPER)   // |P_i| + round((C_local - |P_i|) r) <= budget + min(M, C_local)
    sz.k_max = std::min<int64_t>(sz.C_local, sz.budget + 1 + std::min<int64_t>(sz.M, sz.C_local));
  else if (cfg->sample_mode == PFC_SAMPLE_RANDOM)
    sz.k_max = sz.budget;
  else
    sz.k_max = std::max<int64_t>(sz.budget, std::min<int64_t>(sz.M, sz.C_local));
  sz.k_pad = round_up(sz.k_max, kKPad);
  sz.ltile = c->use_tc ? 128 : 64;
  sz.n_ltiles = (int)(sz.k_pad / sz.ltile);
  sz.ntiles_sel = (int)((sz.C_local + kSelTile - 1) / kSelTile);

  MarginParams& mp = c->mp;
  mp.type = cfg->margin_type;
  mp.s = cfg->scale;
  mp.m = cfg->margin;
  mp.cos_m = (float)std::cos((double)cfg->margin);
  mp.sin_m = (float)std::sin((double)cfg->margin);
  mp.th = (float)std::cos(M_PI - (double)cfg->margin);
  mp.mm = (float)(std::sin((double)cfg->margin) * (double)cfg->margin);

  const size_t d = sz.d, M = sz.M, Mp = sz.M_pad, B = sz.B, kp = sz.k_pad;
  const size_t esz = c->bf16 ? 2 : 4;
  pfc_status s = PFC_OK;
#define ALLOC(p, bytes) \
  if ((s = dalloc(c, &(p), (bytes))) != PFC_OK) { g_init_error = c->err; pfc_destroy(c); return s; }
  if (cfg->param_location == PFC_PARAMS_HOST) {
    for (int t = 0; t < 2; ++t) {
      void* h = nullptr;
      void* dp = nullptr;
      const size_t bytes = (size_t)sz.C_local * d * 4;
      cudaError_t e = cudaHostAlloc(&h, std::max<size_t>(bytes, 16), cudaHostAllocMapped | cudaHostAllocPortable);
      if (e == cudaSuccess) e = cudaHostGetDevicePointer(&dp, h, 0);
      if (e != cudaSuccess) {
        cudaGetLastError();
        if (h) cudaFreeHost(h);
        s = set_err(c, PFC_ERR_OOM, std::string("page-locked host allocation of W / V failed: ") + cudaGetErrorString(e));
        g_init_error = c->err;
        pfc_destroy(c);
        return s;
      }
      c->host_allocs.push_back(h);
      std::memset(h, 0, bytes);
      (t == 0 ? c->W_host : c->V_host) = static_cast<float*>(h);
      (t == 0 ? c->W : c->V) = static_cast<float*>(dp);
    }
  } else {
    ALLOC(c->W, (size_t)sz.C_local * d * 4);
    ALLOC(c->V, (size_t)sz.C_local * d * 4);
  }
  ALLOC(c->xh_local, B * d * 4);
  ALLOC(c->xnorm, B * 4);
  if (cfg->comm_mode == PFC_COMM_NCCL_FUSED || cfg->comm_mode == PFC_COMM_LOOPBACK_FUSED) {
    // the exchange region of the fused collectives holds the all-gather targets X32 and Y (SymLayout)
    if (cfg->comm_mode == PFC_COMM_NCCL_FUSED) {
      // the communicator first (1 rank at world size 1: the fused code path on one GPU)
      ncclResult_t r = ncclSuccess;
      if (k > 1) {
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
        r = ncclCommInitRank(&c->comm, k, id, i);
      } else {
        int dev = cfg->device;
        r = ncclCommInitAll(&c->comm, 1, &dev);
      }
      if (r != ncclSuccess) {
        std::string m = std::string("NCCL communicator: ") + ncclGetErrorString(r);
        pfc_destroy(c);
        return set_err(nullptr, PFC_ERR_NCCL, m);
      }
      std::string m;
      pfc_status fs = fused_nccl_create(c->comm, sz, &c->fnccl, &c->sym, &c->peers, &m);
      if (fs != PFC_OK) {
        pfc_destroy(c);
        return set_err(nullptr, fs, m);
      }
      c->fused_nccl = true;
    } else {
      ALLOC(c->sym, (size_t)sym_layout(sz).bytes);
      cudaMemset(c->sym, 0, (size_t)sym_layout(sz).bytes);
    }
    c->X32 = reinterpret_cast<float*>(c->sym + sym_layout(sz).x32);
    c->Y = reinterpret_cast<int64_t*>(c->sym + sym_layout(sz).y);
  } else {
    ALLOC(c->X32, Mp * d * 4);
    ALLOC(c->Y, M * 8);
  }
  ALLOC(c->Xb, Mp * d * 2);
  if (c->bf16) ALLOC(c->Xh16, Mp * d * 2);
  ALLOC(c->bits, ((sz.C_local + 31) / 32) * 4);
  ALLOC(c->keys, (size_t)sz.ntiles_sel * kSelTile * 4);   // padded to whole compaction tiles (vector loads)
  ALLOC(c->hist, 5120 * 4);
  ALLOC(c->tile_cnt, (size_t)sz.ntiles_sel * 4 * 4);
  ALLOC(c->st, sizeof(SamplerState));
  ALLOC(c->idx, kp * 4);
  if (cfg->param_location == PFC_PARAMS_HOST) {
    const char* e = std::getenv("PFC_HOST_STAGE");
    c->stage = !(e && e[0] == '0');
  }
  if (c->stage) {
    ALLOC(c->Wst, kp * d * 4);
    ALLOC(c->Vst, kp * d * 4);
    ALLOC(c->idx_id, kp * 4);
    launch_iota(c->idx_id, kp, 0);
  }
  ALLOC(c->tcol, M * 4);
  ALLOC(c->Ws, kp * d * esz);
  ALLOC(c->inv_norm, kp * 4);
  ALLOC(c->ct, M * 4);
  ALLOC(c->cosv, Mp * kp * esz);   // class-major [k_pad][M_pad]
  ALLOC(c->partials, M * (size_t)sz.n_ltiles * sizeof(float2));
  ALLOC(c->rowmax, M * 4);
  ALLOC(c->gmax, M * 4);
  ALLOC(c->rowsum, M * 4);
  ALLOC(c->zt, M * 4);
  ALLOC(c->red, (3 * M + 1) * 4);
  ALLOC(c->metrics, 16);
  ALLOC(c->gt, M * 4);
  ALLOC(c->lse, M * 4);
  ALLOC(c->loss_dev, 16);
  ALLOC(c->G, Mp * kp * esz);      // class-major [k_pad][M_pad]
  ALLOC(c->dXh, Mp * d * 4);
  ALLOC(c->dxh_local, B * d * 4);
  c->fused_gather = c->use_tc && logits_gather_supported(sz);
  c->use_dwx = c->fused_gather && dwx_supported(sz);
  if (c->use_tc && !c->fused_gather) ALLOC(c->Ws16, kp * d * 2);
  ALLOC(c->split_ws, (size_t)(c->use_tc ? std::max(dx_split_ws_floats(sz), c->use_dwx ? dwx_ws_floats(sz) : 0) : 1) * 4);
  {
    const char* e = std::getenv("PFC_EFORM");
    // E = e^{s c} must stay finite in bf16/fp32 (s < 88) and f_n = (s/M) e^{-LSE_n}, LSE_n <= s + ln k_i, a
    // normal fp32 number (s + ln k_i < 80): the paper's s = 64 fits up to k_i ~ 1e7 per shard
    const double span = (double)c->cfg.scale + std::log((double)sz.k_max);
    const bool ok = c->cfg.scale <= 80.f && span < 80.0 && !(e && e[0] == '0');
    c->eform = ok && c->use_dwx && sz.d <= 1024;   // dwx.cu sums <= 8 d-tile partials
    c->eform_pair = ok && c->use_tc && !c->fused_gather && logits_pair_enabled(sz) && sz.M_pad <= 16384;
  }
  if (c->eform || c->eform_pair) {
    ALLOC(c->ef_f, Mp * 4);
    ALLOC(c->Xt, Mp * d * 2);
    ALLOC(c->dcorr, kp * 4);
  }
  if (c->eform_pair && dw_sgd_pairx_enabled(sz, 0) && !dw_sgd_full_enabled(sz, 0))
    ALLOC(c->xws, (size_t)dw_sgd_pairx_ws_floats(sz) * 4);
  if (c->eform) {
    ALLOC(c->xch, kp * (size_t)(d / 128) * 4);
    ALLOC(c->cnt, (kp / 128) * 4);
  }
  ALLOC(c->dWh, kp * d * 4);
  ALLOC(c->dotw, kp * 4);
  ALLOC(c->err_dev, 16);
  {
    void* h = nullptr;
    void* dp = nullptr;
    if (cudaHostAlloc(&h, 64, cudaHostAllocMapped) == cudaSuccess && cudaHostGetDevicePointer(&dp, h, 0) == cudaSuccess) {
      c->host_allocs.push_back(h);
      c->err_host = static_cast<int*>(h);
      c->err_host_dev = static_cast<int*>(dp);
      *c->err_host = 0;
    } else {
      cudaGetLastError();
      if (h) cudaFreeHost(h);
    }
  }
  ALLOC(c->step_dev, 16);
  ALLOC(c->lr_dev, 16);
  ALLOC(c->x_in, B * d * 4);
  ALLOC(c->y_in, B * 8);
  ALLOC(c->gx_out, B * d * 4);
#undef ALLOC
  if (!c->W_host) {
    cudaMemset(c->W, 0, (size_t)sz.C_local * d * 4);
    cudaMemset(c->V, 0, (size_t)sz.C_local * d * 4);
  }
  cudaMemset(c->X32, 0, Mp * d * 4);
  cudaMemset(c->Xb, 0, Mp * d * 2);
  if (c->Xh16) cudaMemset(c->Xh16, 0, Mp * d * 2);
  if (c->eform || c->eform_pair) {
    cudaMemset(c->ef_f, 0, Mp * 4);
    cudaMemset(c->Xt, 0, Mp * d * 2);
  }
  cudaMemset(c->dXh, 0, Mp * d * 4);
  cudaMemset(c->err_dev, 0, 16);
  cudaMemset(c->step_dev, 0, 16);
  cudaMemset(c->lr_dev, 0, 16);
  {
    const char* g = std::getenv("PFC_GRAPH");
    c->graph_on = !(g && g[0] == '0');
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::string m = std::string("init memset: ") + cudaGetErrorString(e);
    pfc_destroy(c);
    return set_err(nullptr, PFC_ERR_CUDA, m);
  }
  const char* solo = std::getenv("PFC_NCCL_SOLO");
  if (k == 1 && cfg->comm_mode == PFC_COMM_NCCL && solo && solo[0] == '1') {
    // validation mode: the multi-rank code path (every collective call, graph-captured) on one GPU, where each
    // collective is the identity; results must equal the world-size-1 path
    int dev = cfg->device;
    ncclResult_t r = ncclCommInitAll(&c->comm, 1, &dev);
    if (r != ncclSuccess) {
      std::string m = std::string("ncclCommInitAll: ") + ncclGetErrorString(r);
      pfc_destroy(c);
      return set_err(nullptr, PFC_ERR_NCCL, m);
    }
    c->nccl_solo = true;
  }
  if (k > 1 && cfg->comm_mode == PFC_COMM_NCCL) {   // (PFC_COMM_NCCL_FUSED created its communicator above)
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&c->comm, k, id, i);
    if (r != ncclSuccess) {
      std::string m = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      pfc_destroy(c);
      return set_err(nullptr, PFC_ERR_NCCL, m);
    }
  }
  if (c->comm) {   // side stream + fork/join events of the overlapped dX exchange
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
      pfc_destroy(c);
      return set_err(nullptr, PFC_ERR_CUDA, "side stream / event creation failed");
    }
  }
  *out = c;
  return PFC_OK;
}

pfc_status pfc_destroy(pfc_ctx* c) {
  if (!c) return PFC_OK;
  cudaSetDevice(c->cfg.device);
  cudaDeviceSynchronize();
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->fnccl) fused_nccl_destroy(c->comm, c->fnccl);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (auto& ev : c->prof_ev)
    for (auto& e : ev) cudaEventDestroy(e);
  for (void* p : c->allocs) cudaFree(p);
  for (void* p : c->host_allocs) cudaFreeHost(p);
  delete c;
  return PFC_OK;
}

// ------------------------------------------------------------------------------------------------
// Step phases. Between them sit the three collectives of Alg.1 (all-gather L2, all-reduce L7,
// all-reduce + get_submatrix L12-13 = reduce-scatter), either NCCL or the loopback group.
// ------------------------------------------------------------------------------------------------
namespace {

pfc_status check_fb_args(pfc_ctx* c, const float* x, const int64_t* labels, float* grad_x) {
  if (!x || !labels || !grad_x) return set_err(c, PFC_ERR_CONTRACT, "x, labels and grad_x must be non-NULL");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(grad_x)) & 15)
    return set_err(c, PFC_ERR_CONTRACT, "x and grad_x must be 16-byte aligned");
  return PFC_OK;
}

// Event boundary b of the current step (b = section index; b + 1 closes it).
void mark(pfc_ctx* c, int b, cudaStream_t s) {
  if (!c->prof || !c->prof_cur) return;
  cudaEventRecord((*c->prof_cur)[b], s);
  (*c->prof_cur_set)[b] = true;
}

void prof_begin_step(pfc_ctx* c) {
  if (!c->prof) return;
  if (c->prof_used == c->prof_ev.size()) {
    std::array<cudaEvent_t, PFC_PROF_SECTIONS + 1> ev;
    for (auto& e : ev) cudaEventCreate(&e);
    c->prof_ev.push_back(ev);
    c->prof_set.emplace_back();
  }
  c->prof_cur = &c->prof_ev[c->prof_used];
  c->prof_cur_set = &c->prof_set[c->prof_used];
  c->prof_cur_set->fill(false);
  c->prof_used++;
}

// K1: normalise this rank's features into its all-gather slot; copy labels into theirs.
void phase_a(pfc_ctx* c, const float* x, const int64_t* labels, cudaStream_t s) {
  c->launches += launch_normalize_x(c->sz, x, labels, c->xh_local, c->xnorm, c->X32, c->Y, c->err_dev, c->P(),
                                    c->cfg.ignore_index, s);
}

// K1b, sampler K2-K4, K5, K5b, K6 logits + partial den_i, K7 local row (max, sum).
void phase_b(pfc_ctx* c, bool fused, cudaStream_t s) {
  const Sizes& sz = c->sz;
  const bool bf = c->bf16;
  int n = 0;
  mark(c, 1, s);
  if (bf) n += launch_x_to_bf16(sz, c->X32, c->Xb, c->Xh16, s);
  n += launch_sampler(sz, c->Y, c->cfg.seed, c->step_dev, c->bits, c->keys, c->hist, c->tile_cnt, c->st, c->idx,
                      c->tcol, c->err_dev, s);
  if (c->stage)   // f4: the sampled W / V rows of the host shard into HBM, once
    n += launch_stage_rows(sz, c->W, c->V, c->idx, c->st, c->Wst, c->Vst, /*to_host=*/false, s);
  mark(c, 2, s);
  if (!c->fused_gather)
    n += launch_gather_w(sz, bf, c->Wk(), c->idxk(), c->st, c->Ws, c->Ws16, c->inv_norm, c->err_dev, s);
  n += launch_target_cos(sz, c->X32, c->W, c->Y, c->idx, c->st, c->tile_cnt, c->tcol, c->ct, s);
  mark(c, 3, s);
  int nparts = 0;   // per-row LSE partials the logits kernel leaves (0: one per 128-column tile)
  if (c->fused_gather)
    n += launch_logits_gather_tc(sz, c->Wk(), c->idxk(), c->Xh16, (__nv_bfloat16*)c->Ws, !(fused && c->use_dwx), c->inv_norm,
                                 c->tcol, c->st, c->mp, (__half*)c->cosv, c->partials, c->err_dev,
                                 fused && c->eform, &nparts, s);
  else if (c->use_tc && logits_pair_enabled(sz))
    n += launch_logits_pair_tc(sz, c->Xh16, c->Ws16, c->tcol, c->st, c->mp, (__half*)c->cosv,
                               c->partials, fused && c->eform_pair, &nparts, s);
  else if (c->use_tc)
    n += launch_logits_tc(sz, c->Xh16, c->Ws16, c->tcol, c->ct, c->st, c->mp, (__half*)c->cosv,
                          c->partials, s);
  else
    n += launch_logits_simt(sz, bf, bf ? (const void*)c->Xb : (const void*)c->X32, c->Ws, c->tcol, c->ct, c->st, c->mp,
                            c->cosv, c->partials, s);
  mark(c, 4, s);
  n += launch_row_combine(sz, c->partials, nparts, c->Y, c->ct, c->st, c->mp, c->rowmax, c->rowsum, c->zt, c->P(), s);
  c->launches += n;
}

// after all-reduce MAX: red[n] = l_n e^{m_n - gm_n} (non-target columns), red[M + n] = local z_t
// (fused collectives: gmax is formed here from the peers' row maxima)
void phase_c(pfc_ctx* c, float* gmax, cudaStream_t s) {
  c->launches += launch_prep_sum(c->sz, c->rowmax, gmax, c->rowsum, c->zt, c->tcol, c->Y, c->ct, c->red, c->P(), s);
}

// after all-reduce SUM: LSE, loss, K8 (prob - onehot), K9 dX_hat partial
void phase_d(pfc_ctx* c, const float* gmax, float* loss_out, bool fused, cudaStream_t s) {
  const Sizes& sz = c->sz;
  int n = 0;
  n += launch_finalize(sz, gmax, c->red, c->lse, c->gt, loss_out, c->metrics, c->err_dev, c->P(), c->Y,
                       c->cfg.ignore_index, s);
  mark(c, 5, s);
  if (fused && c->eform) {
    // E-form: no softmax-gradient pass; f, X~ and the target entries, then dW + SGD + dX on E directly
    n += launch_eform_prep(sz, c->X32, c->lse, c->gt, c->tcol, c->ct, c->mp, c->ef_f, c->Xt,
                           (__nv_bfloat16*)c->cosv, c->dcorr, c->metrics + 2, s);
    mark(c, 6, s);
    SgdArgs a{c->Wk(), c->Vk(), c->idxk(), c->inv_norm, c->dotw, c->lr_dev, c->cfg.momentum, c->cfg.weight_decay, 0};
    a.rows = c->stage ? sz.k_pad : sz.C_local;
    EformArgs ef{c->ef_f, c->tcol, c->dcorr, c->xch, c->cnt, c->err_dev, c->mp.s};
    n += launch_dwx_tc(sz, (const __nv_bfloat16*)c->cosv, c->Xt, c->st, a, c->split_ws, c->dXh, &ef, c->P(), s);
    c->launches += n;
    return;
  }
  if (fused && c->eform_pair) {
    // E-form at M > 256: f, X~, the target entries and the radial dots, then dX_hat = f (E' W_s)
    n += launch_eform_prep(sz, c->X32, c->lse, c->gt, c->tcol, c->ct, c->mp, c->ef_f, c->Xt,
                           (__nv_bfloat16*)c->cosv, c->dcorr, c->metrics + 2, s);
    if (!dw_sgd_full_enabled(sz, 0) && !c->xws)   // else the dW + SGD kernel forms the radial dots itself
      n += launch_eform_dotw(sz, (const __nv_bfloat16*)c->cosv, c->ef_f, c->dcorr, c->st, c->mp, c->dotw, s);
    mark(c, 6, s);
    n += launch_dx_tc(sz, (const __nv_bfloat16*)c->cosv, (const __nv_bfloat16*)c->Ws, c->st, c->dXh, c->split_ws,
                      c->ef_f, c->P(), s);
    c->launches += n;
    return;
  }
  n += launch_softmax_grad(sz, c->bf16, c->cosv, c->lse, c->gt, c->tcol, c->ct, c->st, c->mp, c->G,
                           fused && c->use_tc ? c->dotw : nullptr, c->fused_gather ? c->inv_norm : nullptr,
                           c->metrics + 2, s);
  mark(c, 6, s);
  if (fused && c->use_dwx) {
    SgdArgs a{c->Wk(), c->Vk(), c->idxk(), c->inv_norm, c->dotw, c->lr_dev, c->cfg.momentum, c->cfg.weight_decay, 1};
    a.rows = c->stage ? sz.k_pad : sz.C_local;
    n += launch_dwx_tc(sz, (const __nv_bfloat16*)c->G, c->Xb, c->st, a, c->split_ws, c->dXh, nullptr, c->P(), s);
  } else if (c->use_tc)
    n += launch_dx_tc(sz, (const __nv_bfloat16*)c->G, (const __nv_bfloat16*)c->Ws, c->st, c->dXh, c->split_ws,
                      nullptr, c->P(), s);
  else {
    n += launch_dx_simt(sz, c->bf16, c->G, c->Ws, c->st, c->dXh, s);
    if (c->P()) n += launch_push_dx(sz, c->dXh, c->peers, s);   // fused reduce-scatter: the owners' slots
  }
  c->launches += n;
}

// K11 dW_hat (+ K12 when fused); independent of the dX exchange
void phase_e_dw(pfc_ctx* c, bool fused, cudaStream_t s) {
  const Sizes& sz = c->sz;
  int n = 0;
  if (fused && c->use_dwx) {
    // dW + SGD ran inside the dX kernel (phase_d)
  } else if (c->use_tc && fused) {
    SgdArgs a{c->Wk(), c->Vk(), c->idxk(), c->inv_norm, c->dotw, c->lr_dev, c->cfg.momentum, c->cfg.weight_decay,
              c->fused_gather ? 1 : 0};
    if (c->eform_pair) { a.xws = c->xws; a.err = c->err_dev; }   // E-form pair path: radial dots in the dW kernel
    a.rows = c->stage ? sz.k_pad : sz.C_local;
    if (c->eform_pair)   // dW_hat = E'^T X~ (E-form): same contraction, other operands
      n += launch_dw_sgd_tc(sz, (const __nv_bfloat16*)c->cosv, c->Xt, c->st, a, s);
    else
      n += launch_dw_sgd_tc(sz, (const __nv_bfloat16*)c->G, c->Xb, c->st, a, s);
  } else {
    if (c->use_tc)
      n += launch_dw_tc(sz, (const __nv_bfloat16*)c->G, c->Xb, c->st, c->dWh, s);
    else
      n += launch_dw_simt(sz, c->bf16, c->G, c->bf16 ? (const void*)c->Xb : (const void*)c->X32, c->st, c->dWh, s);
    if (fused)
      n += launch_sgd(sz, c->Wk(), c->Vk(), c->dWh, c->idxk(), c->inv_norm, c->st, c->lr_dev, c->cfg.momentum,
                      c->cfg.weight_decay, c->fused_gather ? 1 : 0, s);
  }
  c->launches += n;
}

// f4 staging: the updated sampled rows back into the host shard (after the fused train step's update)
void stage_out(pfc_ctx* c, bool fused, cudaStream_t s) {
  if (c->stage && fused)
    c->launches += launch_stage_rows(c->sz, c->W, c->V, c->idx, c->st, c->Wst, c->Vst, /*to_host=*/true, s);
}

// after reduce-scatter: K10 x-norm backward of this rank's rows, K11 dW_hat (+ K12 when fused)
void phase_e(pfc_ctx* c, const float* dxh, float* grad_x, bool fused, cudaStream_t s) {
  c->launches += launch_xnorm_backward(c->sz, dxh, c->xh_local, c->xnorm, grad_x, c->P(), s);
  mark(c, 8, s);
  phase_e_dw(c, fused, s);
  mark(c, 9, s);
}

pfc_status finish_fb(pfc_ctx* c, bool fused, cudaStream_t s) {
  CUDA_TRY(c, cudaGetLastError());
  c->step += 1;
  c->fb_done = !fused;
  c->last_stream = s;
  if (c->sync_check) {
    if (pfc_status w = wait_stream(c, s)) return w;
    return device_error(c);
  }
  return PFC_OK;
}

}  // namespace

static pfc_status run_step(pfc_ctx* c, const float* x, const int64_t* labels, float* grad_x, float* loss, bool fused,
                           float lr, void* stream);

pfc_status pfc_forward_backward(pfc_ctx* c, const float* x, const int64_t* labels, float* grad_x, float* loss,
                                void* stream) {
  return run_step(c, x, labels, grad_x, loss, false, 0.f, stream);
}

pfc_status pfc_train_step(pfc_ctx* c, const float* x, const int64_t* labels, float* grad_x, float* loss, float lr,
                          void* stream) {
  return run_step(c, x, labels, grad_x, loss, true, lr, stream);
}

// Collectives fused into the kernels (PFC_COMM_NCCL_FUSED, fused_comm.cu): the kernels store into the peers'
// exchange regions, one LSA barrier after each producer.
static void enqueue_step_fused(pfc_ctx* c, const float* x, const int64_t* labels, float* grad_x, float* loss_out,
                               bool fused, cudaStream_t s) {
  const Sizes& sz = c->sz;
  mark(c, 0, s);
  phase_a(c, x, labels, s);                                  // x_hat / labels -> every peer (all-gather)
  c->launches += launch_lsa_barrier(c->fnccl, s);
  phase_b(c, fused, s);                                      // ... K7 row maxima -> every peer's xmax slot
  c->launches += launch_lsa_barrier(c->fnccl, s);
  phase_c(c, c->gmax, s);                                    // global max (rank order); sums -> peers' xred
  c->launches += launch_lsa_barrier(c->fnccl, s);
  phase_d(c, c->gmax, loss_out, fused, s);                   // finalize sums xred; dX rows -> owners' xdx
  mark(c, 7, s);
  if (!(fused && c->use_dwx) && !c->prof_cur && c->side) {
    // barrier + x-norm backward (the reduce-scatter's reduction) on the side stream, overlapping the dW kernel
    cudaEventRecord(c->ev_fork, s);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    c->launches += launch_lsa_barrier(c->fnccl, c->side);
    c->launches += launch_xnorm_backward(sz, nullptr, c->xh_local, c->xnorm, grad_x, c->P(), c->side);
    phase_e_dw(c, fused, s);
    cudaEventRecord(c->ev_join, c->side);
    cudaStreamWaitEvent(s, c->ev_join, 0);
  } else {
    c->launches += launch_lsa_barrier(c->fnccl, s);
    phase_e(c, nullptr, grad_x, fused, s);
  }
  stage_out(c, fused, s);
  c->launches += launch_advance_step(c->step_dev, c->err_dev, c->err_host_dev, s);
}

static void enqueue_step(pfc_ctx* c, const float* x, const int64_t* labels, float* grad_x, float* loss_out, bool fused,
                         cudaStream_t s, ncclResult_t* nres) {
  const Sizes& sz = c->sz;
  const bool multi = sz.world > 1 || c->nccl_solo;
  *nres = ncclSuccess;
  if (c->fused_nccl) {
    enqueue_step_fused(c, x, labels, grad_x, loss_out, fused, s);
    return;
  }
  auto nccl = [&](ncclResult_t r) { if (r != ncclSuccess && *nres == ncclSuccess) *nres = r; };
  mark(c, 0, s);
  phase_a(c, x, labels, s);
  if (multi) {  // Alg.1 L2: X = allgather(x_i) (+ labels)
    nccl(ncclGroupStart());
    nccl(ncclAllGather(c->X32 + (size_t)sz.rank * sz.B * sz.d, c->X32, (size_t)sz.B * sz.d, ncclFloat, c->comm, s));
    nccl(ncclAllGather(c->Y + (size_t)sz.rank * sz.B, c->Y, (size_t)sz.B, ncclInt64, c->comm, s));
    nccl(ncclGroupEnd());
  }
  phase_b(c, fused, s);
  float* gmax = c->rowmax;
  if (multi) {  // Alg.1 L7 (stabilised, R12): global row max, then global sum
    nccl(ncclAllReduce(c->rowmax, c->gmax, sz.M, ncclFloat, ncclMax, c->comm, s));
    gmax = c->gmax;
  }
  phase_c(c, gmax, s);
  if (multi) nccl(ncclAllReduce(c->red, c->red, 3 * sz.M + 1, ncclFloat, ncclSum, c->comm, s));
  phase_d(c, gmax, loss_out, fused, s);
  mark(c, 7, s);
  const float* dxh = c->dXh + (size_t)sz.rank * sz.B * sz.d;
  if (multi && !(fused && c->use_dwx) && !c->prof_cur && c->side) {
    // the dX exchange and the x-norm backward on a side stream, overlapping the dW (+ SGD) kernel, which does
    // not depend on them (fork / join by events: also inside graph capture)
    cudaEventRecord(c->ev_fork, s);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    nccl(ncclReduceScatter(c->dXh, c->dxh_local, (size_t)sz.B * sz.d, ncclFloat, ncclSum, c->comm, c->side));
    c->launches += launch_xnorm_backward(sz, c->dxh_local, c->xh_local, c->xnorm, grad_x, nullptr, c->side);
    phase_e_dw(c, fused, s);
    cudaEventRecord(c->ev_join, c->side);
    cudaStreamWaitEvent(s, c->ev_join, 0);
  } else {
    if (multi) {  // Alg.1 L12-13: allreduce(grad logits w^T) then get_submatrix(i) == reduce-scatter (R16)
      nccl(ncclReduceScatter(c->dXh, c->dxh_local, (size_t)sz.B * sz.d, ncclFloat, ncclSum, c->comm, s));
      dxh = c->dxh_local;
    }
    phase_e(c, dxh, grad_x, fused, s);
  }
  stage_out(c, fused, s);
  c->launches += launch_advance_step(c->step_dev, c->err_dev, c->err_host_dev, s);
}

static pfc_status run_step(pfc_ctx* c, const float* x, const int64_t* labels, float* grad_x, float* loss, bool fused,
                           float lr, void* stream) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  pfc_status a = check_fb_args(c, x, labels, grad_x);
  if (a != PFC_OK) return a;
  if (c->cfg.comm_mode == PFC_COMM_LOOPBACK_FUSED || (c->sz.world > 1 && c->cfg.comm_mode == PFC_COMM_LOOPBACK))
    return set_err(c, PFC_ERR_CONTRACT, "loopback contexts are driven by pfc_group_forward_backward");
  if (pfc_status pe = pending_error(c)) return pe;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float* loss_out = loss ? loss : c->loss_dev;
  if (fused) c->launches += launch_set_scalar(c->lr_dev, lr, s);   // outside any graph: a kernel argument
  tmap_error() = 0;
  ncclResult_t nres = ncclSuccess;
  const bool use_graph = c->graph_on && !c->prof && s != nullptr;
  if (!use_graph) {
    prof_begin_step(c);
    enqueue_step(c, x, labels, grad_x, loss_out, fused, s, &nres);
    if (nres != ncclSuccess) return set_err(c, PFC_ERR_NCCL, ncclGetErrorString(nres));
    if (tmap_error()) return set_err(c, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(tmap_error()) + "): kernels not launched");
    return finish_fb(c, fused, s);
  }
  // CUDA graph of the whole step, cached per (pointers, stream, fused); the first call of a context runs eagerly
  // (one-time kernel attribute setup), later calls capture once and replay.
  for (auto& g : c->graphs) {
    if (g.x == x && g.y == labels && g.gx == grad_x && g.loss == loss_out && g.s == s && g.fused == fused) {
      CUDA_TRY(c, cudaGraphLaunch(g.exec, s));
      c->launches += c->graph_launches;
      return finish_fb(c, fused, s);
    }
  }
  if (c->graph_warm++ == 0 || c->graphs.size() >= 8) {
    prof_begin_step(c);
    enqueue_step(c, x, labels, grad_x, loss_out, fused, s, &nres);
    if (nres != ncclSuccess) return set_err(c, PFC_ERR_NCCL, ncclGetErrorString(nres));
    if (tmap_error()) return set_err(c, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(tmap_error()) + "): kernels not launched");
    return finish_fb(c, fused, s);
  }
  cudaGraph_t graph = nullptr;
  CUDA_TRY(c, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  const int64_t l0 = c->launches;
  c->prof_cur = nullptr;
  enqueue_step(c, x, labels, grad_x, loss_out, fused, s, &nres);
  cudaError_t ce = cudaStreamEndCapture(s, &graph);
  c->graph_launches = c->launches - l0;
  c->launches = l0;
  if (nres != ncclSuccess) { if (graph) cudaGraphDestroy(graph); return set_err(c, PFC_ERR_NCCL, ncclGetErrorString(nres)); }
  if (tmap_error()) {
    if (graph) cudaGraphDestroy(graph);
    return set_err(c, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(tmap_error()) + "): kernels not launched");
  }
  CUDA_TRY(c, ce);
  cudaGraphExec_t exec = nullptr;
  ce = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  CUDA_TRY(c, ce);
  c->graphs.push_back({x, labels, grad_x, loss_out, s, fused, exec});
  CUDA_TRY(c, cudaGraphLaunch(exec, s));
  c->launches += c->graph_launches;
  return finish_fb(c, fused, s);
}

static pfc_status group_step(pfc_ctx** ctxs, int32_t n, const float* const* x, const int64_t* const* labels,
                             float* const* grad_x, float* loss, bool fused, float lr, void* stream);

pfc_status pfc_group_forward_backward(pfc_ctx** ctxs, int32_t n, const float* const* x, const int64_t* const* labels,
                                      float* const* grad_x, float* loss, void* stream) {
  return group_step(ctxs, n, x, labels, grad_x, loss, false, 0.f, stream);
}

pfc_status pfc_group_train_step(pfc_ctx** ctxs, int32_t n, const float* const* x, const int64_t* const* labels,
                                float* const* grad_x, float* loss, float lr, void* stream) {
  return group_step(ctxs, n, x, labels, grad_x, loss, true, lr, stream);
}

static pfc_status group_step(pfc_ctx** ctxs, int32_t n, const float* const* x, const int64_t* const* labels,
                             float* const* grad_x, float* loss, bool fused, float lr, void* stream) {
  if (!ctxs || n < 1 || n > kMaxLoopback || !x || !labels || !grad_x)
    return set_err(nullptr, PFC_ERR_CONTRACT, "bad group arguments (1 <= n <= 16, non-NULL arrays)");
  for (int r = 0; r < n; ++r) {
    pfc_ctx* c = ctxs[r];
    if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "NULL context in group");
    const bool lb = c->cfg.comm_mode == PFC_COMM_LOOPBACK || c->cfg.comm_mode == PFC_COMM_LOOPBACK_FUSED;
    if (c->sz.world != n || c->sz.rank != r || (n > 1 && !lb) || c->cfg.comm_mode != ctxs[0]->cfg.comm_mode)
      return set_err(c, PFC_ERR_CONTRACT, "group contexts must be loopback ranks 0..n-1 of a world of size n");
    if (c->sz.B != ctxs[0]->sz.B || c->sz.d != ctxs[0]->sz.d || c->sz.C != ctxs[0]->sz.C || c->step != ctxs[0]->step)
      return set_err(c, PFC_ERR_CONTRACT, "group contexts disagree on B, d, C or step");
    pfc_status a = check_fb_args(c, x[r], labels[r], grad_x[r]);
    if (a != PFC_OK) return a;
  }
  for (int r = 0; r < n; ++r)
    if (pfc_status pe = pending_error(ctxs[r])) return pe;
  tmap_error() = 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int r = 0; r < n; ++r) ctxs[r]->prof_cur = nullptr;  // no event timing in loopback groups
  if (fused)
    for (int r = 0; r < n; ++r) ctxs[r]->launches += launch_set_scalar(ctxs[r]->lr_dev, lr, s);
  const Sizes& sz = ctxs[0]->sz;
  const size_t rowbytes = (size_t)sz.B * sz.d * 4;
  pfc_ctx* c0 = ctxs[0];
  PtrPack src{}, dst{};
  if (c0->cfg.comm_mode == PFC_COMM_LOOPBACK_FUSED) {
    // collectives fused into the kernels (fused_comm.cu), the ranks' exchange regions being the contexts' own
    // allocations: each phase runs for every rank before the next one consumes the peers' stores (stream order
    // stands in for the LSA barriers of PFC_COMM_NCCL_FUSED)
    for (int r = 0; r < n; ++r) {
      Peers& P = ctxs[r]->peers;
      P = Peers{};
      for (int q = 0; q < n; ++q) P.base[q] = ctxs[q]->sym;
      P.n = n;
      P.rank = r;
      P.lay = sym_layout(ctxs[r]->sz);
    }
    for (int r = 0; r < n; ++r) phase_a(ctxs[r], x[r], labels[r], s);
    for (int r = 0; r < n; ++r) phase_b(ctxs[r], fused, s);
    for (int r = 0; r < n; ++r) phase_c(ctxs[r], ctxs[r]->gmax, s);
    for (int r = 0; r < n; ++r) phase_d(ctxs[r], ctxs[r]->gmax, r == 0 && loss ? loss : ctxs[r]->loss_dev, fused, s);
    for (int r = 0; r < n; ++r) {
      phase_e(ctxs[r], nullptr, grad_x[r], fused, s);
      stage_out(ctxs[r], fused, s);
      ctxs[r]->launches += launch_advance_step(ctxs[r]->step_dev, ctxs[r]->err_dev, ctxs[r]->err_host_dev, s);
    }
    if (tmap_error()) return set_err(c0, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed: kernels not launched");
    for (int r = 0; r < n; ++r) {
      pfc_status f = finish_fb(ctxs[r], fused, s);
      if (f != PFC_OK) return f;
    }
    return PFC_OK;
  }
  for (int r = 0; r < n; ++r) phase_a(ctxs[r], x[r], labels[r], s);
  for (int r = 0; r < n; ++r)      // all-gather: copy rank r's slot into every other rank
    for (int q = 0; q < n; ++q) {
      if (q == r) continue;
      CUDA_TRY(c0, cudaMemcpyAsync(ctxs[q]->X32 + (size_t)r * sz.B * sz.d, ctxs[r]->X32 + (size_t)r * sz.B * sz.d,
                                   rowbytes, cudaMemcpyDefault, s));
      CUDA_TRY(c0, cudaMemcpyAsync(ctxs[q]->Y + (size_t)r * sz.B, ctxs[r]->Y + (size_t)r * sz.B, (size_t)sz.B * 8,
                                   cudaMemcpyDefault, s));
    }
  for (int r = 0; r < n; ++r) phase_b(ctxs[r], fused, s);
  for (int r = 0; r < n; ++r) { src.p[r] = ctxs[r]->rowmax; dst.p[r] = ctxs[r]->gmax; }
  c0->launches += launch_group_reduce(sz.M, src, 0, dst, n, n, 1, s);
  for (int r = 0; r < n; ++r) phase_c(ctxs[r], ctxs[r]->gmax, s);
  for (int r = 0; r < n; ++r) { src.p[r] = ctxs[r]->red; dst.p[r] = ctxs[r]->red; }
  c0->launches += launch_group_reduce(3 * sz.M + 1, src, 0, dst, n, n, 0, s);  // in place: all reads precede writes per element
  for (int r = 0; r < n; ++r) phase_d(ctxs[r], ctxs[r]->gmax, r == 0 && loss ? loss : ctxs[r]->loss_dev, fused, s);
  for (int r = 0; r < n; ++r) src.p[r] = ctxs[r]->dXh;
  for (int r = 0; r < n; ++r) {  // reduce-scatter: owner r sums rows [rB, (r+1)B) over ranks
    PtrPack one{};
    one.p[0] = ctxs[r]->dxh_local;
    c0->launches += launch_group_reduce((int64_t)sz.B * sz.d, src, (int64_t)r * sz.B * sz.d, one, n, 1, 0, s);
  }
  for (int r = 0; r < n; ++r) {
    phase_e(ctxs[r], ctxs[r]->dxh_local, grad_x[r], fused, s);
    stage_out(ctxs[r], fused, s);
    ctxs[r]->launches += launch_advance_step(ctxs[r]->step_dev, ctxs[r]->err_dev, ctxs[r]->err_host_dev, s);
  }
  if (tmap_error()) return set_err(c0, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed: kernels not launched");
  for (int r = 0; r < n; ++r) {
    pfc_status f = finish_fb(ctxs[r], fused, s);
    if (f != PFC_OK) return f;
  }
  return PFC_OK;
}

static pfc_status host_step(pfc_ctx* c, const float* x_host, const int64_t* labels_host, float* grad_x_host,
                            float* loss_host, bool fused, float lr, void* stream, bool sync = true) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  if (!x_host || !labels_host || !grad_x_host) return set_err(c, PFC_ERR_CONTRACT, "NULL host buffer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t xb = (size_t)c->sz.B * c->sz.d * 4;
  CUDA_TRY(c, cudaMemcpyAsync(c->x_in, x_host, xb, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(c->y_in, labels_host, (size_t)c->sz.B * 8, cudaMemcpyHostToDevice, s));
  pfc_status r = run_step(c, c->x_in, c->y_in, c->gx_out, c->loss_dev, fused, lr, stream);
  if (r != PFC_OK) return r;
  CUDA_TRY(c, cudaMemcpyAsync(grad_x_host, c->gx_out, xb, cudaMemcpyDeviceToHost, s));
  if (loss_host) CUDA_TRY(c, cudaMemcpyAsync(loss_host, c->loss_dev, 4, cudaMemcpyDeviceToHost, s));
  if (!sync) {
    c->last_stream = s;
    return PFC_OK;
  }
  return wait_stream(c, s);
}

pfc_status pfc_forward_backward_host_async(pfc_ctx* c, const float* x_host, const int64_t* labels_host,
                                           float* grad_x_host, float* loss_host, void* stream) {
  return host_step(c, x_host, labels_host, grad_x_host, loss_host, false, 0.f, stream, false);
}

pfc_status pfc_train_step_host_async(pfc_ctx* c, const float* x_host, const int64_t* labels_host, float* grad_x_host,
                                     float* loss_host, float lr, void* stream) {
  return host_step(c, x_host, labels_host, grad_x_host, loss_host, true, lr, stream, false);
}

pfc_status pfc_forward_backward_host(pfc_ctx* c, const float* x_host, const int64_t* labels_host, float* grad_x_host,
                                     float* loss_host, void* stream) {
  return host_step(c, x_host, labels_host, grad_x_host, loss_host, false, 0.f, stream);
}

pfc_status pfc_train_step_host(pfc_ctx* c, const float* x_host, const int64_t* labels_host, float* grad_x_host,
                               float* loss_host, float lr, void* stream) {
  return host_step(c, x_host, labels_host, grad_x_host, loss_host, true, lr, stream);
}

pfc_status pfc_step(pfc_ctx* c, float lr, void* stream) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  if (!c->fb_done) return set_err(c, PFC_ERR_CONTRACT, "pfc_step without a preceding pfc_forward_backward");
  if (pfc_status pe = pending_error(c)) return pe;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  c->last_stream = s;
  if (c->prof) {
    prof_begin_step(c);
    mark(c, 9, s);
  }
  c->launches += launch_set_scalar(c->lr_dev, lr, s);
  c->launches += launch_sgd(c->sz, c->Wk(), c->Vk(), c->dWh, c->idxk(), c->inv_norm, c->st, c->lr_dev, c->cfg.momentum,
                            c->cfg.weight_decay, c->fused_gather ? 1 : 0, s);
  stage_out(c, true, s);
  if (c->prof) mark(c, 10, s);
  CUDA_TRY(c, cudaGetLastError());
  c->fb_done = false;
  if (c->sync_check) {
    CUDA_TRY(c, cudaStreamSynchronize(s));
    return device_error(c);
  }
  return PFC_OK;
}

pfc_status pfc_shard_range(const pfc_ctx* c, int64_t* start, int64_t* count) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  if (start) *start = c->sz.a;
  if (count) *count = c->sz.C_local;
  return PFC_OK;
}

pfc_status pfc_sizes(const pfc_ctx* c, int64_t* M, int64_t* k_max) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  if (M) *M = c->sz.M;
  if (k_max) *k_max = c->sz.k_max;
  return PFC_OK;
}

pfc_status pfc_param_ptrs(pfc_ctx* c, float** W, float** V) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  if (W) *W = c->W_host ? c->W_host : c->W;
  if (V) *V = c->V_host ? c->V_host : c->V;
  return PFC_OK;
}

static pfc_status sync_and_check(pfc_ctx* c) {
  CUDA_TRY(c, cudaSetDevice(c->cfg.device));
  if (pfc_status w = wait_stream(c, c->last_stream)) return w;
  CUDA_TRY(c, cudaDeviceSynchronize());
  return device_error(c);
}

pfc_status pfc_check(pfc_ctx* c) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  return sync_and_check(c);
}

pfc_status pfc_get_sampled(pfc_ctx* c, int64_t* idx_host, int64_t capacity, int64_t* k_out) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  pfc_status r = sync_and_check(c);
  if (r != PFC_OK) return r;
  SamplerState h;
  CUDA_TRY(c, cudaMemcpy(&h, c->st, sizeof(h), cudaMemcpyDeviceToHost));
  if (k_out) *k_out = h.k;
  if (!idx_host) return PFC_OK;
  if (capacity < h.k) return set_err(c, PFC_ERR_CONTRACT, "idx capacity < k_i");
  std::vector<int32_t> tmp(h.k);
  CUDA_TRY(c, cudaMemcpy(tmp.data(), c->idx, (size_t)h.k * 4, cudaMemcpyDeviceToHost));
  for (int i = 0; i < h.k; ++i) idx_host[i] = c->sz.a + tmp[i];
  return PFC_OK;
}

pfc_status pfc_get_sampled_grad(pfc_ctx* c, float* dW_host, int64_t capacity_rows) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  if (!c->fb_done) return set_err(c, PFC_ERR_CONTRACT, "no pending gradient (call before pfc_step)");
  pfc_status r = sync_and_check(c);
  if (r != PFC_OK) return r;
  SamplerState h;
  CUDA_TRY(c, cudaMemcpy(&h, c->st, sizeof(h), cudaMemcpyDeviceToHost));
  if (capacity_rows < h.k) return set_err(c, PFC_ERR_CONTRACT, "capacity_rows < k_i");
  float* tmp = nullptr;
  const size_t bytes = (size_t)h.k * c->sz.d * 4;
  CUDA_TRY(c, cudaMalloc(&tmp, std::max<size_t>(bytes, 16)));
  c->launches += launch_raw_grad(c->sz, c->Wk(), c->dWh, c->idxk(), c->inv_norm, c->st, tmp, c->fused_gather ? 1 : 0, 0);
  cudaError_t e = cudaMemcpy(dW_host, tmp, bytes, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  CUDA_TRY(c, e);
  return PFC_OK;
}

pfc_status pfc_get_lse(pfc_ctx* c, float* lse_host, int64_t capacity) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  if (capacity < c->sz.M) return set_err(c, PFC_ERR_CONTRACT, "capacity < M");
  pfc_status r = sync_and_check(c);
  if (r != PFC_OK) return r;
  CUDA_TRY(c, cudaMemcpy(lse_host, c->lse, (size_t)c->sz.M * 4, cudaMemcpyDeviceToHost));
  return PFC_OK;
}

pfc_status pfc_get_metrics(pfc_ctx* c, float* loss, float* ca_pcc) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  pfc_status r = sync_and_check(c);
  if (r != PFC_OK) return r;
  float h[2];
  CUDA_TRY(c, cudaMemcpy(h, c->metrics, sizeof(h), cudaMemcpyDeviceToHost));
  if (loss) *loss = h[0];
  if (ca_pcc) *ca_pcc = h[1];
  return PFC_OK;
}

pfc_status pfc_get_step(const pfc_ctx* c, uint64_t* step) {
  if (!c || !step) return set_err(nullptr, PFC_ERR_CONTRACT, "NULL argument");
  *step = c->step;
  return PFC_OK;
}

pfc_status pfc_set_step(pfc_ctx* c, uint64_t step) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  CUDA_TRY(c, cudaDeviceSynchronize());
  CUDA_TRY(c, cudaMemcpy(c->step_dev, &step, sizeof(step), cudaMemcpyHostToDevice));
  c->step = step;
  c->fb_done = false;
  return PFC_OK;
}

pfc_status pfc_get_state(pfc_ctx* c, float* W_host, float* V_host, uint64_t* step) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  const size_t bytes = (size_t)c->sz.C_local * c->sz.d * sizeof(float);
  CUDA_TRY(c, cudaDeviceSynchronize());
  if (W_host) CUDA_TRY(c, cudaMemcpy(W_host, c->W, bytes, cudaMemcpyDefault));
  if (V_host) CUDA_TRY(c, cudaMemcpy(V_host, c->V, bytes, cudaMemcpyDefault));
  if (step) *step = c->step;
  return device_error(c);
}

pfc_status pfc_set_state(pfc_ctx* c, const float* W_host, const float* V_host, const uint64_t* step) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  const size_t bytes = (size_t)c->sz.C_local * c->sz.d * sizeof(float);
  CUDA_TRY(c, cudaDeviceSynchronize());
  if (W_host) CUDA_TRY(c, cudaMemcpy(c->W, W_host, bytes, cudaMemcpyDefault));
  if (V_host) CUDA_TRY(c, cudaMemcpy(c->V, V_host, bytes, cudaMemcpyDefault));
  if (step) {
    CUDA_TRY(c, cudaMemcpy(c->step_dev, step, sizeof(*step), cudaMemcpyHostToDevice));
    c->step = *step;
  }
  c->fb_done = false;
  return PFC_OK;
}

int64_t pfc_launch_count(const pfc_ctx* c) { return c ? c->launches : 0; }

uint32_t pfc_path_flags(const pfc_ctx* c) {
  if (!c) return 0u;
  return (c->use_tc ? PFC_PATH_TENSOR_CORES : 0u) | (c->fused_gather ? PFC_PATH_FUSED_GATHER : 0u) |
         (c->use_dwx ? PFC_PATH_FUSED_DWX : 0u) | (c->eform || c->eform_pair ? PFC_PATH_EFORM : 0u);
}

static const char* kSectionNames[PFC_PROF_SECTIONS] = {
    "normalize_x", "sampler", "gather_w", "logits_gemm", "row_lse", "softmax_grad", "dx_gemm", "xnorm_backward",
    "dw_gemm", "sgd"};

const char* pfc_profile_section(int32_t i) { return (i >= 0 && i < PFC_PROF_SECTIONS) ? kSectionNames[i] : nullptr; }

pfc_status pfc_profile_enable(pfc_ctx* c, int32_t enable) {
  if (!c) return set_err(nullptr, PFC_ERR_CONTRACT, "ctx is NULL");
  c->prof = enable != 0;
  c->prof_used = 0;
  c->prof_cur = nullptr;
  return PFC_OK;
}

pfc_status pfc_profile_read(pfc_ctx* c, double* ms, int64_t* count) {
  if (!c || !ms || !count) return set_err(c, PFC_ERR_CONTRACT, "NULL argument");
  CUDA_TRY(c, cudaDeviceSynchronize());
  for (size_t st = 0; st < c->prof_used; ++st) {
    auto& ev = c->prof_ev[st];
    auto& set = c->prof_set[st];
    for (int b = 0; b < PFC_PROF_SECTIONS; ++b) {
      if (!set[b] || !set[b + 1]) continue;
      float t = 0.f;
      if (cudaEventElapsedTime(&t, ev[b], ev[b + 1]) == cudaSuccess) {
        ms[b] += t;
        count[b] += 1;
      }
    }
  }
  cudaGetLastError();
  c->prof_used = 0;
  c->prof_cur = nullptr;
  return PFC_OK;
}

pfc_status pfc_sample_shard(int64_t C, int32_t world, int32_t rank, double r, uint64_t seed, uint64_t step,
                            const int64_t* labels, int32_t M, int32_t sample_mode, int64_t* idx_out, int64_t* k_out,
                            void* stream) {
  if (!labels || !idx_out || !k_out || M < 1) return set_err(nullptr, PFC_ERR_CONTRACT, "bad arguments");
  if (world < 1 || rank < 0 || rank >= world || C < world || !(r > 0.0 && r <= 1.0))
    return set_err(nullptr, PFC_ERR_CONFIG, "bad shard configuration");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  Sizes sz{};
  sz.C = C; sz.world = world; sz.rank = rank; sz.M = M;
  sz.C_local = C / world + (rank < C % world ? 1 : 0);
  sz.a = (int64_t)rank * (C / world) + std::min<int64_t>(rank, C % world);
  sz.budget = (int64_t)std::ceil(r * (double)sz.C_local);
  sz.rate = r;
  sz.sample_mode = sample_mode;
  sz.k_max = std::min<int64_t>(sz.C_local, sz.budget + 1 + std::min<int64_t>(M, sz.C_local));
  sz.ntiles_sel = (int)((sz.C_local + kSelTile - 1) / kSelTile);
  uint32_t *bits = nullptr, *keys = nullptr;
  int *hist = nullptr, *tile = nullptr, *err = nullptr;
  SamplerState* st = nullptr;
  int32_t *idx = nullptr, *tcol = nullptr;
  uint64_t* step_dev = nullptr;
  cudaError_t e = cudaSuccess;
  auto A = [&](void** p, size_t b) { if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(b, 16)); };
  A((void**)&bits, ((sz.C_local + 31) / 32) * 4);
  A((void**)&keys, (size_t)sz.ntiles_sel * kSelTile * 4);
  A((void**)&hist, 5120 * 4);
  A((void**)&tile, (size_t)sz.ntiles_sel * 16);
  A((void**)&err, 16);
  A((void**)&st, sizeof(SamplerState));
  A((void**)&idx, sz.k_max * 4);
  A((void**)&tcol, (size_t)M * 4);
  A((void**)&step_dev, 16);
  pfc_status res = PFC_OK;
  if (e != cudaSuccess) {
    res = set_err(nullptr, PFC_ERR_OOM, cudaGetErrorString(e));
  } else {
    cudaMemsetAsync(err, 0, 16, s);
    cudaMemcpyAsync(step_dev, &step, sizeof(step), cudaMemcpyHostToDevice, s);
    launch_sampler(sz, labels, seed, step_dev, bits, keys, hist, tile, st, idx, tcol, err, s);
    launch_idx_to_global(sz.k_max, idx, st, sz.a, idx_out, s);
    SamplerState h{};
    int herr = 0;
    cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) res = set_err(nullptr, PFC_ERR_CUDA, cudaGetErrorString(e));
    else if (herr & ERR_INTERNAL) res = set_err(nullptr, PFC_ERR_CUDA, "sampler consistency check failed");
    *k_out = h.k;
  }
  cudaFree(bits); cudaFree(keys); cudaFree(hist); cudaFree(tile); cudaFree(err); cudaFree(st); cudaFree(idx);
  cudaFree(tcol); cudaFree(step_dev);
  return res;
}

}  // extern "C"
