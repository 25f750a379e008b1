/*
 * pfc.h — C-ABI of the B200-native Partial FC layer (arXiv 2010.05222, /root/reference/PAPER.md).
 *
 * One context per process / rank / GPU. The layer owns one contiguous shard of the class-centre matrix W
 * ("partition W into k sub-matrices w of size d x C/k and place the i-th on the i-th GPU", PAPER.md:102;
 * "evenly divided ... according to the order") together with its momentum buffer V
 * ("each parameter will occupy 12 bytes, as we use momentum SGD").
 *
 * Conventions for every entry point
 *   - Pointers named *_dev are device pointers on cfg.device; *_host are host pointers. All are owned by
 *     the caller and must stay valid until the work enqueued on `stream` has completed.
 *   - `stream` is a cudaStream_t passed as void*. NULL means the legacy default stream.
 *     Work is enqueued asynchronously; no entry point of the hot path synchronises the host.
 *   - Layouts are row-major, dense: x is [B][d] float32, grad_x is [B][d] float32, labels is [B] int64,
 *     W and V are [C_local][d] float32 (row j = class centre a_i + j).
 *   - Collective contract (world_size > 1): every rank calls the hot-path entry points in the same order
 *     with the same B (Alg.1 is a collective program).
 *   - Host-detectable errors are returned synchronously and leave the context unchanged. Errors found on
 *     the device (label outside [0, C), zero-norm row, non-finite loss, an internal consistency check) set a
 *     sticky device word. The last kernel of every step mirrors it into page-locked host memory, and every
 *     hot-path entry point (pfc_forward_backward, pfc_train_step, pfc_step, the *_host and group variants)
 *     checks that mirror first, without synchronising: an error of an earlier, completed step is returned by the
 *     next call. Synchronising calls (pfc_check, pfc_get_*) report it at once; PFC_SYNC_CHECK=1 makes every
 *     step synchronise and report its own error.
 *   - NCCL: host waits poll ncclCommGetAsyncError; an asynchronous error or a collective exceeding
 *     PFC_NCCL_TIMEOUT_S seconds (default 600) aborts the communicator and returns PFC_ERR_NCCL.
 *   - Not re-entrant: one host thread per context.
 */
#ifndef PFC_H_
#define PFC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PFC_OK = 0,
  PFC_ERR_CONFIG = 1,      /* invalid pfc_config (C < world_size, r outside (0,1], bad margin, d % 128 != 0 ...) */
  PFC_ERR_CONTRACT = 2,    /* NULL / misaligned pointer, wrong call order (pfc_step without forward_backward) */
  PFC_ERR_DATA = 3,        /* a label outside [0, C) (device-detected) */
  PFC_ERR_DEGENERATE = 4,  /* a zero-norm feature or class-centre row (norm clamped to 1e-12, reported) */
  PFC_ERR_NUMERIC = 5,     /* non-finite loss */
  PFC_ERR_CUDA = 6,        /* CUDA runtime error (message in pfc_last_error) */
  PFC_ERR_NCCL = 7,        /* NCCL error */
  PFC_ERR_OOM = 8          /* device allocation failed */
} pfc_status;

typedef enum { PFC_MARGIN_NONE = 0, PFC_MARGIN_ARCFACE = 1, PFC_MARGIN_COSFACE = 2 } pfc_margin;

/* Arithmetic of the three contractions. PFC_BF16: bf16 operands on the tcgen05 tensor cores with fp32
 * accumulation, cosines stored as fp16, target cosine refined in fp32. PFC_FP32: fp32 FFMA throughout. */
typedef enum { PFC_FP32 = 0, PFC_BF16 = 1 } pfc_precision;

/* How the world_size ranks exchange data.
 * PFC_COMM_NCCL: one process per GPU, NCCL all-gather / all-reduce / reduce-scatter over NVLink.
 * PFC_COMM_LOOPBACK: all world_size contexts live in ONE process (any devices, typically one GPU) and are
 *   driven together by pfc_group_forward_backward; the collectives are rank-ordered device copies and
 *   rank-ascending sums (the single-matrix form of Alg.1). Used for multi-rank parity on one GPU and for the
 *   per-rank solo timing of the scaling study. pfc_forward_backward rejects such a context when world_size > 1.
 * PFC_COMM_NCCL_FUSED: one process per GPU, the collectives fused into the step's kernels over NVLink peer memory
 *   (Fig.4): the normalisation kernel stores x_hat and the labels straight into
 *   every peer (Alg.1 L2), the row-combine / prep kernels store the row maxima and sums into the peers' slots and
 *   read all ranks' in rank order (Alg.1 L6-7), the dX reduction stores each owner's rows into the
 *   owner's slot (Alg.1 L12-13). The exchange region is an NCCL 2.28 symmetric window (ncclMemAlloc +
 *   ncclCommWindowRegister), synchronised by device-side LSA barriers; all ranks must share one NVLink domain.
 *   At world_size 1 it runs the same kernels and barriers on a 1-rank communicator. Results are deterministic
 *   (rank-ordered reductions) and equal PFC_COMM_LOOPBACK_FUSED's.
 * PFC_COMM_LOOPBACK_FUSED: a loopback group (as PFC_COMM_LOOPBACK, driven by pfc_group_forward_backward) whose
 *   collectives are those fused kernels storing into the other contexts' exchange regions. */
typedef enum {
  PFC_COMM_NCCL = 0,
  PFC_COMM_LOOPBACK = 1,
  PFC_COMM_NCCL_FUSED = 2,
  PFC_COMM_LOOPBACK_FUSED = 3
} pfc_comm_mode;

/* Which classes a shard samples (R1, R23, R24).
 * PFC_SAMPLE_PPRN       north_star rule: every positive + negatives up to k_i = max(ceil(r C_local), |P_i|).
 * PFC_SAMPLE_PPRN_PAPER the paper's step 2: |P_i| positives + round((C_local - |P_i|) r)
 *                       negatives (round half up); k_i differs between ranks.
 * PFC_SAMPLE_RANDOM     fully random (the Fig.3 baseline): ceil(r C_local) classes of the whole
 *                       shard, labels ignored; a row whose positive is not sampled keeps Eq.9's denominator over the
 *                       sampled set and gets no positive pull. */
typedef enum { PFC_SAMPLE_PPRN = 0, PFC_SAMPLE_PPRN_PAPER = 1, PFC_SAMPLE_RANDOM = 2 } pfc_sample_mode;

/* Where the W and V shards live (the paper keeps W in host RAM past GPU memory, PAPER.md:344,
 * PAPER.md:357).
 * PFC_PARAMS_DEVICE  HBM (the default; up to ~100M classes per 8 B200).
 * PFC_PARAMS_HOST    page-locked, device-mapped host memory: the same kernels gather the sampled rows and write
 *                    their updates through the mapping (PCIe / C2C bandwidth instead of HBM); capacity mode for
 *                    shards beyond HBM. The rest of the workspace stays in HBM. */
typedef enum { PFC_PARAMS_DEVICE = 0, PFC_PARAMS_HOST = 1 } pfc_param_location;

typedef struct {
  int64_t num_classes;   /* C >= world_size      */
  int32_t dim;           /* d, multiple of 128 in [128, 1024] (512 in the paper)      */
  int32_t batch;         /* N = B, features per rank, equal on all ranks, >= 1      */
  double sample_rate;    /* r in (0, 1]      */
  float scale;           /* s > 0 (64 in the paper)      */
  int32_t margin_type;   /* pfc_margin      */
  float margin;          /* ArcFace 0 <= m < pi/2 (0.5); CosFace 0 <= m < 1 (0.4)      */
  float momentum;        /* mu in [0, 1)      */
  float weight_decay;    /* lambda >= 0 (the paper is silent; explicit)                                 */
  int32_t precision;     /* pfc_precision                                                               */
  uint64_t seed;         /* keys the Philox negative sampler (R2)                             */
  int32_t rank;          /* i in [0, world_size)                                                        */
  int32_t world_size;    /* k >= 1                                                                      */
  int32_t device;        /* CUDA device ordinal for this rank                                            */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId from pfc_get_unique_id on rank 0, broadcast by the
                                 caller (e.g. over torch.distributed); required iff world_size > 1 and
                                 comm_mode is PFC_COMM_NCCL or PFC_COMM_NCCL_FUSED                        */
  int32_t comm_mode;     /* pfc_comm_mode                                                                */
  int32_t sample_mode;   /* pfc_sample_mode                                                              */
  int32_t param_location; /* pfc_param_location                                                         */
  int32_t ignore_index;  /* 0: every label must be in [0, C) (else PFC_ERR_DATA). 1: a label of -1 marks an
                            ignored row (PyTorch ignore_index = -1, R28): it
                            contributes no loss and receives zero grad_x; the mean of Eq.5 and the gradients
                            divide by the number of rows not ignored (global over the ranks; 1 if all are)     */
} pfc_config;

typedef struct pfc_ctx pfc_ctx;

/* ------------------------------------------------------------------------------------------------------
 * Lifecycle
 * ---------------------------------------------------------------------------------------------------- */

/* Writes a fresh 128-byte NCCL unique id into id_out (host buffer of >= 128 bytes). Call on rank 0 only. */
pfc_status pfc_get_unique_id(void* id_out_host);

/* Validates cfg, selects cfg->device, computes the shard [a_i, a_i + C_local) (balanced, first C mod k
 * ranks get one more row; R6), allocates W and V (zero-filled) and the step workspace, and
 * creates the NCCL communicator when world_size > 1. *out receives the context (NULL on error). */
pfc_status pfc_init(const pfc_config* cfg, pfc_ctx** out);

/* Frees all device memory and the communicator. NULL is a no-op. */
pfc_status pfc_destroy(pfc_ctx* ctx);

/* Text of the last error of ctx (or of the last failed pfc_init when ctx is NULL). Never NULL. */
const char* pfc_last_error(const pfc_ctx* ctx);

/* ------------------------------------------------------------------------------------------------------
 * Hot path
 * ---------------------------------------------------------------------------------------------------- */

/* One forward + backward pass of the sampled model-parallel margin-softmax layer on this rank
 * (Alg.1, with the PPRN sampler of PAPER.md:292-316 and Eq.9):
 *   X = allgather(x / ||x||) and labels; P_i = labels in this shard; k_i = max(ceil(r C_local), |P_i|);
 *   the k_i - |P_i| negatives with the smallest Philox keys (R1-R4); W_s = normalised sampled
 *   rows; logits = s * X W_s^T with the margin at each row's own class; global softmax over
 *   the union of all ranks' samples via all-reduce (Alg.1 L6-7); loss = mean over the global batch
 *   M = k B of the cross-entropy (Eq.5); grad_x = d loss / d x for this rank's B rows (Alg.1 L12-13);
 *   the gradient of the sampled W rows is kept for pfc_step.
 * x_dev      [B][d] float32 features of this rank (any norm > 0).
 * labels_dev [B] int64 global class ids in [0, C).
 * grad_x_dev [B][d] float32 output; may alias nothing else.
 * loss_dev   float32 scalar output (same value on every rank) or NULL.
 * Increments the context's step counter, which keys the sampler of the next call. */
pfc_status pfc_forward_backward(pfc_ctx* ctx, const float* x_dev, const int64_t* labels_dev,
                                float* grad_x_dev, float* loss_dev, void* stream);

/* One forward + backward of ALL ranks of a loopback group (comm_mode == PFC_COMM_LOOPBACK): ctxs[i] is rank
 * i (n == world_size, same config otherwise); x_dev[i], labels_dev[i], grad_x_dev[i] as in
 * pfc_forward_backward for rank i. loss_dev (or NULL) receives the loss. All work goes to `stream`. */
pfc_status pfc_group_forward_backward(pfc_ctx** ctxs, int32_t n, const float* const* x_dev,
                                      const int64_t* const* labels_dev, float* const* grad_x_dev, float* loss_dev,
                                      void* stream);

/* pfc_forward_backward followed by pfc_step(lr), fused: the momentum-SGD update of the sampled rows is applied
 * inside the dW contraction's epilogue (bf16 mode; the fp32 mode runs the same two kernels back to back), so
 * the sampled-row gradient is never written to HBM. Same results as the pair up to
 * rounding; afterwards no gradient is pending (pfc_get_sampled_grad / pfc_step return PFC_ERR_CONTRACT). */
pfc_status pfc_train_step(pfc_ctx* ctx, const float* x_dev, const int64_t* labels_dev, float* grad_x_dev,
                          float* loss_dev, float lr, void* stream);

/* pfc_group_forward_backward + update of every rank, fused as in pfc_train_step. */
pfc_status pfc_group_train_step(pfc_ctx** ctxs, int32_t n, const float* const* x_dev, const int64_t* const* labels_dev,
                                float* const* grad_x_dev, float* loss_dev, float lr, void* stream);

/* The same pass with HOST buffers: copies x and labels host->device and grad_x, loss device->host on
 * `stream` (pinned host memory gives asynchronous copies), then synchronises `stream`. loss_host may be
 * NULL. Used for the end-to-end measurement. */
pfc_status pfc_forward_backward_host(pfc_ctx* ctx, const float* x_host, const int64_t* labels_host,
                                     float* grad_x_host, float* loss_host, void* stream);

/* pfc_train_step with HOST buffers (copies inside, synchronises `stream`): the end-to-end entry point. */
pfc_status pfc_train_step_host(pfc_ctx* ctx, const float* x_host, const int64_t* labels_host, float* grad_x_host,
                               float* loss_host, float lr, void* stream);

/* The two host-buffer entries WITHOUT the final synchronisation: the copies and the step are enqueued on
 * `stream` and the call returns, so a training loop keeps the GPU fed (the next step is enqueued while this one
 * runs). The host buffers must be page-locked (pinned); x_host / labels_host must stay unmodified and
 * grad_x_host / loss_host are valid only after `stream` completes (cudaStreamSynchronize, or pfc_check).
 * Device-detected errors of the step are reported by the next call, as for pfc_train_step. */
pfc_status pfc_forward_backward_host_async(pfc_ctx* ctx, const float* x_host, const int64_t* labels_host,
                                           float* grad_x_host, float* loss_host, void* stream);
pfc_status pfc_train_step_host_async(pfc_ctx* ctx, const float* x_host, const int64_t* labels_host,
                                     float* grad_x_host, float* loss_host, float lr, void* stream);

/* Lazy momentum-SGD update of the rows sampled by the last pfc_forward_backward (DESIGN.md
 * R15): g = (dw_hat - w_hat (w_hat . dw_hat)) / ||w||; v <- mu v + g + lambda w; w <- w - lr v.
 * Rows not sampled are untouched. Returns PFC_ERR_CONTRACT if no forward_backward preceded it or it was
 * already applied. Reports sticky device errors (synchronises `stream`). */
pfc_status pfc_step(pfc_ctx* ctx, float lr, void* stream);

/* ------------------------------------------------------------------------------------------------------
 * Introspection, state and parity (synchronising; not on the hot path)
 * ---------------------------------------------------------------------------------------------------- */

/* Global start a_i and row count C_local of this rank's shard. */
pfc_status pfc_shard_range(const pfc_ctx* ctx, int64_t* start, int64_t* count);

/* Sizes: M = world_size * B, k_max = max(ceil(r C_local), min(M, C_local)) (the workspace bound). */
pfc_status pfc_sizes(const pfc_ctx* ctx, int64_t* M, int64_t* k_max);

/* Pointers to the library-owned W and V shards ([C_local][d] float32): device pointers with
 * PFC_PARAMS_DEVICE, host pointers (page-locked) with PFC_PARAMS_HOST. The caller may read or write them
 * between calls (stream-ordered on the stream it uses; host memory after synchronising it). */
pfc_status pfc_param_ptrs(pfc_ctx* ctx, float** W, float** V);

/* Sampled global class ids of the last forward_backward, ascending (R4), and k_i.
 * idx_host has room for `capacity` entries (>= k_i, else PFC_ERR_CONTRACT with *k_out set). */
pfc_status pfc_get_sampled(pfc_ctx* ctx, int64_t* idx_host, int64_t capacity, int64_t* k_out);

/* Gradient of the loss w.r.t. the raw W rows of the sampled set of the last forward_backward,
 * [k_i][d] float32 in the order of pfc_get_sampled. Must be called before pfc_step. */
pfc_status pfc_get_sampled_grad(pfc_ctx* ctx, float* dW_host, int64_t capacity_rows);

/* Per-row log-sum-exp over the global sampled set (M floats) of the last forward_backward. */
pfc_status pfc_get_lse(pfc_ctx* ctx, float* lse_host, int64_t capacity);

/* Loss (Eq.5) and CA_pcc (Eq.7: mean cos between each feature and its own class centre) of the
 * last forward_backward / train_step, synchronising. Either pointer may be NULL. */
pfc_status pfc_get_metrics(pfc_ctx* ctx, float* loss_host, float* ca_pcc_host);

/* Step counter (number of forward_backward calls since init / set). */
pfc_status pfc_get_step(const pfc_ctx* ctx, uint64_t* step);
pfc_status pfc_set_step(pfc_ctx* ctx, uint64_t step);

/* Checkpoint / resume: copy the whole shard state to or from host memory, synchronising the
 * device first. W_host, V_host: [C_local][d] float32 (row-major, C_local from pfc_shard_range), either may be NULL
 * to skip that tensor; step: the step counter (keys the sampler), NULL to skip. set_state also clears a pending
 * pfc_step. A resumed context continues bit-identically to the one the state was taken from. */
pfc_status pfc_get_state(pfc_ctx* ctx, float* W_host, float* V_host, uint64_t* step);
pfc_status pfc_set_state(pfc_ctx* ctx, const float* W_host, const float* V_host, const uint64_t* step);

/* Synchronises the context's last stream and returns the sticky device error (PFC_OK if none). */
pfc_status pfc_check(pfc_ctx* ctx);

/* Standalone sampler (K2-K4) of shard `rank` of `world_size` (no context), rule `sample_mode` (pfc_sample_mode):
 * labels_dev [M] int64 global labels of the global batch (device), idx_dev receives the k_i sampled global ids
 * ascending (device, room for min(C_local, ceil(r C_local) + 1 + min(M, C_local)) entries), *k_out = k_i (host;
 * synchronises `stream`).
 * Same arithmetic as inside pfc_forward_backward with the given `step`. */
pfc_status pfc_sample_shard(int64_t num_classes, int32_t world_size, int32_t rank, double sample_rate, uint64_t seed,
                            uint64_t step, const int64_t* labels_dev, int32_t M, int32_t sample_mode, int64_t* idx_dev,
                            int64_t* k_out, void* stream);

/* ------------------------------------------------------------------------------------------------------
 * Per-kernel timing (CUDA events recorded on the launching stream between the kernels of the step)
 * ---------------------------------------------------------------------------------------------------- */
#define PFC_PROF_SECTIONS 10
/* Sections: 0 normalize_x (+all-gather), 1 sampler, 2 gather_w (+target cos), 3 logits GEMM, 4 row combine +
 * all-reduces + finalize, 5 softmax_grad, 6 dx GEMM, 7 reduce-scatter + x-norm backward, 8 dw GEMM, 9 sgd. */
/* Enables (1) or disables (0) event recording; clears the accumulators. Not for loopback groups. */
pfc_status pfc_profile_enable(pfc_ctx* ctx, int32_t enable);
/* Synchronises, adds the elapsed time of every recorded step to ms[PFC_PROF_SECTIONS] (milliseconds) and the
 * number of recorded launches to count[PFC_PROF_SECTIONS], then clears the record. */
pfc_status pfc_profile_read(pfc_ctx* ctx, double* ms, int64_t* count);
/* Name of section i, or NULL. */
const char* pfc_profile_section(int32_t i);

/* Number of kernels this library launched since init (each launch counted once). */
int64_t pfc_launch_count(const pfc_ctx* ctx);

/* Kernel path chosen at init for this configuration (bit set = used), for reporting: */
#define PFC_PATH_TENSOR_CORES 1u  /* tcgen05 contractions (bf16 precision on sm_100) */
#define PFC_PATH_FUSED_GATHER 2u  /* gather + bf16 + norms + logits in one kernel (global batch M <= 256):
                                     profile section 3 then holds it and section 2 only the target cosines */
#define PFC_PATH_FUSED_DWX    4u  /* train step: dW + momentum SGD + dX_hat in one kernel (section 6; 8 empty) */
#define PFC_PATH_EFORM        8u  /* train step (bf16, tensor cores, s <= 80 and s + ln k_i < 80; R26): the
                                     logits kernel stores E = exp(s c) (bf16) and the dX / dW + SGD kernels contract
                                     it directly, no softmax-gradient pass. Section 5 then holds the per-row
                                     preparation (with FUSED_DWX) or that plus the radial-dot pass over E (M > 256).
                                     pfc_forward_backward keeps the softmax-gradient form. PFC_EFORM=0 at init
                                     disables. */
/* Returns the PFC_PATH_* bits (0 for a NULL context). */
uint32_t pfc_path_flags(const pfc_ctx* ctx);

/* Library version string. */
const char* pfc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PFC_H_ */
