/*
 * hdc.h -- C ABI of libhdc.so: batched HDC inference on B200 (sm_100a).
 *
 * The operation (ScalableHD, arXiv 2506.09282; PAPER.md line numbers "P:n"):
 *   Alg. 1 "Two-Stage HDC Inference", batch form P:171-190:
 *     Stage I    H = HardSign(X B)        eq. batch_encode
 *                HardSign(v) = +1 if v >= 0 else -1   eq. hardsign
 *     Stage II   S = H C^T                eq. batch_sim
 *                y = argmax_k S[n, k]     eq. pred_batch
 *   with X (N x F), B (F x D, the base HVs), C (K x D, the paper's class matrix M).
 *   Ties in the argmax go to the LOWEST class index (the paper is silent;
 *   DESIGN.md reading R2).  HardSign(-0.0) = +1 (reading R1).
 *
 * Conventions for every entry point:
 *   - All matrices are row-major, fp32, and DEVICE pointers unless the name says
 *     _host.  They are caller-owned; the library never frees or retains them
 *     beyond the call (hdc_model_create copies B and C into its own layout).
 *   - Calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream) and return after enqueue, except hdc_model_create /
 *     hdc_model_destroy which synchronise the device.
 *   - Synchronous argument errors return HDC_ERR_INVALID_VALUE (bad sizes, NULL
 *     required pointer, K > HDC_MAX_K) or HDC_ERR_MISALIGNED (pointer not 4-byte
 *     aligned; labels 4-byte).  Asynchronous device faults surface as
 *     HDC_ERR_CUDA on the next call (cuBLAS convention).
 *   - Non-finite inputs are not checked on the hot path; outputs are then
 *     unspecified.
 *   - Determinism: the same inputs, precision and path give bit-identical
 *     scores and labels (fixed-order reductions; cross-CTA sums only in integers).
 *     The tensor-core kernels (TF32 / BF16 / FP32_TC fused kernel, and the FP32_TC
 *     small-batch kernel) add each row's per-tile Stage II scores EXACTLY, in int64
 *     fixed point, so a row's scores and label do not depend on N, on how a batch is
 *     split into calls or shards, or on the launch configuration.  The fp32 streaming
 *     kernel (small batches) also sums its CTA partials in int64 and adds sign-recheck
 *     corrections as integers: a row's scores do not depend on the other rows of the
 *     batch for a given B stream (N = 1 on sign-exact models streams B's bf16 hi plane,
 *     N >= 2 the fp32 B; the two differ in the last bits of Stage II's fp32 sums, never
 *     in the signs).  The fp32 FFMA large-batch kernel sums D-split partials in fp32 in
 *     an order that depends on N: its scores may differ in the last bits between batch
 *     sizes (labels only at near-ties).
 *   - A model handle is immutable after creation but owns a workspace: calls on
 *     ONE handle must be serialised (one stream at a time); use one handle per
 *     concurrent stream.
 */
#ifndef HDC_H_
#define HDC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HDC_MAX_K 256

typedef enum {
  HDC_OK = 0,
  HDC_ERR_INVALID_VALUE = 1,
  HDC_ERR_MISALIGNED = 2,
  HDC_ERR_UNSUPPORTED = 3,
  HDC_ERR_NO_MEMORY = 4,
  HDC_ERR_CUDA = 5
} hdc_status_t;

/* Arithmetic of Stage I.  The paper keeps B and M in fp32.
 *   HDC_PREC_FP32: HardSign decisions equal those of the exact product X B.  Served by
 *     the HDC_PREC_FP32_TC kernels below (same guarantee, ~12x faster) when K <= 32 and
 *     F <= 100000, else -- or when the environment variable HDC_FP32_FFMA is set at
 *     hdc_model_create -- by the fp32 FFMA kernels: fp32 FFMA accumulation + float64
 *     re-evaluation of every pre-activation whose |v| is within the rigorous fp32 error
 *     bound (F+32) 2^-24 ||x_n|| ||b_d|| (DESIGN.md §4 "sign recheck").
 *   HDC_PREC_TF32 / HDC_PREC_BF16: Stage I on tcgen05 tensor cores with X and B
 *     rounded to tf32 (RNA) / bf16 (RN), fp32 accumulation; no recheck
 *     (approximate H).  Stage II on tcgen05 with C split into bf16 hi + lo.
 *   HDC_PREC_FP32_TC: sign-exact Stage I on the int8 tensor cores: each row of
 *     X and column of B is scaled to a 21-bit integer image split into three
 *     int8 limbs; the six limb products of weight >= 2^-14 accumulate EXACTLY
 *     in int32 (tcgen05 kind::i8); every pre-activation within the rigorous
 *     bound of that image is re-evaluated in float64 -> HardSign decisions
 *     equal those of the exact product.  Stage II on tcgen05 with
 *     C split into bf16 hi + lo (fp32 accumulation); where a re-evaluated sign
 *     differs from the provisional one, S is corrected exactly (int64 fixed point).
 *     Falls back to the HDC_PREC_FP32 kernels (same guarantee) when K > 32 or
 *     F > 100000.  Low-precision modes fall back likewise when K > 64. */
typedef enum {
  HDC_PREC_FP32 = 0,
  HDC_PREC_TF32 = 1,
  HDC_PREC_BF16 = 2,
  HDC_PREC_FP32_TC = 3
} hdc_precision_t;

/* Kernel selection (diagnostics and tests; HDC_PATH_AUTO is the product path).
 *   SMALL: bandwidth-bound D-split kernel (streams B and C once per 32 rows; fp32).
 *   FUSED: large-batch fused kernel (H never leaves the chip).
 * AUTO: SMALL for N <= 32 (N <= 8 for TF32 / BF16 models), else FUSED. */
typedef enum { HDC_PATH_AUTO = 0, HDC_PATH_SMALL = 1, HDC_PATH_FUSED = 2 } hdc_path_t;

typedef struct hdc_model_s* hdc_model_t;

/* One-shot inference (BASELINE north_star "hdc_infer(X, B, C, N, F, D, K) ->
 * labels plus optional scores").  Builds a temporary model (copies B, C),
 * runs, and releases it; the copies and allocations are inside the call, which
 * therefore synchronises the device (like hdc_model_create/destroy).
 *   X [N*F], B [F*D], C [K*D]: inputs.   N >= 0, F >= 1, D >= 1, 1 <= K <= 256.
 *   labels [N] int32 (required when N > 0): y_pred, values in [0, K).
 *   scores [N*K] fp32 (nullable): S. */
hdc_status_t hdc_infer(const float* X, const float* B, const float* C, int64_t N, int64_t F,
                       int64_t D, int64_t K, int32_t* labels, float* scores,
                       hdc_precision_t prec, void* stream);

/* Amortised setup: copies B and C (device pointers) into the model's padded
 * layouts and precomputes per-column norms ||b_d|| (sign recheck) and any
 * low-precision operand copies `prec` needs.  Timed latency excludes this, as
 * the paper's pre-tiled B and J.  Synchronises the device. */
/* (C may be NULL: encoder-only model for hdc_model_encode; K still sets the class count.) */
hdc_status_t hdc_model_create(const float* B, const float* C, int64_t F, int64_t D, int64_t K,
                              hdc_precision_t prec, hdc_model_t* out);

/* Inference on a resident model.  X [N*F] device; labels [N]; scores [N*K] or NULL. */
hdc_status_t hdc_model_infer(hdc_model_t m, const float* X, int64_t N, int32_t* labels,
                             float* scores, void* stream);

/* Same, with an explicit kernel path (see hdc_path_t). */
hdc_status_t hdc_model_infer_path(hdc_model_t m, const float* X, int64_t N, int32_t* labels,
                                  float* scores, hdc_path_t path, void* stream);

/* End-to-end variant on HOST buffers: copies X_host (N*F fp32) to the device,
 * runs hdc_model_infer, copies labels (and scores if non-NULL) back.  The
 * host-to-device copies run on a library-owned copy stream into one of two
 * staging buffers, so back-to-back calls pipeline: the copy of call i + 1 overlaps
 * the inference of call i.  For N > 32 the rows are also processed in up to 8
 * chunks of ~8192, the copy of chunk j + 1 overlapping the inference of chunk j
 * (rows are independent: on the tensor-core kernels the results equal the
 * one-shot call bit for bit; on the fp32 FFMA kernels up to fp32 summation order, see
 * Determinism above).
 * Ordering: the copies of X_host are ordered after this model's previous host-path
 * calls, NOT after other work already queued on `stream` -- X_host must be fully
 * written when the call is made.  Labels / scores are written in `stream` order:
 * directly by the kernels when the host buffers are mapped pinned memory (cudaHostAlloc,
 * or any pinned allocation under unified addressing), else by device-to-host copies.
 * Host buffers should be pinned (cudaHostAlloc) for the copies to be
 * asynchronous; the call returns after enqueue -- synchronise `stream` before
 * reading the outputs or reusing X_host.  Concurrent host-path calls on the same
 * model must be serialised by the caller (they share the staging buffers). */
hdc_status_t hdc_model_infer_host(hdc_model_t m, const float* X_host, int64_t N,
                                  int32_t* labels_host, float* scores_host, void* stream);

/* D-shard piece (Alg. 3's per-worker S_local over its D column blocks):
 * the model holds this rank's D-slice of B and C; writes the partial scores
 * S_partial [N*K] = HardSign(X B_r) C_r^T (no argmax).  The caller sums the
 * partials over ranks (Alg. 3 line `S += S_local`) and calls hdc_argmax. */
hdc_status_t hdc_model_partial_scores(hdc_model_t m, const float* X, int64_t N, float* S_partial,
                                      void* stream);

/* D-shard inference with the reduction inside the kernel (Alg. 3 `S += S_local`, P:336,
 * across GPUs; SURVEY §8 f2 over peer memory): every rank calls this with its D-slice
 * model, the same X (N rows, 1 <= N <= 32), the same `epoch` (a call counter that
 * increases by one per call, identical on all ranks) and `xbufs`, a DEVICE array of
 * `world` pointers: the exchange buffer of each rank, mapped into this process (CUDA IPC
 * / symmetric memory; xbufs[rank] is this rank's own).  Each buffer holds
 * hdc_dshard_exchange_bytes(N, K, world) bytes (world uint32 signal words, padded to 16
 * bytes, then 2 x world slots of 32*K floats: slots are sized for the largest N, so one
 * buffer serves every 1 <= N <= 32 and N may change from call to call) and must be zeroed
 * once before the first call (epoch 1 is the first valid epoch).  The N argument of
 * hdc_dshard_exchange_bytes is only validated (0 is returned outside 1..32).  The small-batch kernel's last CTA stores this
 * rank's partial scores into every rank's buffer (peer stores), release-signals them,
 * waits until all ranks' partials arrived and sums them in rank order, so labels and
 * scores (N*K, optional) are identical on every rank.  One launch, no NCCL.  The ranks'
 * kernels wait on one another: launch them on different GPUs only.
 * Errors: UNSUPPORTED (N > 32, shapes outside the streaming kernel), INVALID_VALUE. */
int64_t hdc_dshard_exchange_bytes(int64_t N, int64_t K, int world);
hdc_status_t hdc_model_infer_dshard(hdc_model_t m, const float* X, int64_t N, int32_t* labels,
                                    float* scores, float* const* xbufs, int rank, int world,
                                    uint32_t epoch, void* stream);

/* Row argmax, lowest index among equal maxima: labels[n] = argmax_k S[n*K+k]. */
hdc_status_t hdc_argmax(const float* S, int64_t N, int64_t K, int32_t* labels, void* stream);

/* ---- Materialised H: encoding, unfused similarity (ablation), single-pass training ----
 * Bit-packed layout of H (N x D signs): row n, column d at word H[n*ldw + d/32],
 * bit d%32; the bit is SET iff h[n,d] = -1 (HardSign).  ldw >= ceil(D/32).
 *
 * Stage I alone, H = HardSign(X B) (eq. batch_encode), written to
 * H [N*ldw] (device, caller-owned, cleared by the call).  The model must use a
 * tensor-core precision; HDC_PREC_FP32_TC gives the exact signs of the fp32 product
 * (float64 re-evaluation of the bound-flagged ones).  A model created
 * with C == NULL is an encoder-only model (hdc_model_infer rejects it).
 * Errors: INVALID_VALUE (null pointers, ldw too small), UNSUPPORTED (FP32 FFMA model,
 * N >= 2^31), MISALIGNED (4-byte alignment). */
hdc_status_t hdc_model_encode(hdc_model_t m, const float* X, int64_t N, uint32_t* H, int64_t ldw,
                              void* stream);

/* Stage II + argmax from a packed H (the unfused variant of Alg. 1 used to measure
 * what fusion saves): S[n,k] = sum_d h[n,d] C[k,d] (d ascending,
 * fp32), labels = lowest-index argmax.  C [K*D] fp32 device; labels [N] and/or
 * scores [N*K] (either may be NULL, not both).  K <= 64. */
hdc_status_t hdc_similarity_packed(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C,
                                   int64_t K, int32_t* labels, float* scores, void* stream);

/* Single-pass training (constrained bundling P:94-105): for labels y [N] in
 * [0, K), counts[k*D+d] += sum_{n: y_n = k} h[n,d] (int32, exact, accumulates: clear it
 * first), and if M != NULL the class HVs M[k*D+d] = HardSign(counts) = +1 / -1 (fp32,
 * ties +1).  Synchronises `stream` to validate the labels (INVALID_VALUE if any is out
 * of range). */
hdc_status_t hdc_bundle_classes(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const int32_t* y,
                                int64_t K, int32_t* counts, float* M, void* stream);

/* Releases the model and its device memory.  Synchronises the device. */
hdc_status_t hdc_model_destroy(hdc_model_t m);

/* Model dimensions (any out pointer may be NULL). */
hdc_status_t hdc_model_dims(hdc_model_t m, int64_t* F, int64_t* D, int64_t* K,
                            hdc_precision_t* prec);

/* Cumulative number of float64 sign re-evaluations performed by all calls on
 * this model since creation; synchronises the device (diagnostic; -1 on error). */
int64_t hdc_model_recheck_count(hdc_model_t m);

/* Number of kernel launches the last call on this model enqueued. */
int32_t hdc_model_last_launch_count(hdc_model_t m);

/* Kernel family that computed the last call on this model (diagnostic; -1 on a NULL
 * model).  The arithmetic differs by family, which is what the parity tests key on:
 *   HDC_KERNEL_SMALL:    fp32 streaming D-split kernel (sign-exact, any precision's model);
 *   HDC_KERNEL_FFMA:     fp32 fused FFMA kernel (sign-exact);
 *   HDC_KERNEL_TC:       fused tcgen05 kernel in the model's precision;
 *   HDC_KERNEL_SMALL_TC: int8 tensor-core streaming D-split kernel (HDC_PREC_FP32_TC models,
 *                        N <= 32; sign-exact). */
typedef enum {
  HDC_KERNEL_NONE = 0,
  HDC_KERNEL_SMALL = 1,
  HDC_KERNEL_FFMA = 2,
  HDC_KERNEL_TC = 3,
  HDC_KERNEL_SMALL_TC = 4
} hdc_kernel_t;
int32_t hdc_model_last_kernel(hdc_model_t m);

/* D-tile width of this model's fused tensor-core kernel (diagnostic): 80 or 160 columns,
 * 0 if the model has no tensor-core path, -1 on a NULL model.  int8 models (fp32_tc, and
 * fp32 when routed) with K <= 16 and padded F >= 768 run the "wide" K4 variant, 160-column
 * tiles of two 80-column sub-tiles; the environment variable HDC_TC_WIDE=0/1,
 * read at model creation, overrides the F threshold (measurements). */
int32_t hdc_model_tc_tile_n(hdc_model_t m);

/* Diagnostics for roofline reporting: when enabled, each call records CUDA
 * events on its stream around its dominant kernel (the fused kernel, or the
 * small-batch launches); hdc_model_last_kernel_ms synchronises on the last
 * call's end event and returns the elapsed milliseconds (-1 if unavailable). */
hdc_status_t hdc_model_set_kernel_timing(hdc_model_t m, int enable);
float hdc_model_last_kernel_ms(hdc_model_t m);

const char* hdc_status_string(hdc_status_t st);
/* Detail for the last failing call on this thread (thread-local, never NULL). */
const char* hdc_last_error(void);
/* Library version string. */
const char* hdc_version(void);

/* Diagnostic (measurement only): read `bytes` bytes of the device buffer `buf` once with
 * 1-D bulk copies, each SM one contiguous range through an 8 x 16 KB shared-memory ring --
 * the one-shot streaming ceiling of a read of that size, against which bench.py reads the
 * small-batch kernels' HBM fraction.  `buf` and `bytes` 16-byte aligned; asynchronous. */
hdc_status_t hdc_diag_stream_read(const void* buf, int64_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HDC_H_ */
