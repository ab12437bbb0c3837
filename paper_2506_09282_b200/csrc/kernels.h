// kernels.h -- internal launch interface between the C ABI (hdc_api.cu) and the
// kernels.  Not installed; the public boundary is include/hdc.h.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace hdc {

// Model operands in the library's own layout (made by hdc_model_create).
struct ModelView {
  int64_t F, D, K;
  int64_t Fp;            // F padded to a multiple of kFPad (zero rows)
  int64_t Dp;            // D padded to a multiple of kDPad (zero columns)
  const float* Bp;       // Fp x Dp fp32, zero-padded rows and columns
  const float* Bt;       // Dp x Fp fp32: B transposed (fp64 sign recheck gathers)
  const float* B4;       // unit-major copy [Dp/4][Fp][4] (small-batch streaming)
  const float* Cp;       // K x Dp fp32, zero-padded columns
  const float* bnorm;    // Dp: ||b_d||_2 rounded up (0 on padding)
  float tau_coef;        // sign_bound_coef(F)
  const uint16_t* B4h = nullptr;   // bf16 hi plane of B4 (K2s sign-exact streaming), or null
  const float* hibound = nullptr;  // Dp: the hi plane's sign-bound coefficient (launch_hi_plane)
};

constexpr int64_t kDPad = 256;  // D padding granule (covers every kernel's D tile)
constexpr int64_t kFPad = 64;   // F padding granule (covers every kernel's K step)

// Workspace for the small-batch kernel's cross-CTA reduction.
struct SmallWorkspace {
  float* S_part;         // [num_sms][32][K]
  unsigned* cnt1;        // [64] last-arriver counters, zero between launches
  unsigned long long* recheck;  // fp64 re-evaluation counter (diagnostic)
  unsigned long long* acc;      // [32][K] int64 fixed-point score sums (K2s), zero between launches
  int shift;                    // fixed point: 2^-shift units (tc_corr_shift)
};

int64_t small_num_ctas(int64_t D, int num_sms);                       // CTAs of K2
int small_max_rows(int64_t F, int64_t D, int64_t K, int num_sms);     // rows per K2 launch

// K2: rows [0, n) of X (n <= small_max_rows), all of D.  Writes S (n x K) to
// `scores` when non-null and argmax labels to `labels` when non-null.
cudaError_t launch_smallbatch(const ModelView& m, const SmallWorkspace& ws, const float* X,
                              int n, float* scores, int32_t* labels, bool recheck, int num_sms,
                              cudaStream_t st);

// K2s (k_smallstream.cu): TMA-streamed small-batch kernel, rows [0, n), n <= 32.
bool smallstream_fits(int64_t F, int64_t D, int64_t K, int n, int num_sms);
// In-kernel D-shard exchange of the small-batch kernel (hdc_model_infer_dshard).
// Slots are sized for kDshardMaxRows rows whatever the call's N, so the slot offsets of
// consecutive calls never depend on N (a rank may run call e+1 while a peer still sums e).
constexpr int kDshardMaxRows = 32;
__host__ __device__ inline int64_t dshard_slot_floats(int64_t K) { return (kDshardMaxRows * K + 3) / 4 * 4; }
struct DshardExchange {
  float* const* bufs;   // device array [world] of the ranks' exchange buffers
  int rank, world;
  uint32_t epoch;
};
// Model setup: B4h = RN_bf16(B4) and hibound[d] (k_smallstream.cu).
cudaError_t launch_hi_plane(const float* B4, const float* Bt, int64_t F, int64_t Fp, int64_t Dp, uint16_t* B4h,
                            float* hibound, cudaStream_t st);
cudaError_t launch_smallstream(const ModelView& m, const SmallWorkspace& ws, const float* X, int n,
                               float* scores, int32_t* labels, bool recheck, int num_sms,
                               cudaStream_t st, const DshardExchange* xc = nullptr);

// Workspace of the fused large-batch kernels (grown with N).
struct FusedWorkspace {
  float* Xt;             // staged X (layout per kernel)
  float* xnorm;          // [Np] ||x_n||_2
  float* S_part;         // [R][Np][K]
  unsigned* cnt;         // [Tn], zero between launches
  unsigned long long* recheck;
};

// K1 + K3 (fp32-exact FFMA fused kernel).
size_t fused_ffma_smem_bytes(int64_t K);
int fused_choose_splits(int64_t Tn, int64_t Td, int num_sms);
cudaError_t launch_prep_x(const float* X, int64_t N, int64_t F, int64_t Fp, float* Xt, float* xnorm,
                          cudaStream_t st);
cudaError_t launch_fused_ffma(const ModelView& m, const FusedWorkspace& ws, const float* X, int64_t N,
                              float* scores, int32_t* labels, bool recheck, int R, cudaStream_t st);

// K4: fused tcgen05 kernel.  mode 0 = bf16, 1 = tf32, 2 = int8x3 (sign-exact), 3 = int8x3
// with 160-column tiles (two 80-column sub-tiles, one accumulator buffer; large F).
struct TcOperands {
  int64_t F, Fp, D, Dp, Dq, K, N_p;  // Dq = D rounded up to cl_d D-tiles; N_p to cl_n x 128 rows
  int cl_n, cl_d;                    // thread-block cluster shape (N-tiles x D-tiles), multicast
  int cl_virt;                       // 1: virtual 1 x cl_d group (no hardware cluster / multicast); 2: CTA pair (cta_group::2)
  const void* A;                     // [NL][N_p][Fp] staged X (limbs / rounded copy)
  const void* B;                     // [NL][Dq][Fp]  B^T (limbs / rounded copy), K-major
  const void* Cil;                   // per D-tile Stage II operand (tc_c_tile_bytes each)
  const float* X;                    // caller's X (fp64 recheck)
  const float* Bt;                   // [Dp][Fp] fp32 (fp64 recheck)
  const int64_t* rowtau;             // [N_p] int8 mode
  const int64_t* coltau;             // [Dq]  int8 mode
  const int32_t* coltau_m;           // [Dq]  int8 mode: ceil(coltau / 2^flag_shift) (tc_flag_shift)
  int flag_shift;
  long long* S_part;                 // [s_part_slots][128][Kp] int64 fixed-point partial scores
  long long* S_acc = nullptr;        // [N_p][Kp] int64 sums of N-tiles split over > 8 CTAs, zero between calls
  int64_t s_part_slots;
  int shift;                         // fixed-point shift of the Stage II sums (tc_corr_shift)
  unsigned* cnt;                     // [N_p / 128]
  unsigned long long* recheck;
  // int8 mode deferred rechecks (tc_recheck_kernel / tc_finalize_kernel)
  const float* Cp;                   // [K][Dp] fp32 class HVs (exact corrections)
  uint2* flags;                      // [flag_cap] (row, d | provisional-negative << 31)
  unsigned long long* flag_count;    // zero between calls
  unsigned long long flag_cap;
  long long* corr;                   // [N_p][Kp] fixed-point corrections, zero between calls
  unsigned* dirty;                   // [N_p], zero between calls
  uint32_t* hout = nullptr;          // encode mode: bit-packed H output (zeroed by the caller)
  int64_t hout_ldw = 0;
};
int tc_tile_n(int mode, int64_t K);   // D-tile width of K4 (80 or 160)
// Cluster shape of K4 for a mode (HDC_TC_CLUSTER="NxD" overrides, for measurements).
void tc_cluster_shape(int mode, int64_t K, int64_t F, int64_t D, int* cl_n, int* cl_d, int* virt);
// Partial-score slots ([128][K] each) K4 needs for Tn x Td tiles with that cluster shape.
int64_t tc_s_part_slots(int64_t Tn, int64_t Td, int cl_n, int cl_d, int virt, int num_sms);
int tc_max_k(int mode);
int64_t tc_kp(int64_t K);
int64_t tc_c_tile_bytes(int mode, int64_t K);
cudaError_t launch_tc_c_tiles(int mode, const float* Cp, int64_t K, int64_t D, int64_t Dp, int64_t Dq,
                              void* out, cudaStream_t st);
int64_t tc_max_fp_int8();
int64_t tc_tau_const(int64_t F);
int tc_flag_shift(int64_t Fp);
cudaError_t launch_tc_coltau_m(const int64_t* coltau, int64_t Dq, int shift, int32_t* out, cudaStream_t st);
cudaError_t launch_tc_limbs(const float* src, int64_t rows, int64_t rows_p, int64_t F, int64_t ld_src,
                            int64_t Fp, int8_t* out, int64_t* tau_part, int64_t tau_const,
                            cudaStream_t st);
cudaError_t launch_tc_round(int mode, const float* src, int64_t rows, int64_t rows_p, int64_t F,
                            int64_t ld_src, int64_t Fp, void* out, cudaStream_t st);
cudaError_t launch_fused_tc(int mode, const TcOperands& o, int64_t N, float* scores, int32_t* labels,
                            int num_sms, cudaStream_t st);
// int8 mode, after launch_fused_tc (which must have written S to `S`): float64 rechecks of
// the listed signs, exact corrections of S and labels of the affected rows.
cudaError_t launch_tc_recheck(const TcOperands& o, int64_t N, float* S, int32_t* labels, int shift,
                              cudaStream_t st);
int tc_corr_shift(const float* Cp, int64_t n, int64_t D);   // fixed-point shift for |C| (synchronous)
// 2-D uint8 tensor map (row-major [outer][inner] bytes) with the given box and swizzle.
bool make_tensor_map_u8(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                        uint32_t box_outer, int swizzle_bytes);

// K2t (k_small_tc.cu): small-batch (n <= 32) sign-exact inference on the int8 tensor cores
// for HDC_PREC_FP32_TC models: each CTA streams the int8 limbs of its D-range of B^T once,
// X's limbs are built in shared memory by every CTA, HardSign + float64 rechecks + Stage II
// in the CTA, partial scores summed exactly in int64 fixed point (2^-shift units) by
// atomics, the last CTA converts and takes the argmax.
struct SmallTcOperands {
  int64_t F, Fp, D, Dp, Dq, K;
  const int8_t* Btc;                 // [3][Dq][Fp] limbs of B^T
  const int64_t* coltau;             // [Dq]
  const float* Bt;                   // [Dp][Fp] fp32 (fp64 recheck)
  const float* Cp;                   // [K][Dp]
  int shift;                         // fixed-point shift (tc_corr_shift)
  unsigned long long* acc;           // [32 K] int64 accumulators, zero between launches
  unsigned* cnt;                     // [1], zero between launches
  unsigned long long* recheck;
  uint8_t* ximg;                     // [small_tc_image_bytes(F)] X limb image workspace
};
int64_t small_tc_image_bytes(int64_t F);
bool small_tc_fits(int64_t F, int64_t D, int64_t K, int n, int num_sms);
cudaError_t launch_small_tc(const SmallTcOperands& o, const float* X, int n, float* scores, int32_t* labels,
                            int num_sms, cudaStream_t st);

// k_packed.cu: unfused Stage II from bit-packed H (ablation) and class bundling (training)
cudaError_t launch_packed_similarity(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C,
                                     int64_t K, int32_t* labels, float* scores, cudaStream_t st);
// k_packed_tc.cu: the same on the tensor cores (bf16 +-1 H unpacked in shared memory, C hi + lo)
cudaError_t launch_packed_similarity_tc(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C,
                                        int64_t K, int32_t* labels, float* scores, int num_sms, cudaStream_t st);
cudaError_t launch_bundle(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const int32_t* y, int64_t K,
                          int32_t* counts, float* M, unsigned* err, cudaStream_t st);

// Diagnostic one-shot read of `bytes` (16-byte aligned buffer) with bulk copies.
cudaError_t launch_stream_read(const void* buf, int64_t bytes, int num_sms, cudaStream_t st);

// K5: labels[r] = lowest-index argmax of S[r, 0:K).
cudaError_t launch_argmax(const float* S, int64_t N, int64_t K, int32_t* labels, cudaStream_t st);

// Model setup helpers.
cudaError_t launch_pad_copy(const float* src, int64_t rows, int64_t cols, float* dst,
                            int64_t dst_cols, cudaStream_t st);
cudaError_t launch_transpose(const float* src, int64_t rows, int64_t cols, float* dst,
                             cudaStream_t st);  // dst[c][r] = src[r][c]
cudaError_t launch_unit_major(const float* Bp, int64_t Fp, int64_t Dp, float* B4, cudaStream_t st);
cudaError_t launch_col_norms(const float* Bp, int64_t F, int64_t Dp, int64_t D, float* out,
                             cudaStream_t st);

}  // namespace hdc
