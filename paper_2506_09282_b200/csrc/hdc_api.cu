// hdc_api.cu -- the C ABI of libhdc.so (include/hdc.h): validation, model
// handles (padded operand layouts, norms), workspaces and kernel dispatch.
//
// Dispatch (the analogue of the paper's S/L variant choice by batch size,
// P:222): N <= 32 -> K2 small-batch D-split kernel; larger N ->
// the fused large-batch kernel (FFMA fp32-exact or tcgen05 by precision).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/hdc.h"
#include "common.cuh"
#include "kernels.h"

using namespace hdc;

namespace {

thread_local std::string g_last_error = "";

hdc_status_t fail(hdc_status_t st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

hdc_status_t cuda_fail(cudaError_t e, const char* where) {
  return fail(HDC_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define HDC_CUDA_TRY(expr, where)                   \
  do {                                              \
    cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Every call on a model runs on the model's device (its buffers and workspaces live there),
// whatever device is current; the caller's current device is restored on return.
struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev && cudaSetDevice(dev) == cudaSuccess) switched = true;
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
};

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

constexpr int64_t kMaxF = int64_t(1) << 20;
constexpr int kSmallMaxN = 32;
constexpr int kSmallMaxNLowp = 8;          // bf16 / tf32 models (see run())
constexpr int64_t kWideMinFp = 768;        // int8 wide K4 from this padded F (tools/gpu/r2_wsweep.py:
                                           // wide/80-column time 1.0-1.02 at F = 640, 0.93-0.95 at 784)
constexpr int kSmallTcMinN = 5;            // fp32_tc models: K2t from this many rows (see run())
constexpr int64_t kInlineRecheckElems = 4000000;   // int8 K4: in-kernel rechecks up to N x Dq (run_fused_tc)
constexpr int kHostChunksMax = 8;        // chunks of the pipelined host-buffer path

}  // namespace

struct hdc_model_s {
  int device = 0;
  int64_t F = 0, D = 0, K = 0, Dp = 0, Fp = 0;
  int num_sms = 148;
  hdc_precision_t prec = HDC_PREC_FP32;
  bool fp32_tc = false;       // HDC_PREC_FP32 served by the sign-exact int8 tensor-core kernels
  bool tc_wide = false;       // int8 K4 in wide mode (160-column tiles, one accumulator; large F)
  float* Bp = nullptr;
  float* Bt = nullptr;
  float* B4 = nullptr;       // unit-major copy of Bp for the small-batch kernel
  uint16_t* B4h = nullptr;   // its bf16 hi plane (K2s sign-exact streaming: half the bytes)
  float* hibound = nullptr;  // [Dp] the hi plane's sign-bound coefficient
  // tensor-core operands (by precision): B^T rounded (bf16/tf32) or int8 limbs
  int64_t Dq = 0;            // D rounded up to cl_d tensor-core D tiles (tc_tile_n)
  int cl_n = 1, cl_d = 1;    // K4 thread-block cluster (multicast) shape
  int cl_virt = 0;           // 1: virtual 1 x cl_d CTA groups (large F: L2 working set); 2: CTA pair
  void* Btc = nullptr;       // [NL][Dq][Fp]
  int64_t* coltau = nullptr; // [Dq] (int8 limbs)
  int32_t* coltau_m = nullptr; // [Dq] K4's coarse column taus (tc_flag_shift)
  void* Cil = nullptr;       // per D-tile Stage II operand (tc_c_tile_bytes each)
  // tensor-core workspace, grown with N
  int64_t tw_rows = 0;
  int64_t tw_slots = 0;      // capacity of S_part_tc in [128][K] slots
  // int8 mode deferred rechecks: listed signs, fixed-point corrections, affected rows
  int corr_shift = 0;
  bool has_c = true;         // false: encoder-only model (created with C == NULL)
  uint2* flags = nullptr;
  unsigned long long* flag_count = nullptr;
  unsigned long long flag_cap = 0;
  long long* corr = nullptr;          // [tw_rows][Kp]
  unsigned* dirty = nullptr;          // [tw_rows]
  float* S_ws = nullptr;              // [tw_rows][K] scores when the caller passes none
  uint32_t* hout = nullptr;           // set only during hdc_model_encode
  int64_t hout_ldw = 0;
  void* Atc = nullptr;       // [NL][Np][Fp]
  int64_t* rowtau = nullptr; // [Np]
  long long* S_part_tc = nullptr;
  long long* S_acc_tc = nullptr;      // [tw_rows][Kp] K4's red.add sums of many-partial N-tiles
  unsigned* cnt_tc = nullptr;
  float* Cp = nullptr;
  float* bnorm = nullptr;
  // small-batch workspace
  unsigned long long* acc_t = nullptr;   // K2t: [32][K] int64 fixed-point score accumulators
  unsigned long long* acc_s = nullptr;   // K2s: the same for the fp32 streaming kernel
  unsigned* cnt_t = nullptr;             // K2t: [1] arrival counter
  uint8_t* ximg_t = nullptr;             // K2t: X limb image
  float* S_part = nullptr;
  unsigned* cnt = nullptr;  // [4] last-arriver counter of K2
  unsigned long long* recheck = nullptr;
  // fused-path workspace, grown on demand with N
  int64_t fw_rows = 0;  // Np capacity
  int fw_R = 0;
  float* Xt = nullptr;
  float* xnorm = nullptr;
  float* S_part_f = nullptr;
  unsigned* cnt_f = nullptr;
  // host-buffer (e2e) staging, grown on demand
  float* Xdev = nullptr;          // host-buffer path: two staging buffers of Xdev_rows x F
  int64_t Xdev_rows = 0;
  int xbuf = 0;                   // staging buffer of the next call
  cudaEvent_t ev_done[2] = {};    // compute that last read staging buffer b
  int32_t* ldev = nullptr;
  float* sdev = nullptr;
  cudaStream_t copy_stream = nullptr;   // host-buffer path: H2D copies, overlapped with compute
  cudaEvent_t ev_h2d[8] = {};
  int32_t last_launches = 0;
  int32_t last_kernel = 0;        // hdc_kernel_t of the last call's dominant kernel
  // diagnostics: CUDA events around the dominant kernel of each call
  bool timing = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void tic(cudaStream_t st) { if (timing) cudaEventRecord(ev0, st); }
  void toc(cudaStream_t st) { if (timing) cudaEventRecord(ev1, st); }

  ModelView view() const {
    ModelView v;
    v.F = F;
    v.D = D;
    v.K = K;
    v.Dp = Dp;
    v.Fp = Fp;
    v.Bp = Bp;
    v.Bt = Bt;
    v.B4 = B4;
    v.Cp = Cp;
    v.bnorm = bnorm;
    v.tau_coef = sign_bound_coef(F);
    v.B4h = B4h;
    v.hibound = hibound;
    return v;
  }
  SmallWorkspace small_ws() const {
    SmallWorkspace w;
    w.S_part = S_part;
    w.cnt1 = cnt;
    w.acc = acc_s;
    w.shift = corr_shift;
    w.recheck = recheck;
    return w;
  }
};

namespace {

hdc_status_t check_dims(int64_t F, int64_t D, int64_t K) {
  if (F < 1 || D < 1 || K < 1) return fail(HDC_ERR_INVALID_VALUE, "F, D, K must be >= 1");
  if (K > HDC_MAX_K) return fail(HDC_ERR_INVALID_VALUE, "K > HDC_MAX_K (256)");
  if (F > kMaxF) return fail(HDC_ERR_UNSUPPORTED, "F > 2^20 (sign-recheck bound validity)");
  if (D > (int64_t(1) << 31) - 4096) return fail(HDC_ERR_UNSUPPORTED, "D > 2^31 - 4096");
  return HDC_OK;
}

void free_model_memory(hdc_model_s* m) {
  if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
  for (int i = 0; i < 2; ++i)
    if (m->ev_done[i]) cudaEventDestroy(m->ev_done[i]);
  for (int i = 0; i < kHostChunksMax; ++i)
    if (m->ev_h2d[i]) cudaEventDestroy(m->ev_h2d[i]);
  if (m->ev0) cudaEventDestroy(m->ev0);
  if (m->ev1) cudaEventDestroy(m->ev1);
  cudaFree(m->Btc);
  cudaFree(m->coltau);
  cudaFree(m->coltau_m);
  cudaFree(m->Cil);
  cudaFree(m->Atc);
  cudaFree(m->rowtau);
  cudaFree(m->S_part_tc);
  cudaFree(m->S_acc_tc);
  cudaFree(m->cnt_tc);
  cudaFree(m->flags);
  cudaFree(m->flag_count);
  cudaFree(m->corr);
  cudaFree(m->dirty);
  cudaFree(m->S_ws);
  cudaFree(m->Bp);
  cudaFree(m->Bt);
  cudaFree(m->B4);
  cudaFree(m->B4h);
  cudaFree(m->hibound);
  cudaFree(m->Xt);
  cudaFree(m->xnorm);
  cudaFree(m->S_part_f);
  cudaFree(m->cnt_f);
  cudaFree(m->Cp);
  cudaFree(m->bnorm);
  cudaFree(m->S_part);
  cudaFree(m->acc_t);
  cudaFree(m->acc_s);
  cudaFree(m->cnt_t);
  cudaFree(m->ximg_t);
  cudaFree(m->cnt);
  cudaFree(m->recheck);
  cudaFree(m->Xdev);
  cudaFree(m->ldev);
  cudaFree(m->sdev);
}

constexpr int64_t kTileM = 128, kTileN = 128;

// Grows the fused workspace to N rows (synchronises only when it grows).
hdc_status_t ensure_fused_ws(hdc_model_s* m, int64_t N, int R) {
  const int64_t Tn = (N + kTileM - 1) / kTileM, Np = Tn * kTileM;
  if (Np <= m->fw_rows && R <= m->fw_R) return HDC_OK;
  const int64_t rows = Np > m->fw_rows ? Np : m->fw_rows;
  const int RR = R > m->fw_R ? R : m->fw_R;
  cudaDeviceSynchronize();
  cudaFree(m->Xt);
  cudaFree(m->xnorm);
  cudaFree(m->S_part_f);
  cudaFree(m->cnt_f);
  m->Xt = nullptr; m->xnorm = nullptr; m->S_part_f = nullptr; m->cnt_f = nullptr;
  m->fw_rows = 0;
  m->fw_R = 0;
  cudaError_t e = cudaMalloc((void**)&m->Xt, sizeof(float) * rows * m->Fp);
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->xnorm, sizeof(float) * rows);
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->S_part_f, sizeof(float) * RR * rows * m->K);
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->cnt_f, sizeof(unsigned) * (rows / kTileM));
  if (e == cudaSuccess) e = cudaMemset(m->cnt_f, 0, sizeof(unsigned) * (rows / kTileM));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HDC_ERR_NO_MEMORY, "fused workspace allocation");
  }
  m->fw_rows = rows;
  m->fw_R = RR;
  return HDC_OK;
}

int tc_mode_of(const hdc_model_s* m) {
  switch (m->prec) {
    case HDC_PREC_BF16: return 0;
    case HDC_PREC_TF32: return 1;
    case HDC_PREC_FP32_TC: return m->tc_wide ? 3 : 2;
    case HDC_PREC_FP32: return m->fp32_tc ? (m->tc_wide ? 3 : 2) : -1;
    default: return -1;
  }
}
int tc_limbs(int mode) { return mode >= 2 ? 3 : 1; }
size_t tc_esz(int mode) { return mode == 0 ? 2 : mode == 1 ? 4 : 1; }

bool tc_eligible(const hdc_model_s* m) {
  const int mode = tc_mode_of(m);
  if (mode < 0 || m->K > tc_max_k(mode)) return false;
  if (mode >= 2 && m->Fp > tc_max_fp_int8()) return false;
  return m->Btc != nullptr;
}

hdc_status_t ensure_tc_ws(hdc_model_s* m, int64_t N) {
  const int mode = tc_mode_of(m);
  const int64_t gm = kTileM * m->cl_n;
  const int64_t Np = (N + gm - 1) / gm * gm;
  int64_t slots = tc_s_part_slots(Np / kTileM, m->Dq / tc_tile_n(mode, m->K), m->cl_n, m->cl_d,
                                  m->cl_virt, m->num_sms);
  if (m->cl_virt == 1 && m->cl_d > 4) {            // run_fused_tc may launch 1 x 4 groups
    const int64_t s4 = tc_s_part_slots(Np / kTileM, m->Dq / tc_tile_n(mode, m->K), 1, 4, 1, m->num_sms);
    if (s4 > slots) slots = s4;
  }
  if (Np <= m->tw_rows && slots <= m->tw_slots) return HDC_OK;
  const int64_t rows = Np > m->tw_rows ? Np : m->tw_rows;
  const int64_t nsl = slots > m->tw_slots ? slots : m->tw_slots;
  cudaDeviceSynchronize();
  cudaFree(m->Atc);
  cudaFree(m->rowtau);
  cudaFree(m->S_part_tc);
  cudaFree(m->S_acc_tc);
  cudaFree(m->cnt_tc);
  cudaFree(m->flags);
  cudaFree(m->flag_count);
  cudaFree(m->corr);
  cudaFree(m->dirty);
  cudaFree(m->S_ws);
  m->Atc = nullptr; m->rowtau = nullptr; m->S_part_tc = nullptr; m->S_acc_tc = nullptr; m->cnt_tc = nullptr;
  m->flags = nullptr; m->flag_count = nullptr; m->corr = nullptr; m->dirty = nullptr; m->S_ws = nullptr;
  m->tw_rows = 0;
  m->tw_slots = 0;
  cudaError_t e = cudaMalloc(&m->Atc, tc_esz(mode) * tc_limbs(mode) * rows * m->Fp);
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->rowtau, sizeof(int64_t) * rows);
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->S_part_tc, sizeof(long long) * nsl * kTileM * tc_kp(m->K));
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->S_acc_tc, sizeof(long long) * rows * tc_kp(m->K));
  if (e == cudaSuccess) e = cudaMemset(m->S_acc_tc, 0, sizeof(long long) * rows * tc_kp(m->K));
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->cnt_tc, sizeof(unsigned) * (rows / kTileM));
  if (e == cudaSuccess) e = cudaMemset(m->cnt_tc, 0, sizeof(unsigned) * (rows / kTileM));
  if (e == cudaSuccess && mode >= 2) {
    // list capacity: ~1/256 of the elements (measured ~1e-4 flagged), at most 4M entries;
    // beyond it the kernel re-evaluates inline (correct, slower)
    const int64_t kp = tc_kp(m->K);
    unsigned long long cap = (unsigned long long)(rows * m->Dq / 256);
    if (cap < (1ull << 16)) cap = 1ull << 16;
    if (cap > (1ull << 22)) cap = 1ull << 22;
    e = cudaMalloc((void**)&m->flags, sizeof(uint2) * cap);
    if (e == cudaSuccess) e = cudaMalloc((void**)&m->flag_count, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(m->flag_count, 0, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc((void**)&m->corr, sizeof(long long) * rows * kp);
    if (e == cudaSuccess) e = cudaMemset(m->corr, 0, sizeof(long long) * rows * kp);
    if (e == cudaSuccess) e = cudaMalloc((void**)&m->dirty, sizeof(unsigned) * rows);
    if (e == cudaSuccess) e = cudaMemset(m->dirty, 0, sizeof(unsigned) * rows);
    m->flag_cap = cap;
  }
  // scores scratch: int8 mode's provisional scores; every mode's split-N-tile sums
  if (e == cudaSuccess) e = cudaMalloc((void**)&m->S_ws, sizeof(float) * rows * m->K);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HDC_ERR_NO_MEMORY, "tensor-core workspace allocation");
  }
  m->tw_rows = rows;
  m->tw_slots = nsl;
  return HDC_OK;
}

hdc_status_t run_fused_tc(hdc_model_s* m, const float* X, int64_t N, int32_t* labels, float* scores,
                          cudaStream_t st) {
  const int mode = tc_mode_of(m);
  hdc_status_t stt = ensure_tc_ws(m, N);
  if (stt != HDC_OK) return stt;
  // one N-tile or less: no CTA pairs over N-tiles (the partner tile would be all padding);
  // single CTAs spread the D-tiles over all SMs instead
  int cl_n = m->cl_n, cl_d = m->cl_d, cl_virt = m->cl_virt;
  if (N <= kTileM && cl_virt != 1) {
    cl_n = 1;
    cl_d = 1;
    cl_virt = 0;
  }
  // large batches on virtual groups: 1 x 4 groups once every group gets >= 8 rows of N-tiles,
  // so the launch takes ranges of whole rows and the groups sweep B's D-groups in step
  // (k_fused_tc.cu launch_mode): cfg5 int8 17.1 -> 16.7-16.8 ms, bf16 6.69 -> 6.07, D = 2000
  // bf16 2.81 -> 1.64; below that 1 x 16 (N = 16384: int8 2.08 vs 2.34 ms)
  if (cl_virt == 1 && cl_d > 4 && !getenv("HDC_TC_CLUSTER") &&
      (N + kTileM - 1) / kTileM >= 8 * (int64_t)(m->num_sms / 4))
    cl_d = 4;
  const int64_t gm = kTileM * cl_n;
  const int64_t Np = (N + gm - 1) / gm * gm;
  cudaError_t e;
  if (mode >= 2)
    e = launch_tc_limbs(X, N, Np, m->F, m->F, m->Fp, (int8_t*)m->Atc, m->rowtau, tc_tau_const(m->F), st);
  else
    e = launch_tc_round(mode, X, N, Np, m->F, m->F, m->Fp, m->Atc, st);
  if (e != cudaSuccess) return cuda_fail(e, "tensor-core operand staging");
  TcOperands o;
  o.F = m->F;
  o.Fp = m->Fp;
  o.D = m->D;
  o.Dp = m->Dp;
  o.Dq = m->Dq;
  o.K = m->K;
  o.N_p = Np;
  o.cl_n = cl_n;
  o.cl_d = cl_d;
  o.cl_virt = cl_virt;
  o.A = m->Atc;
  o.B = m->Btc;
  o.Cil = m->Cil;
  o.X = X;
  o.Bt = m->Bt;
  o.rowtau = m->rowtau;
  o.coltau = m->coltau;
  o.coltau_m = m->coltau_m;
  o.flag_shift = tc_flag_shift(m->Fp);
  o.S_part = m->S_part_tc;
  o.S_acc = m->S_acc_tc;
  o.s_part_slots = m->tw_slots;
  o.shift = m->corr_shift;
  o.cnt = m->cnt_tc;
  o.recheck = m->recheck;
  o.Cp = m->Cp;
  o.flags = m->flags;
  o.flag_count = m->flag_count;
  // int8 mode, small batches (N x Dq <= kInlineRecheckElems, cfg1: ~1 flag per CTA): the
  // fused kernel re-evaluates its flags itself and the recheck / finalize launches are
  // skipped; HDC_TC_INLINE_RECHECK=0/1 overrides (measurements)
  const char* irc = getenv("HDC_TC_INLINE_RECHECK");
  const bool inline_rc = mode >= 2 && (irc ? atoi(irc) != 0 : N * m->Dq <= kInlineRecheckElems);
  o.flag_cap = inline_rc ? 0 : m->flag_cap;
  o.corr = m->corr;
  o.dirty = m->dirty;
  o.hout = m->hout;
  o.hout_ldw = m->hout_ldw;
  // the fused kernel always writes scores (int8 mode: provisional, corrected afterwards;
  // all modes: split N-tiles sum their partials there before the argmax)
  float* S = scores ? scores : m->S_ws;
  m->tic(st);
  e = launch_fused_tc(mode, o, N, S, labels, m->num_sms, st);
  m->toc(st);
  if (e != cudaSuccess) return cuda_fail(e, "fused_tc launch");
  m->last_launches = 2;
  m->last_kernel = HDC_KERNEL_TC;
  if (mode >= 2 && !inline_rc) {
    e = launch_tc_recheck(o, N, S, labels, m->corr_shift, st);
    if (e != cudaSuccess) return cuda_fail(e, "tc recheck launch");
    m->last_launches = 4;
  }
  return HDC_OK;
}

hdc_status_t run_fused(hdc_model_s* m, const float* X, int64_t N, int32_t* labels, float* scores,
                       bool recheck, cudaStream_t st) {
  if (tc_eligible(m)) return run_fused_tc(m, X, N, labels, scores, st);
  // fp32 FFMA path (also serves tensor-core precisions with K > 32: more exact, never less)
  const int64_t Tn = (N + kTileM - 1) / kTileM, Td = (m->D + kTileN - 1) / kTileN;
  const int R = fused_choose_splits(Tn, Td, m->num_sms);
  hdc_status_t stt = ensure_fused_ws(m, N, R);
  if (stt != HDC_OK) return stt;
  FusedWorkspace ws;
  ws.Xt = m->Xt;
  ws.xnorm = m->xnorm;
  ws.S_part = m->S_part_f;
  ws.cnt = m->cnt_f;
  ws.recheck = m->recheck;
  cudaError_t e = launch_prep_x(X, N, m->F, m->Fp, m->Xt, m->xnorm, st);
  if (e != cudaSuccess) return cuda_fail(e, "prep_x launch");
  m->tic(st);
  e = launch_fused_ffma(m->view(), ws, X, N, scores, labels, recheck, R, st);
  m->toc(st);
  if (e != cudaSuccess) return cuda_fail(e, "fused_ffma launch");
  m->last_launches = 2;
  m->last_kernel = HDC_KERNEL_FFMA;
  return HDC_OK;
}

// Runs the selected path over rows [0, N) of X.
hdc_status_t run(hdc_model_s* m, const float* X, int64_t N, int32_t* labels, float* scores,
                 hdc_path_t path, cudaStream_t st) {
  m->last_launches = 0;
  m->last_kernel = HDC_KERNEL_NONE;
  if (N == 0) return HDC_OK;
  const ModelView mv = m->view();
  const bool recheck = (m->prec == HDC_PREC_FP32 || m->prec == HDC_PREC_FP32_TC ||
                        !tc_eligible(m));  // FFMA/small kernels are fp32: keep them sign-exact
  if (path == HDC_PATH_AUTO) {
    // bf16 / tf32 models: the fused tensor-core kernel beats the fp32 streaming kernel
    // from N = 16 at cfg3 (tools/smalln_probe.py: N=16 35 vs 40 us, N=32 41 vs 61 us);
    // fp32 semantics keep the streaming kernel up to 32 rows
    const int64_t small_max = (tc_eligible(m) && (m->prec == HDC_PREC_BF16 || m->prec == HDC_PREC_TF32))
                                  ? kSmallMaxNLowp : kSmallMaxN;
    path = (N <= small_max) ? HDC_PATH_SMALL : HDC_PATH_FUSED;
  }
  if (path == HDC_PATH_FUSED) return run_fused(m, X, N, labels, scores, recheck, st);
  // sign-exact models: the int8 tensor-core small-batch kernel (B streamed as 3-byte limbs,
  // Stage I on the tensor cores) from kSmallTcMinN rows; below it the fp32 streaming kernel,
  // whose single launch beats K2t's two (cfg3: N = 1 18.8 vs 19.8 us, N = 4 20.1 vs 21.6 us;
  // N = 16 28.9 vs 21.9 us, N = 32 43.2 vs 23.9 us).  HDC_SMALL_TC=0/1 forces either.
  const char* stc = getenv("HDC_SMALL_TC");
  const bool want_tc = stc ? (atoi(stc) != 0) : (N >= kSmallTcMinN);
  if (m->acc_t && tc_eligible(m) && N <= kSmallMaxN && want_tc && !getenv("HDC_SMALL_FP32") &&
      small_tc_fits(m->F, m->D, m->K, (int)N, m->num_sms)) {
    SmallTcOperands o;
    o.F = m->F;
    o.Fp = m->Fp;
    o.D = m->D;
    o.Dp = m->Dp;
    o.Dq = m->Dq;
    o.K = m->K;
    o.Btc = (const int8_t*)m->Btc;
    o.coltau = m->coltau;
    o.Bt = m->Bt;
    o.Cp = m->Cp;
    o.shift = m->corr_shift;
    o.acc = m->acc_t;
    o.cnt = m->cnt_t;
    o.recheck = m->recheck;
    o.ximg = m->ximg_t;
    m->tic(st);
    cudaError_t e = launch_small_tc(o, X, (int)N, scores, labels, m->num_sms, st);
    m->toc(st);
    if (e != cudaSuccess) return cuda_fail(e, "small tensor-core launch");
    m->last_launches = 2;
    m->last_kernel = HDC_KERNEL_SMALL_TC;
    return HDC_OK;
  }
  const SmallWorkspace ws = m->small_ws();
  const int chunk = small_max_rows(m->F, m->D, m->K, m->num_sms);
  if (chunk < 1) return fail(HDC_ERR_UNSUPPORTED, "F too large for the small-batch kernel's shared memory");
  m->tic(st);
  for (int64_t r0 = 0; r0 < N; r0 += chunk) {
    const int n = (int)((N - r0) < chunk ? (N - r0) : chunk);
    // K2s (TMA-streamed) when X fits its shared memory, else the register-strip K2
    cudaError_t e = (m->B4 && smallstream_fits(m->F, m->D, m->K, n, m->num_sms) && !getenv("HDC_SMALL_LEGACY"))
                        ? launch_smallstream(mv, ws, X + r0 * m->F, n, scores ? scores + r0 * m->K : nullptr,
                                             labels ? labels + r0 : nullptr, recheck, m->num_sms, st)
                        : launch_smallbatch(mv, ws, X + r0 * m->F, n, scores ? scores + r0 * m->K : nullptr,
                                            labels ? labels + r0 : nullptr, recheck, m->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(e, "smallbatch launch");
    ++m->last_launches;
    m->last_kernel = HDC_KERNEL_SMALL;
  }
  m->toc(st);
  return HDC_OK;
}

hdc_status_t validate_call(hdc_model_s* m, const float* X, int64_t N, const void* out_required,
                           const void* out_optional) {
  if (!m) return fail(HDC_ERR_INVALID_VALUE, "null model");
  if (!m->has_c) return fail(HDC_ERR_INVALID_VALUE, "encoder-only model (created without C)");
  if (N < 0) return fail(HDC_ERR_INVALID_VALUE, "N < 0");
  if (N >= (int64_t(1) << 31)) return fail(HDC_ERR_UNSUPPORTED, "N >= 2^31 (row indices are 32-bit)");
  if (N > 0 && (!X || !out_required)) return fail(HDC_ERR_INVALID_VALUE, "null X or output");
  if (!aligned(X, 4) || !aligned(out_required, 4) || !aligned(out_optional, 4))
    return fail(HDC_ERR_MISALIGNED, "pointers must be 4-byte aligned");
  return HDC_OK;
}

}  // namespace

extern "C" {

const char* hdc_status_string(hdc_status_t st) {
  switch (st) {
    case HDC_OK: return "HDC_OK";
    case HDC_ERR_INVALID_VALUE: return "HDC_ERR_INVALID_VALUE";
    case HDC_ERR_MISALIGNED: return "HDC_ERR_MISALIGNED";
    case HDC_ERR_UNSUPPORTED: return "HDC_ERR_UNSUPPORTED";
    case HDC_ERR_NO_MEMORY: return "HDC_ERR_NO_MEMORY";
    case HDC_ERR_CUDA: return "HDC_ERR_CUDA";
  }
  return "HDC_ERR_UNKNOWN";
}

const char* hdc_last_error(void) { return g_last_error.c_str(); }

const char* hdc_version(void) { return "libhdc 0.2 (sm_100a)"; }

hdc_status_t hdc_diag_stream_read(const void* buf, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && !buf)) return fail(HDC_ERR_INVALID_VALUE, "null buffer or bytes < 0");
  if (!aligned(buf, 16) || bytes % 16) return fail(HDC_ERR_MISALIGNED, "16-byte aligned buffer and size required");
  if (bytes == 0) return HDC_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = launch_stream_read(buf, bytes, sms, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "stream read launch");
  return HDC_OK;
}

hdc_status_t hdc_model_create(const float* B, const float* C, int64_t F, int64_t D, int64_t K,
                              hdc_precision_t prec, hdc_model_t* out) {
  if (!out) return fail(HDC_ERR_INVALID_VALUE, "null out");
  *out = nullptr;
  hdc_status_t st = check_dims(F, D, K);
  if (st != HDC_OK) return st;
  if (!B) return fail(HDC_ERR_INVALID_VALUE, "null B");
  if (!aligned(B, 4) || !aligned(C, 4)) return fail(HDC_ERR_MISALIGNED, "B, C must be 4-byte aligned");
  if (prec < HDC_PREC_FP32 || prec > HDC_PREC_FP32_TC) return fail(HDC_ERR_INVALID_VALUE, "bad precision");
  hdc_model_s* m = new hdc_model_s();
  m->F = F;
  m->D = D;
  m->K = K;
  m->prec = prec;
  // fp32 semantics on the tensor cores: the int8x3 limb kernels make every HardSign decision
  // equal to the exact one, as the FFMA kernels do, at 12x their speed (cfg2: 0.50 vs 6.2 ms);
  // HDC_FP32_FFMA (read here) keeps the fp32 FFMA kernels, which remain the fallback
  // (K > 32, F > 100000) either way
  m->fp32_tc = (prec == HDC_PREC_FP32) && !getenv("HDC_FP32_FFMA");
  m->Dp = round_up(D, kDPad);
  m->Fp = round_up(F, kFPad);
  cudaGetDevice(&m->device);
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, m->device);
  const int64_t G = 1024;  // >= small_num_ctas for any device
  cudaError_t e = cudaSuccess;
#define ALLOC(ptr, bytes)                                           \
  if (e == cudaSuccess) e = cudaMalloc((void**)&(ptr), (size_t)(bytes));
  ALLOC(m->Bp, sizeof(float) * m->Fp * m->Dp);
  ALLOC(m->Bt, sizeof(float) * m->Fp * m->Dp);
  ALLOC(m->B4, sizeof(float) * m->Fp * m->Dp);
  ALLOC(m->Cp, sizeof(float) * K * m->Dp);
  ALLOC(m->bnorm, sizeof(float) * m->Dp);
  ALLOC(m->B4h, sizeof(uint16_t) * m->Fp * m->Dp);
  ALLOC(m->hibound, sizeof(float) * m->Dp);
  ALLOC(m->S_part, sizeof(float) * G * kSmallMaxN * K);
  ALLOC(m->cnt, sizeof(unsigned) * 64);
  ALLOC(m->recheck, sizeof(unsigned long long));
  ALLOC(m->acc_s, sizeof(unsigned long long) * kSmallMaxN * K);
#undef ALLOC
  if (e != cudaSuccess) {
    free_model_memory(m);
    delete m;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? HDC_ERR_NO_MEMORY : HDC_ERR_CUDA,
                std::string("model allocation: ") + cudaGetErrorString(e));
  }
  cudaStream_t st0 = 0;
  if (e == cudaSuccess) e = cudaMemset(m->Bp, 0, sizeof(float) * m->Fp * m->Dp);
  if (e == cudaSuccess) e = launch_pad_copy(B, F, D, m->Bp, m->Dp, st0);
  if (e == cudaSuccess) e = launch_transpose(m->Bp, m->Fp, m->Dp, m->Bt, st0);
  if (e == cudaSuccess) e = launch_unit_major(m->Bp, m->Fp, m->Dp, m->B4, st0);
  m->has_c = C != nullptr;
  if (e == cudaSuccess) e = C ? launch_pad_copy(C, K, D, m->Cp, m->Dp, st0)
                              : cudaMemset(m->Cp, 0, sizeof(float) * K * m->Dp);
  if (e == cudaSuccess) e = launch_col_norms(m->Bp, F, m->Dp, D, m->bnorm, st0);
  if (e == cudaSuccess) e = launch_hi_plane(m->B4, m->Bt, F, m->Fp, m->Dp, m->B4h, m->hibound, st0);
  if (e == cudaSuccess) e = cudaMemset(m->cnt, 0, sizeof(unsigned) * 64);
  if (e == cudaSuccess) e = cudaMemset(m->acc_s, 0, sizeof(unsigned long long) * kSmallMaxN * K);
  // fixed point of the exact cross-CTA score sums (all models) and of the int8 recheck
  // corrections: 2 D max|C| 2^shift < 2^62
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) m->corr_shift = tc_corr_shift(m->Cp, K * m->Dp, D);
  {
    // int8 wide mode (k_fused_tc.cu, mode 3) for large F, where K4 streams its operands
    // faster than the double-buffered 80-column tiles can consume them; HDC_TC_WIDE=0/1
    // overrides (measurements)
    const char* w = getenv("HDC_TC_WIDE");
    m->tc_wide = K <= tc_max_k(3) && (w ? atoi(w) != 0 : m->Fp >= kWideMinFp);
  }
  const int mode = tc_mode_of(m);
  const int64_t tn = tc_tile_n(mode < 0 ? 0 : mode, K);
  tc_cluster_shape(mode < 0 ? 0 : mode, K, F, D, &m->cl_n, &m->cl_d, &m->cl_virt);
  m->Dq = (D + tn * m->cl_d - 1) / (tn * m->cl_d) * (tn * m->cl_d);
  if (e == cudaSuccess && mode >= 0 && K <= tc_max_k(mode) && !(mode >= 2 && m->Fp > tc_max_fp_int8())) {
    e = cudaMalloc(&m->Btc, tc_esz(mode) * tc_limbs(mode) * m->Dq * m->Fp);
    if (e == cudaSuccess && mode >= 2) e = cudaMalloc((void**)&m->coltau, sizeof(int64_t) * m->Dq);
    if (e == cudaSuccess && mode >= 2) e = cudaMalloc((void**)&m->coltau_m, sizeof(int32_t) * m->Dq);
    if (e == cudaSuccess)
      e = cudaMalloc(&m->Cil, (size_t)tc_c_tile_bytes(mode, K) * (m->Dq / tn));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();  // Bt must be complete
    if (e == cudaSuccess) {
      if (mode >= 2) {
        e = launch_tc_limbs(m->Bt, D, m->Dq, F, m->Fp, m->Fp, (int8_t*)m->Btc, m->coltau, 0, st0);
        if (e == cudaSuccess)
          e = launch_tc_coltau_m(m->coltau, m->Dq, tc_flag_shift(m->Fp), m->coltau_m, st0);
      } else {
        e = launch_tc_round(mode, m->Bt, D, m->Dq, F, m->Fp, m->Fp, m->Btc, st0);
      }
    }
    if (e == cudaSuccess) e = launch_tc_c_tiles(mode, m->Cp, K, D, m->Dp, m->Dq, m->Cil, st0);
    if (e == cudaSuccess && mode >= 2) {
      // K2t (small-batch tensor-core kernel) accumulators, zero between launches
      if (e == cudaSuccess) e = cudaMalloc((void**)&m->acc_t, sizeof(unsigned long long) * kSmallMaxN * K);
      if (e == cudaSuccess) e = cudaMemset(m->acc_t, 0, sizeof(unsigned long long) * kSmallMaxN * K);
      if (e == cudaSuccess) e = cudaMalloc((void**)&m->cnt_t, sizeof(unsigned));
      if (e == cudaSuccess) e = cudaMemset(m->cnt_t, 0, sizeof(unsigned));
      if (e == cudaSuccess) e = cudaMalloc((void**)&m->ximg_t, (size_t)small_tc_image_bytes(F));
    }
  }
  if (e == cudaSuccess) e = cudaMemset(m->recheck, 0, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    free_model_memory(m);
    delete m;
    return cuda_fail(e, "model setup");
  }
  *out = m;
  return HDC_OK;
}

hdc_status_t hdc_model_destroy(hdc_model_t m) {
  if (!m) return fail(HDC_ERR_INVALID_VALUE, "null model");
  DeviceGuard dg(m->device);
  cudaDeviceSynchronize();
  free_model_memory(m);
  delete m;
  return HDC_OK;
}

hdc_status_t hdc_model_dims(hdc_model_t m, int64_t* F, int64_t* D, int64_t* K,
                            hdc_precision_t* prec) {
  if (!m) return fail(HDC_ERR_INVALID_VALUE, "null model");
  if (F) *F = m->F;
  if (D) *D = m->D;
  if (K) *K = m->K;
  if (prec) *prec = m->prec;
  return HDC_OK;
}

hdc_status_t hdc_model_infer_path(hdc_model_t m, const float* X, int64_t N, int32_t* labels,
                                  float* scores, hdc_path_t path, void* stream) {
  hdc_status_t st = validate_call(m, X, N, labels, scores);
  if (st != HDC_OK) return st;
  DeviceGuard dg(m->device);
  if (path < HDC_PATH_AUTO || path > HDC_PATH_FUSED) return fail(HDC_ERR_INVALID_VALUE, "bad path");
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return cuda_fail(pe, "pending CUDA error");
  return run(m, X, N, labels, scores, path, (cudaStream_t)stream);
}

hdc_status_t hdc_model_infer(hdc_model_t m, const float* X, int64_t N, int32_t* labels,
                             float* scores, void* stream) {
  return hdc_model_infer_path(m, X, N, labels, scores, HDC_PATH_AUTO, stream);
}

hdc_status_t hdc_model_partial_scores(hdc_model_t m, const float* X, int64_t N, float* S_partial,
                                      void* stream) {
  hdc_status_t st = validate_call(m, X, N, S_partial, nullptr);
  if (st != HDC_OK) return st;
  DeviceGuard dg(m->device);
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return cuda_fail(pe, "pending CUDA error");
  return run(m, X, N, nullptr, S_partial, HDC_PATH_AUTO, (cudaStream_t)stream);
}

int64_t hdc_dshard_exchange_bytes(int64_t N, int64_t K, int world) {
  if (N < 1 || N > kDshardMaxRows || K < 1 || K > HDC_MAX_K || world < 1) return 0;
  // slots sized for kDshardMaxRows rows: one buffer serves every N <= 32, and the slot
  // offsets do not move when N changes between calls
  const int64_t stride = dshard_slot_floats(K), sigpad = (world + 3) / 4 * 4;
  return (int64_t)4 * (sigpad + 2 * world * stride);
}

hdc_status_t hdc_model_infer_dshard(hdc_model_t m, const float* X, int64_t N, int32_t* labels,
                                    float* scores, float* const* xbufs, int rank, int world,
                                    uint32_t epoch, void* stream) {
  hdc_status_t st = validate_call(m, X, N, labels, scores);
  if (st != HDC_OK) return st;
  DeviceGuard dg(m->device);
  if (N < 1 || N > kSmallMaxN) return fail(HDC_ERR_UNSUPPORTED, "D-shard exchange: 1 <= N <= 32");
  if (world < 1 || rank < 0 || rank >= world) return fail(HDC_ERR_INVALID_VALUE, "rank / world");
  if (!xbufs || !aligned(xbufs, 8)) return fail(HDC_ERR_INVALID_VALUE, "null or misaligned xbufs");
  if (!m->B4 || !smallstream_fits(m->F, m->D, m->K, (int)N, m->num_sms) ||
      small_max_rows(m->F, m->D, m->K, m->num_sms) < N)
    return fail(HDC_ERR_UNSUPPORTED, "shapes outside the small-batch streaming kernel");
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return cuda_fail(pe, "pending CUDA error");
  cudaStream_t s = (cudaStream_t)stream;
  const DshardExchange xc{xbufs, rank, world, epoch};
  const bool recheck = true;                   // the streaming kernel is fp32: keep it sign-exact
  m->last_launches = 0;
  m->tic(s);
  cudaError_t e = launch_smallstream(m->view(), m->small_ws(), X, (int)N, scores, labels, recheck,
                                     m->num_sms, s, &xc);
  m->toc(s);
  if (e != cudaSuccess) return cuda_fail(e, "D-shard small-batch launch");
  m->last_launches = 1;
  m->last_kernel = HDC_KERNEL_SMALL;
  return HDC_OK;
}

hdc_status_t hdc_model_infer_host(hdc_model_t m, const float* X_host, int64_t N,
                                  int32_t* labels_host, float* scores_host, void* stream) {
  hdc_status_t st = validate_call(m, X_host, N, labels_host, scores_host);
  if (st != HDC_OK) return st;
  DeviceGuard dg(m->device);
  if (N == 0) return HDC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (N > m->Xdev_rows) {
    cudaDeviceSynchronize();                 // earlier calls may still read the staging buffers
    cudaFree(m->Xdev);
    cudaFree(m->ldev);
    cudaFree(m->sdev);
    m->Xdev = nullptr;
    m->ldev = nullptr;
    m->sdev = nullptr;
    m->Xdev_rows = 0;
    cudaError_t e = cudaMalloc((void**)&m->Xdev, sizeof(float) * 2 * N * m->F);
    if (e == cudaSuccess) e = cudaMalloc((void**)&m->ldev, sizeof(int32_t) * N);
    if (e == cudaSuccess) e = cudaMalloc((void**)&m->sdev, sizeof(float) * N * m->K);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(HDC_ERR_NO_MEMORY, "staging allocation");
    }
    m->Xdev_rows = N;
  }
  if (!m->copy_stream) {
    if (cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      return fail(HDC_ERR_CUDA, "copy stream / event creation");
    for (int i = 0; i < kHostChunksMax; ++i)
      if (cudaEventCreateWithFlags(&m->ev_h2d[i], cudaEventDisableTiming) != cudaSuccess)
        return fail(HDC_ERR_CUDA, "event creation");
    for (int i = 0; i < 2; ++i)
      if (cudaEventCreateWithFlags(&m->ev_done[i], cudaEventDisableTiming) != cudaSuccess)
        return fail(HDC_ERR_CUDA, "event creation");
  }
  // Pipelined, two ways.  (1) Across calls: X goes to one of two staging buffers, so
  // the copy of call i + 1 needs only the compute of call i - 1 (which read that
  // buffer) to be done, and overlaps the compute of call i.  (2) Within a call: chunks,
  // the copy of chunk j + 1 overlapping the inference of chunk j.  Copies run on the
  // model's copy stream in call order; compute and the label copies on `stream`.
  // Rows are independent (Alg. 1 per sample), so chunking changes nothing in the results.
  int nchunks = 1;
  if (N > kSmallMaxN) {
    const char* ev = getenv("HDC_HOST_CHUNK_ROWS");   // diagnostics override
    const int64_t target = ev ? atoll(ev) : 8192;     // rows per chunk (>= a few waves of tiles)
    nchunks = (int)((N + target - 1) / target);
    if (nchunks > kHostChunksMax) nchunks = kHostChunksMax;
  }
  const int64_t per = (N + nchunks - 1) / nchunks;
  const int b = m->xbuf;
  m->xbuf ^= 1;
  // Results go straight into mapped pinned host buffers when the caller's are (the kernels
  // write them over PCIe): no device-to-host copy on the copy engine, which on some
  // systems serves both directions in one queue -- a small label copy would then wait
  // behind the next call's host-to-device copy and stall the compute stream.
  auto mapped = [](void* h) -> void* {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return (a.type == cudaMemoryTypeHost && a.devicePointer) ? a.devicePointer : nullptr;
  };
  int32_t* lab_map = static_cast<int32_t*>(mapped(labels_host));
  float* sc_map = scores_host ? static_cast<float*>(mapped(scores_host)) : nullptr;
  float* xd = m->Xdev + (int64_t)b * m->Xdev_rows * m->F;
  HDC_CUDA_TRY(cudaStreamWaitEvent(m->copy_stream, m->ev_done[b], 0), "stream wait");
  // (same stream: a no-op; another stream: the device labels / scores are not reused early)
  HDC_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_done[b ^ 1], 0), "stream wait");
  int32_t launches = 0;
  for (int i = 0; i < nchunks; ++i) {
    const int64_t r0 = i * per, n = (r0 + per <= N) ? per : N - r0;
    if (n <= 0) break;
    HDC_CUDA_TRY(cudaMemcpyAsync(xd + r0 * m->F, X_host + r0 * m->F, sizeof(float) * n * m->F,
                                 cudaMemcpyHostToDevice, m->copy_stream),
                 "H2D X");
    HDC_CUDA_TRY(cudaEventRecord(m->ev_h2d[i], m->copy_stream), "event record");
    HDC_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_h2d[i], 0), "stream wait");
    int32_t* lab = lab_map ? lab_map + r0 : m->ldev + r0;
    float* sc = scores_host ? (sc_map ? sc_map + r0 * m->K : m->sdev + r0 * m->K) : nullptr;
    st = run(m, xd + r0 * m->F, n, lab, sc, HDC_PATH_AUTO, s);
    if (st != HDC_OK) return st;
    launches += m->last_launches;
    if (!lab_map)
      HDC_CUDA_TRY(cudaMemcpyAsync(labels_host + r0, m->ldev + r0, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s),
                   "D2H labels");
    if (scores_host && !sc_map)
      HDC_CUDA_TRY(cudaMemcpyAsync(scores_host + r0 * m->K, m->sdev + r0 * m->K, sizeof(float) * n * m->K,
                                   cudaMemcpyDeviceToHost, s),
                   "D2H scores");
  }
  HDC_CUDA_TRY(cudaEventRecord(m->ev_done[b], s), "event record");
  m->last_launches = launches;
  return HDC_OK;
}

hdc_status_t hdc_model_encode(hdc_model_t m, const float* X, int64_t N, uint32_t* H, int64_t ldw,
                              void* stream) {
  if (!m) return fail(HDC_ERR_INVALID_VALUE, "null model");
  DeviceGuard dg(m->device);
  if (N < 0) return fail(HDC_ERR_INVALID_VALUE, "N < 0");
  if (N >= (int64_t(1) << 31)) return fail(HDC_ERR_UNSUPPORTED, "N >= 2^31");
  if (N > 0 && (!X || !H)) return fail(HDC_ERR_INVALID_VALUE, "null X or H");
  if (ldw < (m->D + 31) / 32) return fail(HDC_ERR_INVALID_VALUE, "ldw < ceil(D / 32)");
  if (!aligned(X, 4) || !aligned(H, 4)) return fail(HDC_ERR_MISALIGNED, "pointers must be 4-byte aligned");
  const int mode = tc_mode_of(m);
  if (mode < 0 || !m->Btc)
    return fail(HDC_ERR_UNSUPPORTED, "encode needs a tensor-core precision model (fp32_tc, tf32, bf16)");
  if (N == 0) return HDC_OK;
  cudaError_t pe = cudaGetLastError();
  if (pe != cudaSuccess) return cuda_fail(pe, "pending CUDA error");
  cudaStream_t st = (cudaStream_t)stream;
  HDC_CUDA_TRY(cudaMemsetAsync(H, 0, sizeof(uint32_t) * N * ldw, st), "H clear");
  m->hout = H;
  m->hout_ldw = ldw;
  hdc_status_t s2 = run_fused_tc(m, X, N, nullptr, nullptr, st);
  m->hout = nullptr;
  m->hout_ldw = 0;
  return s2;
}

hdc_status_t hdc_similarity_packed(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const float* C,
                                   int64_t K, int32_t* labels, float* scores, void* stream) {
  if (N < 0 || D < 1 || K < 1) return fail(HDC_ERR_INVALID_VALUE, "N >= 0, D >= 1, K >= 1 required");
  if (K > 64) return fail(HDC_ERR_UNSUPPORTED, "K > 64 (unfused ablation kernel)");
  if (ldw < (D + 31) / 32) return fail(HDC_ERR_INVALID_VALUE, "ldw < ceil(D / 32)");
  if (N > 0 && (!H || !C || (!labels && !scores))) return fail(HDC_ERR_INVALID_VALUE, "null pointer");
  if (!aligned(H, 4) || !aligned(C, 4) || !aligned(labels, 4) || !aligned(scores, 4))
    return fail(HDC_ERR_MISALIGNED, "alignment");
  if (N == 0) return HDC_OK;
  // the tensor-core Stage II (the unfused ablation at its own roofline); HDC_PACKED_FFMA
  // keeps round 1's FFMA kernel for comparison
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = getenv("HDC_PACKED_FFMA")
                      ? launch_packed_similarity(H, ldw, N, D, C, K, labels, scores, (cudaStream_t)stream)
                      : launch_packed_similarity_tc(H, ldw, N, D, C, K, labels, scores, sms, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "packed similarity launch");
  return HDC_OK;
}

hdc_status_t hdc_bundle_classes(const uint32_t* H, int64_t ldw, int64_t N, int64_t D, const int32_t* y,
                                int64_t K, int32_t* counts, float* M, void* stream) {
  if (N < 0 || D < 1 || K < 1) return fail(HDC_ERR_INVALID_VALUE, "N >= 0, D >= 1, K >= 1 required");
  if (K > HDC_MAX_K) return fail(HDC_ERR_INVALID_VALUE, "K > HDC_MAX_K");
  if (ldw < (D + 31) / 32) return fail(HDC_ERR_INVALID_VALUE, "ldw < ceil(D / 32)");
  if (!counts || (N > 0 && (!H || !y))) return fail(HDC_ERR_INVALID_VALUE, "null pointer");
  if (!aligned(H, 4) || !aligned(y, 4) || !aligned(counts, 4) || !aligned(M, 4))
    return fail(HDC_ERR_MISALIGNED, "alignment");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned* err = nullptr;
  HDC_CUDA_TRY(cudaMallocAsync((void**)&err, sizeof(unsigned), st), "workspace");
  HDC_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(unsigned), st), "workspace");
  cudaError_t e = launch_bundle(H, ldw, N, D, y, K, counts, M, err, st);
  unsigned herr = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, err, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);      // label validation needs the count
  cudaFreeAsync(err, st);
  if (e != cudaSuccess) return cuda_fail(e, "bundle");
  if (herr) return fail(HDC_ERR_INVALID_VALUE, "labels outside [0, K)");
  return HDC_OK;
}

hdc_status_t hdc_argmax(const float* S, int64_t N, int64_t K, int32_t* labels, void* stream) {
  if (N < 0 || K < 1) return fail(HDC_ERR_INVALID_VALUE, "N >= 0, K >= 1 required");
  if (N > 0 && (!S || !labels)) return fail(HDC_ERR_INVALID_VALUE, "null S or labels");
  if (!aligned(S, 4) || !aligned(labels, 4)) return fail(HDC_ERR_MISALIGNED, "alignment");
  cudaError_t e = launch_argmax(S, N, K, labels, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "argmax launch");
  return HDC_OK;
}

hdc_status_t hdc_infer(const float* X, const float* B, const float* C, int64_t N, int64_t F,
                       int64_t D, int64_t K, int32_t* labels, float* scores,
                       hdc_precision_t prec, void* stream) {
  hdc_model_t m = nullptr;
  hdc_status_t st = hdc_model_create(B, C, F, D, K, prec, &m);
  if (st != HDC_OK) return st;
  st = hdc_model_infer(m, X, N, labels, scores, stream);
  hdc_model_destroy(m);
  return st;
}

int64_t hdc_model_recheck_count(hdc_model_t m) {
  if (!m) return -1;
  DeviceGuard dg(m->device);
  unsigned long long v = 0;
  cudaDeviceSynchronize();
  if (cudaMemcpy(&v, m->recheck, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return (int64_t)v;
}

int32_t hdc_model_last_launch_count(hdc_model_t m) { return m ? m->last_launches : -1; }

int32_t hdc_model_last_kernel(hdc_model_t m) { return m ? m->last_kernel : -1; }

int32_t hdc_model_tc_tile_n(hdc_model_t m) {
  if (!m) return -1;
  return m->Btc ? tc_tile_n(tc_mode_of(m), m->K) : 0;
}

hdc_status_t hdc_model_set_kernel_timing(hdc_model_t m, int enable) {
  if (!m) return fail(HDC_ERR_INVALID_VALUE, "null model");
  DeviceGuard dg(m->device);
  if (enable && !m->ev0) {
    if (cudaEventCreate(&m->ev0) != cudaSuccess || cudaEventCreate(&m->ev1) != cudaSuccess)
      return fail(HDC_ERR_CUDA, "event creation");
  }
  m->timing = enable != 0;
  return HDC_OK;
}

float hdc_model_last_kernel_ms(hdc_model_t m) {
  if (!m || !m->timing || !m->ev0) return -1.f;
  DeviceGuard dg(m->device);
  if (cudaEventSynchronize(m->ev1) != cudaSuccess) return -1.f;
  float ms = -1.f;
  if (cudaEventElapsedTime(&ms, m->ev0, m->ev1) != cudaSuccess) return -1.f;
  return ms;
}

}  // extern "C"
