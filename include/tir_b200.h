/*
 * tir_b200.h — C-ABI of the B200 (sm_100a) tensorized-operator library.
 *
 * This is the drop-in boundary for the reference's intrinsic dispatch path:
 *
 *   tir::run → Interp::dispatch_call → HostKernel(std::vector<TensorView>&)
 *   (/root/reference/proj/src/interp.cc:360-383, include/tir/interp.h:120)
 *
 * A HostKernel registered on tir::ExecContext (interp.cc:147-152) receives the
 * operand views [writes[0], reads...] (interp.cc:371-373) and must compute the
 * intrinsic's semantics *accumulating* into the output window (blockize moves
 * `init` to the outer block, schedule_block.cc:570-603; the reference's own
 * intrinsic test reads C first, tests/test_interp.cc:186). The C++ adapter in
 * paper_2207_04296_b200/adapter/ packs the views and calls the entry points
 * below; nothing here uses torch or C++ types.
 *
 * Operand conventions (following tests/testing/workloads.h):
 *   GMM  A[M,K] fp16 row-major, B[K,N] fp16 row-major (N contiguous, workloads.h:45-51),
 *        C[M,N] fp32 (or fp16) row-major.  C (+)= A·B, fp32 accumulation.
 *   CONV X[N,(D,)(H,)W,CI] fp16 (NLC / NHWC / NDHWC, workloads.h:93-99),
 *        W[(KD,)(KH,)KW,CI/G,CO] fp16 (HWIO-style), Y[N,(OD,)(OH,)OW,CO].
 *        Covers C1D, C2D, C3D, DIL (dilation), GRP (groups), T2D (transposed,
 *        gather form), and DEP (groups == CI == CO, CI/G == 1: W is [KH,KW,C],
 *        workloads.h:132-137).
 *
 * All entry points are thread-safe given distinct streams, never throw, and
 * return a status code; tir_b200_last_error() returns a thread-local message.
 */
#ifndef TIR_B200_H_
#define TIR_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The adapter maps them onto tir::Error kinds (ir.h:33-48). */
#define TIR_B200_OK 0
#define TIR_B200_ERR_VALUE 1       /* bad argument / inexact fp16 input -> "ValueError"    */
#define TIR_B200_ERR_UNSUPPORTED 2 /* legal op the kernels do not cover -> "UnsupportedShape" */
#define TIR_B200_ERR_CUDA 3        /* CUDA runtime / driver failure    -> "CudaError"       */

/* Operator tags (the paper's single-op suite). Informational for GMM..T2D; DEP
 * selects the CUDA-core depthwise kernel. */
typedef enum {
  TIR_B200_GMM = 0,
  TIR_B200_C1D = 1,
  TIR_B200_C2D = 2,
  TIR_B200_C3D = 3,
  TIR_B200_DIL = 4,
  TIR_B200_GRP = 5,
  TIR_B200_T2D = 6,
  TIR_B200_DEP = 7
} tir_b200_op;

/* Convolution geometry. Spatial dims are (D, H, W), outermost first; unused
 * leading dims are 1 (C1D: D = H = 1, C2D: D = 1). Output extents follow
 *   forward:    O = (I + 2p - d(K-1) - 1) / s + 1
 *   transposed: O = (I - 1) s - 2p + d(K-1) + 1        (T2D, gather form)     */
typedef struct {
  int32_t op;         /* tir_b200_op */
  int32_t transposed; /* 1: T2D gather form, out[o] += in[(o+p-k d)/s] w[k] when divisible */
  int64_t n;
  int64_t in_d, in_h, in_w;
  int64_t ci, co;
  int64_t k_d, k_h, k_w;
  int64_t s_d, s_h, s_w;
  int64_t p_d, p_h, p_w;
  int64_t d_d, d_h, d_w; /* dilation */
  int64_t groups;
} tir_b200_conv_desc;

/* Fused epilogue, applied per output element after the
 * reduction, in this order:
 *   v = acc;  v = Yin + v (accumulate);  v = v + bias[col];  v = v + residual[elem];
 *   v = act(v).
 * `bias` is fp32 per output column (GMM: N, conv: CO); `residual` is fp16 with
 * Y's shape and layout (a ResNet / MobileNet shortcut); `relu` selects act:
 *   0 none, 1 ReLU max(v, 0), 2 ReLU6 min(max(v, 0), 6), 3 GELU (erf form).
 * Every field may be 0/NULL. gemm + relu is the reference's gemm_relu_source
 * workload (tests/testing/workloads.h:61-91) as one intrinsic. DEP supports
 * bias and act but not residual. */
#define TIR_B200_ACT_NONE 0
#define TIR_B200_ACT_RELU 1
#define TIR_B200_ACT_RELU6 2
#define TIR_B200_ACT_GELU 3
typedef struct {
  const float* bias;
  int32_t relu;
  const uint16_t* residual;
} tir_b200_epilogue;

/* Library / device facts. */
int tir_b200_version(void);
const char* tir_b200_last_error(void);
/* Number of kernel launches issued by this thread since the last reset
 * (bench.py's gpu_launches evidence). */
int64_t tir_b200_launch_count(void);
void tir_b200_reset_launch_count(void);

/* Relayout scratch is one grow-only device buffer per (device, stream); a
 * CUDA graph captured over a CI % 8 != 0 conv keeps pointing at it, so buffers
 * are never freed implicitly. Call this only when no captured graph or
 * in-flight launch still uses them (it synchronises every device it touched). */
int tir_b200_release_workspaces(void);

/* Planner switches (csrc/options.h): tile shape, pipeline depth,
 * epilogue flavour — never the result. Initialised once from TIR_B200_<NAME>
 * environment variables; these calls change them at run time for the whole
 * process. Returns TIR_B200_ERR_VALUE for an unknown name. */
int tir_b200_set_option(const char* name, int value);
int tir_b200_get_option(const char* name, int* value);

/* Output extents (OD, OH, OW) for a descriptor; validates it. */
int tir_b200_conv_out_shape(const tir_b200_conv_desc* desc, int64_t out_dhw[3]);

/* ---- device-pointer entry points (asynchronous on `stream`, a cudaStream_t) ----
 * accumulate = 1: Y = Yin + op(X, W) (Yin may alias Y); 0: Y = op(X, W).
 * out_f16 = 1: Y is fp16 (round-to-nearest of the fp32 result); else fp32.
 * Yin, when used, is always fp32. */
int tir_b200_gmm(const uint16_t* A, const uint16_t* B, const float* Cin, void* C,
                 int64_t M, int64_t N, int64_t K, int accumulate, int out_f16, void* stream);

int tir_b200_conv(const tir_b200_conv_desc* desc, const uint16_t* X, const uint16_t* W,
                  const float* Yin, void* Y, int accumulate, int out_f16, void* stream);

/* The same with a fused epilogue (epi may be NULL). */
int tir_b200_gmm_ex(const uint16_t* A, const uint16_t* B, const float* Cin, void* C, int64_t M,
                    int64_t N, int64_t K, int accumulate, int out_f16, const tir_b200_epilogue* epi,
                    void* stream);

int tir_b200_conv_ex(const tir_b200_conv_desc* desc, const uint16_t* X, const uint16_t* W,
                     const float* Yin, void* Y, int accumulate, int out_f16,
                     const tir_b200_epilogue* epi, void* stream);

/* ---- host-buffer entry points (synchronous; H2D, compute, D2H) ----
 * These are what the reference-side HostKernel adapter calls: operands live in
 * host memory (the interpreter's TensorValues hold fp16 values as f32, ir.cc:36-47),
 * so inputs are passed as f32 and converted to fp16 on the device; a value that
 * is not exactly representable in fp16 is rejected with TIR_B200_ERR_VALUE.
 * C/Y is read (accumulate = 1) and written as f32. Device buffers and pinned
 * staging are cached per thread. */
int tir_b200_gmm_host_f32(const float* A, const float* B, float* C, int64_t M, int64_t N,
                          int64_t K, int accumulate);

int tir_b200_conv_host_f32(const tir_b200_conv_desc* desc, const float* X, const float* W,
                           float* Y, int accumulate);

/* Same, but with fp16 host inputs (pinned or pageable), the e2e benchmark path. */
int tir_b200_gmm_host(const uint16_t* A, const uint16_t* B, float* C, int64_t M, int64_t N,
                      int64_t K, int accumulate);

int tir_b200_conv_host(const tir_b200_conv_desc* desc, const uint16_t* X, const uint16_t* W,
                       float* Y, int accumulate);

/* ---- network-graph glue, device pointers, asynchronous ----
 * fp16 NHWC / row-major operands, 16-byte aligned, channel / column counts a
 * multiple of 8. The networks' contractions (every conv / GEMM, with bias,
 * residual and activation fused) go through tir_b200_conv_ex / tir_b200_gmm_ex. */
/* Y[n, OH, OW, c] = max over k x k windows (stride s, padding p never wins). */
int tir_b200_maxpool2d(const uint16_t* X, uint16_t* Y, int64_t n, int64_t h, int64_t w, int64_t c,
                       int64_t k, int64_t s, int64_t p, void* stream);
/* Y[n, c] = fp16(sum over hw pixels of X[n, hw, c] / hw), fp32 sum. */
int tir_b200_avgpool_global(const uint16_t* X, uint16_t* Y, int64_t n, int64_t hw, int64_t c,
                            void* stream);
/* Y[r, :] = LayerNorm(X[r, :]) * gamma + beta (fp32 statistics), cols <= 8192. */
int tir_b200_layernorm(const uint16_t* X, uint16_t* Y, const float* gamma, const float* beta,
                       int64_t rows, int64_t cols, float eps, void* stream);
/* Y[r, :] = softmax(scale * X[r, :]) (fp32 internally), cols <= 8192. */
int tir_b200_softmax(const uint16_t* X, uint16_t* Y, int64_t rows, int64_t cols, float scale,
                     void* stream);

/* ---- batched GMM (attention: per-(sequence, head) problems over strided views) ----
 * Problem z = z1 * z2n + z2 (0 <= z1 < z1n, 0 <= z2 < z2n) computes
 *   C[cr + m, cc + n] = epilogue( sum_k A[ar + m, ac + k] * B[br + k, bc + n] )
 * where A [a_rows, lda], B [b_rows, ldb] (N contiguous) and C [c_rows, ldc] are
 * plain row-major fp16 (C fp16 or fp32) tensors and each of ar, ac, br, bc, cr,
 * cc is base + z1 * step1 + z2 * step2 (elements). No copies of the strided
 * per-head views are made. M % 128 == 0, K % 64 == 0 and N % 32 == 0 per
 * problem; bias (if any) is indexed by the problem-local column n. */
typedef struct {
  int64_t z1n, z2n;
  int64_t a_row[3], a_col[3]; /* base, per-z1 step, per-z2 step */
  int64_t b_row[3], b_col[3];
  int64_t c_row[3], c_col[3];
  int64_t b_kmajor; /* 1: B is given transposed, B_z[k, n] = B[br + n, bc + k] (K contiguous,
                       e.g. attention's K rows read straight from the QKV tensor) */
} tir_b200_batch_desc;

int tir_b200_gmm_batched(const uint16_t* A, int64_t a_rows, int64_t lda, const uint16_t* B,
                         int64_t b_rows, int64_t ldb, void* C, int64_t c_rows, int64_t ldc, int64_t M,
                         int64_t N, int64_t K, const tir_b200_batch_desc* batch, int out_f16,
                         const tir_b200_epilogue* epi, void* stream);

/* Frees the calling thread's cached device/pinned buffers. */
void tir_b200_release_host_cache(void);

#ifdef __cplusplus
}
#endif

#endif /* TIR_B200_H_ */
