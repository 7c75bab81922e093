/*
 * qmb.h -- C ABI of the B200-native Quamba W8A8 Mamba-block library (libqmb.so).
 *
 * Drop-in boundary for the reference package `ssmq` (arXiv 2410.13229 reference,
 * paths relative to its pkg/ directory).  Every entry point below replaces one
 * reference function on the quantized block path; the citation names it.
 *
 * Conventions (mirroring the reference's operator contracts):
 *  - All tensor pointers are DEVICE pointers owned by the caller, except the
 *    host weight/table pointers inside qmb_block_desc (copied by create).
 *  - Activations are token-major: row m = b*T + t, features contiguous.
 *  - Scales are passed exactly as the reference holds them (Python float =
 *    IEEE double); the library derives every f32 constant the way numpy does
 *    (np.float32(s_a * s_b * extra), f32(s) as a divisor, f32(f64(q)*s) for
 *    dequantization) so integer outputs are bit-exact.
 *  - Functions enqueue on `stream` and never synchronize.  They return 0 on
 *    success, a negative QMB_E* code for an argument error (message via
 *    qmb_last_error(), text mirrors the reference's ValueError), or a positive
 *    cudaError_t.
 *  - Data-dependent failures the reference raises at run time set bits in the
 *    caller's device word *err_flag (may be NULL): QMB_ERR_NONFINITE for
 *    ValueError("non-finite activation") (quant.py:149-150), QMB_ERR_SCAN for
 *    FloatingPointError("scan divergence") (kernels.py:97-98).  The host shim
 *    checks the word at its next sync point.
 *  - Handles are immutable after create; all functions are reentrant.
 */
#ifndef QMB_H
#define QMB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* qmb_stream_t; /* == cudaStream_t */

#define QMB_ABI_VERSION 1

#define QMB_ERR_NONFINITE 1u
#define QMB_ERR_SCAN 2u

#define QMB_E_ARG (-1)      /* invalid argument (shape/scale/range) */
#define QMB_E_UNSUPP (-2)   /* shape outside what the kernels support */
#define QMB_E_WS (-3)       /* workspace too small */

/* Quantization modes: qblock.py:32-44 (Mode) */
#define QMB_MODE_NAIVE 0
#define QMB_MODE_IN_PERCENTILE 1
#define QMB_MODE_OUT_HADAMARD 2
#define QMB_MODE_FULL 3

/* Activation sites, in ACT_SITES order (qblock.py:57). */
enum {
  QMB_ACT_IN = 0, QMB_ACT_CONV_IN, QMB_ACT_CONV_OUT, QMB_ACT_X, QMB_ACT_B, QMB_ACT_C,
  QMB_ACT_DT_R, QMB_ACT_DT, QMB_ACT_Y, QMB_ACT_Y_HAD, QMB_NUM_ACT
};

/* One int8 weight tensor in the reference's layout (QTensor values + scale). */
typedef struct {
  const int8_t* data; /* host pointer, C-contiguous, reference shape */
  double scale;
} qmb_qweight;

/* Host description of a QuantizedBlock (qblock.py:75-95) + its BlockConfig
 * (ssm.py:21-40) and HadamardPlan (hadamard.py:87-106). */
typedef struct {
  int d_model, d_inner, d_state, d_conv, dt_rank;
  int bit_width;           /* QuantizedBlock.bit_width (2..8) */
  int mode;                /* QMB_MODE_* */
  double act[QMB_NUM_ACT]; /* ScaleEntry.scale per site */
  /* weights, reference shapes (SSMParams docstring, ssm.py:43-54) */
  qmb_qweight a;          /* (d_inner, d_state) */
  qmb_qweight d;          /* (d_inner,) */
  qmb_qweight w_in;       /* (d_model, 2*d_inner) */
  qmb_qweight conv_w;     /* (d_conv, d_inner) */
  qmb_qweight conv_b;     /* (d_inner,) */
  qmb_qweight w_b;        /* (d_inner, d_state) */
  qmb_qweight w_c;        /* (d_inner, d_state) */
  qmb_qweight w_dt_rank;  /* (d_inner, dt_rank) */
  qmb_qweight w_dt;       /* (dt_rank, d_inner) */
  qmb_qweight dt_bias;    /* (d_inner,) */
  qmb_qweight w_out;      /* (d_inner, d_model); used in non-Hadamard modes */
  qmb_qweight w_out_h;    /* (d_inner, d_model) = quantize(H W_out); Hadamard modes */
  int had_p, had_m;       /* d_inner = 2^p * m, m in {1, 12, 20} */
  const int8_t* had_base; /* (m, m) +/-1 host table */
} qmb_block_desc;

typedef struct qmb_block qmb_block;

/* Workspace slots of one prefill (offsets via qmb_block_workspace_layout). */
enum {
  QMB_WS_UPAD = 0, /* int8 [M, Dp]    padded u_q copy (only when d_model % 16) */
  QMB_WS_XQ,       /* int8 [M, E]     in_proj x-half, quantized at conv_in */
  QMB_WS_Z,        /* f32  [M, E]     in_proj z-half; overwritten by gated y */
  QMB_WS_SCANX,    /* int8 [M, Ep]    conv+SiLU output = scan input x */
  QMB_WS_B,        /* int8 [M, N]     x_proj -> b */
  QMB_WS_C,        /* int8 [M, N]     x_proj -> c */
  QMB_WS_DTR,      /* int8 [M, Rp]    x_proj -> dt_r */
  QMB_WS_DELTA,    /* int8 [M, E]     dt_proj+softplus -> delta_q */
  QMB_WS_YQ,       /* int8 [M, Ep]    Hadamard (or direct) quantized y */
  QMB_WS_BCF,      /* f32  [M, 36]    dequantized b | c rows, 4 pad floats (scan operand, N = 16) */
  QMB_WS_ACC32,    /* int32 split-K partials (19 MB, only when M <= 128: decode) */
  QMB_WS_COUNT
};

/* ---- library ---- */
int qmb_abi_version(void);
const char* qmb_last_error(void);

/* ---- block handle: quantize_block's product, uploaded (qblock.py:223-240) ---- */
int qmb_block_create(const qmb_block_desc* desc, qmb_block** out);
void qmb_block_destroy(qmb_block* blk);
size_t qmb_block_workspace_bytes(const qmb_block* blk, long long rows);
int qmb_block_workspace_layout(const qmb_block* blk, long long rows, size_t offsets[QMB_WS_COUNT]);

/* block_forward_q (qblock.py:185-215), batched: u_q [B*T, d_model] int8 at
 * scale u_scale (<= 0 selects act[in]; qblock.py:194 uses u_q.scale) ->
 * out [B*T, d_model] f32.  Optional state outputs for the
 * decode handoff: conv_state_out [B, d_conv-1, d_inner] int8 (last x_q rows),
 * ssm_state_out [B, d_inner, d_state] f32 (final h of scan_core, kernels.py:99).
 * scan_exp: 0 = tabulated exact expf (default), 1 = direct FP64 restatement,
 *   2 = fast mode: approximate exp (MUFU ex2) and contracted FMAs in the
 *   batch-tiled prefill scan (B >= 16), NOT bit-exact -- y within a stated tolerance
 *   of the exact scan; smaller batches and decode run exact. */
int qmb_block_prefill(const qmb_block* blk, const int8_t* u_q, double u_scale, int B, int T, float* out,
                      int8_t* conv_state_out, float* ssm_state_out, int scan_exp,
                      void* workspace, size_t ws_bytes, uint32_t* err_flag, qmb_stream_t stream);

/* Same, accumulating: res[m, :] += block output (bit-identical to the residual
 * add `x_out + x_res` of the next fused_rmsnorm_quant, qblock.py:181, folded into
 * out_proj's epilogue; forward_q's loop (model.py:246-258) then normalizes res
 * directly).  Model-level fusion, not a reference operator. */
int qmb_block_prefill_accum(const qmb_block* blk, const int8_t* u_q, double u_scale, int B, int T, float* res,
                            int8_t* conv_state_out, float* ssm_state_out, int scan_exp,
                            void* workspace, size_t ws_bytes, uint32_t* err_flag, qmb_stream_t stream);
int qmb_block_decode_accum(const qmb_block* blk, const int8_t* u_q, double u_scale, int B, int8_t* conv_state,
                           float* ssm_state, float* res, void* workspace, size_t ws_bytes,
                           uint32_t* err_flag, qmb_stream_t stream);

/* Quantized single-token decode (no reference function: semantics = last row
 * of block_forward_q on the prefix; state carry pinned by test_formats.py:76-94).
 * u_q [B, d_model]; conv_state [B, d_conv-1, d_inner] and ssm_state
 * [B, d_inner, d_state] updated in place; out [B, d_model] f32. */
int qmb_block_decode(const qmb_block* blk, const int8_t* u_q, double u_scale, int B, int8_t* conv_state,
                     float* ssm_state, float* out, void* workspace, size_t ws_bytes,
                     uint32_t* err_flag, qmb_stream_t stream);

/* Prefill with per-stage device timing (CUDA events on `stream`; synchronizes).
 * stage_ms: in_proj, conv, x_proj, dt_proj, scan, output quant, out_proj. */
#define QMB_NUM_STAGES 7
/* Tensor-parallel E-sharding: a handle created from a
 * contiguous channel slice [e0, e0 + d_inner) of a block (w_in's x and z columns,
 * conv, a, d, dt_bias and w_dt's columns of those channels; w_b / w_c / w_dt_rank
 * and w_out(_h) rows of those channels as K-slices; every scale unchanged) runs
 * one layer in four stages around three collectives:
 *   1  in_proj, conv, x_proj partial    -> xacc  [M, 2N + R] int32   (all-reduce SUM)
 *   2  x_proj requant, dt_proj, scan    -> y_local [M, d_inner] f32  (all-gather over channels)
 *   3  Hadamard (FULL plan) of y_full, out_proj partial of the local K-slice
 *                                       -> oacc  [M, D] int32        (all-reduce SUM)
 *   4  out_proj epilogue (+= out if accumulate)
 * The int32 sums are exact in any order: the result is bit-identical to the
 * unsharded qmb_block_prefill / qmb_block_decode.  The same workspace must be
 * passed to every stage of a step; conv_state / ssm_state are the local
 * channels' (decode: in-out; prefill: outputs, nullable). */
typedef struct {
  int stage;                 /* 1..4 */
  int32_t* xacc;             /* [M, 2N + R] */
  float* y_local;            /* [M, d_inner] */
  const float* y_full;       /* [M, e_full] */
  int8_t* yq_full;           /* [M, e_full] scratch */
  long long e_full;          /* full d_inner (multiple of 16) */
  int e0;                    /* first channel of this handle (multiple of 16) */
  int had_p, had_m;          /* full-width Hadamard plan (Hadamard modes) */
  const int8_t* had_base;    /* [had_m, had_m] host pointer */
  int32_t* oacc;             /* [M, d_model] */
} qmb_tp_args;
int qmb_block_tp_stage(const qmb_block* blk, const qmb_tp_args* tp, const int8_t* u_q, double u_scale, int B,
                       int T, int decode, int8_t* conv_state, float* ssm_state, float* out, int accumulate,
                       void* ws, size_t ws_bytes, uint32_t* err_flag, qmb_stream_t stream);

int qmb_block_prefill_profiled(const qmb_block* blk, const int8_t* u_q, double u_scale, int B, int T,
                               float* out, int scan_exp, void* workspace, size_t ws_bytes,
                               uint32_t* err_flag, qmb_stream_t stream, float stage_ms[QMB_NUM_STAGES]);

/* ---- operator mirrors (qblock.py / quant.py / hadamard.py) ---- */

/* fused_rmsnorm_quant (qblock.py:170-182): res = x_out + x_res (x_res may be
 * NULL = zeros); u = rmsnorm(res, gain) (ssm.py:104-107, eps 1e-6);
 * u_q = quantize(u, s_out).  res_out may alias x_res; u_q or y_out may be NULL
 * (y_out receives the f32 normalized rows: the model's final norm). */
int qmb_rmsnorm_residual_quant(const float* x_out, const float* x_res, float* res_out,
                               const float* gain, long long M, int D, double s_out, int bit_width,
                               int8_t* u_q, float* y_out, uint32_t* err_flag, qmb_stream_t stream);

/* quantize (quant.py:142-155) of n f32 values. */
int qmb_quantize(const float* x, long long n, double scale, int bit_width, int8_t* out,
                 uint32_t* err_flag, qmb_stream_t stream);
/* Same for float64 input (numpy divides f64 / f64 then: quantize_weight of the
 * Hadamard-fused f64 weights, qblock.py:236-239). */
int qmb_quantize_f64(const double* x, long long n, double scale, int bit_width, int8_t* out,
                     uint32_t* err_flag, qmb_stream_t stream);

/* qlinear (qblock.py:98-123): x_q [M, K] @ w_q [K, N] (reference layout) with
 * exact int32 accumulation; out = f32(acc) * f32(s_x*s_w*extra) (+ deq bias);
 * s_out > 0 -> requantized int8 out, else f32 out.  Workspace >=
 * qmb_qlinear_workspace_bytes(M, K, N).  path: 0 auto, 1 tcgen05, 2 SIMT GEMV. */
size_t qmb_qlinear_workspace_bytes(long long M, int K, int N);
int qmb_qlinear(const int8_t* x_q, long long M, int K, double s_x, const int8_t* w_q, int N,
                double s_w, const int8_t* bias_q, double s_bias, double s_out, double extra_scale,
                int bit_width, void* out, void* workspace, size_t ws_bytes, int path,
                uint32_t* err_flag, qmb_stream_t stream);

/* fused_qconv (qblock.py:126-143) over B independent sequences of length T:
 * x_q [B*T, C], w_q [K, C], bias_q [C] or NULL -> out [B*T, C] int8. */
int qmb_fused_qconv(const int8_t* x_q, int B, int T, int C, double s_x, const int8_t* w_q, int K,
                    double s_w, const int8_t* bias_q, double s_bias, double s_out, int bit_width,
                    int8_t* out, uint32_t* err_flag, qmb_stream_t stream);

/* quantized_selective_scan (qblock.py:146-167) over B sequences:
 * a_q [D, N], b_q/c_q [B*T, N], d_q [D], dt_q/x_q [B*T, D] -> y [B*T, D] f32.
 * h (nullable) [B, D, N] f32: carried state in (if h_in) and final state out
 * (kernels.py:69-99 h0 / returned h). */
int qmb_selective_scan(const int8_t* a_q, double s_a, const int8_t* b_q, double s_b,
                       const int8_t* c_q, double s_c, const int8_t* d_q, double s_d,
                       const int8_t* dt_q, double s_dt, const int8_t* x_q, double s_x,
                       int B, int T, int D, int N, float* h, int h_in, float* y,
                       void* ws, size_t ws_bytes, uint32_t* err_flag, qmb_stream_t stream);
/* Device workspace qmb_selective_scan needs for d_inner D, d_state N (its
 * dequantized a / d and dequant tables; the library allocates nothing per call). */
size_t qmb_selective_scan_workspace_bytes(int D, int N);

/* hadamard_quantize (hadamard.py:164-166): y [M, n] f32, n = 2^p*m ->
 * out [M, n] int8; y_h (nullable) receives the f32 transform (apply_hadamard). */
int qmb_hadamard_quantize(const float* y, long long M, int p, int m, const int8_t* base,
                          double scale, int bit_width, int8_t* out, float* y_h,
                          uint32_t* err_flag, qmb_stream_t stream);

/* Elementwise restated transcendentals (parity harness): fn 0 np.exp f32,
 * 1 glibc expf, 2 glibc log1pf, 3 softplus (np.logaddexp(x,0)), 4 silu,
 * 5 silu hot-path variant, 6 / 7 the packed (f32x2) silu of the in_proj
 * epilogue, low / high half (5, 6, 7 must equal 4 everywhere). */
int qmb_eval_math(int fn, const float* x, float* y, long long n, qmb_stream_t stream);

/* Exhaustive check: fn_a and fn_b bit-identical on all 2^32 float inputs?
 * Device outputs: *mismatches (count), *first_bad (smallest mismatching bit
 * pattern, 0xffffffff if none). */
int qmb_verify_math(int fn_a, int fn_b, unsigned long long* mismatches, uint32_t* first_bad,
                    qmb_stream_t stream);

/* Measured dense int8 tensor-core peak (TOP/s): back-to-back tcgen05 kind::i8
 * 128x256x32 MMAs on every SM (roofline denominator; synchronizes). */
int qmb_measure_i8_peak(int iters, double* tops);

/* GEMM tuning probe on synthetic operands: average ms of the tcgen05 GEMM at
 * M x N x K with epilogue `mode` (0 f32/TMA store, 1 int8, 2 f32 direct,
 * 3 int8|f32 split as in_proj, 4 softplus+quant). Allocates; synchronizes. */
int qmb_gemm_bench(int M, int N, int K, int mode, int iters, float* ms);

/* Embedding row gather (model.py:249): out[r] = table[tokens[r]]. */
/* The tied f32 LM head final @ embedding^T (model.py:257-258): x [M, K], emb [V, K]
 * -> out [M, V] f32.  Tolerance-only (the reference's BLAS sums in its own order). */
int qmb_lm_head(const float* x, int M, int K, const float* emb, int V, float* out, qmb_stream_t stream);

/* The LM head above 8 rows on the fp16 tensor cores (model.py lm_head_split16, the
 * two GEMMs by cuBLAS): qmb_lm_split16 scales each row of x [M, K] by a power of two
 * s_r (max |x_r s_r| < 2^14) and splits it into fp16 halves, out16 [2M, K] = [hi; lo],
 * inv_scale[r] = 1 / s_r; qmb_lm_combine16 forms out [M, V] =
 * ((p[r] + p[M + r]) + q[r]) * inv_scale[r] * 2^-k from p = [hi; lo] W_hi^T [2M, V] and
 * q = hi W_lo^T [M, V] (W * 2^k = W_hi + W_lo). */
int qmb_lm_split16(const float* x, int M, int K, void* out16, float* inv_scale, qmb_stream_t stream);

/* Greedy next tokens (model.py greedy decoding: numpy.argmax over the vocabulary):
 * out[r] = the first index of the maximum of row r of logits [M, ld] over V columns,
 * a NaN counting as the maximum (first NaN wins). */
int qmb_argmax(const float* logits, int M, int V, long long ld, long long* out, qmb_stream_t stream);
int qmb_lm_combine16(const float* p, const float* q, const float* inv_scale, int M, int V, int k, float* out,
                     qmb_stream_t stream);

int qmb_embed_gather(const float* table, const long long* tokens, long long n, int D, float* out,
                     qmb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* QMB_H */
