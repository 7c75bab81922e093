// qmb_kernels.cuh -- launch interfaces of the non-GEMM kernels.
#pragma once
#include "qmb_common.cuh"
#include "qmb_gemm.cuh"

namespace qmb {

// ---------------------------------------------------------------- RMSNorm
// numpy pairwise-sum plan for a row of length n (loops_utils.h.src pairwise_sum):
// leaves of <= 128 elements in order, and the combine tree in postfix form.
constexpr int RMS_MAX_LEAVES = 160;
struct PairwisePlan {
  int n;
  int nleaves;
  int nops;
  int leaf_start[RMS_MAX_LEAVES];
  short leaf_len[RMS_MAX_LEAVES];
  short ops[2 * RMS_MAX_LEAVES];  // >=0: push leaf i; -1: pop two, push sum
};
bool make_pairwise_plan(int n, PairwisePlan* plan);

// res = x_out + x_res (written to res_out, may alias x_res); u = rmsnorm(res, gain);
// if u_q: u_q = quantize(u, s_out); if y_out: y_out = u (f32).
cudaError_t rmsnorm_residual(const float* x_out, const float* x_res, float* res_out, const float* gain,
                             const PairwisePlan& plan, float eps, float s_out, int qmax, int8_t* u_q, float* y_out,
                             long long M, uint32_t* err, cudaStream_t st);

// ---------------------------------------------------------------- quantize
cudaError_t quantize_f32(const float* x, long long n, float s, int qmax, int8_t* out, uint32_t* err,
                         cudaStream_t st);
// Strided 2D version (rows x cols, row strides in elements).
cudaError_t quantize_f32_2d(const float* x, long long ldx, long long rows, long long cols, float s, int qmax,
                            int8_t* out, long long ldo, uint32_t* err, cudaStream_t st);

// ---------------------------------------------------------------- conv + SiLU + requant
struct ConvParams {
  const int8_t* x;       // [B*T, ldx] int8 (conv input, token-major)
  long long ldx;
  const int8_t* w;       // [K, C] int8 taps (reference layout)
  const float* bias;     // [C] dequantized bias or nullptr
  const int8_t* bias_q;  // alternatively: [C] int8 bias dequantized on the fly as f32(f64(q) * bias_scale)
  double bias_scale;
  int8_t* out;           // [B*T, ldo]
  long long ldo;
  int8_t* state_out;     // [B, K-1, C] last K-1 input rows (zero-padded), or nullptr
  int B, T, C, K;
  float s_conv;          // f32(s_x * s_w)
  float s_out;           // f32(s_out)
  int qmax;
  uint32_t* err;
  float inv_out, silu_thr;  // set by conv_silu_quant (1 / s_out; verified fast-path threshold)
};
// Verified fast-path threshold of quantize(silu(v), s_out) (cached per scale).
float silu_quant_thr(float s_out, int qmax, cudaStream_t st);
cudaError_t conv_silu_quant(const ConvParams& p, cudaStream_t st);
// Decode step: state [B, K-1, C] (in/out), x [B, C] new row -> out [B, C].
cudaError_t conv_step(const int8_t* x, long long ldx, int8_t* state, const int8_t* w, const float* bias,
                      int8_t* out, long long ldo, int B, int C, int K, float s_conv, float s_out, int qmax,
                      uint32_t* err, cudaStream_t st);

// ---------------------------------------------------------------- Hadamard + quant
struct HadParams {
  const float* y;   // [M, ldy]
  long long ldy;
  int8_t* out;      // [M, ldo]
  long long ldo;
  float* yh;        // optional f32 transformed output [M, n] (tests), or nullptr
  long long M;
  int p, m;         // n = 2^p * m
  uint32_t base_rows[20];  // bit k of row o set => B[o][k] = +1
  float s_out;
  int qmax;
  uint32_t* err;
  // set by hadamard_quant: packed {+-1, +-1} sign pairs (index 2*[lo < 0] + [hi < 0])
  unsigned long long sgn2[4];
};
cudaError_t hadamard_quant(const HadParams& p, cudaStream_t st);

// ---------------------------------------------------------------- selective scan
struct ScanParams {
  const int8_t* x;  long long ldx;    // scan input x_q   [B*T, ldx]
  const int8_t* dt; long long lddt;   // delta_q          [B*T, lddt]
  const int8_t* bq; const int8_t* cq; long long ldbc;  // [B*T, ldbc] each
  const float* z;   long long ldz;    // gate input z or nullptr (no gate)
  int z_silu;                         // z already holds silu(z) (computed in the in_proj epilogue)
  float* y;         long long ldy;    // output (may alias z)
  const float* lut_x; const float* lut_dt; const float* lut_b; const float* lut_c;  // 256-entry, index q+128
  const float* a;                     // [E, N] dequantized a (direct-exp path)
  const uint8_t* a_col;               // [E, N] column into exp_lut (LUT path)
  const float* exp_lut; int exp_ncols;  // [128][exp_ncols]: expf(deq_dt[q] * a_col value), q in [0,127]
  const float* exp_tab;               // [E, 128, 16] per-channel expf rows (d_state 16) or nullptr
  const float* d;                     // [E] dequantized d
  float* bcf;                         // [B*T, 2N] scratch for dequantized b | c rows (batch-tiled scan), or null
  // {-0.0f, -0.0f} and {1.0f, 1.0f} as runtime operands: fma.rn.f32x2(a, b, NEGZ) is an
  // exactly rounded product and fma.rn.f32x2(a, ONE, c) an exactly rounded sum; being
  // opaque to ptxas they cannot be folded/contracted (literal constants would be).
  unsigned long long negz2, one2;
  // dequantization of x / dt as fma(q, hi, q * lo) (3 ALU ops instead of a table
  // gather); dq_fast is set only when the host verified it equals
  // f32(f64(q) * s) for every q in [-128, 127] (deq_split in qmb_block.cu)
  float dq_x_hi, dq_x_lo, dq_dt_hi, dq_dt_lo;
  int dq_fast;
  int fast;                           // scan_exp = 2: approximate exp (MUFU ex2) in the batch-tiled
                                      // kernel, not bit-exact (B < 16 and decode stay exact)
  float* h;                           // [B, E, N] carried state (in if h_in, out if h_out)
  int h_in, h_out;
  int B, T, E, N;
  uint32_t* err;
};
// use_lut: 1 = per-layer expf table in shared memory (prefill kernels), 2 = same
// table read through L1 (decode), 0 = direct FP64 glibc-expf restatement.
cudaError_t selective_scan(const ScanParams& p, int use_lut, cudaStream_t st);
// exp_tab[(i * 128 + r) * 16 + j] = glibc_expf(lut_dt[r + 128] * a[i * 16 + j]) (the layer's
// per-channel exp rows, resident with the block handle: decode reads a row per
// channel-step, prefill CTAs copy their 16 channels into shared memory)
cudaError_t build_exp_tab(const float* lut_dt, const float* a, int E, float* exp_tab, cudaStream_t st);
// exp_lut[r * ncols + c] = glibc_expf(lut_dt[r + 128] * a_vals[c]) for r in [0, 127]
cudaError_t build_exp_lut(const float* lut_dt, const float* a_vals, int ncols, float* exp_lut, cudaStream_t st);

// Decode scan with dt_proj fused (x_proj's b | c | dt_r codes as input): see
// decode_scan_kernel.
struct DecodeScanParams {
  const int8_t* x; long long ldx;     // [B, ldx] conv output (scan input) codes
  float* z;                           // [B, E] silu(z) in, gated y out
  const int8_t* bq; const int8_t* cq; const int8_t* dtr; long long ld_dtr;  // x_proj outputs
  const int8_t* w_dt; long long ld_wdt; int R;  // [E, ld_wdt] dt_proj weights (K-major)
  const int8_t* delta; long long ld_delta;       // non-null: dt_proj already ran, its codes [B, ld_delta]
  float dt_scale; const float* dt_bias; const float* qtab; float dt_div, dt_inv;
  const float* lut_x; const float* lut_dt; const float* lut_b; const float* lut_c;
  const float* exp_tab; const float* d;
  float* h;                           // [B, E, 16] carried state (updated)
  int B, E, qmax;
  uint32_t* err;
};
bool decode_scan_ok(int B, int E, int N, int Nx, int R, long long ld_wdt);
cudaError_t decode_scan(const DecodeScanParams& p, cudaStream_t st);

// Tied LM head: out[M, V] = x[M, K] @ emb[V, K]^T, f32 (FFMA2 register-blocked GEMM).
cudaError_t lm_head(const float* x, int M, int K, const float* emb, int V, float* out, cudaStream_t st);
cudaError_t argmax_rows(const float* x, int M, int V, long long ld, long long* out, cudaStream_t st);
cudaError_t lm_split16(const float* x, int M, int K, void* out16, float* inv, cudaStream_t st);
cudaError_t lm_combine16(const float* p, const float* q, const float* inv, int M, int V, int k, float* out,
                         cudaStream_t st);

// Verified softplus+quantize threshold table (QTAB_FLOATS floats at `tab`);
// scratch2: 2 device uint32 words.  Enqueued on `st` (the sweep covers all 2^32 floats).
cudaError_t build_softplus_qtab(float s_div, int qmax, float* tab, uint32_t* scratch2, cudaStream_t st);

// ---------------------------------------------------------------- misc
cudaError_t transpose_i8(const int8_t* src, long long rows, long long cols, long long lds, int8_t* dst,
                         long long ldd, cudaStream_t st);  // dst[c, r] = src[r, c]
cudaError_t embed_gather(const float* table, const long long* tokens, long long n, int D, float* out,
                         cudaStream_t st);
// Elementwise exact transcendentals (for the parity harness).
cudaError_t eval_math(int fn, const float* x, float* y, long long n, cudaStream_t st);
// Bitwise comparison of eval_math functions fa, fb over all 2^32 float inputs
// (device counters: mismatch count, smallest mismatching bit pattern or ~0u).
cudaError_t verify_math(int fa, int fb, unsigned long long* bad, uint32_t* first, cudaStream_t st);

}  // namespace qmb
