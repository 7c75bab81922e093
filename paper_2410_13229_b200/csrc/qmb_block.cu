// qmb_block.cu -- C-ABI entry points (include/qmb.h): the block handle
// (quantize_block's product uploaded to HBM in kernel-native layouts) and the
// prefill / decode orchestration of block_forward_q (qblock.py:185-215).
#include <stdlib.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/qmb.h"
#include "qmb_gemm.cuh"
#include "qmb_kernels.cuh"

using namespace qmb;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return (int)e;
}

#define QMB_CUDA(call, what)                        \
  do {                                              \
    cudaError_t _e = (call);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

inline long long round_up(long long v, long long a) { return (v + a - 1) / a * a; }
inline int qmax_of(int bits) { return (1 << (bits - 1)) - 1; }
// numpy semantics of the reference's scale constants
inline float f32(double v) { return (float)v; }
inline float deq(int q, double s) { return (float)((double)q * s); }
// hi + lo split of a dequantization scale for the scan's ALU dequantization
// fma(q, hi, q * lo); true iff it reproduces f32(f64(q) * s) for every int8 code
// (checked here with the same IEEE single operations the device performs).
inline bool deq_split(double s, float* hi, float* lo) {
  *hi = (float)s;
  *lo = (float)(s - (double)*hi);
  for (int q = -128; q <= 127; ++q) {
    volatile float prod = (float)q * *lo;
    const float v = fmaf((float)q, *hi, prod);
    if (v != deq(q, s)) return false;
  }
  return true;
}

}  // namespace

struct qmb_block {
  int D, E, N, Kc, R, bits, qmax, mode;
  int in_il;  // in_proj output columns x | z interleaved in blocks of in_il (0: not interleaved)
  int Dp, Ep, Rp, Nx;
  bool had;
  int had_p, had_m;
  uint32_t base_rows[20];
  double act[QMB_NUM_ACT];
  double s_w_in, s_conv_w, s_w_b, s_w_c, s_w_dtr, s_w_dt, s_w_out;
  // device (one allocation)
  void* mem;
  int8_t* w_in_t;   // [2E, Dp]
  int8_t* conv_w;   // [Kc, E]
  float* conv_b;    // [E]
  int8_t* w_x_t;    // [Nx, Ep]: rows b | c | dt_r
  int8_t* w_dt_t;   // [E, Rp]
  float* dt_bias;   // [E]
  float* a_deq;     // [E, N]
  uint8_t* a_col;   // [E, N]
  float* exp_lut;   // [128, exp_ncols]
  int exp_ncols;
  float* exp_tab;   // [E, 128, N] expf(deq_dt[level] * a[i][j]) (N == 16 only; else null)
  float* d_deq;     // [E]
  int8_t* w_out_t;  // [D, Ep]
  float* luts;      // [4][256] dequant tables: x, dt, b, c (index q + 128)
  float* sp_qtab;   // [QTAB_FLOATS] verified softplus+quantize thresholds for dt_proj
};

extern "C" int qmb_abi_version(void) { return QMB_ABI_VERSION; }
extern "C" const char* qmb_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------ create
static int check_w(const qmb_qweight& w, const char* name) {
  if (!w.data) return fail(QMB_E_ARG, "missing weight %s", name);
  if (!(w.scale > 0.0)) return fail(QMB_E_ARG, "scale must be positive, got %g", w.scale);
  return 0;
}

extern "C" int qmb_block_create(const qmb_block_desc* d, qmb_block** out) {
  if (!d || !out) return fail(QMB_E_ARG, "null argument");
  *out = nullptr;
  if (d->d_model <= 0 || d->d_inner <= 0 || d->d_state <= 0 || d->d_conv <= 0 || d->dt_rank <= 0)
    return fail(QMB_E_ARG, "block dimensions must be positive");
  if (d->bit_width < 2 || d->bit_width > 8) return fail(QMB_E_UNSUPP, "bit width must be in [2, 8]");
  if (d->mode < 0 || d->mode > 3) return fail(QMB_E_ARG, "unknown mode %d", d->mode);
  if (d->d_state > 64) return fail(QMB_E_UNSUPP, "d_state > 64 is not supported");
  if (d->d_model > 8192) return fail(QMB_E_UNSUPP, "d_model > 8192 is not supported");
  for (int i = 0; i < QMB_NUM_ACT; ++i)
    if (!(d->act[i] > 0.0)) return fail(QMB_E_ARG, "scale must be positive, got %g", d->act[i]);
  const bool had = d->mode == QMB_MODE_OUT_HADAMARD || d->mode == QMB_MODE_FULL;
  int rc;
  if ((rc = check_w(d->a, "a")) || (rc = check_w(d->d, "d")) || (rc = check_w(d->w_in, "w_in")) ||
      (rc = check_w(d->conv_w, "conv_w")) || (rc = check_w(d->conv_b, "conv_b")) || (rc = check_w(d->w_b, "w_b")) ||
      (rc = check_w(d->w_c, "w_c")) || (rc = check_w(d->w_dt_rank, "w_dt_rank")) || (rc = check_w(d->w_dt, "w_dt")) ||
      (rc = check_w(d->dt_bias, "dt_bias")))
    return rc;
  if (had && (rc = check_w(d->w_out_h, "w_out_h"))) return fail(QMB_E_ARG, "fused output weights must be present exactly in Hadamard modes");
  if (!had && (rc = check_w(d->w_out, "w_out"))) return rc;
  if (had) {
    if (!(d->had_m == 1 || d->had_m == 12 || d->had_m == 20) || d->had_p < 0 ||
        ((long long)d->had_m << d->had_p) != d->d_inner)
      return fail(QMB_E_ARG, "plan factorization is inconsistent");
    if (d->d_inner > 32768) return fail(QMB_E_UNSUPP, "Hadamard dimension too large");
    if (d->had_m > 1 && !d->had_base) return fail(QMB_E_ARG, "base matrix shape mismatch");
  }

  qmb_block* b = new qmb_block();
  b->D = d->d_model;
  b->E = d->d_inner;
  b->N = d->d_state;
  b->Kc = d->d_conv;
  b->R = d->dt_rank;
  b->bits = d->bit_width;
  b->qmax = qmax_of(d->bit_width);
  b->mode = d->mode;
  b->had = had;
  b->had_p = d->had_p;
  b->had_m = d->had_m;
  memset(b->base_rows, 0, sizeof(b->base_rows));
  if (had) {
    for (int o = 0; o < d->had_m; ++o)
      for (int k = 0; k < d->had_m; ++k) {
        const int8_t v = d->had_m == 1 ? 1 : d->had_base[o * d->had_m + k];
        if (v != 1 && v != -1) {
          delete b;
          return fail(QMB_E_ARG, "base entries must be +/-1");
        }
        if (v > 0) b->base_rows[o] |= 1u << k;
      }
  }
  memcpy(b->act, d->act, sizeof(b->act));
  b->s_w_in = d->w_in.scale;
  b->s_conv_w = d->conv_w.scale;
  b->s_w_b = d->w_b.scale;
  b->s_w_c = d->w_c.scale;
  b->s_w_dtr = d->w_dt_rank.scale;
  b->s_w_dt = d->w_dt.scale;
  b->s_w_out = had ? d->w_out_h.scale : d->w_out.scale;
  const int D = b->D, E = b->E, N = b->N, Kc = b->Kc, R = b->R;
  b->Dp = (int)round_up(D, 16);
  b->Ep = (int)round_up(E, 16);
  b->Rp = (int)round_up(R, 16);
  b->Nx = 2 * N + R;

  // ---- host-side repack into kernel layouts (K-major B operands, padded K)
  // in_proj columns interleaved x | z in blocks of 64 when E allows, so every
  // 256-column output tile carries half quantize and half silu epilogue work
  b->in_il = (E % 64 == 0) ? 64 : 0;
  std::vector<int8_t> w_in_t((size_t)2 * E * b->Dp, 0);
  for (int n = 0; n < 2 * E; ++n) {
    int src = n;  // reference column of GEMM column n
    if (b->in_il) {
      const int blk = n / b->in_il;
      src = (blk & 1) * E + (blk >> 1) * b->in_il + (n - blk * b->in_il);
    }
    for (int k = 0; k < D; ++k) w_in_t[(size_t)n * b->Dp + k] = d->w_in.data[(size_t)k * 2 * E + src];
  }
  std::vector<int8_t> w_x_t((size_t)b->Nx * b->Ep, 0);
  for (int k = 0; k < E; ++k) {
    for (int n = 0; n < N; ++n) {
      w_x_t[(size_t)n * b->Ep + k] = d->w_b.data[(size_t)k * N + n];
      w_x_t[(size_t)(N + n) * b->Ep + k] = d->w_c.data[(size_t)k * N + n];
    }
    for (int n = 0; n < R; ++n) w_x_t[(size_t)(2 * N + n) * b->Ep + k] = d->w_dt_rank.data[(size_t)k * R + n];
  }
  std::vector<int8_t> w_dt_t((size_t)E * b->Rp, 0);
  for (int k = 0; k < R; ++k)
    for (int n = 0; n < E; ++n) w_dt_t[(size_t)n * b->Rp + k] = d->w_dt.data[(size_t)k * E + n];
  const int8_t* wo = had ? d->w_out_h.data : d->w_out.data;
  std::vector<int8_t> w_out_t((size_t)D * b->Ep, 0);
  for (int k = 0; k < E; ++k)
    for (int n = 0; n < D; ++n) w_out_t[(size_t)n * b->Ep + k] = wo[(size_t)k * D + n];
  std::vector<float> conv_b(E), dt_bias(E), d_deq(E), a_deq((size_t)E * N);
  for (int i = 0; i < E; ++i) {
    conv_b[i] = deq(d->conv_b.data[i], d->conv_b.scale);
    dt_bias[i] = deq(d->dt_bias.data[i], d->dt_bias.scale);
    d_deq[i] = deq(d->d.data[i], d->d.scale);
  }
  // a columns for the tabulated expf: distinct quantized a values
  int col_of[256];
  for (int q = 0; q < 256; ++q) col_of[q] = -1;
  std::vector<float> a_vals;
  std::vector<uint8_t> a_col((size_t)E * N);
  for (size_t k = 0; k < (size_t)E * N; ++k) {
    const int q = d->a.data[k];
    a_deq[k] = deq(q, d->a.scale);
    if (col_of[q + 128] < 0) {
      col_of[q + 128] = (int)a_vals.size();
      a_vals.push_back(a_deq[k]);
    }
    a_col[k] = (uint8_t)col_of[q + 128];
  }
  b->exp_ncols = (int)a_vals.size();
  std::vector<float> luts(4 * 256);
  const double lut_s[4] = {d->act[QMB_ACT_X], d->act[QMB_ACT_DT], d->act[QMB_ACT_B], d->act[QMB_ACT_C]};
  for (int t = 0; t < 4; ++t)
    for (int q = -128; q < 128; ++q) luts[t * 256 + q + 128] = deq(q, lut_s[t]);

  // ---- one device allocation
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (size_t)round_up((long long)bytes, 256);
    return o;
  };
  const size_t o_win = take(w_in_t.size()), o_cw = take((size_t)Kc * E), o_cb = take(E * 4), o_wx = take(w_x_t.size()),
               o_wdt = take(w_dt_t.size()), o_dtb = take(E * 4), o_a = take((size_t)E * N * 4),
               o_acol = take((size_t)E * N), o_lut = take((size_t)128 * b->exp_ncols * 4), o_d = take(E * 4),
               o_wo = take(w_out_t.size()), o_luts = take(4 * 256 * 4), o_avals = take(a_vals.size() * 4),
               o_qtab = take(QTAB_FLOATS * 4), o_scr = take(16),
               o_etab = take(N == 16 ? (size_t)E * 128 * 16 * 4 : 0);
  cudaError_t e = cudaMalloc(&b->mem, off);
  if (e != cudaSuccess) {
    delete b;
    return cuda_fail(e, "qmb_block_create: cudaMalloc");
  }
  char* base = static_cast<char*>(b->mem);
  b->w_in_t = (int8_t*)(base + o_win);
  b->conv_w = (int8_t*)(base + o_cw);
  b->conv_b = (float*)(base + o_cb);
  b->w_x_t = (int8_t*)(base + o_wx);
  b->w_dt_t = (int8_t*)(base + o_wdt);
  b->dt_bias = (float*)(base + o_dtb);
  b->a_deq = (float*)(base + o_a);
  b->a_col = (uint8_t*)(base + o_acol);
  b->exp_lut = (float*)(base + o_lut);
  b->exp_tab = N == 16 ? (float*)(base + o_etab) : nullptr;
  b->d_deq = (float*)(base + o_d);
  b->w_out_t = (int8_t*)(base + o_wo);
  b->luts = (float*)(base + o_luts);
  float* avals_dev = (float*)(base + o_avals);
  b->sp_qtab = (float*)(base + o_qtab);
  uint32_t* scratch = (uint32_t*)(base + o_scr);
  struct Up {
    void* dst;
    const void* src;
    size_t n;
  } ups[] = {
      {b->w_in_t, w_in_t.data(), w_in_t.size()},       {b->conv_w, d->conv_w.data, (size_t)Kc * E},
      {b->conv_b, conv_b.data(), (size_t)E * 4},       {b->w_x_t, w_x_t.data(), w_x_t.size()},
      {b->w_dt_t, w_dt_t.data(), w_dt_t.size()},       {b->dt_bias, dt_bias.data(), (size_t)E * 4},
      {b->a_deq, a_deq.data(), a_deq.size() * 4},      {b->a_col, a_col.data(), a_col.size()},
      {b->d_deq, d_deq.data(), (size_t)E * 4},         {b->w_out_t, w_out_t.data(), w_out_t.size()},
      {b->luts, luts.data(), luts.size() * 4},         {avals_dev, a_vals.data(), a_vals.size() * 4},
  };
  for (auto& u : ups) {
    e = cudaMemcpy(u.dst, u.src, u.n, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(b->mem);
      delete b;
      return cuda_fail(e, "qmb_block_create: upload");
    }
  }
  e = build_exp_lut(b->luts + 256, avals_dev, b->exp_ncols, b->exp_lut, 0);
  if (e == cudaSuccess && b->exp_tab) e = build_exp_tab(b->luts + 256, b->a_deq, E, b->exp_tab, 0);
  if (e == cudaSuccess) e = build_softplus_qtab(f32(d->act[QMB_ACT_DT]), b->qmax, b->sp_qtab, scratch, 0);
  // verified conv silu+quantize fast path for this layer's scale (cached)
  if (e == cudaSuccess) {
    const float t_silu = silu_quant_thr(f32(d->act[QMB_ACT_X]), b->qmax, 0);
    if (getenv("QMB_VERBOSE"))
      fprintf(stderr, "qmb_block_create: verified silu-quant fast-path threshold %.9g (s=%g)\n", t_silu,
              d->act[QMB_ACT_X]);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(b->mem);
    delete b;
    return cuda_fail(e, "qmb_block_create: exp table");
  }
  *out = b;
  return 0;
}

extern "C" void qmb_block_destroy(qmb_block* b) {
  if (!b) return;
  cudaFree(b->mem);
  delete b;
}

// ------------------------------------------------------------------ workspace
static void ws_layout(const qmb_block* b, long long M, size_t off[QMB_WS_COUNT], size_t* total) {
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (size_t)round_up((long long)bytes, 256);
    return r;
  };
  off[QMB_WS_UPAD] = take((b->D % 16) ? (size_t)M * b->Dp : 0);
  off[QMB_WS_XQ] = take((size_t)M * b->E);
  off[QMB_WS_Z] = take((size_t)M * b->E * 4);
  off[QMB_WS_SCANX] = take((size_t)M * b->Ep);
  off[QMB_WS_B] = take((size_t)M * b->N);
  off[QMB_WS_C] = take((size_t)M * b->N);
  off[QMB_WS_DTR] = take((size_t)M * b->Rp);
  off[QMB_WS_DELTA] = take((size_t)M * b->E);
  off[QMB_WS_YQ] = take((size_t)M * b->Ep);
  off[QMB_WS_BCF] = take((size_t)M * 36 * 4);  // BCF_LD-float rows (scan staging pitch)
  off[QMB_WS_ACC32] = take(M <= 4096 ? (size_t)SPLITK_SCRATCH_INTS * 4 : 0);  // split-K scratch (skinny GEMMs)
  *total = o;
}

extern "C" size_t qmb_block_workspace_bytes(const qmb_block* b, long long rows) {
  if (!b || rows < 0) return 0;
  size_t off[QMB_WS_COUNT], total;
  ws_layout(b, rows, off, &total);
  return total;
}

extern "C" int qmb_block_workspace_layout(const qmb_block* b, long long rows, size_t offsets[QMB_WS_COUNT]) {
  if (!b || rows < 0 || !offsets) return fail(QMB_E_ARG, "null argument");
  size_t total;
  ws_layout(b, rows, offsets, &total);
  return 0;
}
// Decode scan: each channel-step reads its 16 exps as one row of the layer's
// resident exp table (3, default); QMB_DECODE_SCAN=0 evaluates the exact expf
// directly in FP64, =2 gathers the compact (level, a-value) table through L1.
static int decode_scan_mode() {
  static const int v = [] {
    const char* e = getenv("QMB_DECODE_SCAN");
    if (e && (e[0] == '0' || e[0] == '2')) return e[0] - '0';
    return 3;  // rows of the resident exp table
  }();
  return v;
}

// Where the gate's silu(z) is evaluated: the in_proj epilogue (default) or the
// scan (QMB_ZSILU_IN_GEMM=0, kept for A/B measurements).  Same f32 values either way.
// QMB_DECODE_SCAN_FUSED=0 keeps dt_proj and the split-K fix-up as separate decode kernels.
static bool decode_scan_enabled() {
  static const bool v = [] {
    const char* e = getenv("QMB_DECODE_SCAN_FUSED");
    return !(e && e[0] == '0');
  }();
  return v;
}

// QMB_DECODE_SCAN2=0: decode from 16 sequences uses scan_tab16 (one thread per channel)
// instead of the two-lane step kernel on dt_proj's codes.
static bool decode_scan2_enabled() {
  static const bool v = [] {
    const char* e = getenv("QMB_DECODE_SCAN2");
    return !(e && e[0] == '0');
  }();
  return v;
}

// QMB_CONV_FUSE=0: the decode conv step as its own kernel after the in_proj GEMV.
static bool conv_fuse_enabled() {
  static const bool v = [] {
    const char* e = getenv("QMB_CONV_FUSE");
    return !(e && e[0] == '0');
  }();
  return v;
}

static bool zsilu_in_gemm() {
  static const bool v = [] {
    const char* e = getenv("QMB_ZSILU_IN_GEMM");
    return !(e && e[0] == '0');
  }();
  return v;
}


// ------------------------------------------------------------------ forward
// Optional per-stage event recording (qmb_block_prefill_profiled).
static thread_local cudaEvent_t* g_prof = nullptr;
#define PROF(i, st)                                   \
  do {                                                \
    if (g_prof) cudaEventRecord(g_prof[(i)], (st));   \
  } while (0)

// Tensor-parallel back half on an E-sharded handle (channels [e0, e0 + E) of the
// full d_inner tp->e_full): stage 3 quantizes the gathered gated y [M, e_full]
// (Hadamard with the FULL plan, qblock.py:211-214) and multiplies the local K-slice
// of y_q with this handle's rows of w_out(_h), leaving exact int32 partial sums in
// tp->oacc [M, D]; stage 4 applies out_proj's epilogue to the all-reduced sums
// (extra scale 1 / e_full, qblock.py:213).  int32 sums are exact in any order, so
// the result is bit-identical to the unsharded block.
static int tp_back(const qmb_block* b, const qmb_tp_args* tp, int B, int T, float* out, bool accum, uint32_t* err,
                   cudaStream_t st, int32_t* acc32, long long M) {
  const int D = b->D, E = b->E;
  const long long Ef = tp->e_full;
  if (Ef % 16 || tp->e0 % 16 || tp->e0 + E > Ef) return fail(QMB_E_ARG, "tensor-parallel channel range is inconsistent");
  if (tp->stage == 3) {
    if (b->had) {
      HadParams hp{};
      hp.y = tp->y_full;
      hp.ldy = Ef;
      hp.out = tp->yq_full;
      hp.ldo = Ef;
      hp.yh = nullptr;
      hp.M = M;
      hp.p = tp->had_p;
      hp.m = tp->had_m;
      if ((hp.m != 1 && hp.m != 12 && hp.m != 20) || ((long long)hp.m << hp.p) != Ef)
        return fail(QMB_E_ARG, "plan factorization is inconsistent");
      for (int o = 0; o < hp.m; ++o) {
        uint32_t row = 0;
        for (int k = 0; k < hp.m; ++k) row |= (tp->had_base[o * hp.m + k] > 0 ? 1u : 0u) << k;
        hp.base_rows[o] = row;
      }
      hp.s_out = f32(b->act[QMB_ACT_Y_HAD]);
      hp.qmax = b->qmax;
      hp.err = err;
      QMB_CUDA(hadamard_quant(hp, st), "tp hadamard");
    } else {
      QMB_CUDA(quantize_f32_2d(tp->y_full, Ef, M, Ef, f32(b->act[QMB_ACT_Y]), b->qmax, tp->yq_full, Ef, err, st),
               "tp y quantize");
    }
    EpiParams rp{};
    rp.nseg = 1;
    rp.qmax = b->qmax;
    rp.err = err;
    rp.seg[0] = EpiSeg{0, D, EPI_F32, 1.0f, 1.0f, nullptr, D, nullptr};
    rp.raw_out = tp->oacc;
    rp.raw_ld = D;
    QMB_CUDA(gemm_i8(tp->yq_full + tp->e0, Ef, b->w_out_t, b->Ep, (int)M, D, E, rp, st, 0, acc32),
             "tp out_proj partial gemm");
    return 0;
  }
  EpiParams ep{};
  ep.nseg = 1;
  ep.qmax = b->qmax;
  ep.err = err;
  const double s_y = b->had ? b->act[QMB_ACT_Y_HAD] : b->act[QMB_ACT_Y];
  const double extra = b->had ? 1.0 / (double)Ef : 1.0;
  ep.seg[0] = EpiSeg{0, D, accum ? EPI_F32_ADDTO : EPI_F32, f32(s_y * b->s_w_out * extra), 1.0f, out, D, nullptr};
  QMB_CUDA(epi_apply_i32(tp->oacc, (int)M, D, ep, st), "tp out_proj finish");
  return 0;
}

// Shared body of prefill (T >= 1 per sequence, h0 = 0) and decode (T = 1 with
// carried conv window and h).
static int block_run(const qmb_block* b, const int8_t* u_q, double u_scale, int B, int T, float* out, int8_t* conv_state,
                     float* ssm_state, bool decode, int8_t* conv_state_out, float* ssm_state_out, int scan_exp,
                     void* ws, size_t ws_bytes, uint32_t* err, cudaStream_t st, bool accum = false,
                     const qmb_tp_args* tp = nullptr) {
  // tensor-parallel stages (qmb_block_tp_stage): 1 = in_proj .. x_proj partial sums,
  // 2 = x_proj finish .. gated y of the local channels, 3 = Hadamard of the gathered
  // y + out_proj partial sums, 4 = out_proj finish
  const int stage = tp ? tp->stage : 0;
  if (tp && (stage < 1 || stage > 4)) return fail(QMB_E_ARG, "tensor-parallel stage must be 1..4");
  if (!b || (!u_q && stage <= 1) || (!out && (stage == 0 || stage == 4))) return fail(QMB_E_ARG, "null argument");
  if (B < 0 || T < 0) return fail(QMB_E_ARG, "batch and length must be non-negative");
  const long long M = (long long)B * T;
  if (M == 0) return 0;
  size_t off[QMB_WS_COUNT], total;
  ws_layout(b, M, off, &total);
  if (!ws || ws_bytes < total) return fail(QMB_E_WS, "workspace too small: need %zu bytes", total);
  char* w = static_cast<char*>(ws);
  int8_t* xq = (int8_t*)(w + off[QMB_WS_XQ]);
  float* z = (float*)(w + off[QMB_WS_Z]);
  int8_t* scanx = (int8_t*)(w + off[QMB_WS_SCANX]);
  int8_t* bq = (int8_t*)(w + off[QMB_WS_B]);
  int8_t* cq = (int8_t*)(w + off[QMB_WS_C]);
  int8_t* dtr = (int8_t*)(w + off[QMB_WS_DTR]);
  int8_t* delta = (int8_t*)(w + off[QMB_WS_DELTA]);
  int8_t* yq = (int8_t*)(w + off[QMB_WS_YQ]);
  float* bcf = (float*)(w + off[QMB_WS_BCF]);
  int32_t* acc32 = M <= 4096 ? (int32_t*)(w + off[QMB_WS_ACC32]) : nullptr;
  const int D = b->D, E = b->E, N = b->N, R = b->R;
  const double s_u = u_scale > 0.0 ? u_scale : b->act[QMB_ACT_IN];

  if (stage >= 3) return tp_back(b, tp, B, T, out, accum, err, st, acc32, M);
  bool fused_dscan = false;
  bool conv_fused = false;
  // in_proj (qblock.py:192-198)
  PROF(0, st);
  if (stage != 2) {
  const int8_t* A = u_q;
  long long lda = D;
  if ((D % 16) || ((uintptr_t)u_q % 16)) {
    int8_t* up = (int8_t*)(w + off[QMB_WS_UPAD]);
    if (D % 16 == 0) up = yq;  // aligned copy target (yq is free until the Hadamard step)
    QMB_CUDA(cudaMemcpy2DAsync(up, b->Dp, u_q, D, D, M, cudaMemcpyDeviceToDevice, st), "u_q pad copy");
    A = up;
    lda = b->Dp;
  }
  {
    EpiParams ep{};
    ep.nseg = 2;
    ep.qmax = b->qmax;
    ep.err = err;
    ep.il = b->in_il;
    const float s_lin = f32(s_u * b->s_w_in);
    ep.seg[0] = EpiSeg{0, E, EPI_QUANT, s_lin, f32(b->act[QMB_ACT_CONV_IN]), xq, E, nullptr};
    // z-half: silu(z) (the gate's factor, ssm.py:110-111) is computed here, in
    // the epilogue that overlaps the MMAs, instead of in the issue-bound scan.
    ep.seg[1] = EpiSeg{E, 2 * E, zsilu_in_gemm() ? EPI_F32_SILU : EPI_F32, s_lin, 1.0f, z, E, nullptr};
    // decode through the GEMV: the conv step runs in its epilogue (one launch fewer)
    conv_fused = !tp && decode && conv_fuse_enabled() &&
                 gemv_selected(A, lda, b->w_in_t, b->Dp, (int)M, D);
    if (conv_fused) {
      EpiConv& cf = ep.cf;
      cf.state = conv_state;
      cf.w = b->conv_w;
      cf.bias = b->conv_b;
      cf.out = scanx;
      cf.ldo = b->Ep;
      cf.s_conv = f32(b->act[QMB_ACT_CONV_IN] * b->s_conv_w);
      cf.s_out = f32(b->act[QMB_ACT_X]);
      cf.inv_out = 1.0f / cf.s_out;
      cf.thr = silu_quant_thr(cf.s_out, b->qmax, st);
      cf.K = b->Kc;
      cf.C = E;
    }
    QMB_CUDA(gemm_i8(A, lda, b->w_in_t, b->Dp, (int)M, 2 * E, D, ep, st, 0, acc32), "in_proj gemm");
  }
  }  // (stage != 2)
  // conv + SiLU + requant (qblock.py:199-201 -> fused_qconv :126-143)
  const float s_conv = f32(b->act[QMB_ACT_CONV_IN] * b->s_conv_w);
  PROF(1, st);
  {
  if (stage == 2) {  // x_proj's requant from the all-reduced int32 sums
    EpiParams ep{};
    ep.nseg = 3;
    ep.qmax = b->qmax;
    ep.err = err;
    const double s_x = b->act[QMB_ACT_X];
    ep.seg[0] = EpiSeg{0, N, EPI_QUANT, f32(s_x * b->s_w_b * 1.0), f32(b->act[QMB_ACT_B]), bq, N, nullptr};
    ep.seg[1] = EpiSeg{N, 2 * N, EPI_QUANT, f32(s_x * b->s_w_c * 1.0), f32(b->act[QMB_ACT_C]), cq, N, nullptr};
    ep.seg[2] = EpiSeg{2 * N, 2 * N + R, EPI_QUANT, f32(s_x * b->s_w_dtr * 1.0), f32(b->act[QMB_ACT_DT_R]), dtr,
                       b->Rp, nullptr};
    QMB_CUDA(epi_apply_i32(tp->xacc, (int)M, b->Nx, ep, st), "x_proj finish");
  } else {
  if (decode && conv_fused) {
    // (done in in_proj's GEMV epilogue)
  } else if (decode) {
    QMB_CUDA(conv_step(xq, E, conv_state, b->conv_w, b->conv_b, scanx, b->Ep, B, E, b->Kc, s_conv,
                       f32(b->act[QMB_ACT_X]), b->qmax, err, st),
             "conv step");
  } else {
    ConvParams cp{};
    cp.x = xq;
    cp.ldx = E;
    cp.w = b->conv_w;
    cp.bias = b->conv_b;
    cp.out = scanx;
    cp.ldo = b->Ep;
    cp.state_out = conv_state_out;
    cp.B = B;
    cp.T = T;
    cp.C = E;
    cp.K = b->Kc;
    cp.s_conv = s_conv;
    cp.s_out = f32(b->act[QMB_ACT_X]);
    cp.qmax = b->qmax;
    cp.err = err;
    QMB_CUDA(conv_silu_quant(cp, st), "conv");
  }
  // x_proj: b, c, dt_r (qblock.py:202-204)
  PROF(2, st);
  {
    EpiParams ep{};
    ep.nseg = 3;
    ep.qmax = b->qmax;
    ep.err = err;
    const double s_x = b->act[QMB_ACT_X];
    ep.seg[0] = EpiSeg{0, N, EPI_QUANT, f32(s_x * b->s_w_b * 1.0), f32(b->act[QMB_ACT_B]), bq, N, nullptr};
    ep.seg[1] = EpiSeg{N, 2 * N, EPI_QUANT, f32(s_x * b->s_w_c * 1.0), f32(b->act[QMB_ACT_C]), cq, N, nullptr};
    ep.seg[2] = EpiSeg{2 * N, 2 * N + R, EPI_QUANT, f32(s_x * b->s_w_dtr * 1.0), f32(b->act[QMB_ACT_DT_R]), dtr,
                       b->Rp, nullptr};
    // decode below 16 sequences: dt_proj + softplus fused into the scan step kernel
    // (16 layers at B = 8: 1.34 vs 1.49 ms; B = 1: 0.62 vs 0.66 ms).  From B = 16 the
    // dt_proj GEMM + batch-tiled scan_tab16 is faster (B = 64: 1.49 vs 1.55 ms).
    fused_dscan = !tp && decode && B < 16 && b->exp_tab && zsilu_in_gemm() && decode_scan_enabled() &&
                  decode_scan_ok(B, E, N, b->Nx, R, b->Rp);
    if (stage == 1) {  // K-sharded x_proj: the exact int32 partial sums, all-reduced by the caller
      EpiParams rp{};
      rp.nseg = 1;
      rp.qmax = b->qmax;
      rp.err = err;
      rp.seg[0] = EpiSeg{0, b->Nx, EPI_F32, 1.0f, 1.0f, nullptr, b->Nx, nullptr};
      rp.raw_out = tp->xacc;
      rp.raw_ld = b->Nx;
      QMB_CUDA(gemm_i8(scanx, b->Ep, b->w_x_t, b->Ep, (int)M, b->Nx, E, rp, st, 0, acc32), "x_proj partial gemm");
      return 0;
    }
    QMB_CUDA(gemm_i8(scanx, b->Ep, b->w_x_t, b->Ep, (int)M, b->Nx, E, ep, st, 0, acc32), "x_proj gemm");
  }
  }  // (stage != 2: conv, x_proj)
  // dt_proj + bias + softplus + quantize (qblock.py:205-206)
  PROF(3, st);
  if (fused_dscan) {
    // dt_proj, softplus, the scan step and the gate in one kernel
    DecodeScanParams dp{};
    dp.x = scanx;
    dp.ldx = b->Ep;
    dp.z = z;
    dp.bq = bq;
    dp.cq = cq;
    dp.dtr = dtr;
    dp.ld_dtr = b->Rp;
    dp.w_dt = b->w_dt_t;
    dp.ld_wdt = b->Rp;
    dp.R = R;
    dp.dt_scale = f32(b->act[QMB_ACT_DT_R] * b->s_w_dt * 1.0);
    dp.dt_bias = b->dt_bias;
    dp.qtab = b->sp_qtab;
    dp.dt_div = f32(b->act[QMB_ACT_DT]);
    dp.dt_inv = 1.0f / dp.dt_div;
    dp.lut_x = b->luts;
    dp.lut_dt = b->luts + 256;
    dp.lut_b = b->luts + 512;
    dp.lut_c = b->luts + 768;
    dp.exp_tab = b->exp_tab;
    dp.d = b->d_deq;
    dp.h = ssm_state;
    dp.B = B;
    dp.E = E;
    dp.qmax = b->qmax;
    dp.err = err;
    QMB_CUDA(decode_scan(dp, st), "decode scan");
    PROF(4, st);
  } else {
    EpiParams ep{};
    ep.nseg = 1;
    ep.qmax = b->qmax;
    ep.err = err;
    ep.seg[0] = EpiSeg{0, E, EPI_SOFTPLUS_Q, f32(b->act[QMB_ACT_DT_R] * b->s_w_dt * 1.0), f32(b->act[QMB_ACT_DT]),
                       delta, E, b->dt_bias, b->sp_qtab};
    QMB_CUDA(gemm_i8(dtr, b->Rp, b->w_dt_t, b->Rp, (int)M, E, R, ep, st, 0, acc32), "dt_proj gemm");
    // scan + D skip + gate (qblock.py:207-210), gated y written over z
    PROF(4, st);
    if (!tp && decode && b->exp_tab && zsilu_in_gemm() && decode_scan2_enabled() &&
        decode_scan_ok(B, E, N, b->Nx, R, b->Rp)) {  // the two-lane step kernel on dt_proj's codes
      DecodeScanParams dp{};
      dp.x = scanx;
      dp.ldx = b->Ep;
      dp.z = z;
      dp.bq = bq;
      dp.cq = cq;
      dp.delta = delta;
      dp.ld_delta = E;
      dp.lut_x = b->luts;
      dp.lut_dt = b->luts + 256;
      dp.lut_b = b->luts + 512;
      dp.lut_c = b->luts + 768;
      dp.exp_tab = b->exp_tab;
      dp.d = b->d_deq;
      dp.h = ssm_state;
      dp.B = B;
      dp.E = E;
      dp.qmax = b->qmax;
      dp.err = err;
      QMB_CUDA(decode_scan(dp, st), "decode scan");
    } else {
    ScanParams sp{};
    sp.x = scanx;
    sp.ldx = b->Ep;
    sp.dt = delta;
    sp.lddt = E;
    sp.bq = bq;
    sp.cq = cq;
    sp.ldbc = N;
    sp.z = z;
    sp.ldz = E;
    sp.z_silu = zsilu_in_gemm() ? 1 : 0;
    sp.y = z;
    sp.ldy = E;
    sp.lut_x = b->luts;
    sp.lut_dt = b->luts + 256;
    sp.lut_b = b->luts + 512;
    sp.lut_c = b->luts + 768;
    sp.a = b->a_deq;
    sp.a_col = b->a_col;
    sp.exp_lut = b->exp_lut;
    sp.exp_ncols = b->exp_ncols;
    sp.exp_tab = b->exp_tab;
    sp.d = b->d_deq;
    sp.bcf = bcf;
    sp.negz2 = kNegZero2;
    sp.one2 = kOne2;
    sp.dq_fast = deq_split(b->act[QMB_ACT_X], &sp.dq_x_hi, &sp.dq_x_lo) &&
                 deq_split(b->act[QMB_ACT_DT], &sp.dq_dt_hi, &sp.dq_dt_lo);
    sp.h = decode ? ssm_state : ssm_state_out;
    sp.h_in = decode ? 1 : 0;
    sp.h_out = (decode || ssm_state_out) ? 1 : 0;
    sp.B = B;
    sp.T = T;
    sp.E = E;
    sp.N = N;
    sp.err = err;
    // 1: tabulated expf in shared memory (prefill), 2: tabulated expf through L1
    // (decode, one step per sequence), 0: direct FP64 glibc-expf restatement;
    // scan_exp 2 = fast mode (approximate exp in the batch-tiled prefill kernel)
    sp.fast = (scan_exp == 2 && !decode) ? 1 : 0;
    const int use_lut = scan_exp == 1 ? 0 : (decode ? decode_scan_mode() : 1);
    QMB_CUDA(selective_scan(sp, use_lut, st), "scan");
    }
  }  // (unfused dt_proj + scan)
  }  // (unfused stages)
  if (stage == 2) {  // the local channels' gated y, all-gathered by the caller
    QMB_CUDA(cudaMemcpy2DAsync(tp->y_local, (size_t)E * 4, z, (size_t)E * 4, (size_t)E * 4, M,
                               cudaMemcpyDeviceToDevice, st),
             "tp y copy");
    return 0;
  }
  // output quantization (qblock.py:211-214)
  PROF(5, st);
  if (b->had) {
    HadParams hp{};
    hp.y = z;
    hp.ldy = E;
    hp.out = yq;
    hp.ldo = b->Ep;
    hp.yh = nullptr;
    hp.M = M;
    hp.p = b->had_p;
    hp.m = b->had_m;
    memcpy(hp.base_rows, b->base_rows, sizeof(hp.base_rows));
    hp.s_out = f32(b->act[QMB_ACT_Y_HAD]);
    hp.qmax = b->qmax;
    hp.err = err;
    QMB_CUDA(hadamard_quant(hp, st), "hadamard");
  } else {
    QMB_CUDA(quantize_f32_2d(z, E, M, E, f32(b->act[QMB_ACT_Y]), b->qmax, yq, b->Ep, err, st), "y quantize");
  }
  // out_proj (qblock.py:213/215)
  PROF(6, st);
  {
    EpiParams ep{};
    ep.nseg = 1;
    ep.qmax = b->qmax;
    ep.err = err;
    const double s_y = b->had ? b->act[QMB_ACT_Y_HAD] : b->act[QMB_ACT_Y];
    const double extra = b->had ? 1.0 / (double)E : 1.0;
    // accum: out += the block output (the next fused_rmsnorm_quant's residual add, qblock.py:181)
    ep.seg[0] = EpiSeg{0, D, accum ? EPI_F32_ADDTO : EPI_F32, f32(s_y * b->s_w_out * extra), 1.0f, out, D, nullptr};
    QMB_CUDA(gemm_i8(yq, b->Ep, b->w_out_t, b->Ep, (int)M, D, E, ep, st, 0, acc32), "out_proj gemm");
  }
  PROF(7, st);
  return 0;
}

extern "C" int qmb_block_prefill_profiled(const qmb_block* b, const int8_t* u_q, double u_scale, int B, int T,
                                          float* out, int scan_exp, void* ws, size_t ws_bytes, uint32_t* err,
                                          qmb_stream_t stream, float stage_ms[QMB_NUM_STAGES]) {
  cudaEvent_t ev[QMB_NUM_STAGES + 1];
  for (int i = 0; i <= QMB_NUM_STAGES; ++i) QMB_CUDA(cudaEventCreate(&ev[i]), "event");
  g_prof = ev;
  // (accumulating out_proj, as every layer of the model's prefill runs it)
  int rc = block_run(b, u_q, u_scale, B, T, out, nullptr, nullptr, false, nullptr, nullptr, scan_exp, ws, ws_bytes,
                     err, (cudaStream_t)stream, true);
  g_prof = nullptr;
  if (rc == 0) {
    QMB_CUDA(cudaEventSynchronize(ev[QMB_NUM_STAGES]), "event sync");
    for (int i = 0; i < QMB_NUM_STAGES; ++i) cudaEventElapsedTime(&stage_ms[i], ev[i], ev[i + 1]);
  }
  for (int i = 0; i <= QMB_NUM_STAGES; ++i) cudaEventDestroy(ev[i]);
  return rc;
}

extern "C" int qmb_block_prefill(const qmb_block* b, const int8_t* u_q, double u_scale, int B, int T, float* out,
                                 int8_t* conv_state_out, float* ssm_state_out, int scan_exp, void* ws,
                                 size_t ws_bytes, uint32_t* err, qmb_stream_t stream) {
  return block_run(b, u_q, u_scale, B, T, out, nullptr, nullptr, false, conv_state_out, ssm_state_out, scan_exp, ws,
                   ws_bytes, err, (cudaStream_t)stream);
}

extern "C" int qmb_block_prefill_accum(const qmb_block* b, const int8_t* u_q, double u_scale, int B, int T,
                                       float* res, int8_t* conv_state_out, float* ssm_state_out, int scan_exp,
                                       void* ws, size_t ws_bytes, uint32_t* err, qmb_stream_t stream) {
  return block_run(b, u_q, u_scale, B, T, res, nullptr, nullptr, false, conv_state_out, ssm_state_out, scan_exp, ws,
                   ws_bytes, err, (cudaStream_t)stream, true);
}

extern "C" int qmb_block_decode_accum(const qmb_block* b, const int8_t* u_q, double u_scale, int B,
                                      int8_t* conv_state, float* ssm_state, float* res, void* ws, size_t ws_bytes,
                                      uint32_t* err, qmb_stream_t stream) {
  if (B == 0) return 0;  // (zero sequences: nothing to advance, like the reference's empty arrays)
  if (!conv_state || !ssm_state) return fail(QMB_E_ARG, "decode requires conv and ssm state");
  return block_run(b, u_q, u_scale, B, 1, res, conv_state, ssm_state, true, nullptr, nullptr, 0, ws, ws_bytes, err,
                   (cudaStream_t)stream, true);
}

extern "C" int qmb_block_decode(const qmb_block* b, const int8_t* u_q, double u_scale, int B, int8_t* conv_state,
                                float* ssm_state, float* out, void* ws, size_t ws_bytes, uint32_t* err,
                                qmb_stream_t stream) {
  if (B == 0) return 0;  // (zero sequences: nothing to advance, like the reference's empty arrays)
  if (!conv_state || !ssm_state) return fail(QMB_E_ARG, "decode requires conv and ssm state");
  return block_run(b, u_q, u_scale, B, 1, out, conv_state, ssm_state, true, nullptr, nullptr, 0, ws, ws_bytes, err,
                   (cudaStream_t)stream);
}

// ------------------------------------------------------------------ operator mirrors
extern "C" int qmb_rmsnorm_residual_quant(const float* x_out, const float* x_res, float* res_out, const float* gain,
                                          long long M, int D, double s_out, int bit_width, int8_t* u_q,
                                          float* y_out, uint32_t* err, qmb_stream_t stream) {
  if (!x_out || !gain) return fail(QMB_E_ARG, "null argument");
  if (u_q && !(s_out > 0.0)) return fail(QMB_E_ARG, "scale must be positive, got %g", s_out);
  if (bit_width < 2 || bit_width > 8) return fail(QMB_E_UNSUPP, "bit width must be in [2, 8]");
  PairwisePlan plan;
  if (!make_pairwise_plan(D, &plan)) return fail(QMB_E_UNSUPP, "row length %d unsupported", D);
  QMB_CUDA(rmsnorm_residual(x_out, x_res, res_out, gain, plan, f32(1e-6), f32(s_out), qmax_of(bit_width), u_q,
                            y_out, M, err, (cudaStream_t)stream),
           "rmsnorm");
  return 0;
}

extern "C" int qmb_quantize(const float* x, long long n, double scale, int bit_width, int8_t* out, uint32_t* err,
                            qmb_stream_t stream) {
  if (!(scale > 0.0)) return fail(QMB_E_ARG, "scale must be positive, got %g", scale);
  if (bit_width < 2 || bit_width > 8) return fail(QMB_E_UNSUPP, "bit width must be in [2, 8]");
  QMB_CUDA(quantize_f32(x, n, f32(scale), qmax_of(bit_width), out, err, (cudaStream_t)stream), "quantize");
  return 0;
}

__global__ void quantize_f64_kernel(const double* __restrict__ x, long long n, double s, int qmax,
                                    int8_t* __restrict__ out, uint32_t* err_flag) {
  uint32_t err = 0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
    const double v = x[k];
    if (!isfinite(v)) {
      err |= QMB_ERR_NONFINITE;
      out[k] = 0;
      continue;
    }
    double q = rint(__ddiv_rn(v, s));
    q = fmin(fmax(q, -(double)qmax), (double)qmax);
    out[k] = (int8_t)(int)q;
  }
  flag_error(err_flag, err);
}

extern "C" int qmb_quantize_f64(const double* x, long long n, double scale, int bit_width, int8_t* out,
                                uint32_t* err, qmb_stream_t stream) {
  if (!(scale > 0.0)) return fail(QMB_E_ARG, "scale must be positive, got %g", scale);
  if (bit_width < 2 || bit_width > 8) return fail(QMB_E_UNSUPP, "bit width must be in [2, 8]");
  if (n <= 0) return 0;
  long long blocks = (n + 255) / 256;
  if (blocks > num_sms() * 16) blocks = num_sms() * 16;
  quantize_f64_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, n, scale, qmax_of(bit_width), out, err);
  QMB_CUDA(cudaGetLastError(), "quantize_f64");
  return 0;
}

__global__ void dequant_kernel(const int8_t* q, int n, double s, float* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = __double2float_rn(__dmul_rn((double)q[k], s));
}

extern "C" size_t qmb_qlinear_workspace_bytes(long long M, int K, int N) {
  const long long Kp = round_up(K, 16);
  // + split-K scratch for decode-size M
  return (size_t)(round_up(M * Kp, 256) + round_up((long long)N * Kp, 256) + round_up((long long)N * 4, 256) +
                  (M <= 4096 ? SPLITK_SCRATCH_INTS * 4 : 0));
}

extern "C" int qmb_qlinear(const int8_t* x_q, long long M, int K, double s_x, const int8_t* w_q, int N, double s_w,
                           const int8_t* bias_q, double s_bias, double s_out, double extra_scale, int bit_width,
                           void* out, void* ws, size_t ws_bytes, int path, uint32_t* err, qmb_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (K > 32768) return fail(QMB_E_ARG, "inner dimension %d exceeds the int32 accumulation bound", K);
  if (M < 0 || K <= 0 || N <= 0) return fail(QMB_E_ARG, "qlinear inner dimensions do not match");
  if (bit_width < 2 || bit_width > 8) return fail(QMB_E_UNSUPP, "bit width must be in [2, 8]");
  if (M == 0) return 0;
  if (ws_bytes < qmb_qlinear_workspace_bytes(M, K, N)) return fail(QMB_E_WS, "workspace too small");
  const long long Kp = round_up(K, 16);
  char* w = static_cast<char*>(ws);
  int8_t* a_pad = (int8_t*)w;
  int8_t* bt = (int8_t*)(w + round_up(M * Kp, 256));
  float* bias = (float*)(w + round_up(M * Kp, 256) + round_up((long long)N * Kp, 256));
  const int8_t* A = x_q;
  long long lda = K;
  if ((K % 16) || ((uintptr_t)x_q % 16)) {
    QMB_CUDA(cudaMemcpy2DAsync(a_pad, Kp, x_q, K, K, M, cudaMemcpyDeviceToDevice, st), "qlinear pad");
    A = a_pad;
    lda = Kp;
  }
  QMB_CUDA(transpose_i8(w_q, K, N, N, bt, Kp, st), "qlinear transpose");
  if (bias_q) {
    dequant_kernel<<<(N + 255) / 256, 256, 0, st>>>(bias_q, N, s_bias, bias);
    QMB_CUDA(cudaGetLastError(), "bias dequant");
  }
  EpiParams ep{};
  ep.nseg = 1;
  ep.qmax = qmax_of(bit_width);
  ep.err = err;
  const float acc_scale = f32(s_x * s_w * extra_scale);
  if (s_out > 0.0)
    ep.seg[0] = EpiSeg{0, N, EPI_QUANT, acc_scale, f32(s_out), out, N, bias_q ? bias : nullptr};
  else
    ep.seg[0] = EpiSeg{0, N, EPI_F32, acc_scale, 1.0f, out, N, bias_q ? bias : nullptr};
  int32_t* acc32 = nullptr;
  if (M <= 4096)  // split-K scratch (skinny products)
    acc32 = (int32_t*)(w + round_up(M * Kp, 256) + round_up((long long)N * Kp, 256) + round_up((long long)N * 4, 256));
  QMB_CUDA(gemm_i8(A, lda, bt, Kp, (int)M, N, K, ep, st, path, acc32), "qlinear gemm");
  return 0;
}

extern "C" int qmb_fused_qconv(const int8_t* x_q, int B, int T, int C, double s_x, const int8_t* w_q, int K,
                               double s_w, const int8_t* bias_q, double s_bias, double s_out, int bit_width,
                               int8_t* out, uint32_t* err, qmb_stream_t stream) {
  if (!(s_out > 0.0)) return fail(QMB_E_ARG, "scale must be positive, got %g", s_out);
  if (B < 0 || T < 0 || C <= 0 || K <= 0) return fail(QMB_E_ARG, "conv channel mismatch");
  ConvParams cp{};
  cp.x = x_q;
  cp.ldx = C;
  cp.w = w_q;
  cp.bias = nullptr;
  cp.bias_q = bias_q;
  cp.bias_scale = s_bias;
  cp.out = out;
  cp.ldo = C;
  cp.state_out = nullptr;
  cp.B = B;
  cp.T = T;
  cp.C = C;
  cp.K = K;
  cp.s_conv = f32(s_x * s_w);
  cp.s_out = f32(s_out);
  cp.qmax = qmax_of(bit_width);
  cp.err = err;
  QMB_CUDA(conv_silu_quant(cp, (cudaStream_t)stream), "conv");
  return 0;
}

__global__ void scan_tables_kernel(const int8_t* a_q, double s_a, const int8_t* d_q, double s_d, int D, int N,
                                   double s_x, double s_dt, double s_b, double s_c, float* luts, float* a, float* d) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < 1024) {
    const int t = k >> 8, q = (k & 255) - 128;
    const double s = t == 0 ? s_x : t == 1 ? s_dt : t == 2 ? s_b : s_c;
    luts[k] = __double2float_rn(__dmul_rn((double)q, s));
  }
  if (k < D * N) a[k] = __double2float_rn(__dmul_rn((double)a_q[k], s_a));
  if (k < D) d[k] = __double2float_rn(__dmul_rn((double)d_q[k], s_d));
}

extern "C" size_t qmb_selective_scan_workspace_bytes(int D, int N) {
  if (D <= 0 || N <= 0) return 0;
  return (1024 + (size_t)D * N + (size_t)D) * sizeof(float);
}

extern "C" int qmb_selective_scan(const int8_t* a_q, double s_a, const int8_t* b_q, double s_b, const int8_t* c_q,
                                  double s_c, const int8_t* d_q, double s_d, const int8_t* dt_q, double s_dt,
                                  const int8_t* x_q, double s_x, int B, int T, int D, int N, float* h, int h_in,
                                  float* y, void* ws, size_t ws_bytes, uint32_t* err, qmb_stream_t stream) {
  if (B < 0 || T < 0 || D <= 0 || N <= 0) return fail(QMB_E_ARG, "scan argument shapes are inconsistent");
  if (N > 64) return fail(QMB_E_UNSUPP, "d_state > 64 is not supported");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t need = qmb_selective_scan_workspace_bytes(D, N);
  if (!ws || ws_bytes < need) return fail(QMB_E_WS, "workspace too small: need %zu bytes", need);
  float* buf = static_cast<float*>(ws);
  float* luts = buf;
  float* a = buf + 1024;
  float* d = a + (size_t)D * N;
  const int total = (int)((size_t)D * N > 1024 ? (size_t)D * N : 1024);
  scan_tables_kernel<<<(total + 255) / 256, 256, 0, st>>>(a_q, s_a, d_q, s_d, D, N, s_x, s_dt, s_b, s_c, luts, a, d);
  QMB_CUDA(cudaGetLastError(), "scan tables");
  ScanParams sp{};
  sp.x = x_q;
  sp.ldx = D;
  sp.dt = dt_q;
  sp.lddt = D;
  sp.bq = b_q;
  sp.cq = c_q;
  sp.ldbc = N;
  sp.z = nullptr;
  sp.ldz = 0;
  sp.y = y;
  sp.ldy = D;
  sp.lut_x = luts;
  sp.lut_dt = luts + 256;
  sp.lut_b = luts + 512;
  sp.lut_c = luts + 768;
  sp.a = a;
  sp.a_col = nullptr;
  sp.exp_lut = nullptr;
  sp.exp_ncols = 0;
  sp.d = d;
  sp.h = h;
  sp.h_in = (h && h_in) ? 1 : 0;
  sp.h_out = h ? 1 : 0;
  sp.B = B;
  sp.T = T;
  sp.E = D;
  sp.N = N;
  sp.err = err;
  QMB_CUDA(selective_scan(sp, 0, st), "scan");
  return 0;
}

extern "C" int qmb_hadamard_quantize(const float* y, long long M, int p, int m, const int8_t* base, double scale,
                                     int bit_width, int8_t* out, float* y_h, uint32_t* err, qmb_stream_t stream) {
  if (!(scale > 0.0)) return fail(QMB_E_ARG, "scale must be positive, got %g", scale);
  if (!(m == 1 || m == 12 || m == 20) || p < 0) return fail(QMB_E_ARG, "plan factorization is inconsistent");
  if (((long long)m << p) > 32768) return fail(QMB_E_UNSUPP, "Hadamard dimension too large");
  HadParams hp{};
  hp.y = y;
  hp.ldy = (long long)m << p;
  hp.out = out;
  hp.ldo = hp.ldy;
  hp.yh = y_h;
  hp.M = M;
  hp.p = p;
  hp.m = m;
  for (int o = 0; o < m; ++o)
    for (int k = 0; k < m; ++k) {
      const int v = (m == 1) ? 1 : base[o * m + k];
      if (v != 1 && v != -1) return fail(QMB_E_ARG, "base entries must be +/-1");
      if (v > 0) hp.base_rows[o] |= 1u << k;
    }
  hp.s_out = f32(scale);
  hp.qmax = qmax_of(bit_width);
  hp.err = err;
  QMB_CUDA(hadamard_quant(hp, (cudaStream_t)stream), "hadamard");
  return 0;
}

extern "C" int qmb_gemm_bench(int M, int N, int K, int mode, int iters, float* ms) {
  if (M <= 0 || N <= 0 || K <= 0 || K % 16 || iters <= 0 || !ms) return fail(QMB_E_ARG, "invalid argument");
  QMB_CUDA(gemm_bench(M, N, K, mode, iters, ms), "gemm bench");
  return 0;
}

extern "C" int qmb_measure_i8_peak(int iters, double* tops) {
  if (iters <= 0 || !tops) return fail(QMB_E_ARG, "invalid argument");
  QMB_CUDA(measure_i8_peak(iters, tops), "i8 peak probe");
  return 0;
}

extern "C" int qmb_eval_math(int fn, const float* x, float* y, long long n, qmb_stream_t stream) {
  if (fn < 0 || fn > 7) return fail(QMB_E_ARG, "unknown function %d", fn);
  QMB_CUDA(eval_math(fn, x, y, n, (cudaStream_t)stream), "eval_math");
  return 0;
}

extern "C" int qmb_verify_math(int fn_a, int fn_b, unsigned long long* mismatches, uint32_t* first_bad,
                               qmb_stream_t stream) {
  if (fn_a < 0 || fn_a > 7 || fn_b < 0 || fn_b > 7) return fail(QMB_E_ARG, "unknown function");
  QMB_CUDA(verify_math(fn_a, fn_b, mismatches, first_bad, (cudaStream_t)stream), "verify_math");
  return 0;
}

extern "C" int qmb_embed_gather(const float* table, const long long* tokens, long long n, int D, float* out,
                                qmb_stream_t stream) {
  QMB_CUDA(embed_gather(table, tokens, n, D, out, (cudaStream_t)stream), "embed");
  return 0;
}

extern "C" int qmb_block_tp_stage(const qmb_block* b, const qmb_tp_args* tp, const int8_t* u_q, double u_scale, int B,
                                  int T, int decode, int8_t* conv_state, float* ssm_state, float* out, int accumulate,
                                  void* ws, size_t ws_bytes, uint32_t* err, qmb_stream_t stream) {
  if (!tp) return fail(QMB_E_ARG, "null argument");
  if (decode && T != 1) return fail(QMB_E_ARG, "decode advances one token per sequence");
  if ((tp->stage == 1 && !tp->xacc) || (tp->stage == 2 && (!tp->xacc || !tp->y_local)) ||
      (tp->stage == 3 && (!tp->y_full || !tp->yq_full || !tp->oacc)) || (tp->stage == 4 && !tp->oacc))
    return fail(QMB_E_ARG, "null argument");
  return block_run(b, u_q, u_scale, B, T, out, decode ? conv_state : nullptr, decode ? ssm_state : nullptr,
                   decode != 0, decode ? nullptr : conv_state, decode ? nullptr : ssm_state, 0, ws, ws_bytes, err,
                   (cudaStream_t)stream, accumulate != 0, tp);
}

extern "C" int qmb_lm_head(const float* x, int M, int K, const float* emb, int V, float* out, qmb_stream_t stream) {
  if (M < 0 || K <= 0 || V < 0 || (M && (!x || !emb || !out))) return fail(QMB_E_ARG, "null argument");
  QMB_CUDA(lm_head(x, M, K, emb, V, out, (cudaStream_t)stream), "lm head");
  return 0;
}

extern "C" int qmb_argmax(const float* logits, int M, int V, long long ld, long long* out, qmb_stream_t stream) {
  if (M < 0 || V <= 0 || ld < V || (M && (!logits || !out))) return fail(QMB_E_ARG, "null argument");
  QMB_CUDA(argmax_rows(logits, M, V, ld, out, (cudaStream_t)stream), "argmax");
  return 0;
}

extern "C" int qmb_lm_split16(const float* x, int M, int K, void* out16, float* inv_scale, qmb_stream_t stream) {
  if (M < 0 || K <= 0 || (M && (!x || !out16 || !inv_scale))) return fail(QMB_E_ARG, "null argument");
  QMB_CUDA(lm_split16(x, M, K, out16, inv_scale, (cudaStream_t)stream), "lm split16");
  return 0;
}

extern "C" int qmb_lm_combine16(const float* p, const float* q, const float* inv_scale, int M, int V, int k,
                                float* out, qmb_stream_t stream) {
  if (M < 0 || V < 0 || (M && V && (!p || !q || !inv_scale || !out))) return fail(QMB_E_ARG, "null argument");
  QMB_CUDA(lm_combine16(p, q, inv_scale, M, V, k, out, (cudaStream_t)stream), "lm combine16");
  return 0;
}
