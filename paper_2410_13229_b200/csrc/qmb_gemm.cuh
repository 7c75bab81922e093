// qmb_gemm.cuh -- int8 x int8 -> int32 GEMM for sm_100a with fused
// dequant/requant epilogues (the reference's qlinear, qblock.py:98-123, and
// the inline in_proj, qblock.py:192-198).
//
// C[m, n] = sum_k A[m, k] * Bt[n, k]      (A: [M, K] K-major, Bt: [N, K] K-major)
// The int32 accumulator is exact, so any summation order matches numpy's
// int32 matmul bit-for-bit; the epilogue then applies the reference's float
// steps in the reference's order (int32 -> f32 RN, * f32 scale, + f32 bias,
// optional softplus, quantize).
#pragma once
#include <climits>
#include <cuda.h>

#include "qmb_common.cuh"

namespace qmb {

enum EpiKind : int {
  EPI_QUANT = 0,     // int8 out = quantize(f32(acc) * s [+ bias])
  EPI_F32 = 1,       // f32 out = f32(acc) * s [+ bias]
  EPI_SOFTPLUS_Q = 2,  // int8 out = quantize(softplus(f32(acc) * s [+ bias]))
  EPI_F32_SILU = 3,    // f32 out = silu(f32(acc) * s [+ bias]) (the gate's silu(z), ssm.py:110-111)
  EPI_F32_ADDTO = 4    // f32 out = (f32(acc) * s [+ bias]) + out (the residual add of the next
                       // fused_rmsnorm_quant, qblock.py:181, folded into out_proj's epilogue)
};
__host__ __device__ __forceinline__ bool epi_is_f32(int kind) {
  return kind == EPI_F32 || kind == EPI_F32_SILU || kind == EPI_F32_ADDTO;
}

struct EpiSeg {
  int n0, n1;           // column range [n0, n1) of the GEMM output this segment covers
  int kind;             // EpiKind
  float acc_scale;      // f32(s_x * s_w * extra)
  float out_div;        // f32(s_out) (quantizing kinds)
  void* out;            // int8* or float*
  long long ld;         // output row stride (elements)
  const float* bias;    // per-column dequantized bias (indexed n - n0) or nullptr
  const float* qtab;    // EPI_SOFTPLUS_Q: verified threshold table (softplus_qtab) or nullptr
  float out_inv;        // 1.0f / out_div (filled in by gemm_i8)
};

// Verified threshold table for quantize(softplus(v)) (monotone non-decreasing):
// tab[0] = -inf, tab[k] = min{v : q(v) >= k} for k = 1..127 (+inf past qmax),
// tab[128] = +inf, and tab[QTAB_LO], tab[QTAB_HI] = the interval of v on which an
// exhaustive sweep over all 2^32 floats at handle creation found the table
// function below to disagree with the exact evaluation (empty: lo > hi); there,
// and for non-finite v, the exact formula is used.  Exact by construction.
constexpr int QTAB_FLOATS = 131;
constexpr int QTAB_LO = 129, QTAB_HI = 130;

// The table function: a fast-math estimate of the level, taken half a level low
// (q0 = rint(sp / s - 1/2) in {q - 1, q} for the true level q), then one threshold
// comparison lifts it (level q <=> tab[q] <= v < tab[q + 1]).  The rint is the
// 1.5 * 2^23 bias add (no conversion-unit op).  Branch-free; the sweep verifies
// exactly this function.
// Returns the level biased by 0x4B400000 (its low byte is the int8 code): the bias
// add's bits index the table directly (a 32-bit shared-window address,
// softplus_tab_bias(tab) = addr(tab) + 4 - 4 * 0x4B400000 mod 2^32) and feed the byte
// packing without an integer conversion.  tab must be in shared memory.
constexpr uint32_t QTAB_BIAS = 4u - 4u * 0x4B400000u;
// bias: QTAB_BIAS, passed at run time by the epilogue (EpiParams::qtab_bias) so that
// ptxas cannot split the constant back off the per-element address
__device__ __forceinline__ uint32_t softplus_tab_bias(const float* tab, uint32_t bias = QTAB_BIAS) {
  return (uint32_t)__cvta_generic_to_shared(tab) + bias;
}
__device__ __forceinline__ uint32_t softplus_quant_table_bits(float v, uint32_t tab_b, float s_inv, float qmaxf) {
  float e, l, t;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(__fmul_rn(v, 1.44269504088896341f)));
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(__fadd_rn(1.0f, e)));
  const float sp = v > 15.0f ? v : __fmul_rn(l, 0.693147180559945309f);
  const float y = fminf(fmaxf(__fmaf_rn(sp, s_inv, -0.5f), 0.0f), qmaxf);
  const uint32_t b = __float_as_uint(__fadd_rn(y, 12582912.0f));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(t) : "r"(tab_b + 4u * b));
  return b + (v >= t ? 1u : 0u);
}
// softplus_quant_table_bits on two values: the float ops as FFMA2s (each half rounded
// like the scalar op, run-time 1.0 / -0.0 operands), the rest per half; bit-identical
// per half to the scalar function the sweep verifies.
__device__ __forceinline__ void softplus_quant_table_bits2(float v0, float v1, uint32_t tab_b,
                                                           unsigned long long sinv2, float qmaxf,
                                                           unsigned long long one2, unsigned long long negz2,
                                                           uint32_t& b0, uint32_t& b1) {
  const float2 a = unpack_f32x2(fma2_rn(pack_f32x2(v0, v1), 0x3FB8AA3B3FB8AA3Bull, negz2));  // v * log2(e)
  float e0, e1, l0, l1, t0, t1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(a.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(a.y));
  const float2 den = unpack_f32x2(fma2_rn(pack_f32x2(e0, e1), one2, one2));  // 1 + e
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l0) : "f"(den.x));
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l1) : "f"(den.y));
  const float2 sl = unpack_f32x2(fma2_rn(pack_f32x2(l0, l1), 0x3F3172183F317218ull, negz2));  // l * ln(2)
  const float sp0 = v0 > 15.0f ? v0 : sl.x, sp1 = v1 > 15.0f ? v1 : sl.y;
  const float2 y = unpack_f32x2(fma2_rn(pack_f32x2(sp0, sp1), sinv2, 0xBF000000BF000000ull));  // sp / s - 1/2
  const float2 bb = unpack_f32x2(fma2_rn(
      pack_f32x2(fminf(fmaxf(y.x, 0.0f), qmaxf), fminf(fmaxf(y.y, 0.0f), qmaxf)), one2, 0x4B4000004B400000ull));
  b0 = __float_as_uint(bb.x);
  b1 = __float_as_uint(bb.y);
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(t0) : "r"(tab_b + 4u * b0));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(t1) : "r"(tab_b + 4u * b1));
  b0 += v0 >= t0 ? 1u : 0u;
  b1 += v1 >= t1 ? 1u : 0u;
}
__device__ __forceinline__ int softplus_quant_table(float v, const float* __restrict__ tab, float s_inv,
                                                    float qmaxf) {
  return (int)(softplus_quant_table_bits(v, softplus_tab_bias(tab), s_inv, qmaxf) - 0x4B400000u);
}

// v needs the exact path (outside the verified domain of the table function)
__device__ __forceinline__ bool softplus_table_miss(float v, float lo, float hi) {
  return !(fabsf(v) <= 3.402823466e38f) || (v >= lo && v <= hi);
}

// Exact path (out of line).  Returns INT_MIN for a non-finite input: no pointer
// argument, so callers keep their error word in a register.
static __device__ __noinline__ int softplus_quant_exact(float v, float s_div, int qmax) {
  uint32_t e = 0;
  const int q = quant_i8(softplus_f32(v), s_div, qmax, e);
  return e ? INT_MIN : q;
}

__device__ __forceinline__ int softplus_quant(float v, const float* __restrict__ qtab, float s_div, float s_inv,
                                              int qmax, uint32_t& err) {
  if (qtab && !softplus_table_miss(v, qtab[QTAB_LO], qtab[QTAB_HI]))
    return softplus_quant_table(v, qtab, s_inv, (float)qmax);
  const int q = softplus_quant_exact(v, s_div, qmax);
  if (q == INT_MIN) {
    err |= QMB_ERR_NONFINITE;
    return 0;
  }
  return q;
}

// Decode GEMV only: the causal conv step of fused_qconv (qblock.py:126-143) fused onto
// in_proj's x columns.  Column i of row b: q = the x code; acc = sum_k w[k][i] x_k over
// the carried window (state [B][K-1][C]) and q; out[b][i] = quantize(silu(f32(acc) *
// s_conv + bias[i]), s_out); the window shifts by q.  state == nullptr: off.
struct EpiConv {
  int8_t* state;
  const int8_t* w;      // [K][C] taps
  const float* bias;    // [C] dequantized conv bias or nullptr
  int8_t* out;          // [B][ldo] scan input codes
  long long ldo;
  float s_conv, s_out, inv_out, thr;
  int K, C;
};

struct EpiParams {
  int nseg;
  int qmax;
  uint32_t* err;
  EpiSeg seg[3];
  int tma_seg;   // segments written through TMA store maps tmC / tmC2 (set by gemm_i8), or -1
  int tma_seg2;
  int il;          // > 0: GEMM columns interleave two segments in blocks of il columns
                   // (block b -> segment b & 1, output column (b >> 1) * il + offset)
  int spin;        // pipeline waits spin (short, latency-bound GEMMs: decode) instead of sleeping
  int small_acc;   // |acc| < 2^22 (K < 256): accumulators convert with i2f_small (set by gemm_i8)
  uint32_t qtab_bias;  // QTAB_BIAS (set by gemm_i8)
  unsigned long long one2, negz2;  // packed {1, 1} / {-0, -0} as run-time operands (set by gemm_i8)
  int splitk;      // > 1: split-K over K blocks; partial int32 sums stored per split
  int32_t* acc32;  // [splitk, M, N] int32 partials; a second kernel sums them and runs the epilogue
  int32_t* raw_out;  // non-null: the exact int32 sums go to raw_out[m * raw_ld + n] instead of any epilogue
  long long raw_ld;  // (single segment [0, N), no interleave; tensor-parallel partial products)
  EpiConv cf;        // decode GEMV: conv step fused onto segment 0 (see EpiConv)
};

// Segment by value with compile-time indices only: a runtime index into the
// param-space array would make the compiler copy it to local memory.
__device__ __forceinline__ EpiSeg pick_seg(const EpiParams& ep, int s) {
  return s == 0 ? ep.seg[0] : (s == 1 ? ep.seg[1] : ep.seg[2]);
}

__device__ __forceinline__ int find_seg(const EpiParams& ep, int n) {
  int s = 0;
#pragma unroll
  for (int i = 1; i < 3; ++i)
    if (i < ep.nseg && n >= ep.seg[i].n0) s = i;
  return s;
}

// GEMM column n -> (segment, output column within the segment)
__device__ __forceinline__ int epi_locate(const EpiParams& ep, int n, int* ocol) {
  if (ep.il > 0) {
    const int blk = n / ep.il;
    *ocol = (blk >> 1) * ep.il + (n - blk * ep.il);
    return blk & 1;
  }
  const int s = find_seg(ep, n);
  *ocol = n - pick_seg(ep, s).n0;
  return s;
}

// Stage the (single) EPI_SOFTPLUS_Q segment's threshold table into shared memory
// (QTAB_FLOATS floats at dst); returns dst, or null when no segment needs it.
// Call from every thread of the CTA, then __syncthreads().
__device__ __forceinline__ const float* stage_qtab(const EpiParams& ep, float* dst) {
  const float* src = nullptr;
  for (int s = 0; s < ep.nseg; ++s)
    if (ep.seg[s].kind == EPI_SOFTPLUS_Q) src = ep.seg[s].qtab;
  if (!src) return nullptr;
  for (int k = threadIdx.x; k < QTAB_FLOATS; k += blockDim.x) dst[k] = src[k];
  return dst;
}

// One output element, scalar path (shared by the SIMT / GEMV / split-K fix-up
// kernels); oc = output column within segment sg.  sqtab: the softplus threshold
// table staged in SHARED memory (the table function reads it with ld.shared), or
// null for the exact evaluation.
__device__ __forceinline__ void epi_store_one(const EpiParams& ep, const EpiSeg& sg, long long m, int oc, int acc,
                                              uint32_t& err, const float* sqtab = nullptr) {
  if (ep.raw_out) {  // raw mode: one segment [0, N), so oc is the GEMM column
    ep.raw_out[m * ep.raw_ld + oc] = acc;
    return;
  }
  float v = __fmul_rn(__int2float_rn(acc), sg.acc_scale);
  if (sg.bias) v = __fadd_rn(v, sg.bias[oc]);
  long long off = m * sg.ld + oc;
  if (epi_is_f32(sg.kind)) {
    float* o = static_cast<float*>(sg.out) + off;
    *o = sg.kind == EPI_F32_SILU ? silu_f32_fast(v) : (sg.kind == EPI_F32_ADDTO ? __fadd_rn(v, *o) : v);
  } else if (sg.kind == EPI_SOFTPLUS_Q) {
    static_cast<int8_t*>(sg.out)[off] = (int8_t)softplus_quant(v, sqtab, sg.out_div, sg.out_inv, ep.qmax, err);
  } else {
    static_cast<int8_t*>(sg.out)[off] = (int8_t)quant_fast(v, sg.out_div, sg.out_inv, ep.qmax, err);
  }
}

}  // namespace qmb

// Host-side launcher API (implemented in qmb_gemm.cu).
namespace qmb {
// A: [M, Kp] with row stride lda bytes; Bt: [N, Kp] with row stride ldb bytes.
// Requirements for the tensor-core path: lda % 16 == 0, ldb % 16 == 0, 16-byte
// aligned base pointers.  Rows beyond M / N and K beyond Kp are zero-filled by TMA.
// acc32_scratch (nullable): int32 scratch of >= SPLITK_SCRATCH_INTS enabling
// split-K for skinny M (decode), where too few output tiles exist to keep the
// SMs streaming weights.
constexpr long long SPLITK_SCRATCH_INTS = 148LL * 128 * 256;
cudaError_t gemm_i8(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int N, int Kp,
                    const EpiParams& ep, cudaStream_t st, int force_path /*0 auto, 1 tc, 2 simt, 3 gemv*/,
                    int32_t* acc32_scratch = nullptr, int* defer_splitk = nullptr);
cudaError_t epi_apply_i32(const int32_t* acc, int M, int N, const EpiParams& ep, cudaStream_t st);
// gemm_i8 will take the decode GEMV (the only path that honours EpiParams::cf)
bool gemv_selected(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int Kp);
// defer_splitk (nullable): when the launch splits K (skinny M with acc32_scratch), skip
// the fix-up kernel and return the split count here (the int32 partials are left in
// acc32_scratch as [split][M][N] for the caller's next kernel); 0 = the epilogue ran.
int num_sms();
// Tiled TMA map of a rank-3 tensor: dims innermost first, byte strides of dims 1, 2;
// elem 1 = uint8, 4 = float32; swizzle 0 / 64 / 128 (bytes).
bool make_tmap_3d(CUtensorMap* tm, int elem, const void* base, const long long dims[3],
                  const long long strides[2], const int box[3], int swizzle);
// Dense int8 tensor-core throughput (TOP/s) of back-to-back 128x256x32 UMMAs on all SMs.
cudaError_t measure_i8_peak(int iters, double* tops);
cudaError_t gemm_bench(int M, int N, int K, int mode, int iters, float* ms_out);
}  // namespace qmb
