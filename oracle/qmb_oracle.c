/*
 * qmb_oracle.c -- CPU restatement of the reference's float/ordering-sensitive
 * primitives on the Quamba W8A8 block path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product (paper_2410_13229_b200/, libqmb.so) never links
 * or calls it.
 *
 * Each function cites the reference call site whose arithmetic it restates
 * (paths relative to the reference's pkg/ directory).  Build with
 *   gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 * (see oracle/Makefile): contraction must stay off because the reference's
 * Cython core is built with -ffp-contract=off (setup.py:14-16) and numpy's
 * SIMD loops use explicit FMAs only where restated below with fma()/fmaf().
 *
 * Third-party arithmetic restated here (not under the reference tree):
 *   - numpy 2.3.5 float32 exp SIMD kernel (AVX2/AVX512 dispatch)  -> np_exp_f32
 *   - glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, FMA ifunc) -> glibc_expf
 *   - glibc 2.39 log1pf (fdlibm float algorithm, s_log1pf.c)       -> glibc_log1pf
 *   - numpy pairwise float32 summation (loops_utils.h.src)         -> pairwise_sum_f32
 * tests/test_oracle_transcendentals.py pins each one against the live
 * numpy / libm of the host it runs on.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static inline double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }

/* ------------------------------------------------------------------------ */
/* numpy float32 exp (SIMD path) -- used by ssm.silu (ssm.py:98-101), which  */
/* feeds fused_qconv (qblock.py:143) and gate (ssm.py:110-111).              */
/* ------------------------------------------------------------------------ */
float np_exp_f32(float x)
{
    if (isnan(x)) return x;
    if (x > 88.72283935546875f) return INFINITY;
    if (x < -103.97208404541015625f) return 0.0f;
    float q = rintf(x * 0x1.715476p+0f);
    float r = fmaf(q, -6.93145752e-1f, x);
    r = fmaf(q, -1.42860677e-6f, r);
    float num = fmaf(fmaf(fmaf(fmaf(fmaf(5.082762527590693718096e-04f, r,
                    6.757896990527504603057e-03f), r,
                    5.114512081637298353406e-02f), r,
                    2.473615434895520810817e-01f), r,
                    7.257664613233124478488e-01f), r,
                    9.999999999980870924916e-01f);
    float den = fmaf(fmaf(2.159509375685829852307e-02f, r,
                    -2.742335390411667452936e-01f), r, 1.0f);
    return ldexpf(num / den, (int)q);
}

/* ------------------------------------------------------------------------ */
/* glibc 2.39 expf -- used by the Cython scan (_core.pyx:59) and by          */
/* np.logaddexp inside softplus (ssm.py:93-95).                              */
/* GCC contracts z = InvLn2N*xd into both consumers (kd and r) -> fma().     */
/* ------------------------------------------------------------------------ */
static const uint64_t EXP2F_T[32] = {
    /* T[i] = bits(RN_double(2^(i/32))) - (i << 47); regenerate with mpmath */
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL,
};

float glibc_expf(float x)
{
    const double InvLn2N = 0x1.71547652b82fep+0 * 32.0;
    const double SHIFT = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / (32.0 * 32.0 * 32.0);
    const double C1 = 0x1.ebfce50fac4f3p-3 / (32.0 * 32.0);
    const double C2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    uint32_t abstop = (f2u(x) >> 20) & 0x7ff;
    if (abstop >= (f2u(88.0f) >> 20)) {
        if (f2u(x) == f2u(-INFINITY)) return 0.0f;
        if (abstop >= (f2u(INFINITY) >> 20)) return x + x;
        if (x > 0x1.62e42ep6f) return INFINITY;
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    double xd = (double)x;
    double kd = fma(InvLn2N, xd, SHIFT);
    uint64_t ki = d2u(kd);
    kd -= SHIFT;
    double r = fma(InvLn2N, xd, -kd);
    uint64_t t = EXP2F_T[ki % 32];
    t += ki << 47;
    double s = u2d(t);
    double y = fma(fma(C0, r, C1), r * r, fma(C2, r, 1.0));
    y = y * s;
    return (float)y;
}

/* ------------------------------------------------------------------------ */
/* glibc 2.39 log1pf (fdlibm float algorithm) -- np.logaddexp (ssm.py:95).   */
/* ------------------------------------------------------------------------ */
float glibc_log1pf(float x)
{
    const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f;
    const float Lp1 = 6.6666668653e-01f, Lp2 = 4.0000000596e-01f,
                Lp3 = 2.8571429849e-01f, Lp4 = 2.2222198546e-01f,
                Lp5 = 1.8183572590e-01f, Lp6 = 1.5313838422e-01f,
                Lp7 = 1.4798198640e-01f;
    float hfsq, f = 0.0f, c = 0.0f, s, z, R, u;
    int32_t k, hx, hu = 0, ax;
    hx = (int32_t)f2u(x);
    ax = hx & 0x7fffffff;
    k = 1;
    if (hx < 0x3ed413d7) {
        if (ax >= 0x3f800000) {
            if (x == -1.0f) return -INFINITY;
            return NAN;
        }
        if (ax < 0x31000000) {
            if (ax < 0x24800000) return x;
            return x - x * x * 0.5f;
        }
        if (hx > 0 || hx <= (int32_t)0xbe95f61f) { k = 0; f = x; hu = 1; }
    } else if (hx >= 0x7f800000) {
        return x + x;
    }
    if (k != 0) {
        if (hx < 0x5a000000) {
            u = 1.0f + x;
            hu = (int32_t)f2u(u);
            k = (hu >> 23) - 127;
            c = (k > 0) ? 1.0f - (u - x) : x - (u - 1.0f);
            c /= u;
        } else {
            u = x;
            hu = (int32_t)f2u(u);
            k = (hu >> 23) - 127;
            c = 0;
        }
        hu &= 0x007fffff;
        if (hu < 0x3504f7) {
            u = u2f((uint32_t)hu | 0x3f800000);
        } else {
            k += 1;
            u = u2f((uint32_t)hu | 0x3f000000);
            hu = (0x00800000 - hu) >> 2;
        }
        f = u - 1.0f;
    }
    hfsq = 0.5f * f * f;
    if (hu == 0) {
        if (f == 0.0f) {
            if (k == 0) return 0.0f;
            c += (float)k * ln2_lo;
            return (float)k * ln2_hi + c;
        }
        R = hfsq * (1.0f - 0.66666666666666666f * f);
        if (k == 0) return f - R;
        return (float)k * ln2_hi - ((R - ((float)k * ln2_lo + c)) - f);
    }
    s = f / (2.0f + f);
    z = s * s;
    R = z * (Lp1 + z * (Lp2 + z * (Lp3 + z * (Lp4 + z * (Lp5 + z * (Lp6 + z * Lp7))))));
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return (float)k * ln2_hi - ((hfsq - (s * (hfsq + R) + ((float)k * ln2_lo + c))) - f);
}

/* softplus = np.logaddexp(x, 0) in float32 (ssm.py:93-95; numpy npy_logaddexpf) */
float softplus_f32(float x)
{
    if (x == 0.0f) return 0.0f + 0.693147180559945309417232121458176568f;
    float tmp = x - 0.0f;
    if (tmp > 0) return x + glibc_log1pf(glibc_expf(-tmp));
    if (tmp <= 0) return 0.0f + glibc_log1pf(glibc_expf(tmp));
    return tmp; /* NaN */
}

/* silu(x) = x / (1 + np.exp(-x)) in float32 (ssm.py:98-101) */
float silu_f32(float x)
{
    return x / (1.0f + np_exp_f32(-x));
}

/* ------------------------------------------------------------------------ */
/* numpy pairwise float32 sum (np.mean in rmsnorm, ssm.py:104-107).          */
/* ------------------------------------------------------------------------ */
float pairwise_sum_f32(const float *a, ptrdiff_t n)
{
    if (n < 8) {
        float res = 0.0f;
        for (ptrdiff_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        float r[8];
        ptrdiff_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        ptrdiff_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum_f32(a, n2) + pairwise_sum_f32(a + n2, n - n2);
    }
}

/* ------------------------------------------------------------------------ */
/* Vector entry points (ctypes).                                            */
/* ------------------------------------------------------------------------ */
void oracle_np_exp_f32(const float *x, float *y, size_t n)
{ for (size_t i = 0; i < n; i++) y[i] = np_exp_f32(x[i]); }

void oracle_glibc_expf(const float *x, float *y, size_t n)
{ for (size_t i = 0; i < n; i++) y[i] = glibc_expf(x[i]); }

void oracle_glibc_log1pf(const float *x, float *y, size_t n)
{ for (size_t i = 0; i < n; i++) y[i] = glibc_log1pf(x[i]); }

void oracle_softplus(const float *x, float *y, size_t n)
{ for (size_t i = 0; i < n; i++) y[i] = softplus_f32(x[i]); }

void oracle_silu(const float *x, float *y, size_t n)
{ for (size_t i = 0; i < n; i++) y[i] = silu_f32(x[i]); }

/* Exhaustive/strided self-check helpers: count mismatches of the restated
 * function against the host libm over bit patterns [lo, hi) with a stride. */
size_t oracle_count_expf_mismatch(uint64_t lo, uint64_t hi, uint64_t stride)
{
    size_t bad = 0;
    for (uint64_t b = lo; b < hi; b += stride) {
        float x = u2f((uint32_t)b);
        float a = glibc_expf(x), r = expf(x);
        if (f2u(a) != f2u(r) && !(isnan(a) && isnan(r))) bad++;
    }
    return bad;
}

size_t oracle_count_log1pf_mismatch(uint64_t lo, uint64_t hi, uint64_t stride)
{
    size_t bad = 0;
    for (uint64_t b = lo; b < hi; b += stride) {
        float x = u2f((uint32_t)b);
        float a = glibc_log1pf(x), r = log1pf(x);
        if (f2u(a) != f2u(r) && !(isnan(a) && isnan(r))) bad++;
    }
    return bad;
}

/* mean of squares per row: np.mean(np.square(x), axis=-1) (ssm.py:106) */
void oracle_mean_sq(const float *x, ptrdiff_t rows, ptrdiff_t n, float *out, float *scratch)
{
    for (ptrdiff_t r = 0; r < rows; r++) {
        const float *row = x + r * n;
        for (ptrdiff_t i = 0; i < n; i++) scratch[i] = row[i] * row[i];
        out[r] = pairwise_sum_f32(scratch, n) / (float)n;
    }
}

/* rmsnorm(x, gain) = x / sqrt(mean(x^2) + eps) * gain  (ssm.py:104-107) */
void oracle_rmsnorm(const float *x, const float *gain, ptrdiff_t rows, ptrdiff_t n,
                    float eps, float *out, float *scratch)
{
    for (ptrdiff_t r = 0; r < rows; r++) {
        const float *row = x + r * n;
        for (ptrdiff_t i = 0; i < n; i++) scratch[i] = row[i] * row[i];
        float ms = pairwise_sum_f32(scratch, n) / (float)n;
        float den = sqrtf(ms + eps);
        for (ptrdiff_t i = 0; i < n; i++) out[r * n + i] = row[i] / den * gain[i];
    }
}

/* ------------------------------------------------------------------------ */
/* Selective scan, float path of _core.selective_scan (_core.pyx:46-65).    */
/* x, delta: (T, D); a: (D, N); b, c: (T, N); d: (D,); h: (D, N) in/out.     */
/* Returns 1 if any output or state value is non-finite (kernels.py:97-98). */
/* ------------------------------------------------------------------------ */
int oracle_selective_scan(const float *x, const float *delta, const float *a,
                          const float *b, const float *c, const float *d,
                          float *h, float *out, ptrdiff_t T, ptrdiff_t D, ptrdiff_t N)
{
    for (ptrdiff_t t = 0; t < T; t++) {
        for (ptrdiff_t i = 0; i < D; i++) {
            float dt = delta[t * D + i];
            float dbx = dt * x[t * D + i];
            float acc = 0.0f;
            for (ptrdiff_t j = 0; j < N; j++) {
                float e = glibc_expf(dt * a[i * N + j]);
                float p1 = h[i * N + j] * e;
                float p2 = dbx * b[t * N + j];
                float hv = p1 + p2;
                h[i * N + j] = hv;
                acc = acc + hv * c[t * N + j];
            }
            out[t * D + i] = acc + d[i] * x[t * D + i];
        }
    }
    int bad = 0;
    for (ptrdiff_t k = 0; k < T * D; k++) if (!isfinite(out[k])) bad = 1;
    for (ptrdiff_t k = 0; k < D * N; k++) if (!isfinite(h[k])) bad = 1;
    return bad;
}

/* ------------------------------------------------------------------------ */
/* Unnormalized Hadamard H_n = kron(H_{2^p}, B_m) along rows of length n.    */
/* apply_hadamard (hadamard.py:128-149): per contiguous m-chunk a sequential */
/* +/-1 base product from +0.0 (the BLAS product at :140 with +/-1 entries   */
/* accumulates exactly this way), then the radix-2 butterfly across the 2^p  */
/* chunks with h ascending (_core.pyx:12-28).  In place, float32.            */
/* ------------------------------------------------------------------------ */
void oracle_hadamard_f32(float *rows, ptrdiff_t nrows, int p, int m,
                         const int8_t *base, float *scratch)
{
    ptrdiff_t blocks = (ptrdiff_t)1 << p, n = blocks * m;
    for (ptrdiff_t r = 0; r < nrows; r++) {
        float *v = rows + r * n;
        if (m > 1) {
            for (ptrdiff_t blk = 0; blk < blocks; blk++) {
                for (int o = 0; o < m; o++) {
                    float acc = 0.0f;
                    for (int k = 0; k < m; k++) {
                        float term = base[o * m + k] > 0 ? v[blk * m + k] : -v[blk * m + k];
                        acc = acc + term;
                    }
                    scratch[blk * m + o] = acc;
                }
            }
            memcpy(v, scratch, (size_t)n * sizeof(float));
        }
        for (ptrdiff_t h = 1; h < blocks; h *= 2) {
            for (ptrdiff_t i = 0; i < blocks; i += 2 * h) {
                for (ptrdiff_t j = i; j < i + h; j++) {
                    for (int l = 0; l < m; l++) {
                        float u = v[j * m + l], w = v[(j + h) * m + l];
                        v[j * m + l] = u + w;
                        v[(j + h) * m + l] = u - w;
                    }
                }
            }
        }
    }
}
