// qmb_gemm.cu -- tcgen05 kind::i8 GEMM (TMA -> smem -> UMMA -> TMEM -> fused
// epilogue) and a warp-per-column dp4a GEMV path for skinny M (decode).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <string.h>
#include <climits>
#include <stdlib.h>
#include <mutex>

#include "qmb_gemm.cuh"

namespace qmb {

// ============================================================ tensor-core path
// Persistent warp-specialized kernel: warp 0 = TMA producer, warp 1 = TMEM
// allocator + single-thread UMMA issuer, EPIW epilogue warps (EPIW/4 per TMEM
// lane quarter, splitting the tile's 32-column chunks).  The accumulator is
// double-buffered in TMEM so the epilogue of tile i overlaps the MMAs of tile
// i+1.  With TMAOUT, the f32 segment is staged through swizzled shared memory
// (32 rows x 16 floats per store) and written with TMA bulk tensor stores.
constexpr int TC_BM = 128;
constexpr int TC_BK = 128;  // bytes of K per stage = one 128B swizzle atom

// CG = 2: CTA pair (cluster of 2, tcgen05 cta_group::2): the pair computes a
// 256 x BN tile; each CTA stages its own 128 rows of A and half (BN/2 rows) of
// B, the leader issues M=256 MMAs over both CTAs' shared memory, and each CTA's
// TMEM receives its 128 rows of the accumulator.  Per output element the
// operand bytes streamed from L2 drop from K(1/BN + 1/128) to K(1/BN + 1/256)
// x ... per CTA (half of B), which is what bounds the large in/out_proj GEMMs.
template <int BN, int EPIW, bool TMAOUT, int CG = 1>
struct TcCfg {
  static constexpr int THREADS = 64 + 32 * EPIW;
  static constexpr int A_BYTES = TC_BM * TC_BK;
  static constexpr int B_BYTES = (BN / CG) * TC_BK;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STG_BYTES = TMAOUT ? EPIW * 4096 : 0;  // 2 x (32 rows x 64 B) per epilogue warp
  static constexpr int BUDGET = 227 * 1024 - 1024 - STG_BYTES - 1024;  // (227 KB: the per-CTA opt-in maximum)
  static constexpr int STAGES = (BUDGET / STAGE_BYTES) > 8 ? 8 : (BUDGET / STAGE_BYTES);
  static constexpr int TMEM_COLS =
      (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM_BYTES =
      1024 /*align slack*/ + STAGES * STAGE_BYTES + STG_BYTES + ((QTAB_FLOATS + 1) & ~1) * 4 + (2 * STAGES + 4) * 8 + 16;
  static_assert(STAGES >= 2, "pipeline too shallow");
};

// int8 epilogue value: softplus+quant is compiled only into the SP kernels (dt_proj)
template <bool SP>
__device__ __forceinline__ int epi_quant(float v, const EpiSeg& g, const float* qtab, int qmax, uint32_t& err) {
  if constexpr (SP) {
    if (g.kind == EPI_SOFTPLUS_Q) return softplus_quant(v, qtab, g.out_div, g.out_inv, qmax, err);
  }
  return quant_fast(v, g.out_div, g.out_inv, qmax, err);
}

// Rare fix-up of one softplus element outside the table's verified domain:
// the exact formula, out of line (scalar argument, so the caller's chunk stays
// in registers).
__device__ __forceinline__ int epi_softplus_fix1(float v, float s_div, int qmax) {
  return softplus_quant_exact(v, s_div, qmax);  // INT_MIN: non-finite (error word set by the caller)
}

// silu of 32 epilogue values: branch-free core, one warp-uniform test, and the
// rare out-of-range inputs (|x| > 80, |x| < 2^-60, non-finite) redone exactly.
// Rows past M (the zero-filled tail of a partial tile, e.g. a decode batch) are
// never stored, so their out-of-range zeros skip the fix-up.
__device__ __forceinline__ void epi_silu32(float (&v)[32], bool row_valid) {
  uint32_t bad = 0;
  float y[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    y[j] = silu_core(v[j]);
    bad |= silu_core_ok(v[j]) ? 0u : (1u << j);
  }
  if (!row_valid) bad = 0;
  if (bad) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (bad & (1u << j)) y[j] = silu_f32_cold(v[j]);
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = y[j];
}

// quantize 32 finite values (quant_fast semantics) into packed int8, branch-free
// except for one test and free of conversion-unit ops; near-tie elements take the
// exact division.
__device__ __forceinline__ void epi_quant32_plain(const float (&v)[32], float s, float inv, int qmax, uint32_t& err,
                                                  uint32_t (&packed)[8]) {
  const float hi = (float)qmax;
  uint32_t miss = 0;
  int q[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {  // (v finite: an int32 accumulator times a finite scale)
    float d;
    q[j] = quant_level_magic(__fmul_rn(v[j], inv), hi + 1.0f, qmax, &d);
    miss |= (d < 0.499755859375f) ? 0u : (1u << j);
  }
  if (miss) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (miss & (1u << j)) {
        float r = quant_slow_rint(v[j], s);
        if (r != r) {
          err |= QMB_ERR_NONFINITE;
          r = 0.0f;
        }
        q[j] = (int)fminf(fmaxf(r, -hi), hi);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 32; j += 4)
    packed[j / 4] = (uint32_t)(q[j] & 0xff) | ((uint32_t)(q[j + 1] & 0xff) << 8) | ((uint32_t)(q[j + 2] & 0xff) << 16) |
                    ((uint32_t)(q[j + 3] & 0xff) << 24);
}

// Compact TMA-store chunk (CTA-pair kernels): the 32-column chunk is processed as four
// 8-column sub-chunks in a rolled loop, each loaded from TMEM, converted, finished
// (bias, residual add, silu or quantize) and staged, so the per-kind code is a
// few hundred instructions: with the x and z chunks of a tile interleaved, the
// fully unrolled 32-wide paths did not fit the instruction cache together.
__device__ __forceinline__ void epi_silu8(float (&v)[8], bool row_valid, unsigned long long one2,
                                          unsigned long long negz2) {
  uint32_t bad = 0;
  float y[8];
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float2 r = unpack_f32x2(silu_core2(pack_f32x2(v[j], v[j + 1]), one2, negz2));
    y[j] = r.x;
    y[j + 1] = r.y;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) bad |= silu_core_ok(v[j]) ? 0u : (1u << j);
  if (!row_valid) bad = 0;
  if (bad) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (bad & (1u << j)) y[j] = silu_f32_cold(v[j]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = y[j];
}

template <int EPIW>
__device__ __forceinline__ void epi_chunk_sub8(const EpiParams& ep, const EpiSeg& sg, uint32_t taddr, float* stg,
                                               int oc, long long m, int M, int lane, const CUtensorMap* map,
                                               int row0, uint32_t& err) {
  const bool f32 = epi_is_f32(sg.kind);
  const float hi = (float)ep.qmax;
  if (lane == 0) bulk_wait_read0();  // the staging buffer's previous store has been read
  __syncwarp();
  uint8_t* hb8 = reinterpret_cast<uint8_t*>(stg);
  const int sw32 = (lane >> 2) & 1;
#pragma unroll 1
  for (int g = 0; g < 4; ++g) {
    uint32_t r8[8];
    tmem_ld_32x32b_x8(taddr + 8 * g, r8);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __fmul_rn(__int2float_rn((int)r8[j]), sg.acc_scale);
    if (sg.bias) {
      const float4* bp = reinterpret_cast<const float4*>(sg.bias + oc + 8 * g);
      const float4 b0 = __ldg(bp), b1 = __ldg(bp + 1);
      v[0] = __fadd_rn(v[0], b0.x), v[1] = __fadd_rn(v[1], b0.y), v[2] = __fadd_rn(v[2], b0.z);
      v[3] = __fadd_rn(v[3], b0.w), v[4] = __fadd_rn(v[4], b1.x), v[5] = __fadd_rn(v[5], b1.y);
      v[6] = __fadd_rn(v[6], b1.z), v[7] = __fadd_rn(v[7], b1.w);
    }
    if (f32) {
      if (sg.kind == EPI_F32_ADDTO && m < M) {
        const float4* op = reinterpret_cast<const float4*>(static_cast<const float*>(sg.out) + m * sg.ld + oc + 8 * g);
        const float4 o0 = op[0], o1 = op[1];
        v[0] = __fadd_rn(v[0], o0.x), v[1] = __fadd_rn(v[1], o0.y), v[2] = __fadd_rn(v[2], o0.z);
        v[3] = __fadd_rn(v[3], o0.w), v[4] = __fadd_rn(v[4], o1.x), v[5] = __fadd_rn(v[5], o1.y);
        v[6] = __fadd_rn(v[6], o1.z), v[7] = __fadd_rn(v[7], o1.w);
      }
      if (sg.kind == EPI_F32_SILU) epi_silu8(v, m < M, ep.one2, ep.negz2);
      // 32 rows x 16 floats per half, 64B rows, SWIZZLE_64B: quad q of a row at q ^ ((row >> 1) & 3)
      float* hb = stg + (g >> 1) * 512;
      const int qa = (g & 1) * 2;
      *reinterpret_cast<float4*>(hb + lane * 16 + ((qa ^ ((lane >> 1) & 3)) * 4)) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(hb + lane * 16 + (((qa + 1) ^ ((lane >> 1) & 3)) * 4)) =
          make_float4(v[4], v[5], v[6], v[7]);
    } else {  // EPI_QUANT (v finite)
      uint32_t miss = 0;
      int q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float d;
        q[j] = quant_level_magic(__fmul_rn(v[j], sg.out_inv), hi + 1.0f, ep.qmax, &d);
        miss |= (d < 0.499755859375f) ? 0u : (1u << j);
      }
      if (miss) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (miss & (1u << j)) {
            float rr = quant_slow_rint(v[j], sg.out_div);
            if (rr != rr) {
              err |= QMB_ERR_NONFINITE;
              rr = 0.0f;
            }
            q[j] = (int)fminf(fmaxf(rr, -hi), hi);
          }
        }
      }
      const uint32_t w0 = (uint32_t)(q[0] & 0xff) | ((uint32_t)(q[1] & 0xff) << 8) | ((uint32_t)(q[2] & 0xff) << 16) |
                          ((uint32_t)(q[3] & 0xff) << 24);
      const uint32_t w1 = (uint32_t)(q[4] & 0xff) | ((uint32_t)(q[5] & 0xff) << 8) | ((uint32_t)(q[6] & 0xff) << 16) |
                          ((uint32_t)(q[7] & 0xff) << 24);
      // 32 rows x 32 B, SWIZZLE_32B: 16B chunk c of row r at chunk c ^ ((r >> 2) & 1)
      *reinterpret_cast<uint2*>(hb8 + lane * 32 + (((g >> 1) ^ sw32) * 16) + (g & 1) * 8) = make_uint2(w0, w1);
    }
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (f32) {
      tma_store_2d(map, stg, oc, row0);
      tma_store_2d(map, stg + 512, oc + 16, row0);
    } else {
      tma_store_2d(map, hb8, oc, row0);
    }
    bulk_commit();
  }
}

// 32 epilogue values -> 32 int8 (packed little-endian)
template <bool SP>
__device__ __forceinline__ void epi_quant32(const float (&v)[32], const EpiSeg& g, const float* qtab, int qmax,
                                            uint32_t& err, uint32_t (&packed)[8], uint32_t qtab_bias,
                                            unsigned long long one2, unsigned long long negz2) {
  if constexpr (SP) {
    if (g.kind == EPI_SOFTPLUS_Q && qtab) {
      const float lo = qtab[QTAB_LO], hi = qtab[QTAB_HI], qmaxf = (float)qmax;
      const uint32_t tab_b = softplus_tab_bias(qtab, qtab_bias);
      const unsigned long long sinv2 = pack_f32x2(g.out_inv, g.out_inv);
      float chk = 0.0f;  // NaN-sticky: becomes NaN iff some v is not finite
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        uint32_t b[4];
        softplus_quant_table_bits2(v[j], v[j + 1], tab_b, sinv2, qmaxf, one2, negz2, b[0], b[1]);
        softplus_quant_table_bits2(v[j + 2], v[j + 3], tab_b, sinv2, qmaxf, one2, negz2, b[2], b[3]);
#pragma unroll
        for (int t = 0; t < 4; ++t) chk = __fmaf_rn(v[j + t], 0.0f, chk);
        packed[j / 4] = __byte_perm(__byte_perm(b[0], b[1], 0x40), __byte_perm(b[2], b[3], 0x40), 0x5410);
      }
      bool miss = !(chk == 0.0f);
      if (lo <= hi) {  // a disagreement interval exists (uniform; typically empty)
#pragma unroll
        for (int j = 0; j < 32; ++j) miss |= (v[j] >= lo && v[j] <= hi);
      }
      if (miss) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (softplus_table_miss(v[j], lo, hi)) {
            int q = epi_softplus_fix1(v[j], g.out_div, qmax);
            if (q == INT_MIN) {
              err |= QMB_ERR_NONFINITE;
              q = 0;
            }
            const int sh = 8 * (j & 3);
            packed[j >> 2] = (packed[j >> 2] & ~(0xffu << sh)) | ((uint32_t)(q & 0xff) << sh);
          }
        }
      }
      return;
    }
  }
  if (SP) {  // 16-warp kernels (<= 112 registers): per-element form
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      uint32_t w = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int q = epi_quant<SP>(v[j + t], g, qtab, qmax, err);
        w |= ((uint32_t)(q & 0xff)) << (8 * t);
      }
      packed[j / 4] = w;
    }
    return;
  }
  epi_quant32_plain(v, g.out_div, g.out_inv, qmax, err, packed);
}

// Ragged / misaligned chunk (segment boundary inside the chunk, tails, odd
// strides): element-wise stores.  Out of line: it is the cold path.  It
// re-reads the chunk from TMEM itself (all 32 lanes call it: tcgen05.ld is
// warp-collective), so the hot path never has to materialize its registers
// in local memory for it.
template <bool SP>
__device__ __noinline__ uint32_t epi_chunk_scalar(const EpiParams& ep, uint32_t taddr, int nb, int N, long long m,
                                                  int M, const float* qtab) {
  uint32_t r[32], err = 0;
  tmem_ld_32x32b_x32(taddr, r);
  if (m >= M) return 0;
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    const int n = nb + j;
    if (n >= N) break;
    int oc;
    const EpiSeg sj = pick_seg(ep, epi_locate(ep, n, &oc));
    float v = __fmul_rn(__int2float_rn((int)r[j]), sj.acc_scale);
    if (sj.bias) v = __fadd_rn(v, sj.bias[oc]);
    const long long off = m * sj.ld + oc;
    if (epi_is_f32(sj.kind)) {
      float* o = static_cast<float*>(sj.out) + off;
      *o = sj.kind == EPI_F32_SILU ? silu_f32_fast(v) : (sj.kind == EPI_F32_ADDTO ? __fadd_rn(v, *o) : v);
    }
    else
      static_cast<int8_t*>(sj.out)[off] = (int8_t)epi_quant<SP>(v, sj, qtab, ep.qmax, err);
  }
  return err;
}

template <int BN, int EPIW, bool TMAOUT, int CG = 1>
__global__ void __launch_bounds__(TcCfg<BN, EPIW, TMAOUT, CG>::THREADS, 1)
    gemm_i8_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2, int M,
                      int N, int Kp, const __grid_constant__ EpiParams ep) {
  using C = TcCfg<BN, EPIW, TMAOUT, CG>;
  constexpr int TILE_M = TC_BM * CG;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;  // CTA's row half of the pair tile
  const bool leader = rank == 0;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned by offsetting the shared array itself (keeps LDS/STS addressing)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sStg = smem + STAGES * C::STAGE_BYTES;  // 1024-aligned
  float* sQtab = reinterpret_cast<float*>(sStg + C::STG_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sQtab + ((QTAB_FLOATS + 1) & ~1));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (TMAOUT && ep.tma_seg >= 0) tma_prefetch_desc(&tmC);
    if (TMAOUT && ep.tma_seg2 >= 0) tma_prefetch_desc(&tmC2);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], CG);  // (pair: used in the leader only; one arrive per CTA)
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], EPIW * CG);  // one per epilogue warp (pair: the leader's counts both CTAs')
    }
    fence_barrier_init();
  }
  // softplus threshold table of the (single) EPI_SOFTPLUS_Q segment -> smem
  const float* qtab_g = nullptr;
  for (int s = 0; s < ep.nseg; ++s)
    if (ep.seg[s].kind == EPI_SOFTPLUS_Q) qtab_g = ep.seg[s].qtab;
  if (qtab_g)
    for (int k = threadIdx.x; k < QTAB_FLOATS; k += blockDim.x) sQtab[k] = qtab_g[k];
  if (warp == 1) {
    if (CG == 2)
      tmem_alloc_pair(tslot, C::TMEM_COLS);
    else
      tmem_alloc(tslot, C::TMEM_COLS);
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // peer barriers initialized before any remote arrive / TMA completion
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_trigger();  // (decode chains: the next kernel may start its prologue)

  const int num_m = (M + TILE_M - 1) / TILE_M;
  const int num_n = (N + BN - 1) / BN;
  const int splitk = ep.splitk > 1 ? ep.splitk : 1;
  const int num_tiles = num_m * num_n * splitk;
  const int num_k_all = (Kp + TC_BK - 1) / TC_BK;
  const int kper = (num_k_all + splitk - 1) / splitk;
  // tile -> (m block, n block, K split): splits of one output tile are adjacent
  auto tile_coords = [&](int tile, int& m0, int& n0, int& kb0, int& kb1) {
    const int sk = tile % splitk, mn = tile / splitk;
    m0 = (mn / num_n) * TILE_M;
    n0 = (mn % num_n) * BN;
    kb0 = sk * kper;
    kb1 = min(num_k_all, kb0 + kper);
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // The weights (B) do not depend on the previous kernel: under PDL the first
      // tile's first STAGES B loads are issued before the dependency wait, their A
      // halves after it.
      int pre = 0;
      if (CG == 1 && (int)blockIdx.x < num_tiles) {
        int m0, n0, kb0, kb1;
        tile_coords(blockIdx.x, m0, n0, kb0, kb1);
        for (int kb = kb0; kb < kb1 && pre < STAGES; ++kb, ++pre) {
          mbar_arrive_expect_tx(&full[pre], C::STAGE_BYTES);
          tma_load_2d(sB + pre * C::B_BYTES, &tmB, &full[pre], kb * TC_BK, n0);
        }
      }
      pdl_wait();
      int it = 0;
      for (int tile = blockIdx.x / CG; tile < num_tiles; tile += gridDim.x / CG) {
        int m0, n0, kb0, kb1;
        tile_coords(tile, m0, n0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          if (it < pre) {  // B already in flight; stage / phase advance as in the main path
            tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * TC_BK, m0);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if (ep.spin) mbar_wait(&empty[stage], phase ^ 1); else mbar_wait_sleep(&empty[stage], phase ^ 1);
          if (CG == 2) {
            // both CTAs' bytes complete on the leader's barrier
            if (leader)
              mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            else
              mbar_arrive_remote(&full[stage], 0);
            tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * TC_BK, m0 + (int)rank * TC_BM);
            tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * TC_BK, n0 + (int)rank * (BN / 2));
          } else {
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * TC_BK, m0);
            tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * TC_BK, n0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = umma_idesc_i8(TILE_M, BN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x / CG; tile < num_tiles; tile += gridDim.x / CG, ++it) {
        const int buf = it & 1;
        const uint32_t use = (uint32_t)(it >> 1);
        if (ep.spin) mbar_wait(&tempty[buf], (use & 1) ^ 1); else mbar_wait_sleep(&tempty[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(buf * BN);
        int m0, n0, kb0, kb1;
        tile_coords(tile, m0, n0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (ep.spin) mbar_wait(&full[stage], phase); else mbar_wait_sleep(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 32; ++k) {
            if (CG == 2)
              umma_i8_pair(d, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                           (kb > kb0 || k > 0) ? 1u : 0u);
            else
              umma_i8(d, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
          }
          if (CG == 2)
            umma_commit_pair(&empty[stage]);
          else
            umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (CG == 2)
          umma_commit_pair(&tfull[buf]);
        else
          umma_commit(&tfull[buf]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 2;                 // epilogue warp index
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int part = ew / 4;                 // which 1/(EPIW/4) slice of the column chunks
    constexpr int PARTS = EPIW / 4;
    const int row = quarter * 32 + lane;
    constexpr int CHUNKS = BN / 32;
    float* stg = reinterpret_cast<float*>(sStg + (TMAOUT ? ew * 4096 : 0));
    const float* qtab = qtab_g ? sQtab : nullptr;
    uint32_t err = 0;
    int it = 0;
    pdl_wait();
    for (int tile = blockIdx.x / CG; tile < num_tiles; tile += gridDim.x / CG, ++it) {
      const int buf = it & 1;
      const uint32_t use = (uint32_t)(it >> 1);
      int m0, n0, kb0, kb1;
      tile_coords(tile, m0, n0, kb0, kb1);
      m0 += (int)rank * TC_BM;  // this CTA's rows of the pair tile
      if (ep.spin) mbar_wait(&tfull[buf], use & 1); else mbar_wait_sleep(&tfull[buf], use & 1);
      tc_fence_after();
      const long long m = (long long)m0 + row;
      const uint32_t tcol = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * BN);
      // 8 epilogue warps (up to 232 registers): the next chunk's TMEM load is in
      // flight while this one is processed; 12 / 16 warps (<= 128 / 112 registers): plain loads
      // The PARTS warps of a lane quarter take alternating 32-column chunks (so an
      // interleaved two-segment tile, ep.il, gives each the same mix of work).
      constexpr bool SUB8 = CG == 2 && TMAOUT && EPIW != 16;  // compact sub-chunk path (epi_chunk_sub8)
      constexpr bool PF = EPIW <= 8 && !SUB8;
      uint32_t rn[32];
      if (PF && part < CHUNKS) tmem_ld_32x32b_x32_nowait(tcol + part * 32, rn);
#pragma unroll 1
      for (int c = part; c < CHUNKS; c += PARTS) {
        if (SUB8 && splitk == 1 && !ep.raw_out) {
          const int nb = n0 + c * 32;
          if (nb >= N) continue;
          int oc;
          const int s = epi_locate(ep, nb, &oc);
          const EpiSeg sg = pick_seg(ep, s);
          const int slot = s == ep.tma_seg ? 0 : (s == ep.tma_seg2 ? 1 : -1);
          if (slot >= 0 && oc + 32 <= sg.n1 - sg.n0 && nb + 32 <= N &&
              (epi_is_f32(sg.kind) || sg.kind == EPI_QUANT)) {
            epi_chunk_sub8<EPIW>(ep, sg, tcol + c * 32, stg, oc, m, M, lane, slot == 0 ? &tmC : &tmC2,
                                 m0 + quarter * 32, err);
            continue;
          }
        }
        uint32_t r[32];
        if (PF) {
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = rn[j];
          if (c + PARTS < CHUNKS) tmem_ld_32x32b_x32_nowait(tcol + (c + PARTS) * 32, rn);
        } else {
          tmem_ld_32x32b_x32(tcol + c * 32, r);
        }
        const int nb = n0 + c * 32;
        if (nb >= N) continue;  // warp-uniform
        if (splitk > 1 || ep.raw_out) {  // split-K partial -> acc32[split][M][N] (summed exactly afterwards),
          if (m < M) {                   // or the raw int32 sums -> raw_out (tensor-parallel partials)
            int32_t* dst = splitk > 1 ? ep.acc32 + ((long long)(tile % splitk) * M + m) * N + nb
                                      : ep.raw_out + m * ep.raw_ld + nb;
            if (nb + 32 <= N && (N % 4) == 0 && (splitk > 1 || ep.raw_ld % 4 == 0)) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<int4*>(dst + j) = make_int4((int)r[j], (int)r[j + 1], (int)r[j + 2], (int)r[j + 3]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < N) dst[j] = (int)r[j];
            }
          }
          continue;
        }
        int oc;  // output column of this chunk within its segment
        const int s = epi_locate(ep, nb, &oc);
        const EpiSeg sg = pick_seg(ep, s);
        const int segw = sg.n1 - sg.n0;
        const int slot = TMAOUT ? (s == ep.tma_seg ? 0 : (s == ep.tma_seg2 ? 1 : -1)) : -1;
        if (TMAOUT && slot >= 0 && oc + 32 <= segw && nb + 32 <= N) {
          // 32 rows x 32 cols through swizzled smem -> TMA store (rows >= M are clipped by TMA)
          const CUtensorMap* map = slot == 0 ? &tmC : &tmC2;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j)  // (16-warp softplus kernels: short-K accumulators off the XU)
            v[j] = __fmul_rn((EPIW == 16 && ep.small_acc) ? i2f_small((int)r[j]) : __int2float_rn((int)r[j]),
                             sg.acc_scale);
          if (sg.bias) {
            const float4* bp = reinterpret_cast<const float4*>(sg.bias + oc);
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 bb = __ldg(bp + j / 4);
              v[j] = __fadd_rn(v[j], bb.x);
              v[j + 1] = __fadd_rn(v[j + 1], bb.y);
              v[j + 2] = __fadd_rn(v[j + 2], bb.z);
              v[j + 3] = __fadd_rn(v[j + 3], bb.w);
            }
          }
          if (epi_is_f32(sg.kind)) {
            if (EPIW <= 12 && sg.kind == EPI_F32_SILU) epi_silu32(v, m < M);
            if (sg.kind == EPI_F32_ADDTO && m < M) {  // += the row's current values
              const float4* op = reinterpret_cast<const float4*>(static_cast<const float*>(sg.out) + m * sg.ld + oc);
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 o4 = op[j / 4];
                v[j] = __fadd_rn(v[j], o4.x);
                v[j + 1] = __fadd_rn(v[j + 1], o4.y);
                v[j + 2] = __fadd_rn(v[j + 2], o4.z);
                v[j + 3] = __fadd_rn(v[j + 3], o4.w);
              }
            }
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float* hb = stg + h * 512;  // 32 rows x 16 floats, 64B rows, SWIZZLE_64B
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int pos = q ^ ((lane >> 1) & 3);
                *reinterpret_cast<float4*>(hb + lane * 16 + pos * 4) = make_float4(
                    v[h * 16 + q * 4], v[h * 16 + q * 4 + 1], v[h * 16 + q * 4 + 2], v[h * 16 + q * 4 + 3]);
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(map, stg, oc, m0 + quarter * 32);
              tma_store_2d(map, stg + 512, oc + 16, m0 + quarter * 32);
              bulk_commit();
            }
          } else {
            uint32_t packed[8];
            epi_quant32<EPIW == 16>(v, sg, qtab, ep.qmax, err, packed, ep.qtab_bias, ep.one2, ep.negz2);
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
            // 32 rows x 32 B, SWIZZLE_32B: 16B chunk c of row r at chunk c ^ ((r >> 2) & 1)
            uint8_t* hb = reinterpret_cast<uint8_t*>(stg);
            const int sw = (lane >> 2) & 1;
            *reinterpret_cast<uint4*>(hb + lane * 32 + (0 ^ sw) * 16) =
                make_uint4(packed[0], packed[1], packed[2], packed[3]);
            *reinterpret_cast<uint4*>(hb + lane * 32 + (1 ^ sw) * 16) =
                make_uint4(packed[4], packed[5], packed[6], packed[7]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(map, hb, oc, m0 + quarter * 32);
              bulk_commit();
            }
          }
          continue;
        }
        const bool f32out = epi_is_f32(sg.kind);
        const long long ldb_bytes = sg.ld * (f32out ? 4 : 1);
        const bool fast = (oc + 32 <= segw) && (nb + 32 <= N) && ((oc & 15) == 0) && (ldb_bytes % 16 == 0) &&
                          ((reinterpret_cast<uintptr_t>(sg.out) & 15) == 0);
        if (!fast) {  // warp-uniform
          tmem_wait_ld();  // the prefetched registers must be final before a call may save them
          err |= epi_chunk_scalar<EPIW == 16>(ep, tcol + c * 32, nb, N, m, M, qtab);
          continue;
        }
        if (m >= M) continue;
        {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j)  // (16-warp softplus kernels: short-K accumulators off the XU)
            v[j] = __fmul_rn((EPIW == 16 && ep.small_acc) ? i2f_small((int)r[j]) : __int2float_rn((int)r[j]),
                             sg.acc_scale);
          if (sg.bias) {
            const float4* bp = reinterpret_cast<const float4*>(sg.bias + oc);
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 bb = __ldg(bp + j / 4);
              v[j] = __fadd_rn(v[j], bb.x);
              v[j + 1] = __fadd_rn(v[j + 1], bb.y);
              v[j + 2] = __fadd_rn(v[j + 2], bb.z);
              v[j + 3] = __fadd_rn(v[j + 3], bb.w);
            }
          }
          if (f32out) {
            if (EPIW <= 12 && sg.kind == EPI_F32_SILU) epi_silu32(v, m < M);
            float4* o = reinterpret_cast<float4*>(static_cast<float*>(sg.out) + m * sg.ld + oc);
            if (sg.kind == EPI_F32_ADDTO) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 o4 = o[j / 4];
                v[j] = __fadd_rn(v[j], o4.x);
                v[j + 1] = __fadd_rn(v[j + 1], o4.y);
                v[j + 2] = __fadd_rn(v[j + 2], o4.z);
                v[j + 3] = __fadd_rn(v[j + 3], o4.w);
              }
            }
#pragma unroll
            for (int j = 0; j < 32; j += 4) o[j / 4] = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
            uint32_t packed[8];
            epi_quant32<EPIW == 16>(v, sg, qtab, ep.qmax, err, packed, ep.qtab_bias, ep.one2, ep.negz2);
            uint4* o = reinterpret_cast<uint4*>(static_cast<int8_t*>(sg.out) + m * sg.ld + oc);
            o[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
            o[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // one arrive per epilogue warp (all its TMEM loads have completed)
        if (CG == 2 && !leader)
          mbar_arrive_remote(&tempty[buf], 0);
        else
          mbar_arrive(&tempty[buf]);
      }
    }
    if (TMAOUT && lane == 0) bulk_wait0();
    flag_error(ep.err, err);
  }

  tc_fence_before();
  if (CG == 2)
    cluster_sync();  // no CTA of the pair leaves while remote arrivals / MMAs may still target it
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_pair(tbase, C::TMEM_COLS);
    else
      tmem_dealloc(tbase, C::TMEM_COLS);
  }
}

// ============================================================ SIMT GEMV path
// One warp per output column n and a block of up to MB rows; lanes split K in
// 16-byte slices; the int32 warp reduction is exact in any order.
template <int MB>
__global__ void __launch_bounds__(256) gemm_i8_simt_kernel(const int8_t* __restrict__ A, long long lda,
                                                           const int8_t* __restrict__ Bt, long long ldb, int M,
                                                           int N, int Kp, EpiParams ep, int vec) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = blockIdx.x * (blockDim.x >> 5) + warp;
  const int m0 = blockIdx.y * MB;
  if (n >= N) return;
  int acc[MB];
#pragma unroll
  for (int i = 0; i < MB; ++i) acc[i] = 0;
  const int8_t* brow = Bt + (long long)n * ldb;
  if (vec) {
    for (int k = lane * 16; k + 16 <= Kp; k += 32 * 16) {
      const int4 b = __ldg(reinterpret_cast<const int4*>(brow + k));
#pragma unroll
      for (int i = 0; i < MB; ++i) {
        if (m0 + i < M) {
          const int4 a = __ldg(reinterpret_cast<const int4*>(A + (long long)(m0 + i) * lda + k));
          acc[i] = __dp4a(a.x, b.x, acc[i]);
          acc[i] = __dp4a(a.y, b.y, acc[i]);
          acc[i] = __dp4a(a.z, b.z, acc[i]);
          acc[i] = __dp4a(a.w, b.w, acc[i]);
        }
      }
    }
    for (int k = (Kp / 16) * 16 + lane; k < Kp; k += 32) {
#pragma unroll
      for (int i = 0; i < MB; ++i)
        if (m0 + i < M) acc[i] += (int)A[(long long)(m0 + i) * lda + k] * (int)brow[k];
    }
  } else {
    for (int k = lane; k < Kp; k += 32) {
      const int b = brow[k];
#pragma unroll
      for (int i = 0; i < MB; ++i)
        if (m0 + i < M) acc[i] += (int)A[(long long)(m0 + i) * lda + k] * b;
    }
  }
#pragma unroll
  for (int i = 0; i < MB; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  }
  uint32_t err = 0;
  int oc;
  const EpiSeg sg = pick_seg(ep, epi_locate(ep, n, &oc));
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    if (lane == i && m0 + i < M) epi_store_one(ep, sg, m0 + i, oc, acc[i], err);
  }
  flag_error(ep.err, err);
}

// ============================================================ decode GEMV (M <= 8)
// Decode-size products stream every weight byte once and do ~M int8 MACs per byte:
// HBM-bound, so this path is built for bytes in flight rather than tensor-core
// throughput.  CTA = GV_WC x WK warps; warp (wc, wk) owns 4 output columns
// n0 + 4 wc .. + 3 and the K slice wk (lanes take 16 consecutive bytes each, 512 B
// of K per warp-iteration).  The weight rows are K-major [N][ldb], so a warp's
// loads are four fully-used 512-byte segments; GV_LA slices stay in flight per
// warp (a register ring, each slot refilled as it is consumed), and the first
// slice is issued before griddepcontrol.wait (weights never depend on the
// previous kernel of a decode chain).  The M <= MB activation rows are staged in
// shared memory once per CTA.  Per-warp int32 sums: xor-shuffle tree, then the
// WK K-slices through shared memory -- exact in any order.  The epilogue is the
// same per-element code as every other path (epi_store_one).
constexpr int GV_WC = 4;  // column warps per CTA (16 columns)

// in_proj x column (row m, channel oc) -> its code, then the fused conv step (EpiConv)
__device__ __forceinline__ void gemv_conv_x(const EpiParams& ep, const EpiSeg& sg, int m, int oc, int acc,
                                            uint32_t& err) {
  float v = __fmul_rn(__int2float_rn(acc), sg.acc_scale);
  if (sg.bias) v = __fadd_rn(v, sg.bias[oc]);
  const int q = quant_fast(v, sg.out_div, sg.out_inv, ep.qmax, err);  // = EPI_QUANT
  const EpiConv& cf = ep.cf;
  int8_t* st = cf.state + (long long)m * (cf.K - 1) * cf.C + oc;
  int ca = 0;  // int8 x int8 -> int32: exact in any order
  for (int k = 0; k + 1 < cf.K; ++k) ca += (int)cf.w[(long long)k * cf.C + oc] * (int)st[(long long)k * cf.C];
  ca += (int)cf.w[(long long)(cf.K - 1) * cf.C + oc] * q;
  float real = __fmul_rn(__int2float_rn(ca), cf.s_conv);
  if (cf.bias) real = __fadd_rn(real, cf.bias[oc]);
  float d;
  int y = silu_quant_level(real, cf.inv_out, (float)ep.qmax + 1.0f, ep.qmax, &d);
  if (!(d < cf.thr)) {
    y = silu_quant_exact(real, cf.s_out, ep.qmax);
    if (y == INT_MIN) {
      err |= QMB_ERR_NONFINITE;
      y = 0;
    }
  }
  cf.out[(long long)m * cf.ldo + oc] = (int8_t)y;
  for (int k = 0; k + 2 < cf.K; ++k) st[(long long)k * cf.C] = st[(long long)(k + 1) * cf.C];
  if (cf.K > 1) st[(long long)(cf.K - 2) * cf.C] = (int8_t)q;
}

template <int MB, int WK>
__global__ void __launch_bounds__(32 * GV_WC * WK) gemv_i8_kernel(const int8_t* __restrict__ A, long long lda,
                                                                 const int8_t* __restrict__ Bt, long long ldb, int M,
                                                                 int N, int Kp, EpiParams ep) {
  extern __shared__ __align__(16) uint8_t gv_smem[];
  int8_t* sA = reinterpret_cast<int8_t*>(gv_smem);                         // [MB][Kp]
  int* sRed = reinterpret_cast<int*>(gv_smem + ((MB * Kp + 15) & ~15));   // [WK][4 GV_WC][MB]
  __shared__ float sQt[QTAB_FLOATS];
  const float* qt = stage_qtab(ep, sQt);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wc = warp % GV_WC, wk = warp / GV_WC;
  const int n0 = (blockIdx.x * GV_WC + wc) * 4;
  const int nslices = Kp / 512 + ((Kp & 511) ? 1 : 0);
  const int per = (nslices + WK - 1) / WK;
  const int s0 = wk * per, s1 = min(nslices, s0 + per);
  const int8_t* brow[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) brow[j] = Bt + (long long)min(n0 + j, N - 1) * ldb;
  auto ldw = [&](int sl, int4 (&w)[4]) {
    const int k = sl * 512 + lane * 16;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w[j] = (sl < s1 && k < Kp) ? __ldg(reinterpret_cast<const int4*>(brow[j] + k)) : make_int4(0, 0, 0, 0);
  };
  int4 wcur[4];
  ldw(s0, wcur);  // before the dependency wait
  pdl_wait();
  pdl_trigger();
  for (int k = threadIdx.x * 16; k < MB * Kp; k += blockDim.x * 16) {
    const int m = k / Kp, kk = k - m * Kp;
    *reinterpret_cast<int4*>(sA + k) =
        m < M ? *reinterpret_cast<const int4*>(A + (long long)m * lda + kk) : make_int4(0, 0, 0, 0);
  }
  __syncthreads();
  int acc[4][MB];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int m = 0; m < MB; ++m) acc[j][m] = 0;
  // GV_LA slices (512 B x 4 columns each) in flight per warp: a register ring,
  // refilled as each slice is used (fewer for many rows: their accumulators)
  constexpr int GV_LA = 2;  // (deeper rings measured slower: fewer CTAs resident per SM)
  int4 wr[GV_LA - 1][4];
#pragma unroll
  for (int u = 0; u < GV_LA - 1; ++u) ldw(s0 + 1 + u, wr[u]);
  for (int sl = s0; sl < s1; sl += GV_LA) {
#pragma unroll
    for (int u = 0; u < GV_LA; ++u) {
      int4 wc[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) wc[j] = u == 0 ? wcur[j] : wr[u - 1][j];
      // refill this ring slot with the slice GV_LA ahead
      if (u == 0) ldw(sl + GV_LA, wcur); else ldw(sl + u + GV_LA, wr[u - 1]);
      const int k = (sl + u) * 512 + lane * 16;
      if (sl + u < s1 && k < Kp) {
#pragma unroll
        for (int m = 0; m < MB; ++m) {
          const int4 a = *reinterpret_cast<const int4*>(sA + m * Kp + k);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[j][m] = __dp4a(a.x, wc[j].x, acc[j][m]);
            acc[j][m] = __dp4a(a.y, wc[j].y, acc[j][m]);
            acc[j][m] = __dp4a(a.z, wc[j].z, acc[j][m]);
            acc[j][m] = __dp4a(a.w, wc[j].w, acc[j][m]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int m = 0; m < MB; ++m)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j][m] += __shfl_xor_sync(0xffffffffu, acc[j][m], o);
  if (WK > 1) {
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int m = 0; m < MB; ++m) sRed[(wk * 4 * GV_WC + 4 * wc + j) * MB + m] = acc[j][m];
    }
    __syncthreads();
  }
  // output (column j of this warp, row m) -> lane 8 j + m ... (MB <= 8)
  if (wk == 0) {
    const int j = lane >> 3, m = lane & 7;
    if (m < MB && m < M && n0 + j < N) {
      int v = 0;
      if (WK > 1) {
#pragma unroll
        for (int w = 0; w < WK; ++w) v += sRed[(w * 4 * GV_WC + 4 * wc + j) * MB + m];
      } else {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int mm = 0; mm < MB; ++mm)
            if (jj == j && mm == m) v = acc[jj][mm];
      }
      uint32_t err = 0;
      int oc;
      const int s = epi_locate(ep, n0 + j, &oc);
      const EpiSeg sg = pick_seg(ep, s);
      if (ep.cf.state && s == 0)
        gemv_conv_x(ep, sg, m, oc, v, err);
      else
        epi_store_one(ep, sg, m, oc, v, err, qt);
      flag_error(ep.err, err);
    }
  }
}

template <int MB>
static cudaError_t launch_gemv_mb(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int N,
                                  int Kp, const EpiParams& ep, cudaStream_t st) {
  const int ctas = (N + 4 * GV_WC - 1) / (4 * GV_WC);
  const int nslices = (Kp + 511) / 512;
  // K split across warps when there are too few column CTAs to keep every SM streaming
  const int wk = (ctas >= 2 * num_sms() || nslices < 2) ? 1 : (ctas * 2 >= num_sms() || nslices < 4 ? 2 : 4);
  const size_t smem = (size_t)((MB * Kp + 15) & ~15) + (size_t)4 * 4 * GV_WC * MB * 4;
  if (wk == 1) {
    cudaError_t e = ensure_smem_attr((const void*)gemv_i8_kernel<MB, 1>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(M <= 128, gemv_i8_kernel<MB, 1>, dim3((unsigned)ctas), dim3(32 * GV_WC), smem, st, A, lda, Bt,
                      ldb, M, N, Kp, ep);
  }
  if (wk == 2) {
    cudaError_t e = ensure_smem_attr((const void*)gemv_i8_kernel<MB, 2>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(M <= 128, gemv_i8_kernel<MB, 2>, dim3((unsigned)ctas), dim3(64 * GV_WC), smem, st, A, lda, Bt,
                      ldb, M, N, Kp, ep);
  }
  cudaError_t e = ensure_smem_attr((const void*)gemv_i8_kernel<MB, 4>, smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(M <= 128, gemv_i8_kernel<MB, 4>, dim3((unsigned)ctas), dim3(128 * GV_WC), smem, st, A, lda, Bt,
                    ldb, M, N, Kp, ep);
}

static bool gemv_ok(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int Kp) {
  return M >= 1 && M <= 8 && Kp % 16 == 0 && lda % 16 == 0 && ldb % 16 == 0 && (uintptr_t)A % 16 == 0 &&
         (uintptr_t)Bt % 16 == 0 && (size_t)8 * Kp <= 160 * 1024;
}

static cudaError_t launch_gemv(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int N, int Kp,
                               const EpiParams& ep, cudaStream_t st) {
  if (M <= 1) return launch_gemv_mb<1>(A, lda, Bt, ldb, M, N, Kp, ep, st);
  if (M <= 2) return launch_gemv_mb<2>(A, lda, Bt, ldb, M, N, Kp, ep, st);
  if (M <= 4) return launch_gemv_mb<4>(A, lda, Bt, ldb, M, N, Kp, ep, st);
  return launch_gemv_mb<8>(A, lda, Bt, ldb, M, N, Kp, ep, st);
}

// ============================================================ int8 tensor peak probe
// One CTA per SM issues back-to-back M=128 x N=256 x K=32 kind::i8 MMAs on
// resident smem operands (no TMA, no epilogue): the measured int8 dense peak
// used as the roofline denominator for the GEMMs.
__global__ void __launch_bounds__(128, 1) umma_i8_peak_kernel(int iters, int* sink) {
  extern __shared__ uint8_t psm_raw[];
  uint8_t* psm = psm_raw + ((1024u - (smem_u32(psm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t done_bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<int*>(psm)[i] = 0x01010101;
  if (threadIdx.x == 0) {
    mbar_init(&done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_i8(128, 256);
    const uint32_t a0 = smem_u32(psm), b0 = smem_u32(psm + 128 * 128);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) umma_i8(t, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc, 1);
    }
    umma_commit(&done_bar);
    mbar_wait(&done_bar, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(t, r);
    if (threadIdx.x == 0) sink[blockIdx.x] = (int)r[0];
    tmem_dealloc(t, 256);
  }
}

// ============================================================ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static bool make_tmap_i8(CUtensorMap* tm, const void* base, long long rows, long long cols, long long ld_bytes,
                         int box_cols, int box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_3d(CUtensorMap* tm, int elem, const void* base, const long long dims[3],
                  const long long strides[2], const int box[3], int swizzle) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[3] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2]};
  cuuint64_t gstride[2] = {(cuuint64_t)strides[0], (cuuint64_t)strides[1]};
  cuuint32_t bx[3] = {(cuuint32_t)box[0], (cuuint32_t)box[1], (cuuint32_t)box[2]};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(tm, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 3,
                   const_cast<void*>(base), gdim, gstride, bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// Store map for one epilogue segment: f32 as 32x16 boxes (SWIZZLE_64B), int8 as
// 32x32 boxes (SWIZZLE_32B), matching the kernel's staging layouts.
static bool make_tmap_store(CUtensorMap* tm, const EpiSeg& s, long long rows) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  const bool f32 = epi_is_f32(s.kind);
  cuuint64_t gdim[2] = {(cuuint64_t)(s.n1 - s.n0), (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(s.ld * (f32 ? 4 : 1))};
  cuuint32_t box[2] = {f32 ? 16u : 32u, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, s.out, gdim, gstride,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, f32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool tma_storable(const EpiSeg& g) {
  const long long eb = epi_is_f32(g.kind) ? 4 : 1;
  return (g.n0 % 32) == 0 && ((g.ld * eb) % 16) == 0 && ((uintptr_t)g.out % 16) == 0 && g.n1 - g.n0 >= 32;
}

template <int BN, int EPIW, bool TMAOUT, int CG = 1>
static cudaError_t launch_tc(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int N, int Kp,
                             EpiParams ep, cudaStream_t st) {
  using C = TcCfg<BN, EPIW, TMAOUT, CG>;
  CUtensorMap tmA, tmB, tmC, tmC2;
  if (!make_tmap_i8(&tmA, A, M, Kp, lda, TC_BK, TC_BM)) return cudaErrorInvalidValue;
  if (!make_tmap_i8(&tmB, Bt, N, Kp, ldb, TC_BK, BN / CG)) return cudaErrorInvalidValue;
  memset(&tmC, 0, sizeof(tmC));
  memset(&tmC2, 0, sizeof(tmC2));
  if (TMAOUT) {
    if (ep.tma_seg >= 0 && !make_tmap_store(&tmC, ep.seg[ep.tma_seg], M)) return cudaErrorInvalidValue;
    if (ep.tma_seg2 >= 0 && !make_tmap_store(&tmC2, ep.seg[ep.tma_seg2], M)) return cudaErrorInvalidValue;
  } else {
    ep.tma_seg = ep.tma_seg2 = -1;
  }
  {
    cudaError_t e = ensure_smem_attr((const void*)gemm_i8_tc_kernel<BN, EPIW, TMAOUT, CG>, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  const int tiles = ((M + TC_BM * CG - 1) / (TC_BM * CG)) * ((N + BN - 1) / BN) * (ep.splitk > 1 ? ep.splitk : 1);
  const int slots = num_sms() / CG;
  const int grid = (tiles < slots ? tiles : slots) * CG;
  if (CG == 1)
    return launch_pdl(M <= 128, gemm_i8_tc_kernel<BN, EPIW, TMAOUT, CG>, dim3((unsigned)grid), dim3(C::THREADS),
                      (size_t)C::SMEM_BYTES, st, tmA, tmB, tmC, tmC2, M, N, Kp, ep);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_i8_tc_kernel<BN, EPIW, TMAOUT, CG>, tmA, tmB, tmC, tmC2, M, N, Kp, ep);
}
// QMB_GEMM_PAIR=0 disables the CTA-pair kernel (A/B measurements).
static bool gemm_pair_enabled() {
  static const bool v = [] {
    const char* e = getenv("QMB_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}
// The in_proj silu(z) epilogue runs on 12 warps (measured 3% faster than 8;
// 16 exceed the register budget). QMB_SILU12=0 selects 8 (A/B).
static bool silu12_enabled() {
  static const bool v = [] {
    const char* e = getenv("QMB_SILU12");
    return !(e && e[0] == '0');
  }();
  return v;
}
template <int BN, int CG = 1>
static cudaError_t launch_tc_bn(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int N, int Kp,
                                EpiParams ep, cudaStream_t st) {
  bool heavy = false;
  ep.tma_seg = ep.tma_seg2 = -1;
  for (int s = 0; s < ep.nseg; ++s) {
    const EpiSeg& g = ep.seg[s];
    // (silu(z) stays on 8 warps: measured faster than 16, whose register budget spills it)
    if (g.kind == EPI_SOFTPLUS_Q) heavy = true;
    if (!tma_storable(g) || ep.raw_out) continue;
    if (ep.tma_seg < 0)
      ep.tma_seg = s;
    else if (ep.tma_seg2 < 0)
      ep.tma_seg2 = s;
  }
  const bool tma = ep.tma_seg >= 0;
  if (heavy) {
    for (int s = 0; s < ep.nseg; ++s)
      if (ep.seg[s].kind == EPI_F32_SILU) return cudaErrorNotSupported;  // silu is compiled for 8 warps only
    if (tma) return launch_tc<BN, 16, true, CG>(A, lda, Bt, ldb, M, N, Kp, ep, st);
    return launch_tc<BN, 16, false, CG>(A, lda, Bt, ldb, M, N, Kp, ep, st);
  }
  if (CG == 2 && tma && silu12_enabled()) {  // the silu(z) epilogue on 12 warps (3 per TMEM lane quarter)
    for (int s = 0; s < ep.nseg; ++s)
      if (ep.seg[s].kind == EPI_F32_SILU) return launch_tc<BN, 12, true, CG>(A, lda, Bt, ldb, M, N, Kp, ep, st);
  }
  if (tma) return launch_tc<BN, 8, true, CG>(A, lda, Bt, ldb, M, N, Kp, ep, st);
  return launch_tc<BN, 8, false, CG>(A, lda, Bt, ldb, M, N, Kp, ep, st);
}

cudaError_t measure_i8_peak(int iters, double* tops) {
  const int grid = num_sms();
  int* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, grid * sizeof(int));
  if (e != cudaSuccess) return e;
  const int smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(umma_i8_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  umma_i8_peak_kernel<<<grid, 128, smem>>>(iters / 4, sink);  // warm-up
  cudaEventRecord(e0);
  umma_i8_peak_kernel<<<grid, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *tops = 2.0 * 128.0 * 256.0 * 128.0 * (double)iters * grid / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

// GEMM microbenchmark on synthetic operands (tuning tool): mode 0 = f32 out
// (TMA store), 1 = int8 requant out, 2 = f32 out without TMA store, 3 = two
// segments (int8 | f32) like in_proj, 4 = softplus+quant with a dummy table.
__global__ void bench_fill_kernel(int8_t* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = (int8_t)(h >> 24);
  }
}

cudaError_t gemm_bench(int M, int N, int K, int mode, int iters, float* ms_out) {
  // mode + 10: SIMT GEMV path; mode + 20: tensor-core path with split-K scratch (decode-like);
  // mode + 100: L2 flushed (256 MB memset) before every timed launch; mode + 1000: random
  // int8 operands (default: all ones)
  const bool rnd = mode >= 1000;
  mode %= 1000;
  const bool cold = mode >= 100;
  mode %= 100;
  const int path = mode >= 10 && mode < 20 ? 2 : 1;
  const bool use_splitk = mode >= 20;
  mode %= 10;
  void* flush = nullptr;
  if (cold && cudaMalloc(&flush, 256u << 20) != cudaSuccess) return cudaErrorMemoryAllocation;
  int32_t* acc32 = nullptr;
  if (use_splitk && cudaMalloc(&acc32, SPLITK_SCRATCH_INTS * 4) != cudaSuccess) return cudaErrorMemoryAllocation;
  if (acc32) cudaMemset(acc32, 0, SPLITK_SCRATCH_INTS * 4);
  int8_t *A = nullptr, *B = nullptr;
  void* C = nullptr;
  float* tab = nullptr;
  cudaError_t e = cudaMalloc(&A, (size_t)M * K);
  if (e == cudaSuccess) e = cudaMalloc(&B, (size_t)N * K);
  if (e == cudaSuccess) e = cudaMalloc(&C, (size_t)M * N * 4 + 256);
  if (e == cudaSuccess) e = cudaMalloc(&tab, QTAB_FLOATS * 4);
  if (e != cudaSuccess) return e;
  if (rnd) {
    bench_fill_kernel<<<1184, 256>>>(A, (size_t)M * K, 12345u);
    bench_fill_kernel<<<1184, 256>>>(B, (size_t)N * K, 777u);
  } else {
    cudaMemset(A, 1, (size_t)M * K);
    cudaMemset(B, 1, (size_t)N * K);
  }
  float h_tab[QTAB_FLOATS];
  h_tab[0] = -INFINITY;
  for (int k = 1; k < 128; ++k) h_tab[k] = logf(expm1f((k - 0.5f) * 0.01f));  // ~softplus^-1 level bounds
  h_tab[128] = INFINITY;
  h_tab[QTAB_LO] = INFINITY;
  h_tab[QTAB_HI] = -INFINITY;
  cudaMemcpy(tab, h_tab, sizeof(h_tab), cudaMemcpyHostToDevice);
  EpiParams ep{};
  ep.qmax = 127;
  ep.err = nullptr;
  ep.nseg = 1;
  if (mode == 0 || mode == 2) {
    ep.seg[0] = EpiSeg{0, N, EPI_F32, 1e-3f, 1.0f, C, mode == 2 ? (long long)N + 4 : (long long)N, nullptr};
  } else if (mode == 1) {
    ep.seg[0] = EpiSeg{0, N, EPI_QUANT, 1e-3f, 0.05f, C, N, nullptr};
  } else if (mode == 3) {
    ep.nseg = 2;
    ep.seg[0] = EpiSeg{0, N / 2, EPI_QUANT, 1e-3f, 0.05f, C, N / 2, nullptr};
    ep.seg[1] = EpiSeg{N / 2, N, EPI_F32, 1e-3f, 1.0f, static_cast<char*>(C) + (size_t)M * N, N / 2, nullptr};
  } else if (mode == 5) {  // in_proj with the gate's silu(z) in the epilogue
    ep.nseg = 2;
    ep.seg[0] = EpiSeg{0, N / 2, EPI_QUANT, 1e-3f, 0.05f, C, N / 2, nullptr};
    ep.seg[1] = EpiSeg{N / 2, N, EPI_F32_SILU, 1e-3f, 1.0f, static_cast<char*>(C) + (size_t)M * N, N / 2, nullptr};
  } else {
    ep.seg[0] = EpiSeg{0, N, EPI_SOFTPLUS_Q, 1e-3f, 0.01f, C, N, nullptr, tab};
  }
  if (mode == 2) {  // force the non-TMA f32 path: ld not 16B-multiple-aligned is avoided; use a misaligned base
    ep.seg[0].ld = N;
    ep.seg[0].out = static_cast<char*>(C) + 4;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  e = gemm_i8(A, K, B, K, M, N, K, ep, 0, path, acc32);
  float ms = 0;
  if (cold) {
    for (int i = 0; i < iters && e == cudaSuccess; ++i) {
      cudaMemsetAsync(flush, i & 0xff, 256u << 20, 0);
      cudaEventRecord(e0);
      e = gemm_i8(A, K, B, K, M, N, K, ep, 0, path, acc32);
      cudaEventRecord(e1);
      if (e == cudaSuccess) e = cudaEventSynchronize(e1);
      float t = 0;
      cudaEventElapsedTime(&t, e0, e1);
      ms += t;
    }
  } else {
    cudaEventRecord(e0);
    for (int i = 0; i < iters && e == cudaSuccess; ++i) e = gemm_i8(A, K, B, K, M, N, K, ep, 0, path, acc32);
    cudaEventRecord(e1);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  *ms_out = ms / iters;
  if (flush) cudaFree(flush);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  cudaFree(tab);
  if (acc32) cudaFree(acc32);
  return e;
}

// Epilogue of a split-K GEMM: the exact int32 sums in acc32 [M, N] through the
// same per-element float steps as the fused epilogue.
__global__ void epi_apply_kernel(const int32_t* __restrict__ acc, int splitk, int M, int N, EpiParams ep) {
  __shared__ float sQt[QTAB_FLOATS];
  const float* qt = stage_qtab(ep, sQt);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  uint32_t err = 0;
  const long long total = (long long)M * N;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    const long long m = k / N;
    const int n = (int)(k - m * N);
    // int32 sums are exact in any order: 8 independent partial chains keep the loads in flight
    int s8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int sk = 0;
    for (; sk + 8 <= splitk; sk += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) s8[u] += __ldg(acc + (sk + u) * total + k);
    }
    for (; sk < splitk; ++sk) s8[0] += __ldg(acc + sk * total + k);
    const int s = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    int oc;
    const EpiSeg sg = pick_seg(ep, epi_locate(ep, n, &oc));
    epi_store_one(ep, sg, m, oc, s, err, qt);
  }
  flag_error(ep.err, err);
}



// Split-K fix-up for many splits (decode x_proj: 40): 8 threads per output element,
// each summing every 8th split with independent loads (one round trip), then the
// eight partial sums through shared memory -- int32, exact in any order.
constexpr int EPW_T = 256, EPW_G = 8;
__global__ void __launch_bounds__(EPW_T) epi_apply_wide_kernel(const int32_t* __restrict__ acc, int splitk, int M,
                                                               int N, EpiParams ep) {
  __shared__ float sQt[QTAB_FLOATS];
  __shared__ int sPart[EPW_G][EPW_T / EPW_G];
  const float* qt = stage_qtab(ep, sQt);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  uint32_t err = 0;
  const long long total = (long long)M * N;
  const int g = threadIdx.x / (EPW_T / EPW_G), e = threadIdx.x % (EPW_T / EPW_G);
  for (long long base = (long long)blockIdx.x * (EPW_T / EPW_G); base < total;
       base += (long long)gridDim.x * (EPW_T / EPW_G)) {
    const long long k = base + e;
    int s = 0;
    if (k < total) {
      int v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int sk = g + u * EPW_G;
        v[u] = sk < splitk ? __ldg(acc + sk * total + k) : 0;
      }
      for (int sk = g + 8 * EPW_G; sk < splitk; sk += EPW_G) s += __ldg(acc + sk * total + k);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    sPart[g][e] = s;
    __syncthreads();
    if (g == 0 && k < total) {
      int t = 0;
#pragma unroll
      for (int u = 0; u < EPW_G; ++u) t += sPart[u][e];
      const long long m = k / N;
      const int n = (int)(k - m * N);
      int oc;
      const EpiSeg sg = pick_seg(ep, epi_locate(ep, n, &oc));
      epi_store_one(ep, sg, m, oc, t, err, qt);
    }
    __syncthreads();
  }
  flag_error(ep.err, err);
}

// The epilogue of `ep` over exact int32 sums acc [M, N] (row stride N): the
// tensor-parallel finish after an all-reduce of partial products.
cudaError_t epi_apply_i32(const int32_t* acc, int M, int N, const EpiParams& ep_in, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  EpiParams ep = ep_in;
  ep.splitk = 1;
  ep.acc32 = nullptr;
  ep.qtab_bias = QTAB_BIAS;
  ep.one2 = kOne2;
  ep.negz2 = kNegZero2;
  for (int s = 0; s < ep.nseg; ++s) ep.seg[s].out_inv = 1.0f / ep.seg[s].out_div;  // RN f32 reciprocal
  const long long total = (long long)M * N;
  long long blocks = (total + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  return launch_pdl(M <= 128, epi_apply_kernel, dim3((unsigned)blocks), dim3(256), 0, st, acc, 1, M, N, ep);
}

template <int BN>
static cudaError_t launch_tc_choose(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int N,
                                    int Kp, EpiParams ep, cudaStream_t st, int32_t* acc32, int* defer = nullptr) {
  const int tiles = ((M + TC_BM - 1) / TC_BM) * ((N + BN - 1) / BN);
  const int num_k = (Kp + TC_BK - 1) / TC_BK;
  int splitk = 1;
  if (acc32 && tiles * 2 <= num_sms() && num_k > 1) {
    splitk = num_sms() / tiles;
    if (splitk > num_k) splitk = num_k;
    while (splitk > 1 && (long long)splitk * M * N > SPLITK_SCRATCH_INTS) --splitk;  // partials fit the scratch
    const int kper = (num_k + splitk - 1) / splitk;  // no empty splits
    splitk = (num_k + kper - 1) / kper;
  }
  if (splitk <= 1) {
    ep.splitk = 1;
    return launch_tc_bn<BN>(A, lda, Bt, ldb, M, N, Kp, ep, st);
  }
  EpiParams sp = ep;
  sp.splitk = splitk;
  sp.acc32 = acc32;
  sp.tma_seg = sp.tma_seg2 = -1;
  cudaError_t e = launch_tc<BN, 8, false>(A, lda, Bt, ldb, M, N, Kp, sp, st);
  if (e != cudaSuccess) return e;
  if (defer) {  // the caller's next kernel sums the splitk partials and runs the epilogue
    *defer = splitk;
    return cudaSuccess;
  }
  ep.splitk = 1;
  const long long total = (long long)M * N;
  if (splitk >= 2 * EPW_G) {  // many splits: 8 threads per output (one load round trip)
    long long blocks = (total + EPW_T / EPW_G - 1) / (EPW_T / EPW_G);
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    return launch_pdl(true, epi_apply_wide_kernel, dim3((unsigned)blocks), dim3(EPW_T), 0, st,
                      (const int32_t*)acc32, splitk, M, N, ep);
  }
  long long blocks = (total + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  return launch_pdl(true, epi_apply_kernel, dim3((unsigned)blocks), dim3(256), 0, st, (const int32_t*)acc32, splitk, M,
                    N, ep);
}

// Fewest 256 x 256 pair tiles for which the CTA-pair kernel is used (QMB_PAIR_MIN).
// Default 40: below one tile per SM pair the pair tile's doubled operand reuse still
// beats a wave of 128 x 128 single-CTA tiles (2.8B out_proj at M = 1024, 40 pair
// tiles: 36 vs 41 us); at 16-24 pair tiles it loses (130M out_proj 21 vs 18 us).
static int pair_min_tiles() {
  static const int v = [] {
    const char* e = getenv("QMB_PAIR_MIN");
    return e ? atoi(e) : 0;
  }();
  return v > 0 ? v : 40;
}

static bool pair128_enabled() {
  static const bool v = [] {
    const char* e = getenv("QMB_PAIR128");
    return !(e && e[0] == '0');
  }();
  return v;
}

static bool gemm_spin() {
  static const bool v = [] {
    const char* e = getenv("QMB_GEMM_SPIN");
    return e && e[0] == '1';
  }();
  return v;
}

static bool gemv_enabled() {
  static const bool v = [] {
    const char* e = getenv("QMB_GEMV");
    return !(e && !strcmp(e, "0"));
  }();
  return v;
}

bool gemv_selected(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int Kp) {
  return gemv_enabled() && gemv_ok(A, lda, Bt, ldb, M, Kp);
}

cudaError_t gemm_i8(const int8_t* A, long long lda, const int8_t* Bt, long long ldb, int M, int N, int Kp,
                    const EpiParams& ep_in, cudaStream_t st, int force_path, int32_t* acc32, int* defer) {
  if (defer) *defer = 0;
  if (M <= 0 || N <= 0) return cudaSuccess;
  EpiParams ep = ep_in;
  ep.splitk = 1;
  ep.acc32 = nullptr;
  ep.spin = (M <= TC_BM && gemm_spin()) ? 1 : 0;  // QMB_GEMM_SPIN=1: spinning pipeline waits for decode GEMMs
  ep.small_acc = (long long)Kp * 128 * 128 < (1LL << 22) ? 1 : 0;
  ep.qtab_bias = QTAB_BIAS;
  ep.one2 = kOne2;
  ep.negz2 = kNegZero2;
  for (int s = 0; s < ep.nseg; ++s) ep.seg[s].out_inv = 1.0f / ep.seg[s].out_div;  // RN f32 reciprocal
  const bool tc_ok = (lda % 16 == 0) && (ldb % 16 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)Bt % 16 == 0) &&
                     Kp > 0;
  int path = force_path;
  // decode-size M: the streaming GEMV (path 3); QMB_GEMV=0 keeps the tensor-core split-K path
  if (path == 0 && gemv_enabled() && gemv_ok(A, lda, Bt, ldb, M, Kp)) path = 3;
  if (ep.cf.state && path != 3) return cudaErrorInvalidValue;  // (only the GEMV fuses the conv step)
  if (path == 3) {
    if (!gemv_ok(A, lda, Bt, ldb, M, Kp)) return cudaErrorInvalidValue;
    return launch_gemv(A, lda, Bt, ldb, M, N, Kp, ep, st);
  }
  if (path == 0) path = (tc_ok && (M > 16 || acc32)) ? 1 : 2;
  if (path == 1 && !tc_ok) return cudaErrorInvalidValue;
  if (path == 1) {
    // split-K when there are too few output tiles to keep the SMs streaming (decode;
    // x_proj / out_proj of a short prefill), as far as the partials fit the scratch
    if ((long long)M * N * 2 > SPLITK_SCRATCH_INTS) acc32 = nullptr;
    // skinny M: one wave of 96-column tiles beats two waves of 64-column ones
    if (M <= TC_BM && N > 192 && (N + 63) / 64 > num_sms() && (N + 95) / 96 <= num_sms())
      return launch_tc_choose<96>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
    // Column tile: the largest BN that still gives >= 1 wave, else the smallest.
    if (N <= 32) return launch_tc_choose<32>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
    if (N <= 64) return launch_tc_choose<64>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
    if (N <= 128) return launch_tc_choose<128>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
    if (N <= 192) return launch_tc_choose<192>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
    const long long m_tiles = (M + TC_BM - 1) / TC_BM;
    // CTA pairs (256 x 256 tiles) once there are enough pair tiles for every SM pair
    if (gemm_pair_enabled() && ((M + 255) / 256) * ((N + 255) / 256) >= pair_min_tiles()) {
      // few waves of 256 x 256 pair tiles (short prefills) of an epilogue-bound GEMM (dt_proj's
      // softplus, K = dt_rank): 256 x 128 tiles when they fill the last wave clearly better.
      // B = 1 / 2 x T = 1024: dt_proj 23.5 -> 21.3 / 29.7 -> 27.2 us; in_proj and out_proj lose
      // (46 -> 53 us, 50 -> 54 us: half-width tiles cost more than the wave balance gains),
      // so they keep 256 x 256 (profiles/r02/pair128_ab.log; QMB_PAIR128=0: off)
      bool heavy = false;
      for (int s = 0; s < ep.nseg; ++s) heavy |= ep.seg[s].kind == EPI_SOFTPLUS_Q;
      const long long slots = num_sms() / 2;
      auto wave_eff = [&](long long t) { return (double)t / (double)(((t + slots - 1) / slots) * slots); };
      const long long t256 = ((M + 255) / 256) * ((N + 255) / 256), t128 = ((M + 255) / 256) * ((N + 127) / 128);
      if (heavy && pair128_enabled() && wave_eff(t128) > wave_eff(t256) + 0.1)
        return launch_tc_bn<128, 2>(A, lda, Bt, ldb, M, N, Kp, ep, st);
      return launch_tc_bn<256, 2>(A, lda, Bt, ldb, M, N, Kp, ep, st);
    }
    if (m_tiles * ((N + 255) / 256) >= num_sms())
      return launch_tc_choose<256>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
    if (m_tiles * ((N + 127) / 128) >= num_sms())
      return launch_tc_choose<128>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
    return launch_tc_choose<64>(A, lda, Bt, ldb, M, N, Kp, ep, st, acc32, defer);
  }
  const int vec = ((lda % 16) == 0 && (ldb % 16) == 0 && ((uintptr_t)A % 16) == 0 && ((uintptr_t)Bt % 16) == 0);
  constexpr int MB = 8;
  dim3 grid((N + 7) / 8, (M + MB - 1) / MB);
  gemm_i8_simt_kernel<MB><<<grid, 256, 0, st>>>(A, lda, Bt, ldb, M, N, Kp, ep, vec);
  return cudaGetLastError();
}

}  // namespace qmb
