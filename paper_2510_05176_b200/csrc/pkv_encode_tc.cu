// K1-TC: persistent fp16 prefill encoder (d = 128, G = 128, P <= 32, 2/4-bit).
//
// Same contract as encode_span_kernel (pkv_encode.cu) -- the reference's
// _commit_span (engine.py:201-252) with match_many (patterns.py:206-221),
// decide (gate.py:174-188), quantize_group and pack_codes (quant.py:70-146) --
// and bit-identical outputs, re-organised so that almost every instruction
// touches data in registers:
//
//  * one persistent CTA per SM, 16 warps: warps 0-7 run the K pipeline and
//    warps 8-15 the V pipeline over the same (unit, span) work items, each with
//    its own TMA stream (cp.async.bulk.tensor.3d, 128-byte swizzle) of 32 KB
//    span tiles, so one side's loads and latencies hide under the other's math;
//  * nearest pattern: one tcgen05.mma chain per span-side computes x . m'_p
//    (m' = channel-centered pattern split hi + lo in fp16, fp32 accumulator in
//    TMEM).  The L2-nearest pattern is the guess g; the exact fp32 d_mm to g
//    comes out of the residual pass; every other pattern is pruned by two exact
//    lower bounds on d_mm -- Popoviciu (osc(v)^2 >= 4 Var(v), Var from the GEMM)
//    and a two-channel probe |v_a - v_b| <= osc(v) -- with rigorous fp error
//    margins.  Survivors (rare) get the full fp32 distance, near ties the
//    reference's fp64 argmin (lowest index on ties);
//  * residuals, extrema and codes in mma-fragment register layout (ldmatrix from
//    the swizzled tile); per-token (V) reductions need 2 shuffles; K's
//    per-channel groups run on a residual tile in a transposed warp layout; V
//    codes move to the V^T fragment layout with movmatrix;
//  * exact fp64 group extrema from fp32 "keys" (value with the element index in
//    the low mantissa bits) plus a count of the elements inside the fp32 error
//    window; codes by a magic-number round z = fma(v - lo, 1/s, 1.5*2^23) whose
//    distance to the rounding boundary is checked per element pair (fp64
//    recompute of the reference sequence inside the guard band).
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "pkv_common.cuh"
#include "pkv_sm100.cuh"

namespace pkv {
namespace fe {

using namespace sm100;

constexpr int NTHR = 512;   // 16 warps: 0-7 K pipeline, 8-15 V pipeline
constexpr int GT = 256;     // threads per side group
constexpr int PM = 32;      // max patterns per side on this path
constexpr int MR = 144;     // permuted fp32 pattern row: 4 lane segments of 36 floats (bank skew)
constexpr int RS = 136;     // K residual tile row stride (floats): conflict-free float2 columns
constexpr float MAGIC = 12582912.f;  // 1.5 * 2^23
#define FE_INF __int_as_float(0x7f800000)
#define FE_NAN __int_as_float(0x7fc00000)
constexpr float TWO_M13 = 1.220703125e-04f;
constexpr float TWO_M15 = 3.0517578125e-05f;
constexpr float TWO_M17 = 7.62939453125e-06f;
constexpr float TWO_M22 = 2.384185791015625e-07f;

// ---- shared memory map (bytes from a 1024-aligned base) ---------------------------------
constexpr int SZ_X = 32768;                       // one side's span tile [2 halves][128 rows][128 B]
constexpr int OFF_X = 0;                          // X[side]
constexpr int SZ_B = 16384;                       // centered hi [2][32][128 B] then lo [2][32][128 B]
constexpr int OFF_B = OFF_X + 2 * SZ_X;
constexpr int SZ_M = PM * MR * 4;                 // permuted fp32 table
constexpr int OFF_M = OFF_B + 2 * SZ_B;
constexpr int OFF_R = OFF_M + 2 * SZ_M;           // K residual tile [128][RS] f32
constexpr int OFF_KW = OFF_R + 128 * RS * 4;      // K code words [8 tiles][32 lanes][<= 8]
constexpr int OFF_TOK = OFF_KW + 8 * 32 * 8 * 4;  // per side: guess, cand, dg, xabs, fidx, ed
constexpr int SZ_TOK = 6 * 128 * 4;
constexpr int OFF_PAT = OFF_TOK + 2 * SZ_TOK;     // per side: bb, mn, pm, mabsr [4][32], mabsc[128], flags[4]
constexpr int SZ_PAT = (4 * 32 + 128 + 4) * 4;
constexpr int OFF_KQ = OFF_PAT + 2 * SZ_PAT;     // K per-channel exact params: lo64[128], scale64[128]
constexpr int OFF_BAR = OFF_KQ + 2 * 128 * 8;     // xfull[2], mma[2] (8 B each) + tmem addr
constexpr int SMEM_BYTES = OFF_BAR + 64 + 1024;   // + alignment slack

struct Tok {
  int* guess; uint32_t* cand; float* dg; float* xabs; int* fidx; float* ed;
  __device__ Tok(unsigned char* sb, int side) {
    unsigned char* p = sb + OFF_TOK + side * SZ_TOK;
    guess = reinterpret_cast<int*>(p);
    cand = reinterpret_cast<uint32_t*>(p + 512);
    dg = reinterpret_cast<float*>(p + 1024);
    xabs = reinterpret_cast<float*>(p + 1536);
    fidx = reinterpret_cast<int*>(p + 2048);
    ed = reinterpret_cast<float*>(p + 2560);
  }
};
struct Pat {
  float* bb;     // ||m'_p||^2 (+inf for p >= P)
  float* mn;     // ||m'_p||
  float* pm;     // m_a - m_b at the probe channels
  float* mabsr;  // max_c |m_pc|
  float* mabsc;  // max_p |m_pc| (K)
  int* flags;    // [0] P, [1] L2 bound disabled, [2] probe a, [3] probe b
  __device__ Pat(unsigned char* sb, int side) {
    float* p = reinterpret_cast<float*>(sb + OFF_PAT + side * SZ_PAT);
    bb = p; mn = p + 32; pm = p + 64; mabsr = p + 96; mabsc = p + 128;
    flags = reinterpret_cast<int*>(p + 256);
  }
};

struct Args {
  DevCache c;
  int nb;            // blocks in this launch (first_block .. first_block + nb)
  int first_block;
  const __half* src[2];  // K, V inputs [U][rows][128]
  int64_t unit_stride;   // elements between units
  int64_t nitems;        // U * nb
  double yq;             // RN(1 / qmax)
};

__device__ __forceinline__ void bar_group(int g) { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(GT) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// 32 lanes x 8 columns of 32-bit: thread i gets lane (base + i), 8 consecutive columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ float h2f_lo(uint32_t v) { return __half2float(__ushort_as_half((unsigned short)(v & 0xffffu))); }
__device__ __forceinline__ float h2f_hi(uint32_t v) { return __half2float(__ushort_as_half((unsigned short)(v >> 16))); }
// value with its low mantissa bits replaced by an element index
__device__ __forceinline__ float fkey(float v, uint32_t idx, uint32_t mask) {
  return __uint_as_float((__float_as_uint(v) & mask) | idx);
}
__device__ __forceinline__ double warp_sum_dd(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// x tile element (fp16) at (row, channel) of a 128B-swizzled [2][128][64] tile
__device__ __forceinline__ float xt_at(const unsigned char* xt, int row, int ch) {
  const int h = ch >> 6, c = ch & 63;
  const unsigned char* p = xt + h * 16384 + row * 128 + ((((c >> 3) ^ (row & 7)) << 4) | ((c & 7) << 1));
  return __half2float(*reinterpret_cast<const __half*>(p));
}
// position of channel c in a permuted fp32 pattern row: lane q's 32 channels
// (16j + 8hc + 2q + e) are contiguous at q*36 + 4j + 2hc + e
__device__ __forceinline__ int mpos(int c) {
  const int j = c >> 4, hc = (c >> 3) & 1, q = (c >> 1) & 3, e = c & 1;
  return q * 36 + 4 * j + 2 * hc + e;
}

// exact division by the integer qmax (Markstein: y = RN(1/b), q0 = RN(a y),
// r = a - b q0 exact by FMA, RN(q0 + r y) = RN(a / b) for normal operands)
__device__ __forceinline__ double div_qmax(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
}

struct GroupQ {   // one quantization group: exact params + fp32 fast-path constants
  double lo, scale;
  float lo32, inv, hg;  // hg = 1/2 - guard
};
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// R >= max |r| over the group, M >= max |m| over the pattern entries it used
__device__ __forceinline__ GroupQ make_group(double lo, double hi, int qmax, double yq, float R, float M) {
  GroupQ g;
  g.lo = lo;
  g.scale = div_qmax(__dsub_rn(hi, lo), (double)qmax, yq);
  g.lo32 = (float)lo;
  g.inv = 0.f;
  if (g.scale == 0.0) { g.hg = 0.5f; return g; }              // all codes 0 (quant.py:105-106)
  if (!(g.scale > 1e-30)) { g.hg = -1.f; return g; }          // degenerate: every code exact
  g.inv = rcp_approx((float)g.scale);
  const float span = (float)(hi - lo);
  // |rl*inv - (v64 - lo64)/scale| <= 2^-24 (2R + M + span)/scale + 2^-22.4 qmax + 2^-25, x2 margin
  const float guard = 1.1920928955078125e-07f * ((2.f * R + M + span) * g.inv + 2.f * (float)qmax + 2.f);
  g.hg = 0.5f - guard;
  return g;
}
// fast code of one element: z holds MAGIC + code in its low byte; bad when the fp32
// quotient lies inside the guard band of a rounding boundary
__device__ __forceinline__ float zcode(float r, float lo32, float inv, float hg, bool& bad) {
  const float rl = __fsub_rn(r, lo32);
  const float z = __fmaf_rn(rl, inv, MAGIC);
  const float k = __fsub_rn(z, MAGIC);
  const float d = __fmaf_rn(rl, inv, -k);
  bad |= fabsf(d) > hg;
  return z;
}
__device__ __forceinline__ uint32_t zpair(float z0, float z1) {
  return __byte_perm(__float_as_uint(z0), __float_as_uint(z1), 0x5410);
}

// ---- rare paths: kept out of line so the hot loop stays in the instruction cache --------
// reference code sequence quant.py:103-109 in IEEE fp64 for the input element *xp
// (minus pattern value *mp unless RAW)
__device__ __noinline__ uint32_t exact_code_at(const __half* xp, const double* mp, double lo, double scale, int qmax) {
  if (scale == 0.0) return 0u;
  double v = (double)__half2float(*xp);
  if (mp) v = __dsub_rn(v, *mp);
  const double t = __dadd_rn(__ddiv_rn(__dsub_rn(v, lo), scale), 0.5);
  const int c = (int)floor(t);
  return (uint32_t)(c < 0 ? 0 : (c > qmax ? qmax : c));
}
__device__ __noinline__ bool gate_div_le(double flat, double raw, double thr) { return __ddiv_rn(flat, raw) <= thr; }
// exact fl(flat / raw) <= thr (gate.py:180-188); a division only within 2^-50 of the threshold
__device__ __forceinline__ bool gate_le(double flat, double raw, double thr) {
  const double t1 = __fma_rn(-thr, raw, flat);  // sign of flat - thr*raw, exact
  if (t1 <= 0.0) return true;
  if (t1 > flat * 8.881784197001252e-16) return false;
  return gate_div_le(flat, raw, thr);
}

// fp64 re-match of token row t over the whole table (patterns.py:217-221): lane q of the
// row's quad takes patterns p = q (mod 4); lowest index on ties.  Whole warp calls.
__device__ __noinline__ int refine64(const unsigned char* X, int t, const double* p64, int P, int q) {
  double bv = __longlong_as_double(0x7ff0000000000000LL);
  int bi = 0x7fffffff;
  for (int p = q; p < P; p += 4) {
    const double* m = p64 + (int64_t)p * 128;
    double mx = -bv, mn = bv;
#pragma unroll 2
    for (int ch = 0; ch < 128; ++ch) {
      const double d = __dsub_rn((double)xt_at(X, t, ch), m[ch]);
      mx = fmax(mx, d);
      mn = fmin(mn, d);
    }
    const double v = __dsub_rn(mx, mn);
    if (v < bv) { bv = v; bi = p; }
  }
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    if (v2 < bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
  }
  return bi;
}
// lane-local keyed extrema of the residual of rows g (+8) against pattern rows p0, p1
// (same arithmetic and keys as resid_pass)
__device__ __noinline__ void cand_stats(const unsigned char* X, const float* M, int gw, int lane, int p0, int p1,
                                        float* out) {
  const int g = lane >> 2, q = lane & 3;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int t = 16 * gw + g + 8 * h;
    const float* mr = M + (h ? p1 : p0) * MR + q * 36;
    float mx = -FE_INF, mn = FE_INF;
#pragma unroll 4
    for (int e = 0; e < 32; ++e) {
      const int j = e >> 2, k = e & 3;
      const int ch = 16 * j + 8 * (k >> 1) + 2 * q + (k & 1);
      const float key = fkey(__fsub_rn(xt_at(X, t, ch), mr[e]), (uint32_t)e, 0xffffffe0u);
      mx = fmaxf(mx, key);
      mn = fminf(mn, key);
    }
    out[2 * h] = mx;
    out[2 * h + 1] = mn;
  }
}
// V row: lane-local fp64 extrema over the elements whose key lies in the error window
__device__ __noinline__ void v_slow_extrema(const __half* xrow, const double* mrow, const float* mr32, int q,
                                            float hib, float lob, double* omx, double* omn) {
  double dmx = -__longlong_as_double(0x7ff0000000000000LL), dmn = -dmx;
  for (int e = 0; e < 32; ++e) {
    const int j = e >> 2, k = e & 3;
    const int ch = 16 * j + 8 * (k >> 1) + 2 * q + (k & 1);
    const float xv = __half2float(xrow[ch]);
    const float key = fkey(__fsub_rn(xv, mr32[e]), (uint32_t)e, 0xffffffe0u);
    if (key >= hib || key <= lob) {
      const double v64 = __dsub_rn((double)xv, mrow[ch]);
      if (key >= hib) dmx = fmax(dmx, v64);
      if (key <= lob) dmn = fmin(dmn, v64);
    }
  }
  *omx = dmx;
  *omn = dmn;
}
// K channel: lane-local fp64 extrema over its 16 tokens whose key lies in the window
__device__ __noinline__ void k_slow_extrema(const float* R, const int* fidx, const __half* xsrc, const double* p64,
                                            int ch, int g, float hib, float lob, double* omx, double* omn) {
  double dmx = -__longlong_as_double(0x7ff0000000000000LL), dmn = -dmx;
  for (int e = 0; e < 16; ++e) {
    const int tt = e >> 1, h = e & 1, t = 16 * tt + 8 * h + g;
    const float key = fkey(R[t * RS + ch], (uint32_t)e, 0xfffffff0u);
    if (key >= hib || key <= lob) {
      const double v64 = __dsub_rn((double)__half2float(xsrc[(int64_t)t * 128 + ch]), p64[(int64_t)fidx[t] * 128 + ch]);
      if (key >= hib) dmx = fmax(dmx, v64);
      if (key <= lob) dmn = fmin(dmn, v64);
    }
  }
  *omx = dmx;
  *omn = dmn;
}

// ---------------------------------------------------------------------------------------
// pattern staging for (unit u, side): permuted fp32 table, centered hi/lo B operand,
// per-pattern scalars.  Called by the side group between group barriers.
// ---------------------------------------------------------------------------------------
__device__ void stage_patterns(const Args& A, int side, int u, unsigned char* sb, int gtid) {
  const DevCache& c = A.c;
  const int P = side == 0 ? c.nk[u] : c.nv[u];
  const float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * c.Dp;
  const double* p64 = (side == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * 128;
  float* M = reinterpret_cast<float*>(sb + OFF_M + side * SZ_M);
  unsigned char* B = sb + OFF_B + side * SZ_B;
  Pat pt(sb, side);
  const int pa = c.probe[((int64_t)u * 2 + side) * 16 + 0], pbc = c.probe[((int64_t)u * 2 + side) * 16 + 1];
  if (gtid == 0) pt.flags[1] = 0;
  for (int i = gtid; i < PM * 128; i += GT) {
    const int p = i >> 7, ch = i & 127;
    M[p * MR + mpos(ch)] = p < P ? p32[(int64_t)p * c.Dp + ch] : 0.f;
  }
  if (side == 0 && gtid < 128) {
    float m = 0.f;
    for (int p = 0; p < P; ++p) m = fmaxf(m, fabsf(p32[(int64_t)p * c.Dp + gtid]));
    pt.mabsc[gtid] = m;
  }
  bar_group(side);  // flags[1] reset visible
  // one warp per pattern (8 warps x 4): mean in fp64, centered hi/lo fp16 rows
  const int w = gtid >> 5, lane = gtid & 31;
  for (int p = w; p < PM; p += 8) {
    double mv[4], s = 0.0;
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mv[i] = p < P ? p64[(int64_t)p * 128 + lane + 32 * i] : 0.0;
      s += mv[i];
      amax = fmaxf(amax, fabsf((float)mv[i]));
    }
    s = warp_sum_dd(s);
    const double mean = s / 128.0;
    double ss = 0.0;
    int bad = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int ch = lane + 32 * i;
      const double mc = p < P ? mv[i] - mean : 0.0;
      if (fabs(mc) > 60000.0) bad = 1;
      ss = fma(mc, mc, ss);
      const __half hi = __double2half(mc);
      const __half lo = __double2half(mc - (double)__half2float(hi));
      const int h = ch >> 6, cc = ch & 63;
      const int off = h * 4096 + p * 128 + ((((cc >> 3) ^ (p & 7)) << 4) | ((cc & 7) << 1));
      *reinterpret_cast<__half*>(B + off) = hi;
      *reinterpret_cast<__half*>(B + 8192 + off) = lo;
    }
    ss = warp_sum_dd(ss);
    amax = warp_max_f(amax);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&pt.flags[1], 1);
    if (lane == 0) {
      pt.bb[p] = p < P ? (float)ss : FE_INF;
      pt.mn[p] = p < P ? (float)sqrt(ss) : 0.f;
      pt.pm[p] = p < P ? (float)__dsub_rn(p64[(int64_t)p * 128 + pa], p64[(int64_t)p * 128 + pbc]) : 0.f;
      pt.mabsr[p] = amax;
    }
  }
  if (gtid == 0) {
    pt.flags[0] = P;
    pt.flags[2] = pa;
    pt.flags[3] = pbc;
  }
  fence_proxy_async();  // generic-proxy writes of B -> tensor-core reads
}

// ---------------------------------------------------------------------------------------
// residual pass of one warp over its 16 tokens (rows g, g+8) against pattern rows
// idx[0], idx[1]: r = x - m in fragment layout, keyed extrema, x extrema
// ---------------------------------------------------------------------------------------
struct RowStats {
  float kmx[2], kmn[2];   // lane-local keyed extrema of r (5-bit element index)
  float xmx[2], xmn[2];   // lane-local extrema of x
};
__device__ __forceinline__ void resid_pass(const unsigned char* X, const float* M, int gw, int lane, const int idx[2],
                                           float (&r)[2][8][4], RowStats& st) {
  const int q = lane & 3;
  const uint32_t xbase = smem_u32(X);
  const int lrow = 16 * gw + (lane & 7) + 8 * ((lane >> 3) & 1);
  const int lchk = lane >> 4;
  const float* m0p = M + idx[0] * MR + q * 36;
  const float* m1p = M + idx[1] * MR + q * 36;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    st.kmx[h] = -FE_INF; st.kmn[h] = FE_INF; st.xmx[h] = -FE_INF; st.xmn[h] = FE_INF;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t a0, a1, a2, a3;
    const uint32_t addr = xbase + (j >> 2) * 16384 + lrow * 128 + ((((2 * (j & 3) + lchk) ^ (lrow & 7))) << 4);
    ldsm_x4(addr, a0, a1, a2, a3);
    const float4 m0 = *reinterpret_cast<const float4*>(m0p + 4 * j);
    const float4 m1 = *reinterpret_cast<const float4*>(m1p + 4 * j);
    const float x0[4] = {h2f_lo(a0), h2f_hi(a0), h2f_lo(a2), h2f_hi(a2)};
    const float x1[4] = {h2f_lo(a1), h2f_hi(a1), h2f_lo(a3), h2f_hi(a3)};
    r[0][j][0] = __fsub_rn(x0[0], m0.x); r[0][j][1] = __fsub_rn(x0[1], m0.y);
    r[0][j][2] = __fsub_rn(x0[2], m0.z); r[0][j][3] = __fsub_rn(x0[3], m0.w);
    r[1][j][0] = __fsub_rn(x1[0], m1.x); r[1][j][1] = __fsub_rn(x1[1], m1.y);
    r[1][j][2] = __fsub_rn(x1[2], m1.z); r[1][j][3] = __fsub_rn(x1[3], m1.w);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float* xx = h ? x1 : x0;
      const float k0 = fkey(r[h][j][0], 4 * j + 0, 0xffffffe0u), k1 = fkey(r[h][j][1], 4 * j + 1, 0xffffffe0u);
      const float k2 = fkey(r[h][j][2], 4 * j + 2, 0xffffffe0u), k3 = fkey(r[h][j][3], 4 * j + 3, 0xffffffe0u);
      st.kmx[h] = fmax3(st.kmx[h], k0, k1); st.kmx[h] = fmax3(st.kmx[h], k2, k3);
      st.kmn[h] = fmin3(st.kmn[h], k0, k1); st.kmn[h] = fmin3(st.kmn[h], k2, k3);
      st.xmx[h] = fmax3(st.xmx[h], xx[0], xx[1]); st.xmx[h] = fmax3(st.xmx[h], xx[2], xx[3]);
      st.xmn[h] = fmin3(st.xmn[h], xx[0], xx[1]); st.xmn[h] = fmin3(st.xmn[h], xx[2], xx[3]);
    }
  }
}
__device__ __forceinline__ float qmax4(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float qmin4(float v) {
  v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fminf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
// bound on |d32 - d64| for a distance taken from keyed fp32 extrema (K1-TC):
// key error 2^-18 |r|, fp32 residual error 2^-24 (|r| + 2|m|), subtraction 2^-24 |d|
__device__ __forceinline__ float derr(float kmx, float kmn, float M) {
  return 7.62939453125e-06f * (fabsf(kmx) + fabsf(kmn)) + 4.76837158203125e-07f * M;
}

// ---------------------------------------------------------------------------------------
// one side's pipeline (SIDE 0 = K on warps 0-7, 1 = V on warps 8-15)
// ---------------------------------------------------------------------------------------
template <int BITS, int SIDE>
__device__ __forceinline__ void run_side(const Args& A, unsigned char* sb, const CUtensorMap* tm, uint32_t tmem_base,
                                         int64_t i0, int64_t i1) {
  const DevCache& c = A.c;
  constexpr int QMAX = (1 << BITS) - 1;
  constexpr int HS = 8 / BITS;
  constexpr int WL = 128 * BITS / 64;  // words per lane per tile
  const int gtid = threadIdx.x & (GT - 1), gw = gtid >> 5, lane = gtid & 31, g = lane >> 2, q = lane & 3;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + OFF_BAR);
  uint64_t* xfull = bars + SIDE;
  uint64_t* mmab = bars + 2 + SIDE;
  unsigned char* X = sb + OFF_X + SIDE * SZ_X;
  unsigned char* B = sb + OFF_B + SIDE * SZ_B;
  const float* M = reinterpret_cast<const float*>(sb + OFF_M + SIDE * SZ_M);
  Tok tk(sb, SIDE);
  Pat pt(sb, SIDE);
  const __half* src = A.src[SIDE];
  unsigned* stats = c.stats;

  auto issue = [&](int64_t item) {
    const int uu = (int)(item / A.nb);
    const int bb = A.first_block + (int)(item % A.nb);
    const int row = (int)(c.blk_start[bb] - c.blk_start[A.first_block]);
    fence_proxy_async();
    mbar_arrive_expect_tx(xfull, 2 * 16384);
    tma_load_3d(X, tm, xfull, 0, row, uu);
    tma_load_3d(X + 16384, tm, xfull, 64, row, uu);
  };
  if (gtid == 0 && i0 < i1) issue(i0);

  int cur_u = -1;
  uint32_t k = 0;
  for (int64_t it = i0; it < i1; ++it, ++k) {
    const int u = (int)(it / A.nb);
    const int b = A.first_block + (int)(it % A.nb);
    const int L = c.blk_len[b];
    const int64_t start = c.blk_start[b];
    const int64_t xrow0 = start - c.blk_start[A.first_block];  // source row of token 0
    const __half* xsrc = src + (int64_t)u * A.unit_stride + xrow0 * 128;
    const double* p64 = (SIDE == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * 128;
    if (u != cur_u) {
      bar_group(SIDE);
      stage_patterns(A, SIDE, u, sb, gtid);
      bar_group(SIDE);
      cur_u = u;
    }
    const int P = pt.flags[0];
    const uint32_t ph = k & 1;
    const uint32_t tcol = tmem_base + SIDE * 64 + ph * 32;
    mbar_wait(xfull, ph);
    if (gtid == 0) {
      tc_fence_after();
      const uint32_t idesc = idesc_f16_f32(128, 32);
      const uint64_t da0 = smem_desc_k_sw128(X), da1 = smem_desc_k_sw128(X + 16384);
      const uint64_t dh0 = smem_desc_k_sw128(B), dh1 = smem_desc_k_sw128(B + 4096);
      const uint64_t dl0 = smem_desc_k_sw128(B + 8192), dl1 = smem_desc_k_sw128(B + 12288);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // 8 x K=16 over d = 128: D += x.hi, D += x.lo
        const uint64_t o = 2 * (kk & 3);  // +32 B per K step inside the 128-B swizzle atom
        mma_f16_ss(tcol, (kk < 4 ? da0 : da1) + o, (kk < 4 ? dh0 : dh1) + o, idesc, kk > 0 ? 1u : 0u);
        mma_f16_ss(tcol, (kk < 4 ? da0 : da1) + o, (kk < 4 ? dl0 : dl1) + o, idesc, 1u);
      }
      mma_commit(mmab);
    }

    // ---- A. guess = argmin_p ||m'_p||^2 - 2 x.m'_p (thread per token, warps 0-3) ----------
    const int tt_ = 32 * gw + lane;  // token of this thread in stages A/C
    int guess = 0;
    float Cg = 0.f, px = 0.f;
    if (gw < 4) {
      mbar_wait(mmab, ph);
      tc_fence_after();
      float best = FE_INF;
#pragma unroll
      for (int p0 = 0; p0 < 32; p0 += 16) {
        uint32_t v[8], w[8];
        tmem_ld8(tcol + p0 + ((uint32_t)(32 * gw) << 16), v);
        tmem_ld8(tcol + p0 + 8 + ((uint32_t)(32 * gw) << 16), w);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          best = fminf(best, fkey(__fmaf_rn(-2.f, __uint_as_float(v[i]), pt.bb[p0 + i]), p0 + i, 0xffffffe0u));
          best = fminf(best, fkey(__fmaf_rn(-2.f, __uint_as_float(w[i]), pt.bb[p0 + 8 + i]), p0 + 8 + i, 0xffffffe0u));
        }
      }
      guess = (int)(__float_as_uint(best) & 31u);
      if (guess >= P) guess = 0;
      Cg = best;
      px = __fsub_rn(xt_at(X, tt_, pt.flags[2]), xt_at(X, tt_, pt.flags[3]));
      tk.guess[tt_] = guess;
      tc_fence_before();
    }
    bar_group(SIDE);

    // ---- B. residual pass against the guess (all 8 warps, 16 tokens each) -------------
    const int t0 = 16 * gw + g;
    int idx[2] = {tk.guess[t0], tk.guess[t0 + 8]};
    float r[2][8][4];
    RowStats st;
    resid_pass(X, M, gw, lane, idx, r, st);
    float kmx[2], kmn[2], xmx[2], xmn[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      kmx[h] = qmax4(st.kmx[h]); kmn[h] = qmin4(st.kmn[h]);
      xmx[h] = qmax4(st.xmx[h]); xmn[h] = qmin4(st.xmn[h]);
      if (q == 0) {
        tk.dg[t0 + 8 * h] = __fsub_rn(kmx[h], kmn[h]);
        tk.ed[t0 + 8 * h] = derr(kmx[h], kmn[h], pt.mabsr[idx[h]]);
        tk.xabs[t0 + 8 * h] = fmaxf(fabsf(xmx[h]), fabsf(xmn[h]));
      }
    }
    bar_group(SIDE);

    // ---- C. prune every other pattern by exact lower bounds (thread per token) ----------
    if (gw < 4) {
      tc_fence_after();
      const float dg = tk.dg[tt_], xa = tk.xabs[tt_];
      const float T2 = tk.ed[tt_];                  // >= |dg - d64(guess)|
      const float dhi = __fadd_rn(dg, T2) * 1.0000002f;
      const float dlo = fmaxf(__fsub_rn(dg, T2), 0.f) * 0.9999998f;
      // Popoviciu: osc^2 >= 4 C / d; C_q >= C'_q - C'_g + C_g, C_g >= osc_g^2 / 2
      const float theta = __fmaf_rn(32.f * dhi, dhi, -0.5f * dlo * dlo) * 1.000001f;
      const float kap = TWO_M13 * 11.3137085f * xa;  // 2 x (tensor-core + split error) / ||m'||, ||x|| <= sqrt(d) |x|max
      const float rhs = theta + Cg + kap * pt.mn[guess] + TWO_M17 * fabsf(Cg);
      const bool nol2 = pt.flags[1] != 0;
      const float pmx = SIDE == 0 ? c.kpmax[u] : c.vpmax[u];
      const float pb = __fadd_rn(dhi, 4.76837158203125e-07f * (xa + pmx));  // probe: 2^-21 (|x| + |m|) rounding
      uint32_t mask = 0;
#pragma unroll 1
      for (int p0 = 0; p0 < 32; p0 += 8) {
        uint32_t v[8];
        tmem_ld8(tcol + p0 + ((uint32_t)(32 * gw) << 16), v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int p = p0 + i;
          const float bbp = pt.bb[p];
          const float cp = __fmaf_rn(-2.f, __uint_as_float(v[i]), bbp);
          const float lhs = __fmaf_rn(-TWO_M22, bbp, __fmaf_rn(-kap, pt.mn[p], __fmaf_rn(-TWO_M17, fabsf(cp), cp)));
          const bool l2ok = nol2 || !(lhs > rhs);
          const bool prok = fabsf(__fsub_rn(px, pt.pm[p])) <= pb;
          mask |= (uint32_t)(l2ok && prok && p < P) << p;
        }
      }
      tc_fence_before();
      mask &= ~(1u << guess);
      tk.cand[tt_] = mask;
      if (stats && mask) atomicAdd(&stats[2], (unsigned)__popc(mask));
    }
    bar_group(SIDE);

    // ---- D. survivors: full fp32 distance, top-2 with error bounds, fp64 re-match ---------
    {
      uint32_t cm[2] = {tk.cand[t0], tk.cand[t0 + 8]};
      if (__any_sync(0xffffffffu, (cm[0] | cm[1]) != 0)) {
        float best[2], bestE[2], low[2];
        int bi[2] = {idx[0], idx[1]};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          best[h] = __fsub_rn(kmx[h], kmn[h]);
          bestE[h] = derr(kmx[h], kmn[h], pt.mabsr[idx[h]]);
          low[h] = FE_INF;  // min over the other evaluated patterns of d - err
        }
        while (__any_sync(0xffffffffu, (cm[0] | cm[1]) != 0)) {
          int pc[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            pc[h] = cm[h] ? __ffs(cm[h]) - 1 : -1;
            cm[h] &= cm[h] - 1;
          }
          float s4[4];
          cand_stats(X, M, gw, lane, pc[0] >= 0 ? pc[0] : idx[0], pc[1] >= 0 ? pc[1] : idx[1], s4);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float cx = qmax4(s4[2 * h]), cn = qmin4(s4[2 * h + 1]);
            if (pc[h] >= 0) {
              const float d = __fsub_rn(cx, cn), e = derr(cx, cn, pt.mabsr[pc[h]]);
              if (d < best[h] || (d == best[h] && pc[h] < bi[h])) {
                low[h] = fminf(low[h], best[h] - bestE[h]);
                best[h] = d; bestE[h] = e; bi[h] = pc[h];
              } else {
                low[h] = fminf(low[h], d - e);
              }
            }
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool amb = low[h] <= best[h] + bestE[h];
          if (__any_sync(0xffffffffu, amb)) {
            const int ri = refine64(X, t0 + 8 * h, p64, P, q);
            if (amb) {
              bi[h] = ri;
              if (stats && q == 0) atomicAdd(&stats[0], 1u);
            }
          }
        }
        const bool chg = bi[0] != idx[0] || bi[1] != idx[1];
        if (__any_sync(0xffffffffu, chg)) {
          idx[0] = bi[0]; idx[1] = bi[1];
          resid_pass(X, M, gw, lane, idx, r, st);
#pragma unroll
          for (int h = 0; h < 2; ++h) { kmx[h] = qmax4(st.kmx[h]); kmn[h] = qmin4(st.kmn[h]); }
        }
      }
      if (q == 0) { tk.fidx[t0] = idx[0]; tk.fidx[t0 + 8] = idx[1]; }
    }
    bar_group(SIDE);  // the x tile is free: prefetch the next item's span
    if (gtid == 0 && it + 1 < i1) issue(it + 1);

    if constexpr (SIDE == 0) {
      // ================= K: per-channel groups over the span's tokens =================
      float* R = reinterpret_cast<float*>(sb + OFF_R);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = t0 + 8 * h;
        const bool ok = t < L;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          *reinterpret_cast<float2*>(R + t * RS + 16 * j + 2 * q) =
              ok ? make_float2(r[h][j][0], r[h][j][1]) : make_float2(FE_NAN, FE_NAN);
          *reinterpret_cast<float2*>(R + t * RS + 16 * j + 8 + 2 * q) =
              ok ? make_float2(r[h][j][2], r[h][j][3]) : make_float2(FE_NAN, FE_NAN);
        }
      }
      bar_group(SIDE);
      const int c0 = 16 * gw + 2 * q;  // channels c0, c0+1, c0+8, c0+9 (k = 0..3)
      float rr[8][2][4];
      float lmx[4], lmn[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) { lmx[kk] = -FE_INF; lmn[kk] = FE_INF; }
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = 16 * tt + 8 * h + g;
          const float2 a = *reinterpret_cast<const float2*>(R + t * RS + c0);
          const float2 bq = *reinterpret_cast<const float2*>(R + t * RS + c0 + 8);
          rr[tt][h][0] = a.x; rr[tt][h][1] = a.y; rr[tt][h][2] = bq.x; rr[tt][h][3] = bq.y;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const float key = fkey(rr[tt][h][kk], 2 * tt + h, 0xfffffff0u);
            lmx[kk] = fmaxf(lmx[kk], key);
            lmn[kk] = fminf(lmn[kk], key);
          }
        }
      double* KQ = reinterpret_cast<double*>(sb + OFF_KQ);
      float qlo[4], qinv[4], qhg[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int ch = c0 + (kk & 1) + 8 * (kk >> 1);
        float gmx = lmx[kk], gmn = lmn[kk];
#pragma unroll
        for (int o = 4; o <= 16; o <<= 1) {
          gmx = fmaxf(gmx, __shfl_xor_sync(0xffffffffu, gmx, o));
          gmn = fminf(gmn, __shfl_xor_sync(0xffffffffu, gmn, o));
        }
        const float Rm = fmaxf(fabsf(gmx), fabsf(gmn));
        const float Mc = pt.mabsc[ch];
        // |key - r64| <= 2^-19 |r| + 2^-24 |r| + 2^-23 |m|: window of twice that
        const float tolx = TWO_M17 * Rm + 4.76837158203125e-07f * Mc;
        const float hib = gmx - tolx, lob = gmn + tolx;
        int cnt = 0;
#pragma unroll
        for (int tt = 0; tt < 8; ++tt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float key = fkey(rr[tt][h][kk], 2 * tt + h, 0xfffffff0u);
            cnt += (key >= hib) + (key <= lob);
          }
#pragma unroll
        for (int o = 4; o <= 16; o <<= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        const uint32_t qm = 0x11111111u << q;
        const uint32_t bmx = __ballot_sync(0xffffffffu, lmx[kk] == gmx) & qm;
        const uint32_t bmn = __ballot_sync(0xffffffffu, lmn[kk] == gmn) & qm;
        const bool fast = cnt == 2 && __popc(bmx) == 1 && __popc(bmn) == 1;
        double hi64, lo64;
        if (__all_sync(0xffffffffu, fast)) {
          const int gx = (__ffs(bmx) - 1) >> 2, gn = (__ffs(bmn) - 1) >> 2;
          const uint32_t ix = __float_as_uint(gmx) & 15u, in_ = __float_as_uint(gmn) & 15u;
          const int tx = 16 * (int)(ix >> 1) + 8 * (int)(ix & 1) + gx;
          const int tn = 16 * (int)(in_ >> 1) + 8 * (int)(in_ & 1) + gn;
          hi64 = __dsub_rn((double)__half2float(xsrc[(int64_t)tx * 128 + ch]), p64[(int64_t)tk.fidx[tx] * 128 + ch]);
          lo64 = __dsub_rn((double)__half2float(xsrc[(int64_t)tn * 128 + ch]), p64[(int64_t)tk.fidx[tn] * 128 + ch]);
        } else {  // several elements inside the error window somewhere: fp64 over all of them
          double dmx, dmn;
          k_slow_extrema(R, tk.fidx, xsrc, p64, ch, g, hib, lob, &dmx, &dmn);
#pragma unroll
          for (int o = 4; o <= 16; o <<= 1) {
            dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
            dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
          }
          hi64 = dmx; lo64 = dmn;
          if (stats && lane == q && !fast) atomicAdd(&stats[3], 1u);
        }
        const GroupQ gg = make_group(lo64, hi64, QMAX, A.yq, Rm, Mc);
        qlo[kk] = gg.lo32; qinv[kk] = gg.inv; qhg[kk] = gg.hg;
        if (g == 0) { KQ[ch] = gg.lo; KQ[128 + ch] = gg.scale; }
      }
      __syncwarp();
      // codes (pairs of channels c0+{0,1} / c0+{8,9} per token), K fragment words
      uint32_t* KW = reinterpret_cast<uint32_t*>(sb + OFF_KW);
      const int slot0 = 2 * (gw % HS);
      const int wbase = 2 * (gw / HS);
      const int swz = (lane / (32 / WL)) & (WL - 1);
      uint32_t badm = 0;  // bit 2e + pr: element pair pr of (tt, h) = e lies in a guard band
#pragma unroll
      for (int tt = 0; tt < 8; ++tt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = 16 * tt + 8 * h + g;
          bool bad0 = false, bad1 = false;
          const float z0 = zcode(rr[tt][h][0], qlo[0], qinv[0], qhg[0], bad0);
          const float z1 = zcode(rr[tt][h][1], qlo[1], qinv[1], qhg[1], bad0);
          const float z2 = zcode(rr[tt][h][2], qlo[2], qinv[2], qhg[2], bad1);
          const float z3 = zcode(rr[tt][h][3], qlo[3], qinv[3], qhg[3], bad1);
          uint32_t p0 = zpair(z0, z1), p1 = zpair(z2, z3);
          if (t >= L) { p0 = 0u; p1 = 0u; bad0 = bad1 = false; }
          badm |= ((uint32_t)bad0 << (2 * (2 * tt + h))) | ((uint32_t)bad1 << (2 * (2 * tt + h) + 1));
          const uint32_t part = (p0 << (slot0 * BITS)) | (p1 << ((slot0 + 1) * BITS));
          atomicOr(&KW[(tt * 32 + lane) * WL + ((h + wbase) ^ swz)], part);
        }
      if (badm) {  // rare: the reference's fp64 sequence decides inside the guard band
#pragma unroll 1
        while (badm) {
          const int bit = __ffs(badm) - 1;
          badm &= badm - 1;
          const int e = bit >> 1, pr = bit & 1, tt = e >> 1, h = e & 1;
          const int t = 16 * tt + 8 * h + g, ch = c0 + 8 * pr;
          const double* mrow = p64 + (int64_t)tk.fidx[t] * 128;
          const __half* xrow = xsrc + (int64_t)t * 128;
          const uint32_t pv = exact_code_at(xrow + ch, mrow + ch, KQ[ch], KQ[128 + ch], QMAX) |
                              (exact_code_at(xrow + ch + 1, mrow + ch + 1, KQ[ch + 1], KQ[128 + ch + 1], QMAX) << 16);
          const int sh = (slot0 + pr) * BITS;
          uint32_t* wp = &KW[(tt * 32 + lane) * WL + ((h + wbase) ^ swz)];
          atomicAnd(wp, ~(((uint32_t)QMAX | ((uint32_t)QMAX << 16)) << sh));
          atomicOr(wp, pv << sh);
          if (stats) atomicAdd(&stats[1], 1u);
        }
      }
      // params
      const int64_t blk = (int64_t)u * c.NBcap + b;
      if (g == 0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int ch = c0 + (kk & 1) + 8 * (kk >> 1);
          c.kparam64[blk * 256 + ch] = KQ[128 + ch];
          c.kparam64[blk * 256 + 128 + ch] = KQ[ch];
          c.kparam32[blk * 2 * c.Dp + ch] = (float)KQ[128 + ch];
          c.kparam32[blk * 2 * c.Dp + c.Dp + ch] = (float)KQ[ch];
        }
      }
      if (gtid < L) c.kidx[blk * c.GP + gtid] = (int16_t)tk.fidx[gtid];
      bar_group(SIDE);
      // K words -> HBM (16 B per thread-chunk), clear for the next item
      uint4* dst = reinterpret_cast<uint4*>(c.kcodes + blk * c.blk_bytes);
      for (int ci = gtid; ci < 8 * 32 * WL / 4; ci += GT) {
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int wi = 4 * ci + e, tl = wi / WL, w = wi % WL, ln = tl & 31;
          const int a = tl * WL + (w ^ ((ln / (32 / WL)) & (WL - 1)));
          wv[e] = KW[a];
          KW[a] = 0u;
        }
        dst[ci] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
    } else {
      // ================= V: per-token groups over channels =================
      const int64_t blk = (int64_t)u * c.NBcap + b;
      uint32_t words[WL];
#pragma unroll
      for (int w = 0; w < WL; ++w) words[w] = 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = t0 + 8 * h;
        const float xa = fmaxf(fabsf(xmx[h]), fabsf(xmn[h]));
        const float Mr = pt.mabsr[idx[h]];
        const float Rm = fmaxf(fabsf(kmx[h]), fabsf(kmn[h]));
        // |key - r64| <= 2^-18 |r| + 2^-24 |r| + 2^-23 |m|: window of twice that
        const float tolx = 1.52587890625e-05f * Rm + 4.76837158203125e-07f * Mr;
        const float hib = kmx[h] - tolx, lob = kmn[h] + tolx;
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float key = fkey(r[h][j][e], 4 * j + e, 0xffffffe0u);
            cnt += (key >= hib) + (key <= lob);
          }
        cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
        const uint32_t gm = 0xfu << (4 * g);
        const uint32_t bmx = __ballot_sync(0xffffffffu, st.kmx[h] == kmx[h]) & gm;
        const uint32_t bmn = __ballot_sync(0xffffffffu, st.kmn[h] == kmn[h]) & gm;
        const double* mrow = p64 + (int64_t)idx[h] * 128;
        const __half* xrow = xsrc + (int64_t)t * 128;
        double hi64, lo64;
        const bool fast = cnt == 2 && __popc(bmx) == 1 && __popc(bmn) == 1;
        if (__all_sync(0xffffffffu, fast)) {
          const int qx = (__ffs(bmx) - 1) & 3, qn = (__ffs(bmn) - 1) & 3;
          const uint32_t ix = __float_as_uint(kmx[h]) & 31u, in_ = __float_as_uint(kmn[h]) & 31u;
          const int chx = 16 * (int)(ix >> 2) + 8 * (int)((ix >> 1) & 1) + 2 * qx + (int)(ix & 1);
          const int chn = 16 * (int)(in_ >> 2) + 8 * (int)((in_ >> 1) & 1) + 2 * qn + (int)(in_ & 1);
          hi64 = __dsub_rn((double)__half2float(xrow[chx]), mrow[chx]);
          lo64 = __dsub_rn((double)__half2float(xrow[chn]), mrow[chn]);
        } else {
          double dmx, dmn;
          v_slow_extrema(xrow, mrow, M + idx[h] * MR + q * 36, q, hib, lob, &dmx, &dmn);
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
            dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
          }
          hi64 = dmx; lo64 = dmn;
          if (stats && q == 0 && t < L && !fast) atomicAdd(&stats[3], 1u);
        }
        // gate (gate.py:180-188; --no-v-gate flattens, engine.py:235-237)
        const double raw = __dsub_rn((double)xmx[h], (double)xmn[h]);
        const double flat = __dsub_rn(hi64, lo64);
        const bool flatten = c.use_vgate ? (raw > 0.0 && gate_le(flat, raw, c.thr)) : true;
        if (!flatten) {  // RAW payload: the exact input row (rare)
          hi64 = (double)xmx[h]; lo64 = (double)xmn[h];
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) r[h][j][e] = __half2float(xrow[16 * j + 8 * (e >> 1) + 2 * q + (e & 1)]);
        }
        const GroupQ gqv = flatten ? make_group(lo64, hi64, QMAX, A.yq, Rm, Mr) : make_group(lo64, hi64, QMAX, A.yq, xa, 0.f);
        // codes -> pairs (token row, channel pair), exact fix-ups, movmatrix -> V^T fragment words
        uint32_t pp[16];
        uint32_t badm = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          bool bad0 = false, bad1 = false;
          const float z0 = zcode(r[h][j][0], gqv.lo32, gqv.inv, gqv.hg, bad0);
          const float z1 = zcode(r[h][j][1], gqv.lo32, gqv.inv, gqv.hg, bad0);
          const float z2 = zcode(r[h][j][2], gqv.lo32, gqv.inv, gqv.hg, bad1);
          const float z3 = zcode(r[h][j][3], gqv.lo32, gqv.inv, gqv.hg, bad1);
          pp[2 * j] = zpair(z0, z1);
          pp[2 * j + 1] = zpair(z2, z3);
          badm |= ((uint32_t)bad0 << (2 * j)) | ((uint32_t)bad1 << (2 * j + 1));
        }
        if (t >= L) {
          badm = 0;
#pragma unroll
          for (int i = 0; i < 16; ++i) pp[i] = 0u;
        }
        if (badm) {  // rare: the reference's fp64 sequence decides inside the guard band
          const double* mr = flatten ? mrow : nullptr;
#pragma unroll 1
          while (badm) {
            const int i = __ffs(badm) - 1;
            badm &= badm - 1;
            const int ca = 16 * (i >> 1) + 8 * (i & 1) + 2 * q;
            const uint32_t pv = exact_code_at(xrow + ca, mr ? mr + ca : nullptr, gqv.lo, gqv.scale, QMAX) |
                                (exact_code_at(xrow + ca + 1, mr ? mr + ca + 1 : nullptr, gqv.lo, gqv.scale, QMAX) << 16);
#pragma unroll
            for (int k2 = 0; k2 < 16; ++k2) pp[k2] = k2 == i ? pv : pp[k2];
            if (stats) atomicAdd(&stats[1], 1u);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t t0v = movm_t(pp[2 * j]), t1v = movm_t(pp[2 * j + 1]);  // hiRow 0 / 1 of sub-tile j
          const int s0 = 2 * (j % HS);
          words[h + 2 * (j / HS)] |= (t0v << (s0 * BITS)) | (t1v << ((s0 + 1) * BITS));
        }
        if (q == 0 && t < L) {
          const int64_t tok = (int64_t)u * c.Tcap + start + t;
          const int64_t slot = blk * c.GP + t;
          c.vparam64[2 * tok] = gqv.scale;
          c.vparam64[2 * tok + 1] = gqv.lo;
          c.vparam32[2 * slot] = (float)gqv.scale;
          c.vparam32[2 * slot + 1] = (float)gqv.lo;
          c.vidx[slot] = (int16_t)(flatten ? idx[h] : RAW);
          if (c.keep_diag && c.vdiag) { c.vdiag[2 * tok] = raw; c.vdiag[2 * tok + 1] = flat; }
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(c.vcodes + blk * c.blk_bytes + (size_t)(gw * 32 + lane) * WL * 4);
#pragma unroll
      for (int w = 0; w < WL; w += 4) dst[w / 4] = make_uint4(words[w], words[w + 1], words[w + 2], words[w + 3]);
    }
  }
}

template <int BITS>
__global__ void __launch_bounds__(NTHR, 1)
encode_tc_kernel(const Args A, const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-aligned base, derived from the shared array itself so every access stays an LDS/STS
  unsigned char* sb = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + OFF_BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sb + OFF_BAR + 32);
  uint32_t* KW = reinterpret_cast<uint32_t*>(sb + OFF_KW);
  for (int i = tid; i < 8 * 32 * 8; i += NTHR) KW[i] = 0u;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
  }
  if (warp == 0) tmem_alloc<128>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int64_t per = A.nitems / gridDim.x, rem = A.nitems % gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * per + min((int64_t)blockIdx.x, rem);
  const int64_t i1 = i0 + per + ((int64_t)blockIdx.x < rem ? 1 : 0);
  if (warp < 8) run_side<BITS, 0>(A, sb, &tmK, tmem, i0, i1);
  else run_side<BITS, 1>(A, sb, &tmV, tmem, i0, i1);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_free<128>(tmem);
}

// TMA descriptor of a [U][rows][128] fp16 tensor (unit stride in elements), 64 x 128 x 1 boxes
static bool make_tmap3(CUtensorMap* map, const void* base, uint64_t rows, uint64_t units, int64_t unit_stride) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess || !p)
      return false;
    fn = reinterpret_cast<EncodeFn>(p);
  }
  const cuuint64_t dims[3] = {128, rows, units};
  const cuuint64_t strides[2] = {128 * 2, (cuuint64_t)unit_stride * 2};
  const cuuint32_t box[3] = {64, 128, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace fe

// Host launcher: returns cudaErrorNotSupported when the cache/config is outside this
// kernel's envelope (the caller then runs encode_span_kernel).
cudaError_t launch_encode_tc(const DevCache& c, int max_p, const __half* k, const __half* v, int64_t rows,
                             int64_t unit_stride, int first_block, int nblocks, cudaStream_t st) {
  const char* env = getenv("PKV_ENCODE_TC");
  if (env && env[0] == '0') return cudaErrorNotSupported;
  if (nblocks <= 0) return cudaSuccess;
  if (c.D != 128 || c.Dp != 128 || c.G != 128 || c.ntile_blk != 8 || !(c.bits == 2 || c.bits == 4) || !c.use_kp ||
      !c.use_vp || c.use_kgate || max_p < 1 || max_p > fe::PM || !c.prune)
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) return cudaErrorNotSupported;
  if ((unit_stride * 2) % 16 || rows >= (1ll << 31)) return cudaErrorNotSupported;
  CUtensorMap tk, tv;
  memset(&tk, 0, sizeof tk);
  memset(&tv, 0, sizeof tv);
  if (!fe::make_tmap3(&tk, k, (uint64_t)rows, (uint64_t)c.U, unit_stride) ||
      !fe::make_tmap3(&tv, v, (uint64_t)rows, (uint64_t)c.U, unit_stride))
    return cudaErrorNotSupported;
  fe::Args a;
  a.c = c;
  a.nb = nblocks;
  a.first_block = first_block;
  a.src[0] = k;
  a.src[1] = v;
  a.unit_stride = unit_stride;
  a.nitems = (int64_t)c.U * nblocks;
  a.yq = 1.0 / (double)((1 << c.bits) - 1);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const int grid = (int)std::min<int64_t>(nsm, a.nitems);
  if (c.bits == 2) {
    cudaFuncSetAttribute(fe::encode_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, fe::SMEM_BYTES);
    fe::encode_tc_kernel<2><<<grid, fe::NTHR, fe::SMEM_BYTES, st>>>(a, tk, tv);
  } else {
    cudaFuncSetAttribute(fe::encode_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, fe::SMEM_BYTES);
    fe::encode_tc_kernel<4><<<grid, fe::NTHR, fe::SMEM_BYTES, st>>>(a, tk, tv);
  }
  return cudaGetLastError();
}

}  // namespace pkv
