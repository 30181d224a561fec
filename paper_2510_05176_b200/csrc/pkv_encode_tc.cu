// K1-TC: persistent fp16 prefill encoder (d = 128, G = 128, P <= 32, 2/4-bit).
//
// Same contract as encode_span_kernel (pkv_encode.cu) -- the reference's
// _commit_span (engine.py:201-252) with match_many (patterns.py:206-221),
// decide (gate.py:174-188), quantize_group and pack_codes (quant.py:70-146) --
// and bit-identical outputs, re-organised so that almost every instruction
// touches data in registers:
//
//  * one persistent CTA per SM, 16 warps in four 4-warp subgroups, all on ONE side (K or V)
//    at a time: chunks of 32 (unit, span) items come from per-side global queues, every CTA
//    starts on K and moves to V as K drains (a K phase, then a V phase: one code path per SM,
//    so the hot code stays in the instruction caches); each subgroup streams its own 32 KB
//    span tiles (cp.async.bulk.tensor.3d, 128-byte swizzle), the last warp out of a tile
//    issuing the next item's TMA;
//  * nearest pattern: one tcgen05.mma chain per span computes x . m'_p (m' = channel-centered
//    pattern split hi + lo in fp16, fp32 accumulator in TMEM).  The L2-nearest pattern is the
//    guess g; the exact fp32 d_mm to g comes out of the residual pass; every other pattern is
//    pruned by an exact lower bound on d_mm with rigorous fp error margins -- V: Popoviciu
//    (osc(v)^2 >= 4 Var(v), Var from the GEMM); K: the residual range over the 8 widest-
//    spread channels (4 first, the other 4 only for survivors).  Survivors (rare) get the full
//    fp32 distance, near ties the reference's fp64 argmin (lowest index on ties);
//  * residuals, extrema and codes in mma-fragment register layout (ldmatrix from the
//    swizzled tile); per-token (V) reductions need 2 shuffles; K's per-channel groups run on
//    a residual tile in a transposed warp layout; V codes move to the V^T fragment layout
//    with movmatrix;
//  * exact fp64 group extrema from fp32 "keys" (value with the element index in the low
//    mantissa bits) plus a one-predicate count of the elements inside the fp32 error windows;
//    codes by a magic-number round z = fma(v - lo, 1/s, 1.5*2^23) whose distance to the
//    rounding boundary is checked per element pair (fp64 recompute of the reference sequence
//    inside the guard band).  DESIGN.md section 3 (K1-TC) has the error bounds and the
//    measurements behind each choice.
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "pkv_common.cuh"
#include "pkv_sm100.cuh"

namespace pkv {
namespace fe {

using namespace sm100;

constexpr int NTHR = 512;   // 16 warps: four 4-warp subgroups, all on the CTA's side (K or V)
constexpr int PM = 32;      // max patterns per side on this path
constexpr float MAGIC = 12582912.f;  // 1.5 * 2^23
#define FE_INF __int_as_float(0x7f800000)
#define FE_NAN __int_as_float(0x7fc00000)
constexpr float TWO_M13 = 1.220703125e-04f;
constexpr float TWO_M17 = 7.62939453125e-06f;
constexpr float TWO_M22 = 2.384185791015625e-07f;

// ---- shared memory map (bytes from a 1024-aligned base) ---------------------------------
// A CTA works on ONE side at a time: its four 4-warp subgroups (sgi = warp / 4) take turns
// over the items of a chunk and share the side's pattern tables.  Chunks (<= CHUNK items of
// one unit) come from a per-side global queue; a CTA starts on its TPC's side (by default
// every TPC starts on K: a K phase, then a V phase) and moves to the other side's queue when
// its own runs dry.  One side per SM (and TPC) keeps the hot code in the instruction caches:
// K and V warps on one SM thrash them (~30% of stall samples were no_instruction), a TPC
// holding a K and a V CTA runs ~1.5x slower.
constexpr int SZ_X = 32768;                       // span tile [2 halves][128 rows][128 B], SW128
constexpr int OFF_X = 0;                          // X[sgi]
constexpr int SZ_B = 16384;                       // centered hi [2][32][128 B] then lo [2][32][128 B]
constexpr int OFF_B = OFF_X + 4 * SZ_X;           // B[side] (K CTAs: B[1] holds KW[2], KW[3])
constexpr int SZ_M = PM * 128 * 4;                // fp32 table, lane-permuted rows (mslot)
constexpr int OFF_M = OFF_B + 2 * SZ_B;           // M[side]
constexpr int NSC = 9;                            // scratch arrays of 128 words per subgroup
constexpr int SZ_SC = NSC * 128 * 4;
constexpr int OFF_SC = OFF_M + 2 * SZ_M;          // SC[sgi]
constexpr int NPRB = 8;    // K probe channels of the pruning bound
constexpr int NFLAG = (2 + NPRB + 3) / 4 * 4;      // P, no-L2, probe channels
constexpr int SZ_PAT = (4 * 32 + 128 + NFLAG + NPRB * 32) * 4;  // bb, mn, (spare), mabsr [4][32], mabsc[128], flags, pm4[32][NPRB]
constexpr int OFF_PAT = OFF_SC + 4 * SZ_SC;       // PAT[side]
constexpr int OFF_BAR = OFF_PAT + 2 * SZ_PAT;     // xfull[4], mma[4], release counters[4], tmem addr,
                                                  // chunk item counter at +84, chunk ring[2] at +96,
                                                  // per-subgroup next item [4] at +104
constexpr int OFF_KW = OFF_BAR + 128;             // 2-bit K code words KW[0], KW[1]: [8 tiles][32 lanes][4]
constexpr int SZ_KW = 8 * 32 * 4 * 4;
static_assert(2 * SZ_KW <= SZ_B, "KW[2..3] live in the unused B[1] of a K CTA");
__host__ __device__ constexpr int smem_bytes(int bits) { return OFF_KW + (bits == 2 ? 2 * SZ_KW : 0) + 1024; }
static_assert(smem_bytes(2) <= 232448 && smem_bytes(4) <= 232448, "shared memory budget");

// per-subgroup scratch: token arrays (index t) during the token stage, then per-group arrays
// (index = token for V, channel for K) for the scalar pass
#define SMEM_PTR(p) __builtin_assume(__isShared(p))
struct Scr {   // per-subgroup scratch, 9 arrays of 128 words
  unsigned char* base;
  __device__ explicit Scr(unsigned char* sb, int sgi) : base(sb + OFF_SC + sgi * SZ_SC) {}
  __device__ int* guess() const { return reinterpret_cast<int*>(base); }             // token stage
  __device__ float* lo32() const { return reinterpret_cast<float*>(base); }          // scalar pass (alias)
  __device__ uint32_t* cand() const { return reinterpret_cast<uint32_t*>(base + 512); }
  __device__ float* inv() const { return reinterpret_cast<float*>(base + 512); }     // scalar pass (alias)
  __device__ float* hg() const { return reinterpret_cast<float*>(base + 1024); }     // 1/2 - guard
  __device__ float* kmx() const { return reinterpret_cast<float*>(base + 1536); }    // keyed residual max
  __device__ float* kmn() const { return reinterpret_cast<float*>(base + 2048); }    // keyed residual min
  __device__ float* xmx() const { return reinterpret_cast<float*>(base + 2560); }    // x max (token)
  __device__ float* xmn() const { return reinterpret_cast<float*>(base + 3072); }    // x min (token)
  __device__ int* fidx() const { return reinterpret_cast<int*>(base + 3584); }       // final pattern per token
  // bit 0 unique extrema (bits 1-7 / 8-14 arg-max / arg-min), bit 1<<16 exact fp64 extrema stored
  // in (kmx, xmx) / (kmn, xmn) as double halves (K), bit 15 flatten (V)
  __device__ int* info() const { return reinterpret_cast<int*>(base + 4096); }
};
struct Pat {   // per-side pattern scalars
  unsigned char* base;
  __device__ explicit Pat(unsigned char* sb, int side) : base(sb + OFF_PAT + side * SZ_PAT) {}
  __device__ float* bb() const { return reinterpret_cast<float*>(base); }            // ||m'_p||^2 (+inf past P)
  __device__ float* mn() const { return reinterpret_cast<float*>(base + 128); }      // ||m'_p||
  __device__ float* pm4() const { return reinterpret_cast<float*>(base + 1024 + 4 * NFLAG); }  // K: m32 at the probe channels
  __device__ float* mabsr() const { return reinterpret_cast<float*>(base + 384); }   // max_c |m_pc|
  __device__ float* mabsc() const { return reinterpret_cast<float*>(base + 512); }   // max_p |m_pc| (K)
  __device__ int* flags() const { return reinterpret_cast<int*>(base + 1024); }      // P, no-L2, probe channels [2..5]
};

struct Args {
  DevCache c;
  int nb;            // blocks in this launch (first_block .. first_block + nb)
  int first_block;
  const __half* src[2];  // K, V inputs [U][rows][128]
  int64_t unit_stride;   // elements between units
  int64_t nitems;        // U * nb
  double yq;             // RN(1 / qmax)
  int k_tpc;             // TPCs [0, k_tpc) start on K, the rest on V
  int chunk[2];          // items per chunk (K, V)
  int cpu[2];            // chunks per unit
  int nchunks[2];        // U * cpu
};

__device__ __forceinline__ void bar_side() { asm volatile("bar.sync 1, %0;" ::"n"(NTHR) : "memory"); }
__device__ __forceinline__ void bar_sub(int sgi) { asm volatile("bar.sync %0, %1;" ::"r"(3 + sgi), "n"(128) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
// an .aligned warp instruction: tells ptxas the warp is converged here, so the shuffles that
// follow in an out-of-line function need no divergence-tolerant (WARPSYNC.COLLECTIVE) copies
__device__ __forceinline__ void warp_converged() {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(0u));  // result unused
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
// x - m for an fp16 x (low / high half of v) and an fp32 m in ONE instruction (FHADD: the
// mixed-precision sub.rn.f32.f16 converts x exactly and rounds once -- the same value as
// converting and then subtracting, without the conversion instruction)
__device__ __forceinline__ float subh_lo(uint32_t v, float m) {
  float d;
  asm("sub.rn.f32.f16 %0, %1, %2;" : "=f"(d) : "h"((unsigned short)(v & 0xffffu)), "f"(m));
  return d;
}
__device__ __forceinline__ float subh_hi(uint32_t v, float m) {
  float d;
  asm("sub.rn.f32.f16 %0, %1, %2;" : "=f"(d) : "h"((unsigned short)(v >> 16)), "f"(m));
  return d;
}
// running fp16 extrema of packed x (exact: max/min commute with the exact fp16 -> fp32
// conversion; NaN lanes lose to numbers as in fmaxf), converted once at the end
__device__ __forceinline__ __half2 u2h2(uint32_t v) { return *reinterpret_cast<const __half2*>(&v); }
__device__ __forceinline__ float h2max(__half2 h) { return fmaxf(__low2float(h), __high2float(h)); }
__device__ __forceinline__ float h2min(__half2 h) { return fminf(__low2float(h), __high2float(h)); }
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
// fp32 pattern row p, lane-permuted: lane q's 32 channels (16j + 8hc + 2q + e) form segment
// q; chunk j (channels 16j + {0,1,8,9} + 2q) sits at slot j ^ 2q ^ (p & 1), so the four
// lanes of a row read distinct bank groups (and rows of different parity interleave)
__device__ __forceinline__ int mslot(int p, int q, int j) { return q * 32 + 4 * ((j ^ (2 * q) ^ (p & 1)) & 7); }
__device__ __forceinline__ int mpos(int p, int c) {
  const int j = c >> 4, hc = (c >> 3) & 1, q = (c >> 1) & 3, e = c & 1;
  return mslot(p, q, j) + 2 * hc + e;
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
// two elements at once on the packed fp32 pipe (FADD2 / FFMA2: lane-wise the same IEEE RN
// operations as zcode -- r - lo == r + (-lo), |d| > hg <=> |d| - hg > 0 without underflow to
// zero); per-element params (K: two channels) with nhg = -hg
__device__ __forceinline__ float2 zcode2(float2 r, float2 nlo, float2 inv, float2 nhg, bool& bad) {
  const float2 rl = __fadd2_rn(r, nlo);
  const float2 z = __ffma2_rn(rl, inv, make_float2(MAGIC, MAGIC));
  const float2 k = __fadd2_rn(z, make_float2(-MAGIC, -MAGIC));
  const float2 d = __ffma2_rn(rl, inv, make_float2(-k.x, -k.y));
  const float2 e = __fadd2_rn(make_float2(fabsf(d.x), fabsf(d.y)), nhg);
  bad |= fmaxf(e.x, e.y) > 0.f;  // fmaxf skips a NaN element (token past the span), as zcode's compare does
  return z;
}
// shared params (V: one token)
__device__ __forceinline__ float2 zcode2s(float2 r, float2 nlo, float2 inv, float hg, bool& bad) {
  const float2 rl = __fadd2_rn(r, nlo);
  const float2 z = __ffma2_rn(rl, inv, make_float2(MAGIC, MAGIC));
  const float2 k = __fadd2_rn(z, make_float2(-MAGIC, -MAGIC));
  const float2 d = __ffma2_rn(rl, inv, make_float2(-k.x, -k.y));
  bad |= fmaxf(fabsf(d.x), fabsf(d.y)) > hg;
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
  SMEM_PTR(X);
  warp_converged();
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
// ---------------------------------------------------------------------------------------
// pattern staging for (unit u, side): permuted fp32 table, centered hi/lo B operand,
// per-pattern scalars.  Called by all threads of the CTA between CTA barriers.
// ---------------------------------------------------------------------------------------
__device__ void stage_patterns(const Args& A, int side, int u, unsigned char* sb, int gtid) {
  const DevCache& c = A.c;
  const int P = side == 0 ? c.nk[u] : c.nv[u];
  const float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * c.Dp;
  const double* p64 = (side == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * 128;
  float* M = reinterpret_cast<float*>(sb + OFF_M + side * SZ_M);
  unsigned char* B = sb + OFF_B + side * SZ_B;
  Pat pt(sb, side);
  const int* prb = c.probe + ((int64_t)u * 2 + side) * 16;  // channels by pattern spread (probe_kernel)
  if (gtid == 0) pt.flags()[1] = 0;
  for (int i = gtid; i < PM * 128; i += NTHR) {
    const int p = i >> 7, ch = i & 127;
    M[p * 128 + mpos(p, ch)] = p < P ? p32[(int64_t)p * c.Dp + ch] : 0.f;
  }
  if (side == 0 && gtid < 128) {
    float m = 0.f;
    for (int p = 0; p < P; ++p) m = fmaxf(m, fabsf(p32[(int64_t)p * c.Dp + gtid]));
    pt.mabsc()[gtid] = m;
  }
  bar_side();  // flags[1] reset visible
  // one warp per pattern (16 warps x 2): mean in fp64, centered hi/lo fp16 rows
  const int w = gtid >> 5, lane = gtid & 31;
  warp_converged();
  for (int p = w; p < PM; p += NTHR / 32) {
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
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&pt.flags()[1], 1);
    if (lane == 0) {
      pt.bb()[p] = p < P ? (float)ss : FE_INF;
      pt.mn()[p] = p < P ? (float)sqrt(ss) : 0.f;
      if (side == 0)
#pragma unroll
        for (int j = 0; j < NPRB; ++j) pt.pm4()[NPRB * p + j] = p < P ? (float)p64[(int64_t)p * 128 + prb[j]] : 0.f;
      pt.mabsr()[p] = amax;
    }
  }
  if (gtid == 0) {
    pt.flags()[0] = P;
#pragma unroll
    for (int j = 0; j < NPRB; ++j) pt.flags()[2 + j] = prb[j];
  }
  fence_proxy_async();  // generic-proxy writes of B -> tensor-core reads
}

// ---------------------------------------------------------------------------------------
// residual pass of one warp over a 16-token tile (rows tb + g, tb + g + 8) against pattern
// rows idx[0], idx[1]: r = x - m in mma-fragment layout, keyed extrema, x extrema
// ---------------------------------------------------------------------------------------
struct RowStats {
  float kmx[2], kmn[2];   // lane-local keyed extrema of r (5-bit element index)
  float xmx[2], xmn[2];   // lane-local extrema of x
};
// KEYED: extrema of keys (the owner's index in the low bits, V); else plain extrema of r (K
// tokens need only max - min; the keyed error bound derr covers both)
template <bool STORE, bool KEYED = true>
__device__ __forceinline__ void resid_tile(const unsigned char* X, const float* M, int tb, int lane, const int idx[2],
                                           float (&r)[2][8][4], RowStats& st) {
  const int q = lane & 3;
  const uint32_t xbase = smem_u32(X);
  const int lrow = tb + (lane & 7) + 8 * ((lane >> 3) & 1);
  const int lchk = lane >> 4;
  const float* m0p = M + idx[0] * 128 + q * 32;
  const float* m1p = M + idx[1] * 128 + q * 32;
  const int sw0 = (2 * q) ^ (idx[0] & 1), sw1 = (2 * q) ^ (idx[1] & 1);
  __half2 hx[2], hn[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    st.kmx[h] = -FE_INF; st.kmn[h] = FE_INF;
    hx[h] = u2h2(0xfc00fc00u); hn[h] = u2h2(0x7c007c00u);  // -inf / +inf
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t a0, a1, a2, a3;
    const uint32_t addr = xbase + (j >> 2) * 16384 + lrow * 128 + ((((2 * (j & 3) + lchk) ^ (lrow & 7))) << 4);
    ldsm_x4(addr, a0, a1, a2, a3);
    const float4 m0 = *reinterpret_cast<const float4*>(m0p + 4 * (j ^ sw0));
    const float4 m1 = *reinterpret_cast<const float4*>(m1p + 4 * (j ^ sw1));
    const float rv[2][4] = {{subh_lo(a0, m0.x), subh_hi(a0, m0.y), subh_lo(a2, m0.z), subh_hi(a2, m0.w)},
                            {subh_lo(a1, m1.x), subh_hi(a1, m1.y), subh_lo(a3, m1.z), subh_hi(a3, m1.w)}};
    hx[0] = __hmax2(hx[0], __hmax2(u2h2(a0), u2h2(a2))); hn[0] = __hmin2(hn[0], __hmin2(u2h2(a0), u2h2(a2)));
    hx[1] = __hmax2(hx[1], __hmax2(u2h2(a1), u2h2(a3))); hn[1] = __hmin2(hn[1], __hmin2(u2h2(a1), u2h2(a3)));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float k0 = KEYED ? fkey(rv[h][0], 4 * j + 0, 0xffffffe0u) : rv[h][0];
      const float k1 = KEYED ? fkey(rv[h][1], 4 * j + 1, 0xffffffe0u) : rv[h][1];
      const float k2 = KEYED ? fkey(rv[h][2], 4 * j + 2, 0xffffffe0u) : rv[h][2];
      const float k3 = KEYED ? fkey(rv[h][3], 4 * j + 3, 0xffffffe0u) : rv[h][3];
      if constexpr (STORE) {  // the keys (or r when not KEYED)
        r[h][j][0] = k0; r[h][j][1] = k1; r[h][j][2] = k2; r[h][j][3] = k3;
      }
      st.kmx[h] = fmax3(st.kmx[h], k0, k1); st.kmx[h] = fmax3(st.kmx[h], k2, k3);
      st.kmn[h] = fmin3(st.kmn[h], k0, k1); st.kmn[h] = fmin3(st.kmn[h], k2, k3);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) { st.xmx[h] = h2max(hx[h]); st.xmn[h] = h2min(hn[h]); }
}

__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& a0, uint32_t& a1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(a0), "=r"(a1) : "r"(addr));
}
// one 8-token row-set (rows tb + g) of a tile against pattern row p: r in fragment layout
// (channels 16j + 8hc + 2q + e at r[j][2hc + e]), keyed extrema, x extrema
__device__ __forceinline__ void resid_row(const unsigned char* X, const float* M, int tb, int lane, int p,
                                          float (&r)[8][4], float& kmx, float& kmn, float& xmx, float& xmn) {
  const int q = lane & 3;
  const uint32_t xbase = smem_u32(X);
  // x2: matrices (rows 0-7, ch lo 8) and (rows 0-7, ch hi 8) of a 16-channel block
  const int lrow = tb + (lane & 7);
  const int lchk = (lane >> 3) & 1;
  const float* mp = M + p * 128 + q * 32;
  const int sw = (2 * q) ^ (p & 1);
  kmx = -FE_INF; kmn = FE_INF;
  __half2 hx = u2h2(0xfc00fc00u), hn = u2h2(0x7c007c00u);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t a0, a1;
    ldsm_x2(xbase + (j >> 2) * 16384 + lrow * 128 + ((((2 * (j & 3) + lchk) ^ (lrow & 7))) << 4), a0, a1);
    const float4 m = *reinterpret_cast<const float4*>(mp + 4 * (j ^ sw));
    r[j][0] = subh_lo(a0, m.x); r[j][1] = subh_hi(a0, m.y); r[j][2] = subh_lo(a1, m.z); r[j][3] = subh_hi(a1, m.w);
    hx = __hmax2(hx, __hmax2(u2h2(a0), u2h2(a1))); hn = __hmin2(hn, __hmin2(u2h2(a0), u2h2(a1)));
    const float k0 = fkey(r[j][0], 4 * j + 0, 0xffffffe0u), k1 = fkey(r[j][1], 4 * j + 1, 0xffffffe0u);
    const float k2 = fkey(r[j][2], 4 * j + 2, 0xffffffe0u), k3 = fkey(r[j][3], 4 * j + 3, 0xffffffe0u);
    kmx = fmax3(kmx, k0, k1); kmx = fmax3(kmx, k2, k3);
    kmn = fmin3(kmn, k0, k1); kmn = fmin3(kmn, k2, k3);
  }
  xmx = h2max(hx); xmn = h2min(hn);
}
__device__ __forceinline__ float qmax4(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float qmin4(float v) {
  v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fminf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
// cnt += (key >= hib || key <= lob): two compares into one predicate and a predicated add
__device__ __forceinline__ void win_or(int& cnt, float key, float hib, float lob) {
  asm("{\n .reg .pred p;\n setp.ge.f32 p, %1, %2;\n setp.le.or.f32 p, %1, %3, p;\n @p add.s32 %0, %0, 1;\n}"
      : "+r"(cnt) : "f"(key), "f"(hib), "f"(lob));
}
// bound on |d32 - d64| for a distance taken from keyed fp32 extrema (K1-TC):
// key error 2^-18 |r|, fp32 residual error 2^-24 (|r| + 2|m|), subtraction 2^-24 |d|
__device__ __forceinline__ float derr(float kmx, float kmn, float M) {
  return 7.62939453125e-06f * (fabsf(kmx) + fabsf(kmn)) + 4.76837158203125e-07f * M;
}

// ---- rare paths (out of line) -----------------------------------------------------------
// lane-local keyed extrema of a tile's two rows against candidate pattern rows
__device__ __noinline__ void cand_stats(const unsigned char* X, const float* M, int tb, int lane, int p0, int p1,
                                        float* out) {
  SMEM_PTR(X); SMEM_PTR(M);
  float r[2][8][4];
  RowStats st;
  const int idx[2] = {p0, p1};
  resid_tile<false, false>(X, M, tb, lane, idx, r, st);  // candidates compare plain distances
  out[0] = st.kmx[0]; out[1] = st.kmn[0]; out[2] = st.kmx[1]; out[3] = st.kmn[1];
}
// fp64 extrema of V row t over the elements whose key (fragment-layout index) lies in the
// error window -- same fp32 arithmetic and keys as resid_tile, one thread
__device__ __noinline__ void v_exact_slow(const unsigned char* X, const float* M, int t, int p, const double* mrow,
                                          float hib, float lob, double* hi, double* lo) {
  SMEM_PTR(X); SMEM_PTR(M);
  double dmx = -__longlong_as_double(0x7ff0000000000000LL), dmn = -dmx;
  for (int ch = 0; ch < 128; ++ch) {
    const int j = ch >> 4, q = (ch >> 1) & 3, k = 2 * ((ch >> 3) & 1) + (ch & 1);
    const float xv = xt_at(X, t, ch);
    const float key = fkey(__fsub_rn(xv, M[p * 128 + mslot(p, q, j) + k]), (uint32_t)(4 * j + k), 0xffffffe0u);
    if (key >= hib || key <= lob) {
      const double v64 = __dsub_rn((double)xv, mrow[ch]);
      if (key >= hib) dmx = fmax(dmx, v64);
      if (key <= lob) dmn = fmin(dmn, v64);
    }
  }
  *hi = dmx;
  *lo = dmn;
}
// exact code of one element from the stored fp64 params (read back through L2)
__device__ __noinline__ uint32_t exact_code_p(const __half* xp, const double* mp, const double* par_lo,
                                              const double* par_scale, int qmax) {
  return exact_code_at(xp, mp, __ldcg(par_lo), __ldcg(par_scale), qmax);
}

// ---------------------------------------------------------------------------------------
// B-pass of one 16-token tile against pattern rows idx[]: keyed extrema (and, for V, the
// count of elements inside the fp32 error window of each extremum plus their owners)
// ---------------------------------------------------------------------------------------
template <bool VS>
__device__ __noinline__ void b_tile(const unsigned char* X, const float* M, Pat pt, Scr sc, int tb,
                                    int lane, int i0, int i1) {
  SMEM_PTR(X); SMEM_PTR(M); SMEM_PTR(pt.base); SMEM_PTR(sc.base);
  const int g = lane >> 2, q = lane & 3, t0 = tb + g;
  const int idx[2] = {i0, i1};
  float r[2][8][4];
  RowStats st;
  resid_tile<VS, VS>(X, M, tb, lane, idx, r, st);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float kx = qmax4(st.kmx[h]), kn = qmin4(st.kmn[h]);
    const float xx = qmax4(st.xmx[h]), xn = qmin4(st.xmn[h]);
    int inf = 0;
    if constexpr (VS) {
      const float Rm = fmaxf(fabsf(kx), fabsf(kn));
      // |key - r64| <= 2^-18 |r| + 2^-24 |r| + 2^-23 |m|: window of twice that
      const float tolx = 1.52587890625e-05f * Rm + 4.76837158203125e-07f * pt.mabsr()[idx[h]];
      const float hib = kx - tolx, lob = kn + tolx;
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          win_or(cnt, r[h][j][e], hib, lob);  // r holds the keys
        }
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
      const uint32_t gm = 0xfu << (4 * g);
      const uint32_t bmx = __ballot_sync(0xffffffffu, st.kmx[h] == kx) & gm;
      const uint32_t bmn = __ballot_sync(0xffffffffu, st.kmn[h] == kn) & gm;
      if (cnt == 2 && hib > lob && __popc(bmx) == 1 && __popc(bmn) == 1) {  // disjoint windows
        const int qx = (__ffs(bmx) - 1) & 3, qn = (__ffs(bmn) - 1) & 3;
        const uint32_t ix = __float_as_uint(kx) & 31u, in_ = __float_as_uint(kn) & 31u;
        const int chx = 16 * (int)(ix >> 2) + 8 * (int)((ix >> 1) & 1) + 2 * qx + (int)(ix & 1);
        const int chn = 16 * (int)(in_ >> 2) + 8 * (int)((in_ >> 1) & 1) + 2 * qn + (int)(in_ & 1);
        inf = 1 | (chx << 1) | (chn << 8);
      }
    }
    __syncwarp();  // every lane's reads of this token's kmx/kmn (stage D) precede the store
    if (q == 0) {
      const int t = t0 + 8 * h;
      sc.kmx()[t] = kx; sc.kmn()[t] = kn; sc.xmx()[t] = xx; sc.xmn()[t] = xn;
      if constexpr (VS) sc.info()[t] = inf;
    }
  }
}

// ---------------------------------------------------------------------------------------
// token stage of one warp over its 32 tokens (its TMEM lane quarter): guess, exact lower
// bounds, survivors, fp64 re-match.  Leaves the final pattern index in sc.fidx() and the
// keyed statistics of the final residual in sc.kmx()/kmn/xmx/xmn(/info).
// ---------------------------------------------------------------------------------------
// A non-finite score row means a non-finite x element: every pattern column accumulates
// x_c * m'_c over all channels and Inf * 0 = NaN, while finite fp16 x and m' cannot overflow
// fp32 (|x.m'| <= 128 * 65504^2).  Rare path: scan the token's row for the first bad channel.
__device__ __noinline__ void nonfinite_row(const unsigned char* X, int t, bool flagged, int side, int u,
                                           int64_t start, unsigned long long* bad) {
  SMEM_PTR(X);
  if (!flagged) return;
  for (int ch = 0; ch < 128; ++ch)
    if (!isfinite(xt_at(X, t, ch))) {
      atomicMin(bad, nf_key(u, side, start + t, ch));
      return;
    }
}

template <int SIDE>
__device__ __noinline__ void token_stage(Scr sc, Pat pt, const unsigned char* X, const float* M,
                                         uint64_t* mmab, uint32_t ph, uint32_t tcol, int w, int lane, int P, float pmx,
                                         const double* p64, unsigned* stats, int u, int64_t start, int L,
                                         unsigned long long* bad) {
  SMEM_PTR(X); SMEM_PTR(M); SMEM_PTR(pt.base); SMEM_PTR(sc.base);
  warp_converged();
  const int g = lane >> 2, q = lane & 3;
  const int tt_ = 32 * w + lane;  // this thread's token in stages A/C
  const uint32_t tl = tcol + ((uint32_t)(32 * w) << 16);
  // ---- A. guess = argmin_p ||m'_p||^2 - 2 x.m'_p --------------------------------------
  mbar_wait(mmab, ph);
  tc_fence_after();
  float best = FE_INF;
#pragma unroll
  for (int p0 = 0; p0 < 32; p0 += 16) {
    uint32_t v[8], v2[8];
    tmem_ld8(tl + p0, v);
    tmem_ld8(tl + p0 + 8, v2);
    tmem_ld_wait();
    if (p0 == 0) {  // fused finiteness check of the token's x row (engine.py:136-138)
      const bool nf = !(fabsf(__uint_as_float(v[0])) <= 3.0e38f);
      if (__any_sync(0xffffffffu, nf)) nonfinite_row(X, tt_, nf && tt_ < L, SIDE, u, start, bad);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      best = fminf(best, fkey(__fmaf_rn(-2.f, __uint_as_float(v[i]), pt.bb()[p0 + i]), p0 + i, 0xffffffe0u));
      best = fminf(best, fkey(__fmaf_rn(-2.f, __uint_as_float(v2[i]), pt.bb()[p0 + 8 + i]), p0 + 8 + i, 0xffffffe0u));
    }
  }
  int guess = (int)(__float_as_uint(best) & 31u);
  if (guess >= P) guess = 0;
  const float Cg = best;
  float x4[NPRB];  // K: x at the probe channels
  if constexpr (SIDE == 0) {
#pragma unroll
    for (int j = 0; j < NPRB; ++j) x4[j] = xt_at(X, tt_, pt.flags()[2 + j]);
  }
  sc.guess()[tt_] = guess;
  __syncwarp();
  // ---- B. keyed residual extrema against the guess, per 16-token tile -----------------
#pragma unroll 1
  for (int tile = 0; tile < 2; ++tile) {
    const int tb = 32 * w + 16 * tile;
    b_tile<SIDE == 1>(X, M, pt, sc, tb, lane, sc.guess()[tb + g], sc.guess()[tb + g + 8]);
  }
  __syncwarp();
  // ---- C. prune every other pattern by an exact lower bound (thread per token) --------
  // K: the range of the residual over the NPRB widest-spread channels (d_mm >= that range;
  //    the Popoviciu bound rarely prunes K).  V: Popoviciu from the GEMM.
  {
    const float kx = sc.kmx()[tt_], kn = sc.kmn()[tt_];
    const float dg = __fsub_rn(kx, kn), xa = fmaxf(fabsf(sc.xmx()[tt_]), fabsf(sc.xmn()[tt_]));
    const float T2 = derr(kx, kn, pt.mabsr()[guess]);  // >= |dg - d64(guess)|
    const float dhi = __fadd_rn(dg, T2) * 1.0000002f;
    uint32_t mask = 0;
    if constexpr (SIDE == 0) {
      // |r32 - r64| <= 2^-23 (|x| + |m|) per probe residual, + 2^-24 relative on the range:
      // inside the 2^-21 (|x|max + |m|max) slack
      const float pb = __fadd_rn(dhi, 4.76837158203125e-07f * (xa + pmx));
      // the first 4 probes prune almost every (token, pattern); the rest are evaluated only
      // when a lane of the warp still keeps the pattern
#pragma unroll 4
      for (int p = 0; p < 32; ++p) {
        const float4 m4 = *reinterpret_cast<const float4*>(pt.pm4() + NPRB * p);
        const float r0 = __fsub_rn(x4[0], m4.x), r1 = __fsub_rn(x4[1], m4.y);
        const float r2 = __fsub_rn(x4[2], m4.z), r3 = __fsub_rn(x4[3], m4.w);
        float hi = fmaxf(fmax3(r0, r1, r2), r3), lo = fminf(fmin3(r0, r1, r2), r3);
        bool keep = __fsub_rn(hi, lo) <= pb && p < P;
        if (__any_sync(0xffffffffu, keep)) {
#pragma unroll
          for (int j = 4; j < NPRB; j += 4) {
            const float4 n4 = *reinterpret_cast<const float4*>(pt.pm4() + NPRB * p + j);
            const float s0 = __fsub_rn(x4[j], n4.x), s1 = __fsub_rn(x4[j + 1], n4.y);
            const float s2 = __fsub_rn(x4[j + 2], n4.z), s3 = __fsub_rn(x4[j + 3], n4.w);
            hi = fmaxf(hi, fmax3(s0, s1, s2)); hi = fmaxf(hi, s3);
            lo = fminf(lo, fmin3(s0, s1, s2)); lo = fminf(lo, s3);
          }
          keep = keep && __fsub_rn(hi, lo) <= pb;
        }
        mask |= (uint32_t)keep << p;
      }
    } else {
      const float dlo = fmaxf(__fsub_rn(dg, T2), 0.f) * 0.9999998f;
      // Popoviciu: osc^2 >= 4 C / d; C_q >= C'_q - C'_g + C_g, C_g >= osc_g^2 / 2
      const float theta = __fmaf_rn(32.f * dhi, dhi, -0.5f * dlo * dlo) * 1.000001f;
      const float kap = TWO_M13 * 11.3137085f * xa;  // 2 x (tensor-core + split error) / ||m'||, ||x|| <= sqrt(d) |x|max
      const float rhs = theta + Cg + kap * pt.mn()[guess] + TWO_M17 * fabsf(Cg);
      const bool nol2 = pt.flags()[1] != 0;
#pragma unroll 1
      for (int p0 = 0; p0 < 32; p0 += 8) {
        uint32_t v[8];
        tmem_ld8(tl + p0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int p = p0 + i;
          const float bbp = pt.bb()[p];
          const float cp = __fmaf_rn(-2.f, __uint_as_float(v[i]), bbp);
          const float lhs = __fmaf_rn(-TWO_M22, bbp, __fmaf_rn(-kap, pt.mn()[p], __fmaf_rn(-TWO_M17, fabsf(cp), cp)));
          mask |= (uint32_t)((nol2 || !(lhs > rhs)) && p < P) << p;
        }
      }
    }
    tc_fence_before();
    mask &= ~(1u << guess);
    sc.cand()[tt_] = mask;
    if (stats && mask) atomicAdd(&stats[2], (unsigned)__popc(mask));
  }
  __syncwarp();
  // ---- D. survivors: full fp32 distance, top-2 with error bounds, fp64 re-match ---------
#pragma unroll 1
  for (int tile = 0; tile < 2; ++tile) {
    const int tb = 32 * w + 16 * tile, t0 = tb + g;
    const int gi[2] = {sc.guess()[t0], sc.guess()[t0 + 8]};
    int idx[2] = {gi[0], gi[1]};
    uint32_t cm[2] = {sc.cand()[t0], sc.cand()[t0 + 8]};
    if (__any_sync(0xffffffffu, (cm[0] | cm[1]) != 0)) {
      float bst[2], bstE[2], low[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float kx = sc.kmx()[t0 + 8 * h], kn = sc.kmn()[t0 + 8 * h];
        bst[h] = __fsub_rn(kx, kn);
        bstE[h] = derr(kx, kn, pt.mabsr()[gi[h]]);
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
        cand_stats(X, M, tb, lane, pc[0] >= 0 ? pc[0] : gi[0], pc[1] >= 0 ? pc[1] : gi[1], s4);
        warp_converged();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float cx = qmax4(s4[2 * h]), cn = qmin4(s4[2 * h + 1]);
          if (pc[h] >= 0) {
            const float d = __fsub_rn(cx, cn), e = derr(cx, cn, pt.mabsr()[pc[h]]);
            if (d < bst[h] || (d == bst[h] && pc[h] < idx[h])) {
              low[h] = fminf(low[h], bst[h] - bstE[h]);
              bst[h] = d; bstE[h] = e; idx[h] = pc[h];
            } else {
              low[h] = fminf(low[h], d - e);
            }
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool amb = low[h] <= bst[h] + bstE[h];
        if (__any_sync(0xffffffffu, amb)) {
          const int ri = refine64(X, t0 + 8 * h, p64, P, q);
          if (amb) {
            idx[h] = ri;
            if (stats && q == 0) atomicAdd(&stats[0], 1u);
          }
        }
      }
      // statistics of the final residual where the winner moved
      if (__any_sync(0xffffffffu, idx[0] != gi[0] || idx[1] != gi[1])) {
        b_tile<SIDE == 1>(X, M, pt, sc, tb, lane, idx[0], idx[1]);
      }
    }
    __syncwarp();  // the tile's guess/cand reads precede their reuse as row offsets
    if (q == 0) {
      sc.fidx()[t0] = idx[0]; sc.fidx()[t0 + 8] = idx[1];
      if constexpr (SIDE == 0) {  // K: the final row's float offsets for even / odd channel chunks
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int pp = idx[h], pl = pp & 1;
          sc.guess()[t0 + 8 * h] = pp * 128 + 4 * pl;  // mslot: (c ^ pl) = c + pl for even c
          reinterpret_cast<int*>(sc.cand())[t0 + 8 * h] = pp * 128 - 4 * pl;  // c - pl for odd c
        }
      }
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------------------
// K: per-channel groups over the span's 128 tokens.  Warp w takes channel chunks 2w, 2w+1;
// in a chunk lane (g, q) holds channels 16jb + 2q + {0,1,8,9} of tokens 16tt + 8h + g.
// ---------------------------------------------------------------------------------------
// r of the lane's 16 tokens x 4 channels of chunk jb (NaN for tokens past the span)
template <bool FULL>
__device__ __forceinline__ void k_load(const unsigned char* X, const float* M, const int (&fi)[16], int jb, int g,
                                       int q, int L, float (&rr)[16][4]) {
  const int c0 = 16 * jb + 2 * q;
  const int hsel = (c0 >> 6) * 16384, ck = (c0 & 63) >> 3, cw = (c0 & 7) << 1;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int t = 16 * (e >> 1) + 8 * (e & 1) + g;
    const unsigned char* rowp = X + hsel + t * 128 + cw;
    const uint32_t xa = *reinterpret_cast<const uint32_t*>(rowp + ((ck ^ (t & 7)) << 4));
    const uint32_t xb = *reinterpret_cast<const uint32_t*>(rowp + (((ck + 1) ^ (t & 7)) << 4));
    // mslot(p, q, jb) = q*32 + 4 ((jb ^ 2q) & 7) + (+-4 (p & 1), folded into fi[e])
    const float4 m = *reinterpret_cast<const float4*>(M + fi[e] + q * 32 + 4 * ((jb ^ (2 * q)) & 7));
    rr[e][0] = subh_lo(xa, m.x); rr[e][1] = subh_hi(xa, m.y); rr[e][2] = subh_lo(xb, m.z); rr[e][3] = subh_hi(xb, m.w);
    if (!FULL && t >= L) rr[e][0] = rr[e][1] = rr[e][2] = rr[e][3] = FE_NAN;
  }
}
// K pass of chunk jb: keyed extrema per channel, window counts and unique owners (for the
// exact fp64 params of the scalar pass) and the codes, from fp32 params of the keyed extrema:
// their error (2^-19 |r| key precision + fp32 residual error) is inside the guard, so every
// code outside the guard band equals the reference's; guard-band pairs are returned (bit
// 2e + pr) for the exact fix-up once the fp64 params exist.  *anyslow: a channel of the chunk
// has several elements inside the fp32 error window of an extremum (k_slow resolves it).
template <int BITS, bool FULL>
__device__ __noinline__ uint32_t k_pass(const unsigned char* X, const float* M, Pat pt, Scr sc, int jb, int lane,
                                        int L, uint32_t* KW, uint32_t* wreg, int* anyslow) {
  SMEM_PTR(X); SMEM_PTR(M); SMEM_PTR(pt.base); SMEM_PTR(sc.base); SMEM_PTR(KW);
  warp_converged();
  constexpr int QMAX = (1 << BITS) - 1;
  constexpr int HS = 8 / BITS;
  const int g = lane >> 2, q = lane & 3;
  // per token: float offset of its pattern row (token stage D), parity-adjusted for this chunk
  const int* moff = (jb & 1) ? reinterpret_cast<const int*>(sc.cand()) : sc.guess();
  int fi[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) fi[e] = moff[16 * (e >> 1) + 8 * (e & 1) + g];
  float rr[16][4];
  k_load<FULL>(X, M, fi, jb, g, q, L, rr);
  // keys replace r from here on: the codes below absorb their 2^-19 |r| error in the guard
#pragma unroll
  for (int e = 0; e < 16; ++e)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) rr[e][kk] = fkey(rr[e][kk], e, 0xfffffff0u);
  // all warp collectives first (no divergent code between them), then the per-channel results
  float lmx[4], lmn[4], gmx[4], gmn[4], hib[4], lob[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    lmx[kk] = -FE_INF; lmn[kk] = FE_INF;
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
      lmx[kk] = fmax3(lmx[kk], rr[e][kk], rr[e + 1][kk]);
      lmn[kk] = fmin3(lmn[kk], rr[e][kk], rr[e + 1][kk]);
    }
    gmx[kk] = lmx[kk]; gmn[kk] = lmn[kk];
  }
#pragma unroll
  for (int o = 4; o <= 16; o <<= 1)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      gmx[kk] = fmaxf(gmx[kk], __shfl_xor_sync(0xffffffffu, gmx[kk], o));
      gmn[kk] = fminf(gmn[kk], __shfl_xor_sync(0xffffffffu, gmn[kk], o));
    }
  int cnt[4];
  float qlo[4], qinv[4], qhg[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int ch = 16 * jb + 2 * q + (kk & 1) + 8 * (kk >> 1);
    const float Rm = fmaxf(fabsf(gmx[kk]), fabsf(gmn[kk])), Mc = pt.mabsc()[ch];
    // |key - r64| <= 2^-19 |r| + 2^-24 |r| + 2^-23 |m|: window of twice that
    const float tolx = TWO_M17 * Rm + 4.76837158203125e-07f * Mc;
    hib[kk] = gmx[kk] - tolx; lob[kk] = gmn[kk] + tolx;
    // elements in either window (one predicate per element); equals the two windows' total
    // count when they are disjoint (hib > lob, required by the fast test below)
    cnt[kk] = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) win_or(cnt[kk], rr[e][kk], hib[kk], lob[kk]);
    // fp32 params from the keyed extrema, codes from the keys; |y - y_exact| <= inv (4 2^-19 R +
    // 2^-21 (R + M) + 2^-23 span)
    // + qmax 2^-22 + 2^-24, doubled (K1-TC)
    const float span = __fsub_rn(gmx[kk], gmn[kk]);
    qlo[kk] = gmn[kk];
    if (span > 4.f * (3.814697265625e-06f * Rm + 4.76837158203125e-07f * (Rm + Mc))) {
      qinv[kk] = (float)QMAX * rcp_approx(span);
      qhg[kk] = 0.5f - (qinv[kk] * (1.52587890625e-05f * Rm + 9.5367431640625e-07f * (Rm + Mc) +
                                    2.384185791015625e-07f * span) +
                        4.76837158203125e-07f * (float)QMAX + 1.1920928955078125e-07f);
    } else {  // (nearly) constant group: every code exact
      qinv[kk] = 0.f;
      qhg[kk] = -1.f;
    }
  }
#pragma unroll
  for (int o = 4; o <= 16; o <<= 1)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) cnt[kk] += __shfl_xor_sync(0xffffffffu, cnt[kk], o);
  const uint32_t qm = 0x11111111u << q;
  uint32_t bmx[4], bmn[4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    bmx[kk] = __ballot_sync(0xffffffffu, lmx[kk] == gmx[kk]) & qm;
    bmn[kk] = __ballot_sync(0xffffffffu, lmn[kk] == gmn[kk]) & qm;
  }
  bool slow = false;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int ch = 16 * jb + 2 * q + (kk & 1) + 8 * (kk >> 1);
    const bool fast = cnt[kk] == 2 && hib[kk] > lob[kk] && __popc(bmx[kk]) == 1 && __popc(bmn[kk]) == 1;
    const int gx = (__ffs(bmx[kk]) - 1) >> 2, gn = (__ffs(bmn[kk]) - 1) >> 2;
    const uint32_t ix = __float_as_uint(gmx[kk]) & 15u, in_ = __float_as_uint(gmn[kk]) & 15u;
    const int tx = 16 * (int)(ix >> 1) + 8 * (int)(ix & 1) + gx;
    const int tn = 16 * (int)(in_ >> 1) + 8 * (int)(in_ & 1) + gn;
    const int inf = fast ? (1 | (tx << 1) | (tn << 8)) : 0;
    slow |= !fast;
    if (g == 0) {
      sc.kmx()[ch] = gmx[kk]; sc.kmn()[ch] = gmn[kk];
      sc.info()[ch] = inf;
    }
  }
  *anyslow = __any_sync(0xffffffffu, slow);
  // codes (pairs of channels c0+{0,1} / c0+{8,9} per token) -> K fragment words
  const int slot0 = 2 * (jb % HS);
  const int wbase = 2 * (jb / HS);
  uint32_t badm = 0;
  const float2 nlo01 = make_float2(-qlo[0], -qlo[1]), nlo23 = make_float2(-qlo[2], -qlo[3]);
  const float2 inv01 = make_float2(qinv[0], qinv[1]), inv23 = make_float2(qinv[2], qinv[3]);
  const float2 nhg01 = make_float2(-qhg[0], -qhg[1]), nhg23 = make_float2(-qhg[2], -qhg[3]);
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int t = 16 * (e >> 1) + 8 * (e & 1) + g;
    bool bad0 = false, bad1 = false;
    const float2 z01 = zcode2(make_float2(rr[e][0], rr[e][1]), nlo01, inv01, nhg01, bad0);
    const float2 z23 = zcode2(make_float2(rr[e][2], rr[e][3]), nlo23, inv23, nhg23, bad1);
    uint32_t p0 = zpair(z01.x, z01.y), p1 = zpair(z23.x, z23.y);
    if (!FULL && t >= L) { p0 = 0u; p1 = 0u; bad0 = bad1 = false; }
    badm |= ((uint32_t)bad0 << (2 * e)) | ((uint32_t)bad1 << (2 * e + 1));
    const uint32_t part = (p0 << (slot0 * BITS)) | (p1 << ((slot0 + 1) * BITS));
    if constexpr (BITS == 2) {
      atomicOr(&KW[((e >> 1) * 32 + lane) * 4 + (((e & 1) + wbase) ^ ((lane >> 3) & 3))], part);
    } else {
      wreg[e] |= part;
    }
  }
  return badm;
}
// Guard-band pairs of chunk jb (bits of badm).  The common route defers them to kfix_kernel
// (k_defer below, in line at the call site); this exact in-line fix runs only for pairs the
// full fix list could not take.  2 bits: into the shared code words KW before they are copied
// out; 4 bits: into the lane's own global code words right after it stored them (the register
// words are never passed by pointer -- that put them in local memory for the whole K pass).
template <int BITS>
__device__ __noinline__ void k_fix(const double* kparam64, const Scr sc, int jb, int lane, uint32_t badm,
                                   const __half* xsrc, const double* p64, int64_t blk, uint32_t* KW, uint32_t* gw,
                                   unsigned* stats) {
  SMEM_PTR(sc.base);
  constexpr int QMAX = (1 << BITS) - 1;
  constexpr int HS = 8 / BITS;
  constexpr int WLK = 16 * BITS / 8;
  const int g = lane >> 2, q = lane & 3;
  const int c0 = 16 * jb + 2 * q;
  const int slot0 = 2 * (jb % HS), wbase = 2 * (jb / HS);
  const double* kp = kparam64 + blk * 256;
  while (badm) {
    const int bit = __ffs(badm) - 1;
    badm &= badm - 1;
    const int e = bit >> 1, pr = bit & 1;
    const int t = 16 * (e >> 1) + 8 * (e & 1) + g, ch = c0 + 8 * pr;
    const double* mrow = p64 + (int64_t)sc.fidx()[t] * 128;
    const __half* xrow = xsrc + (int64_t)t * 128;
    const uint32_t pv = exact_code_p(xrow + ch, mrow + ch, kp + 128 + ch, kp + ch, QMAX) |
                        (exact_code_p(xrow + ch + 1, mrow + ch + 1, kp + 128 + ch + 1, kp + ch + 1, QMAX) << 16);
    const int sh = (slot0 + pr) * BITS;
    const uint32_t clr = ~(((uint32_t)QMAX | ((uint32_t)QMAX << 16)) << sh);
    uint32_t* wp = BITS == 2 ? &KW[((e >> 1) * 32 + lane) * 4 + (((e & 1) + wbase) ^ ((lane >> 3) & 3))]
                             : gw + ((e >> 1) * 32 + lane) * WLK + (e & 1) + wbase;
    atomicAnd(wp, clr);
    atomicOr(wp, pv << sh);
    if (stats) atomicAdd(&stats[1], 1u);
  }
}
// the deferral itself: one 64-bit entry per pair (block, token, channel, global word, shift),
// one slot each from the cache's counter; returns the pairs the full list did not take
template <int BITS>
__device__ __forceinline__ uint32_t k_defer(uint32_t badm, int jb, int lane, int64_t blk, unsigned long long* fix,
                                            int fixcap, int* fixcnt) {
  constexpr int HS = 8 / BITS;
  constexpr int WLK = 16 * BITS / 8;
  const int g = lane >> 2, q = lane & 3;
  const int slot0 = 2 * (jb % HS), wbase = 2 * (jb / HS);
  // slots: one atomic per warp for all of its lanes' pairs (every lane calls)
  const int n = __popc(badm);
  if (!__any_sync(0xffffffffu, n != 0)) return 0u;
  int incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int base = 0;
  if (lane == 31) base = fix ? atomicAdd(fixcnt, incl) : fixcap;
  int slot = __shfl_sync(0xffffffffu, base, 31) + incl - n;
  while (badm) {
    const int bit = __ffs(badm) - 1;
    if (slot >= fixcap) return badm;
    badm &= badm - 1;
    const int e = bit >> 1, pr = bit & 1;
    const int t = 16 * (e >> 1) + 8 * (e & 1) + g, ch = 16 * jb + 2 * q + 8 * pr;
    const int word = ((e >> 1) * 32 + lane) * WLK + (e & 1) + wbase;
    fix[slot++] = (unsigned long long)(uint32_t)blk | ((unsigned long long)t << 32) | ((unsigned long long)ch << 39) |
                  ((unsigned long long)word << 46) | ((unsigned long long)((slot0 + pr) * BITS) << 58);
  }
  return 0u;
}
// groups of chunk jb with several elements inside the fp32 error window: exact fp64 extrema
// over the window, stored as double halves in (kmx, xmx) / (kmn, xmn) with info = 1 << 16.
// Only the slow channels are visited, each by the whole warp (lane = 4 tokens), so a chunk
// with one slow channel costs 4 element steps per lane instead of 16 per channel quad.
template <bool FULL>
__device__ __noinline__ void k_slow(const unsigned char* X, const float* M, Pat pt, Scr sc, int jb, int lane, int L,
                                    const double* p64, unsigned* stats) {
  SMEM_PTR(X); SMEM_PTR(M); SMEM_PTR(pt.base); SMEM_PTR(sc.base);
  warp_converged();
  uint32_t todo = __ballot_sync(0xffffffffu, lane < 16 && !(sc.info()[16 * jb + (lane & 15)] & 1)) & 0xffffu;
  __syncwarp();  // every lane's info read precedes the stores below
#pragma unroll 1
  while (todo) {
    const int cc = __ffs(todo) - 1;
    todo &= todo - 1;
    const int ch = 16 * jb + cc;
    const float gmx = sc.kmx()[ch], gmn = sc.kmn()[ch];
    const float Rm = fmaxf(fabsf(gmx), fabsf(gmn));
    const float tolx = TWO_M17 * Rm + 4.76837158203125e-07f * pt.mabsc()[ch];
    const float hib = gmx - tolx, lob = gmn + tolx;
    // the channel's slot in k_pass's layout: ch = 16 jb + 2q + {0,1,8,9}
    const int q = (ch >> 1) & 3, k4 = 2 * ((ch >> 3) & 1) + (ch & 1);
    double dmx = -__longlong_as_double(0x7ff0000000000000LL), dmn = -dmx;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = lane + 32 * i;
      const int e = 2 * (t >> 4) + ((t >> 3) & 1);  // k_pass element index of token t (key bits)
      const int p = sc.fidx()[t];
      const float xv = xt_at(X, t, ch);
      const float key = fkey(__fsub_rn(xv, M[p * 128 + mslot(p, q, jb) + k4]), (uint32_t)e, 0xfffffff0u);
      const bool in = (FULL || t < L) && (key >= hib || key <= lob);
      const double v64 = in ? __dsub_rn((double)xv, p64[(int64_t)p * 128 + ch]) : 0.0;
      if (in && key >= hib) dmx = fmax(dmx, v64);
      if (in && key <= lob) dmn = fmin(dmn, v64);
    }
#pragma unroll
    for (int o = 1; o <= 16; o <<= 1) {
      dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
      dmn = fmin(dmn, __shfl_xor_sync(0xffffffffu, dmn, o));
    }
    __syncwarp();  // every lane's kmx / kmn reads of this channel precede the store
    if (lane == 0) {
      sc.kmx()[ch] = __int_as_float(__double2hiint(dmx)); sc.xmx()[ch] = __int_as_float(__double2loint(dmx));
      sc.kmn()[ch] = __int_as_float(__double2hiint(dmn)); sc.xmn()[ch] = __int_as_float(__double2loint(dmn));
      sc.info()[ch] = 1 << 16;
      if (stats) atomicAdd(&stats[3], 1u);
    }
  }
}
// K scalar pass: one thread per channel -- exact fp64 extrema, params, fast-path constants
template <int BITS>
__device__ __forceinline__ void k_scalar(const Args& A, const unsigned char* X, const float* M, const Pat& pt,
                                         const Scr& sc, int ch, int L, const double* p64, int64_t blk,
                                         unsigned* stats) {
  const DevCache& c = A.c;
  const float gmx = sc.kmx()[ch], gmn = sc.kmn()[ch];
  const int inf = sc.info()[ch];
  const float Rm = fmaxf(fabsf(gmx), fabsf(gmn)), Mc = pt.mabsc()[ch];
  double hi64, lo64;
  float R = Rm;
  if (inf & 1) {
    const int tx = (inf >> 1) & 127, tn = (inf >> 8) & 127;
    hi64 = __dsub_rn((double)xt_at(X, tx, ch), p64[(int64_t)sc.fidx()[tx] * 128 + ch]);
    lo64 = __dsub_rn((double)xt_at(X, tn, ch), p64[(int64_t)sc.fidx()[tn] * 128 + ch]);
  } else {  // exact extrema from the slow pass (info == 1 << 16)
    hi64 = __hiloint2double(__float_as_int(gmx), __float_as_int(sc.xmx()[ch]));
    lo64 = __hiloint2double(__float_as_int(gmn), __float_as_int(sc.xmn()[ch]));
    R = fmaxf(fabsf((float)hi64), fabsf((float)lo64));
  }
  const GroupQ gg = make_group(lo64, hi64, (1 << BITS) - 1, A.yq, R, Mc);
  sc.lo32()[ch] = gg.lo32; sc.inv()[ch] = gg.inv; sc.hg()[ch] = gg.hg;
  c.kparam64[blk * 256 + ch] = gg.scale;
  c.kparam64[blk * 256 + 128 + ch] = gg.lo;
  c.kparam32[blk * 2 * c.Dp + ch] = (float)gg.scale;
  c.kparam32[blk * 2 * c.Dp + c.Dp + ch] = (float)gg.lo;
}
// ---------------------------------------------------------------------------------------
// V: per-token groups over channels
// ---------------------------------------------------------------------------------------
// scalar pass: one thread per token -- exact fp64 extrema, gate, params, fast-path constants
template <int BITS>
__device__ __forceinline__ void v_scalar(const Args& A, const unsigned char* X, const float* M, const Pat& pt,
                                         const Scr& sc, int t, int L, int64_t start, int u, int64_t blk,
                                         const double* p64, unsigned* stats) {
  const DevCache& c = A.c;
  const int idx = sc.fidx()[t];
  const float kx = sc.kmx()[t], kn = sc.kmn()[t], xx = sc.xmx()[t], xn = sc.xmn()[t];
  int inf = sc.info()[t];
  const float xa = fmaxf(fabsf(xx), fabsf(xn)), Mr = pt.mabsr()[idx];
  const float Rm = fmaxf(fabsf(kx), fabsf(kn));
  const double* mrow = p64 + (int64_t)idx * 128;
  double hi64, lo64;
  if (inf & 1) {
    const int chx = (inf >> 1) & 127, chn = (inf >> 8) & 127;
    hi64 = __dsub_rn((double)xt_at(X, t, chx), mrow[chx]);
    lo64 = __dsub_rn((double)xt_at(X, t, chn), mrow[chn]);
  } else {
    const float tolx = 1.52587890625e-05f * Rm + 4.76837158203125e-07f * Mr;
    v_exact_slow(X, M, t, idx, mrow, kx - tolx, kn + tolx, &hi64, &lo64);
    if (stats && t < L) atomicAdd(&stats[3], 1u);
  }
  // gate (gate.py:180-188; --no-v-gate flattens, engine.py:235-237)
  const double raw = __dsub_rn((double)xx, (double)xn);
  const double flat = __dsub_rn(hi64, lo64);
  const bool flatten = c.use_vgate ? (raw > 0.0 && gate_le(flat, raw, c.thr)) : true;
  const GroupQ gq = flatten ? make_group(lo64, hi64, (1 << BITS) - 1, A.yq, Rm, Mr)
                            : make_group((double)xn, (double)xx, (1 << BITS) - 1, A.yq, xa, 0.f);
  sc.lo32()[t] = gq.lo32; sc.inv()[t] = gq.inv; sc.hg()[t] = gq.hg;
  sc.info()[t] = inf | (flatten ? (1 << 15) : 0);
  if (t < L) {
    const int64_t tok = (int64_t)u * c.Tcap + start + t;
    const int64_t slot = blk * c.GP + t;
    c.vparam64[2 * tok] = gq.scale;
    c.vparam64[2 * tok + 1] = gq.lo;
    c.vparam32[2 * slot] = (float)gq.scale;
    c.vparam32[2 * slot + 1] = (float)gq.lo;
    c.vidx[slot] = (int16_t)(flatten ? idx : RAW);
    if (c.keep_diag && c.vdiag) { c.vdiag[2 * tok] = raw; c.vdiag[2 * tok + 1] = flat; }
  }
}
// codes pass of two 8-token row-sets (rows rb + g and rb + 8 + g, rb a multiple of 16): codes,
// exact fix-ups, movmatrix to the V^T fragment layout, the two row-sets' interleaved words of
// the tile in one 64-bit store each (two independent row-sets per call: twice the ILP of one)
template <int BITS>
__device__ __noinline__ void v_codes(uint8_t* vcodes, const double* vparam64, int blk_bytes, int64_t Tcap,
                                     const unsigned char* X, const float* M, Scr sc, int rb, int lane, int L, int u,
                                     int64_t start, int64_t blk, const __half* xsrc, const double* p64,
                                     unsigned* stats, unsigned long long* fix, int fixcap, int* fixcnt) {
  SMEM_PTR(X); SMEM_PTR(M); SMEM_PTR(sc.base);
  constexpr int QMAX = (1 << BITS) - 1;
  constexpr int HS = 8 / BITS;
  constexpr int WL = 128 * BITS / 64;
  const int g = lane >> 2, q = lane & 3;
  uint32_t pp[2][16];
  uint32_t badm[2];
  int idx[2];
  bool flatten[2];
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    const int t = rb + 8 * n + g;
    idx[n] = sc.fidx()[t];
    flatten[n] = (sc.info()[t] >> 15) & 1;
    const float lo32 = sc.lo32()[t], inv = sc.inv()[t], hg = sc.hg()[t];
    float r[8][4];
    float d0, d1, d2, d3;
    resid_row(X, M, rb + 8 * n, lane, idx[n], r, d0, d1, d2, d3);
    if (!flatten[n]) {  // RAW payload: the exact input row (rare)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) r[j][e] = xt_at(X, t, 16 * j + 8 * (e >> 1) + 2 * q + (e & 1));
    }
    badm[n] = 0;
    const float2 nlo2 = make_float2(-lo32, -lo32), inv2 = make_float2(inv, inv);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      bool bad0 = false, bad1 = false;
      const float2 z01 = zcode2s(make_float2(r[j][0], r[j][1]), nlo2, inv2, hg, bad0);
      const float2 z23 = zcode2s(make_float2(r[j][2], r[j][3]), nlo2, inv2, hg, bad1);
      pp[n][2 * j] = zpair(z01.x, z01.y);
      pp[n][2 * j + 1] = zpair(z23.x, z23.y);
      badm[n] |= ((uint32_t)bad0 << (2 * j)) | ((uint32_t)bad1 << (2 * j + 1));
    }
    if (t >= L) {
      badm[n] = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) pp[n][i] = 0u;
    }
  }
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    if (badm[n]) {  // rare: the reference's fp64 sequence decides inside the guard band (deferred
                    // to kfix_kernel through the fix list; in line when the list is full)
      const int t = rb + 8 * n + g;
      const double* mr = flatten[n] ? p64 + (int64_t)idx[n] * 128 : nullptr;
      const __half* xrow = xsrc + (int64_t)t * 128;
      const double* vp = vparam64 + 2 * ((int64_t)u * Tcap + start + t);
      uint32_t bm = badm[n];
#pragma unroll 1
      while (bm) {
        const int i = __ffs(bm) - 1;
        bm &= bm - 1;
        const int ca = 16 * (i >> 1) + 8 * (i & 1) + 2 * q;
        const int fs = fix ? atomicAdd(fixcnt, 1) : fixcap;
        if (fs < fixcap) {  // V entry: block, token, first channel of the pair, side bit 63
          fix[fs] = (unsigned long long)(uint32_t)blk | ((unsigned long long)t << 32) | ((unsigned long long)ca << 39) |
                    (1ull << 63);
          continue;
        }
        const uint32_t pv = exact_code_p(xrow + ca, mr ? mr + ca : nullptr, vp + 1, vp, QMAX) |
                            (exact_code_p(xrow + ca + 1, mr ? mr + ca + 1 : nullptr, vp + 1, vp, QMAX) << 16);
#pragma unroll
        for (int k2 = 0; k2 < 16; ++k2) pp[n][k2] = k2 == i ? pv : pp[n][k2];
        if (stats) atomicAdd(&stats[1], 1u);
      }
    }
  }
  uint32_t words[2][WL / 2];
#pragma unroll
  for (int n = 0; n < 2; ++n) {
#pragma unroll
    for (int i = 0; i < WL / 2; ++i) words[n][i] = 0u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t t0v = movm_t(pp[n][2 * j]), t1v = movm_t(pp[n][2 * j + 1]);  // hiRow 0 / 1 of sub-tile j
      const int s0 = 2 * (j % HS);
      words[n][j / HS] |= (t0v << (s0 * BITS)) | (t1v << ((s0 + 1) * BITS));
    }
  }
  uint2* dst = reinterpret_cast<uint2*>(vcodes + blk * blk_bytes + (size_t)((rb >> 4) * 32 + lane) * WL * 4);
#pragma unroll
  for (int i = 0; i < WL / 2; ++i) dst[i] = make_uint2(words[0][i], words[1][i]);
}

// ---------------------------------------------------------------------------------------
// one subgroup (4 warps) of a side: its items of every unit in the CTA's range
// ---------------------------------------------------------------------------------------
template <int BITS, int SIDE>
__device__ __forceinline__ void run_sub(const Args& A, unsigned char* sb, const CUtensorMap* tm, uint32_t tmem,
                                        uint32_t& k) {
  const DevCache& c = A.c;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sg = warp >> 2, w = warp & 3, sgi = sg;
  const int gtid = threadIdx.x, st = 32 * w + lane;
  unsigned char* X = sb + OFF_X + sgi * SZ_X;
  unsigned char* B = sb + OFF_B + SIDE * SZ_B;
  const float* M = reinterpret_cast<const float*>(sb + OFF_M + SIDE * SZ_M);
  uint32_t* KW = reinterpret_cast<uint32_t*>(sb + (sg < 2 ? OFF_KW + sg * SZ_KW : OFF_B + SZ_B + (sg - 2) * SZ_KW));
  uint64_t* xfull = reinterpret_cast<uint64_t*>(sb + OFF_BAR) + sgi;
  uint64_t* mmab = reinterpret_cast<uint64_t*>(sb + OFF_BAR + 32) + sgi;
  int* rel = reinterpret_cast<int*>(sb + OFF_BAR + 64) + sgi;
  Scr sc(sb, sgi);
  Pat pt(sb, SIDE);
  const int nb = A.nb;
  unsigned* stats = c.stats;
  int* ring = reinterpret_cast<int*>(sb + OFF_BAR + 96);
  auto chunk_items = [&](int ch, int64_t& b0, int64_t& b1) {
    b0 = b1 = 0;
    if (ch >= A.nchunks[SIDE]) return;
    const int uu = ch / A.cpu[SIDE], pc = ch % A.cpu[SIDE];
    b0 = (int64_t)uu * nb + pc * A.chunk[SIDE];
    b1 = (int64_t)uu * nb + min(nb, (pc + 1) * A.chunk[SIDE]);
  };
  const int64_t row0 = c.blk_start[A.first_block];
  auto issue = [&](int64_t item) {
    const int uu = (int)(item / nb);
    const int bb = A.first_block + (int)(item % nb);
    const int row = (int)(c.blk_start[bb] - row0);
    fence_proxy_async();
    mbar_arrive_expect_tx(xfull, 2 * 16384);
    tma_load_3d(X, tm, xfull, 0, row, uu);
    tma_load_3d(X + 16384, tm, xfull, 64, row, uu);
  };
  int staged = -1;
  // Items of a chunk: the first four statically (item i0 + sg, its TMA issued during the
  // previous chunk), the rest dynamically -- the last warp out of an item takes the chunk's next
  // item from a shared counter, issues its TMA and publishes it to the subgroup -- so the
  // subgroups finish a chunk together instead of waiting for the one with the costliest static
  // share (measured: ~1 item of idle per subgroup and 32-item chunk).
  int* cnext = reinterpret_cast<int*>(sb + OFF_BAR + 84);
  int* snext = reinterpret_cast<int*>(sb + OFF_BAR + 104) + sgi;
  int pending = -1;  // item whose TMA this subgroup already issued
  for (;;) {
    const int cur = ring[0], nx = ring[1];
    if (cur >= A.nchunks[SIDE]) break;
    int64_t i0, i1, j0, j1;
    chunk_items(cur, i0, i1);
    chunk_items(nx, j0, j1);
    const int u = cur / A.cpu[SIDE];
    if (u != staged) {
      stage_patterns(A, SIDE, u, sb, gtid);
      bar_side();
      staged = u;
    }
    const int P = pt.flags()[0];
    const float pmx = SIDE == 0 ? c.kpmax[u] : c.vpmax[u];
    const double* p64 = (SIDE == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * 128;
    for (int64_t it = i0 + sg; it < i1; ++k) {
      // first item of the chunk not prefetched: every warp is past the chunk barrier, x is free
      if (pending != (int)it && w == 0 && lane == 0) issue(it);
      const int b = A.first_block + (int)(it % nb);
      const uint32_t ph = k & 1;
      const uint32_t tcol = tmem + sgi * 64 + ph * 32;
      // span metadata: loads issued before the x wait, consumed after the token stage
      int L;
      int64_t start;
      asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(L) : "l"(c.blk_len + b));
      asm volatile("ld.global.nc.s64 %0, [%1];" : "=l"(start) : "l"(c.blk_start + b));
      mbar_wait(xfull, ph);
      if (w == 0 && lane == 0) {
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
      token_stage<SIDE>(sc, pt, X, M, mmab, ph, tcol, w, lane, P, pmx, p64, stats, u, start, L, c.bad);
      const __half* xsrc = A.src[SIDE] + (int64_t)u * A.unit_stride + (start - row0) * 128;
      const int64_t blk = (int64_t)u * c.NBcap + b;
      if constexpr (SIDE == 0) {
        bar_sub(sgi);  // every token's final pattern index
        if (st < L) c.kidx[blk * c.GP + st] = (int16_t)sc.fidx()[st];
        uint32_t wreg[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) wreg[e] = 0u;
        uint32_t badm[2];
        int slow[2];
#pragma unroll
        for (int jc = 0; jc < 2; ++jc)
          badm[jc] = L == 128 ? k_pass<BITS, true>(X, M, pt, sc, 2 * w + jc, lane, L, KW, wreg, &slow[jc])
                              : k_pass<BITS, false>(X, M, pt, sc, 2 * w + jc, lane, L, KW, wreg, &slow[jc]);
#pragma unroll
        for (int jc = 0; jc < 2; ++jc)
          if (slow[jc]) {
            __syncwarp();
            if (L == 128) k_slow<true>(X, M, pt, sc, 2 * w + jc, lane, L, p64, stats);
            else k_slow<false>(X, M, pt, sc, 2 * w + jc, lane, L, p64, stats);
          }
        bar_sub(sgi);  // per-channel statistics of all 128 channels
        k_scalar<BITS>(A, X, M, pt, sc, st, L, p64, blk, stats);
        bar_sub(sgi);  // per-channel fp64 params in HBM
        uint32_t ovf[2];
#pragma unroll
        for (int jc = 0; jc < 2; ++jc) ovf[jc] = k_defer<BITS>(badm[jc], 2 * w + jc, lane, blk, c.fix, c.fixcap, c.work + 2);
        uint32_t* gw = reinterpret_cast<uint32_t*>(c.kcodes + blk * c.blk_bytes);
        if constexpr (BITS == 2) {
#pragma unroll
          for (int jc = 0; jc < 2; ++jc)
            if (ovf[jc]) k_fix<BITS>(c.kparam64, sc, 2 * w + jc, lane, ovf[jc], xsrc, p64, blk, KW, gw, stats);
        } else {  // word h + 2w of lane (tile tt) holds chunks 2w, 2w+1
#pragma unroll
          for (int e = 0; e < 16; ++e) gw[((e >> 1) * 32 + lane) * 8 + (e & 1) + 2 * w] = wreg[e];
#pragma unroll
          for (int jc = 0; jc < 2; ++jc)
            if (ovf[jc]) k_fix<BITS>(c.kparam64, sc, 2 * w + jc, lane, ovf[jc], xsrc, p64, blk, KW, gw, stats);
        }
      } else {
        v_scalar<BITS>(A, X, M, pt, sc, st, L, start, u, blk, p64, stats);
        __syncwarp();
#pragma unroll 1
        for (int rs = 0; rs < 2; ++rs)
          v_codes<BITS>(c.vcodes, c.vparam64, c.blk_bytes, c.Tcap, X, M, sc, 32 * w + 16 * rs, lane, L, u, start, blk, xsrc,
                        p64, stats, c.fix, c.fixcap, c.work + 2);
      }
      // release the x tile; the last warp out takes the subgroup's next item (this chunk's
      // counter, else its static first item of the next chunk) and starts that span's TMA
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(rel, 1) == 3) {
          *rel = 0;
          const int nn = atomicAdd(cnext, 1);
          const int64_t nxt = nn < i1 ? nn : (j0 + sg < j1 ? j0 + sg : -1);
          *snext = nn < i1 ? nn : 0x7fffffff;
          if (nxt >= 0) issue(nxt);
        }
      }
      bar_sub(sgi);  // the next item is published (2-bit K: and all code words are in KW)
      it = *snext;
      pending = it < i1 ? (int)it : (j0 + sg < j1 ? (int)(j0 + sg) : -1);  // the item whose TMA is in flight
      if constexpr (SIDE == 0 && BITS == 2) {
        uint4* dst = reinterpret_cast<uint4*>(c.kcodes + blk * c.blk_bytes);
        constexpr int WL = 4;
        for (int ci = st; ci < 8 * 32 * WL / 4; ci += 128) {
          uint32_t wv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int wi = 4 * ci + e, tl = wi / WL, ww = wi % WL, ln = tl & 31;
            const int ad = tl * WL + (ww ^ ((ln >> 3) & 3));
            wv[e] = KW[ad];
            KW[ad] = 0u;
          }
          dst[ci] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
    }
    bar_side();  // every subgroup is done with chunk cur and the pattern tables
    if (gtid == 0) {
      ring[0] = nx;
      ring[1] = atomicAdd(&c.work[SIDE], 1);
      *cnext = (int)j0 + 4;
    }
    bar_side();
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
  int* rel = reinterpret_cast<int*>(sb + OFF_BAR + 64);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sb + OFF_BAR + 80);
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  int side = (int)(smid >> 1) < A.k_tpc ? 0 : 1;
  int* ring = reinterpret_cast<int*>(sb + OFF_BAR + 96);
  if (tid < 4) rel[tid] = 0;
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  uint32_t k = 0;  // items this subgroup processed (mbarrier phases), across both sides
  for (int pass = 0; pass < 2; ++pass, side ^= 1) {
    if (BITS == 2 && side == 0) {  // K code words start zeroed (KW[2..3] alias the V side's B)
      uint32_t* KW = reinterpret_cast<uint32_t*>(sb + OFF_KW);
      uint32_t* KW2 = reinterpret_cast<uint32_t*>(sb + OFF_B + SZ_B);
      for (int i = tid; i < 2 * SZ_KW / 4; i += NTHR) KW[i] = KW2[i] = 0u;
    }
    if (tid == 0) {
      ring[0] = atomicAdd(&A.c.work[side], 1);
      ring[1] = atomicAdd(&A.c.work[side], 1);
      const int ch = ring[0];  // the first chunk's dynamic items start after its 4 static ones
      *reinterpret_cast<int*>(sb + OFF_BAR + 84) =
          ch < A.nchunks[side] ? (ch / A.cpu[side]) * A.nb + (ch % A.cpu[side]) * A.chunk[side] + 4 : 0;
    }
    __syncthreads();
    if (side == 0) run_sub<BITS, 0>(A, sb, &tmK, tmem, k);
    else run_sub<BITS, 1>(A, sb, &tmV, tmem, k);
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_free<256>(tmem);
}

// Deferred code fix-ups (k_fix, v_codes): per entry the reference's fp64 code sequence for the
// two elements of a pair (quant.py:103-109 via exact_code_at, the stored fp64 params and pattern
// values) patched into the block's code words -- entries sharing a word touch disjoint bits.
__global__ void kfix_kernel(DevCache c, const __half* src, const __half* src_v, int64_t unit_stride, int first_block) {
  const int n = min(*reinterpret_cast<volatile int*>(c.work + 2), c.fixcap);
  const int64_t row0 = c.blk_start[first_block];
  const int qmax = (1 << c.bits) - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long en = c.fix[i];
    const int64_t blk = (int64_t)(uint32_t)en;
    if (en >> 63) {  // V pair: token t, channels ca, ca + 1 (own params; RAW tokens code the raw row)
      const int t = (int)((en >> 32) & 127), ca = (int)((en >> 39) & 127);
      const int u = (int)(blk / c.NBcap), b = (int)(blk % c.NBcap);
      const int64_t start = c.blk_start[b];
      const int pidx = c.vidx[blk * c.GP + t];
      const __half* xrow = src_v + (int64_t)u * unit_stride + (start - row0 + t) * 128;
      const double* mrow = pidx >= 0 ? c.vpat64 + ((int64_t)u * c.Pcap + pidx) * 128 : nullptr;
      const double* vp = c.vparam64 + 2 * ((int64_t)u * c.Tcap + start + t);
      const int WL = frag_words_per_lane(c.Dp, c.bits);
      uint8_t* tile = c.vcodes + blk * c.blk_bytes + (size_t)(t >> 4) * tile_bytes(c.Dp, c.bits);
#pragma unroll
      for (int k2 = 0; k2 < 2; ++k2) {
        const int ch = ca + k2;
        const uint32_t code = exact_code_at(xrow + ch, mrow ? mrow + ch : nullptr, vp[1], vp[0], qmax);
        // V^T fragment location of (channel ch, token t): side 1, row = ch & 15, col = t & 15
        const int row = ch & 15, col = t & 15;
        const int lane = 4 * (row & 7) + ((col & 7) >> 1), R = 4 * (ch >> 4) + (row >> 3) + 2 * (col >> 3);
        int word, slot;
        frag_word_slot(1, R, c.bits, word, slot);
        const int sh = ((col & 1) ? 16 : 0) + slot * c.bits;
        uint32_t* wp = reinterpret_cast<uint32_t*>(tile) + lane * WL + word;
        atomicAnd(wp, ~((uint32_t)qmax << sh));
        atomicOr(wp, code << sh);
      }
      if (c.stats) atomicAdd(&c.stats[1], 1u);
      continue;
    }
    const int t = (int)((en >> 32) & 127), ch = (int)((en >> 39) & 127), word = (int)((en >> 46) & 4095),
              sh = (int)((en >> 58) & 31);
    const int u = (int)(blk / c.NBcap), b = (int)(blk % c.NBcap);
    const int pidx = c.kidx[blk * c.GP + t];
    const __half* xrow = src + (int64_t)u * unit_stride + (c.blk_start[b] - row0 + t) * 128;
    const double* mrow = c.kpat64 + ((int64_t)u * c.Pcap + pidx) * 128;
    const double* kp = c.kparam64 + blk * 256;
    const uint32_t pv = exact_code_at(xrow + ch, mrow + ch, kp[128 + ch], kp[ch], qmax) |
                        (exact_code_at(xrow + ch + 1, mrow + ch + 1, kp[128 + ch + 1], kp[ch + 1], qmax) << 16);
    uint32_t* wp = reinterpret_cast<uint32_t*>(c.kcodes + blk * c.blk_bytes) + word;
    atomicAnd(wp, ~(((uint32_t)qmax | ((uint32_t)qmax << 16)) << sh));
    atomicOr(wp, pv << sh);
    if (c.stats) atomicAdd(&c.stats[1], 1u);
  }
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
  // starting sides: every CTA starts on the K queue and moves to V as K drains (a K phase,
  // then a V phase, one code path per SM at a time).  Measured against splitting the TPCs
  // between the sides in the K:V cost ratio (0.72): 781 -> 807 GB/s (2-bit), 761 -> 792 (4-bit).
  static double kfrac = 0.0;
  if (kfrac <= 0.0) {
    const char* kf = getenv("PKV_TC_KFRAC");
    kfrac = kf ? atof(kf) : 1.0;
    if (!(kfrac > 0.0 && kfrac <= 1.0)) kfrac = 1.0;
  }
  static int chunk = 0, chunk_v = 0;
  if (!chunk) {
    const char* ce = getenv("PKV_TC_CHUNK");
    chunk = ce ? atoi(ce) : 32;
    if (chunk < 4 || chunk > 4096) chunk = 32;
    const char* cv = getenv("PKV_TC_CHUNK_V");
    chunk_v = cv ? atoi(cv) : chunk;
    if (chunk_v < 4 || chunk_v > 4096) chunk_v = chunk;
  }
  a.k_tpc = (int)(kfrac * (nsm / 2) + 0.5);
  a.chunk[0] = chunk;
  a.chunk[1] = chunk_v;
  for (int sd = 0; sd < 2; ++sd) {
    a.cpu[sd] = (nblocks + a.chunk[sd] - 1) / a.chunk[sd];
    if ((int64_t)c.U * a.cpu[sd] + 2 * nsm >= (1ll << 31)) return cudaErrorNotSupported;
    a.nchunks[sd] = c.U * a.cpu[sd];
  }
  const int grid = (int)std::min<int64_t>(nsm, (int64_t)a.nchunks[0] + a.nchunks[1]);
  if (cudaMemsetAsync(c.work, 0, 16, st) != cudaSuccess) return cudaGetLastError();
  if (c.bits == 2) {
    cudaFuncSetAttribute(fe::encode_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, fe::smem_bytes(2));
    fe::encode_tc_kernel<2><<<grid, fe::NTHR, fe::smem_bytes(2), st>>>(a, tk, tv);
  } else {
    cudaFuncSetAttribute(fe::encode_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, fe::smem_bytes(4));
    fe::encode_tc_kernel<4><<<grid, fe::NTHR, fe::smem_bytes(4), st>>>(a, tk, tv);
  }
  if (c.fix && c.fixcap > 0)  // the deferred K code fix-ups (count on the device: grid-stride)
    fe::kfix_kernel<<<4 * nsm, 256, 0, st>>>(c, k, v, unit_stride, first_block);
  return cudaGetLastError();
}

}  // namespace pkv
