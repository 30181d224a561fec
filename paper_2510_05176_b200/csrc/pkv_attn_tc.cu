// K3-TC decode attention on tcgen05 (semantics: softmax over `committed_matrices` + the
// exact window, engine.py:255-303; the reference has no attention).
//
// K is never materialised and nothing is dequantized to floating point: the packed 2/4-bit
// codes go to the tensor cores as INTEGERS (tcgen05.mma kind::i8, s32 accumulate in TMEM).
//   q.k_t = sum_c (q_c s_c) code_tc + q.z_b + (q.M)[kidx_t]
// * A_K (TMEM, lane = token, 128 K-bytes): one LOP3 per 4 codes turns the mma-fragment words
//   of the cache (pkv_common.cuh) into u8 "planes" (code << 2m at 2 bits, << 4m at 4 bits),
//   stored with tcgen05.st.16x128b -- the fragment rows (g, g+8) are exactly that shape's rows.
// * B_QK (smem, MN-major, [channel][NG heads x 4 bytes]): x = rint(q_c s_c 2^E 4^-m) as four
//   signed base-256 digits, one N column per (head, digit); E per (block, head) from the block's
//   max scale, so |x| < 2^29 and the integer products are exact.  score = sum_d 256^d D[t][h,d].
// * A_V (TMEM, lane = channel, 128 token bytes): the V^T fragment words, one PRMT + 4 LOP3 per
//   lane and tile; B_PV (smem) = u32 digits of p_t s_t 2^Ev per (token, head); D_O accumulates
//   sum_t p_t s_t code_t in TMEM across blocks (exact integers, flushed to fp32 registers only
//   when the running max or Ev changes).
// * pattern weights W_p = sum_{t: vidx_t = p} p_t by a one-hot MMA (A = one-hot [P x tokens] u8 in
//   smem, B = u32 digits of p_t 2^31) accumulated in TMEM; sum_p W_p M'_p once per chunk.
// One CTA of 128 (GQA <= 4) or 256 threads (two head halves) per (unit, chunk of <= 256 blocks);
// a thread is a token in the softmax
// phase and a channel in the B_QK / output phase; thread 0 issues the MMAs.  Per block: two
// named barriers, one QK and one PV/W commit.  Partials (o, m, l) have the legacy K3 format and
// are merged (with the window) by attn_merge_kernel.
#include "pkv_common.cuh"
#include "pkv_sm100.cuh"
#include <cfloat>
#include <cstdlib>

namespace pkv {
namespace atc {
using namespace sm100;

constexpr float TH = 2.f;          // on a rescale, m_ref = block max + TH (log2 units)
constexpr int MAX_BPC = 256;       // blocks per chunk: keeps the s32 D_O digits below 2^31
constexpr int MAXP = 256;          // patterns per side served (one-hot M tiles of 128)

template <int NT>
__device__ __forceinline__ void bar_sync1() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st16x128x8(uint32_t ta, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void st16x128x4(uint32_t ta, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ uint64_t desc_none(const void* base, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm100 descriptor version; layout 0 = no swizzle
  return d;
}
// kind::i8 instruction descriptor: D s32, A/B u8 (0) or s8 (1), K- (0) or MN-major (1)
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_s, int b_s, int a_mn, int b_mn) {
  return (2u << 4) | ((uint32_t)a_s << 7) | ((uint32_t)b_s << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2, ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// smallest e with |v| < 2^e for a finite v != 0 (normal range)
__device__ __forceinline__ int ceil_exp(float v) { return (int)((__float_as_uint(v) >> 23) & 255u) - 126; }
__device__ __forceinline__ int fkey(float f) {  // float order as signed-int order
  const int k = __float_as_int(f);
  return k >= 0 ? k : k ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float funkey(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7FFFFFFF); }

// K-byte position of channel c in the K operand (A_K rows / B_QK rows) and its plane shift
template <int BITS>
__device__ __forceinline__ int kpos_k(int c, int& shift) {
  if (BITS == 2) {
    const int m = 2 * ((c & 31) >> 4) + ((c & 15) >> 3), byte = 2 * (c & 1) + ((c & 63) >> 5);
    shift = 2 * m;
    return 16 * (4 * (c >> 6) + m) + 4 * ((c & 7) >> 1) + byte;
  } else {
    const int m = (c & 15) >> 3, byte = 2 * (c & 1) + ((c & 31) >> 4);
    shift = 4 * m;
    return 16 * (2 * (c >> 5) + m) + 4 * ((c & 7) >> 1) + byte;
  }
}
// K-byte position of token slot t in the V operand (A_V columns / B_PV, B_W, one-hot rows)
__device__ __forceinline__ int kpos_v(int t) {
  const int tp = t & 15;
  return 16 * (t >> 4) + 4 * ((tp & 7) >> 1) + (tp & 1) + 2 * (tp >> 3);
}
// plane shift of channel c (= TMEM lane of A_V) in the V operand
template <int BITS>
__device__ __forceinline__ int vshift(int c) {
  return BITS == 2 ? 2 * ((c & 31) >> 3) : 4 * ((c >> 3) & 1);
}

struct Smem {  // dynamic shared memory carve (byte offsets)
  int bqk, bpv, bw, onehot, qm, sq, stats, red;
  int total;
};
__host__ __device__ inline Smem carve(int NG, int MT, int pkcap, int bpc) {
  Smem s;
  const int bb = 128 * 16 * (NG / 4);
  s.bqk = 0;
  s.bpv = s.bqk + bb;
  s.bw = s.bpv + bb;
  s.onehot = s.bw + bb;
  s.qm = s.onehot + MT * 16384;
  s.sq = s.qm + ((pkcap * NG * 4 + 15) & ~15);
  s.stats = s.sq + NG * 128 * 4;                       // [bpc][NG] c1, [bpc][NG] qz, [bpc] 2^-e_s
  s.red = s.stats + (((2 * NG + 1) * bpc * 4 + 15) & ~15);
  s.total = s.red + 1024;
  return s;
}
// scratch inside `red` (32-bit words); q = TMEM lane quarter (warp % 4), h = head
constexpr int R_FLAG = 0;     // [8] per-warp slow-path votes (even blocks)
constexpr int R_FLAG1 = 8;    // [8] votes of odd blocks: a warp may write block b + 1's vote while a
                              // slower warp still reads block b's (no barrier in between)
constexpr int R_BMAX = 16;    // [4 q][8 h] block max keys (also the prologue's max |q|)
constexpr int R_SVM = 48;     // [4 q] max V scale
constexpr int R_EQ = 52;      // [8 h] e_q per head
constexpr int R_LS = 60;      // [4 q][8 h] final l
constexpr int R_ZS = 92;      // [4 q][8 h] final z
constexpr int R_BAR = 124;    // 2 mbarriers (8-byte aligned)
constexpr int R_TMEM = 128;   // TMEM base

// NG query-head slots per KV head (4 or 8) in HH = NG / 4 head halves: thread (hh, tq) of the
// 128 * HH threads is token / channel / TMEM lane tq for the 4 heads 4 hh .. 4 hh + 3, so every
// thread carries the per-head state of 4 heads whatever the GQA group size (8 heads on one
// thread halved the warps per SM and doubled each thread's softmax chain).
template <int BITS, int NG>
__global__ void __launch_bounds__(32 * NG, NG == 4 ? 4 : 2) attn_tc_kernel(DevCache c, AttnArgs a, int pkcap, int MT) {
  constexpr int HH = NG / 4;                 // head halves
  constexpr int NT = 128 * HH;               // threads
  constexpr int N = 4 * NG;                  // MMA N: heads x base-256 digits
  constexpr uint32_t C_AK = 0, C_AV = 32, C_DS = 64, C_DO = 64 + N, C_DW = 64 + 2 * N;
  constexpr uint32_t TCOLS = NG == 4 ? 128 : 256;
  constexpr int NWK = 16 * BITS / 8;         // K fragment words per lane per tile (4 or 8)
  constexpr int TB = 16 * 128 * BITS / 8;    // bytes per 16-token tile
  constexpr int KT = 2 / HH;                 // K tiles per warp per block
  constexpr int VT = 8 / HH;                 // V tiles per warp per block
  constexpr uint32_t ID_QK = idesc_i8(128, N, 0, 1, 0, 1);
  constexpr uint32_t ID_PV = idesc_i8(128, N, 0, 0, 0, 1);
  // the window merge (attn_merge_kernel, launched programmatically dependent) may start its
  // window rows once every chunk CTA is resident; it waits for this grid before the partials
  asm volatile("griddepcontrol.launch_dependents;");
  const int u = blockIdx.y, chunk = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tq = HH == 1 ? tid : tid & 127, hh = HH == 1 ? 0 : tid >> 7, wq = HH == 1 ? warp : warp & 3;
  const int h0 = 4 * hh;                     // this thread's first head
  const int G = a.G, D = c.D;
  const int Pk = c.use_kp ? c.nk[u] : 0, Pv = c.use_vp ? c.nv[u] : 0;
  const int ntile = c.ntile_blk;
  const int b0 = a.blk0 + chunk * a.bpc, b1 = min(a.blk0 + a.nb, b0 + a.bpc);
  const int nit = max(b1 - b0, 0);

  extern __shared__ __align__(1024) unsigned char sm[];
  const Smem L = carve(NG, MT, pkcap, a.bpc);
  uint8_t* bqk = sm + L.bqk;
  uint8_t* bpv = sm + L.bpv;
  uint8_t* bw = sm + L.bw;
  uint8_t* onehot = sm + L.onehot;
  float* qm = reinterpret_cast<float*>(sm + L.qm);
  float* sq = reinterpret_cast<float*>(sm + L.sq);
  float* st_c1 = reinterpret_cast<float*>(sm + L.stats);   // [bpc][NG] score factor
  float* st_qz = st_c1 + a.bpc * NG;                        // [bpc][NG] scale_log2 * q.z_b (-inf: h >= G)
  float* st_si = st_qz + a.bpc * NG;                        // [bpc] 2^-e_s
  int* ri = reinterpret_cast<int*>(sm + L.red);
  float* rf = reinterpret_cast<float*>(ri);
  uint64_t* mbS = reinterpret_cast<uint64_t*>(ri + R_BAR);
  uint64_t* mbPV = mbS + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(ri + R_TMEM);

  // ---- prologue ---------------------------------------------------------------------------
  if (warp == 0) tmem_alloc<TCOLS>(tslot);
  if (tid == 0) {
    mbar_init(mbS, 1);
    mbar_init(mbPV, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < NG * 128; i += NT) {
    const int h = i >> 7, ch = i & 127;
    sq[i] = (h < G && ch < D) ? a.q[((int64_t)u * G + h) * D + ch] : 0.f;
  }
  for (int i = tid; i < MT * 1024; i += NT) reinterpret_cast<uint4*>(onehot)[i] = make_uint4(0, 0, 0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t T = *tslot;
  const uint32_t lrow = (uint32_t)(32 * wq) << 16;  // this warp's TMEM lane quarter
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(sq[(h0 + i) * 128 + tq])));
    if (lane == 0) ri[R_BMAX + wq * 8 + h0 + i] = (int)m;
  }
  __syncthreads();
  // channel role constants: B_QK row, q o 4^-m scaled so |x| < 2^29
  int kshift;
  const int kposc = kpos_k<BITS>(tq, kshift);
  float qf[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) m = max(m, (unsigned)ri[R_BMAX + w * 8 + h0 + i]);
    const int eq = m ? ceil_exp(__uint_as_float(m)) : 0;
    if (tq == 0) ri[R_EQ + h0 + i] = eq;
    qf[i] = ldexpf(sq[(h0 + i) * 128 + tq], 29 - eq - kshift);
  }
  // q.M table (scale_log2 folded in)
  for (int p = tid; p < Pk; p += NT) {
    const float4* m4 = reinterpret_cast<const float4*>(c.kpat32 + ((int64_t)u * c.Pcap + p) * c.Dp);
    float acc[NG];
#pragma unroll
    for (int h = 0; h < NG; ++h) acc[h] = 0.f;
    for (int i = 0; i < 32; ++i) {
      const float4 mv = __ldg(m4 + i);
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        const float4 qv = reinterpret_cast<const float4*>(sq + h * 128)[i];
        acc[h] = fmaf(qv.x, mv.x, fmaf(qv.y, mv.y, fmaf(qv.z, mv.z, fmaf(qv.w, mv.w, acc[h]))));
      }
    }
#pragma unroll
    for (int h = 0; h < NG; ++h) qm[p * NG + h] = acc[h] * a.scale_log2;
  }
  __syncthreads();  // R_EQ
  // per-block statistics of the chunk (thread per block): max K scale -> e_s, q.z_b per head
  const int64_t ubase = (int64_t)u * c.NBcap;
  for (int i = tid; i < nit; i += NT) {
    const float4* sp = reinterpret_cast<const float4*>(c.kparam32 + (ubase + b0 + i) * 2 * c.Dp);
    const float4* zp = sp + c.Dp / 4;
    float smax = 0.f, qz[NG];
#pragma unroll
    for (int h = 0; h < NG; ++h) qz[h] = 0.f;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const float4 s4 = __ldg(sp + j), z4 = __ldg(zp + j);
      smax = fmaxf(fmaxf(smax, fmaxf(s4.x, s4.y)), fmaxf(s4.z, s4.w));
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        const float4 qv = reinterpret_cast<const float4*>(sq + h * 128)[j];
        qz[h] = fmaf(qv.x, z4.x, fmaf(qv.y, z4.y, fmaf(qv.z, z4.z, fmaf(qv.w, z4.w, qz[h]))));
      }
    }
    const int es = smax > 0.f ? ceil_exp(smax) : 0;
    st_si[i] = ldexpf(1.f, -es);
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      st_c1[i * NG + h] = ldexpf(a.scale_log2, ri[R_EQ + h] + es - 29);
      st_qz[i * NG + h] = h < G ? qz[h] * a.scale_log2 : -INFINITY;
    }
  }

  // ---- per-thread streaming state -------------------------------------------------------------
  // this unit's arenas from this thread's view; a block adds (32-bit) b * stride.  K: warp (wq, hh)
  // owns tiles 2 wq + hh KT .. + KT - 1 (TMEM lanes 16 (tile % 2) of its quarter); V: the warp's
  // channel quarter of tiles hh VT .. hh VT + VT - 1 (A_V columns 4 VT hh ..)
  const uint32_t bbytes = (uint32_t)c.blk_bytes, gp = (uint32_t)c.GP, kps = 2u * (uint32_t)c.Dp;
  const int kt0 = 2 * wq + hh * KT, vt0 = hh * VT;
  const uint8_t* klane = c.kcodes + ubase * c.blk_bytes + kt0 * TB + lane * (4 * NWK);
  const uint8_t* vlane = c.vcodes + ubase * c.blk_bytes + vt0 * TB + lane * (8 * BITS) + (BITS == 2 ? 8 * (wq >> 1) : 8 * wq);
  const bool has_slot = tq < c.GP;
  const int16_t* kidx_u = c.kidx + ubase * c.GP + tq;
  const int16_t* vidx_u = c.vidx + ubase * c.GP + tq;
  const float2* vp_u = reinterpret_cast<const float2*>(c.vparam32) + ubase * c.GP + tq;
  const float* ks_u = c.kparam32 + ubase * 2 * c.Dp + tq;
  uint32_t kw[KT][NWK];  // K fragment words of this warp's tiles (block b + 1)
  uint2 vw[VT];          // V fragment words, this warp's channel quarter of its tiles (block b)
  float s_nx = 0.f;      // K scale of channel tq (block b + 1)
  int kidx_t = RAW, vidx_t = RAW, kidx_n = RAW, vidx_n = RAW, L_t = 128, L_n = 128;
  float vs_t = 0.f, vz_t = 0.f, vs_n = 0.f, vz_n = 0.f;
  // the blocks load in order (K two ahead, V and metadata one ahead): running pointers
  const uint8_t* kptr = klane + (size_t)b0 * bbytes;
  const float* sptr = ks_u + (size_t)b0 * kps;
  const uint8_t* vptr = vlane + (size_t)b0 * bbytes;
  const int* lptr = c.blk_len + b0;
  uint32_t mo = (uint32_t)b0 * gp;
  auto load_k = [&]() {
    const uint8_t* p = kptr;
    kptr += bbytes;
#pragma unroll
    for (int i = 0; i < KT; ++i) {
      if (ntile == 8 || kt0 + i < ntile) {
#pragma unroll
        for (int j = 0; j < NWK / 4; ++j) {
          const uint4 x = __ldg(reinterpret_cast<const uint4*>(p + i * TB) + j);
          kw[i][4 * j] = x.x; kw[i][4 * j + 1] = x.y; kw[i][4 * j + 2] = x.z; kw[i][4 * j + 3] = x.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < NWK; ++j) kw[i][j] = 0u;
      }
    }
    s_nx = __ldg(sptr);
    sptr += kps;
  };
  auto load_v = [&]() {
    const uint8_t* p = vptr;
    vptr += bbytes;
    if (ntile == 8) {
#pragma unroll
      for (int ti = 0; ti < VT; ++ti) vw[ti] = __ldg(reinterpret_cast<const uint2*>(p + ti * TB));
    } else {
#pragma unroll
      for (int ti = 0; ti < VT; ++ti)
        vw[ti] = vt0 + ti < ntile ? __ldg(reinterpret_cast<const uint2*>(p + ti * TB)) : make_uint2(0u, 0u);
    }
  };
  auto load_meta = [&]() {  // token tq of the next block -> the *_n registers
    L_n = __ldg(lptr++);
    const uint32_t o = mo;
    mo += gp;
    if (has_slot) {
      kidx_n = __ldg(kidx_u + o);
      vidx_n = __ldg(vidx_u + o);
      const float2 vp = __ldg(vp_u + o);
      vs_n = vp.x; vz_n = vp.y;
    } else {
      kidx_n = RAW; vidx_n = RAW; vs_n = 0.f; vz_n = 0.f;
    }
  };
  auto next_meta = [&]() { kidx_t = kidx_n; vidx_t = vidx_n; vs_t = vs_n; vz_t = vz_n; L_t = L_n; };
  // K planes of the loaded block -> A_K, B_QK row of channel tq, this thread's heads (block local index i)
  auto k_side = [&](int i) {
    constexpr int NP = BITS == 2 ? 4 : 2;  // planes per word
#pragma unroll
    for (int t2 = 0; t2 < KT; ++t2) {
      uint32_t r[16];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {  // repeat rr: word pair (2 (rr / NP), +1), plane rr % NP
        const int wi = 2 * (rr / NP), m = rr % NP;
        const uint32_t mask = BITS == 2 ? (0x03030303u << (2 * m)) : (m ? 0xF0F0F0F0u : 0x0F0F0F0Fu);
        r[2 * rr] = kw[t2][wi] & mask;
        r[2 * rr + 1] = kw[t2][wi + 1] & mask;
      }
      st16x128x8(T + lrow + ((uint32_t)(16 * ((kt0 + t2) & 1)) << 16) + C_AK, r);
    }
    const float t = s_nx * st_si[i];
    uint32_t x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = ((uint32_t)__float2int_rn(qf[j] * t) + 0x80808080u) ^ 0x80808080u;
    *reinterpret_cast<uint4*>(bqk + hh * 2048 + kposc * 16) = make_uint4(x[0], x[1], x[2], x[3]);
  };

  float mref[4], lsum[4], zsum[4], Of[4], Wf[2][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mref[i] = -FLT_MAX; lsum[i] = 0.f; zsum[i] = 0.f; Of[i] = 0.f; Wf[0][i] = 0.f; Wf[1][i] = 0.f;
  }
  int Ev = 0;
  float evs31 = INFINITY;  // 2^(Ev - 31); +inf until the first V block sets Ev
  bool fresh = true;
  const int vsh = vshift<BITS>(tq);
  const int kposv = kpos_v(tq);
  const int oh_base = (kposv >> 4) * 2048 + (kposv & 15);  // this token's byte in a one-hot tile
  int oh_off = -1;  // this token's one-hot byte (cleared after the block's W MMA; head half 0)
  // descriptors (thread 0 issues every MMA)
  const uint64_t dqk = desc_none(bqk, 128, 2048), dpv = desc_none(bpv, 128, 2048), dbw = desc_none(bw, 128, 2048);
  const uint64_t doh = desc_none(onehot, 2048, 128);

  // flush the TMEM sums (this thread's 16 head-digit columns) into fp32 registers (current Ev),
  // then scale everything by alpha
  auto flush = [&](const float (&alpha)[4]) {
    if (!fresh) {
      uint32_t v[16];
      tmem_ld16(T + lrow + C_DO + 16 * hh, v);
      tmem_ld_wait();
      const float so = ldexpf(1.f, -Ev - vsh);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float x = (float)(int)v[4 * i + 3];
        x = fmaf(x, 256.f, (float)(int)v[4 * i + 2]);
        x = fmaf(x, 256.f, (float)(int)v[4 * i + 1]);
        x = fmaf(x, 256.f, (float)(int)v[4 * i]);
        Of[i] = fmaf(x, so, Of[i]);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        if (mt >= MT) break;
        tmem_ld16(T + lrow + C_DW + N * mt + 16 * hh, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float x = (float)(int)v[4 * i + 3];
          x = fmaf(x, 256.f, (float)(int)v[4 * i + 2]);
          x = fmaf(x, 256.f, (float)(int)v[4 * i + 1]);
          x = fmaf(x, 256.f, (float)(int)v[4 * i]);
          Wf[mt][i] = fmaf(x, 4.656612873077393e-10f, Wf[mt][i]);  // 2^-31
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      Of[i] *= alpha[i]; lsum[i] *= alpha[i]; zsum[i] *= alpha[i];
      Wf[0][i] *= alpha[i]; Wf[1][i] *= alpha[i];
    }
    fresh = true;
  };

  __syncthreads();  // block statistics
  if (nit > 0) {
    load_k();
    load_v();
    load_meta();
    next_meta();
    k_side(0);
    if (nit > 1) load_k();
    st_wait();
    fence_proxy_async();
    tc_fence_before();
  }
  __syncthreads();
  if (nit > 0 && tid == 0) {
    tc_fence_after();
#pragma unroll
    for (int k = 0; k < 4; ++k) mma_ts(T + C_DS, T + C_AK + 8 * k, dqk + 32 * k, ID_QK, k > 0);
    mma_commit(mbS);
  }

  // ---- block loop: QK(b) was issued by the previous iteration --------------------------------
  for (int it = 0; it < nit; ++it) {
    const bool more = it + 1 < nit;
    // (i) scores of token tq, heads h0 .. h0 + 3
    float lg[4];
    {
      mbar_wait(mbS, it & 1);
      tc_fence_after();
      uint32_t v[16];
      tmem_ld16(T + lrow + C_DS + 16 * hh, v);
      float add[4];
      if (kidx_t >= 0 && kidx_t < Pk) {
        const float4 x = *reinterpret_cast<const float4*>(qm + kidx_t * NG + h0);
        add[0] = x.x; add[1] = x.y; add[2] = x.z; add[3] = x.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) add[i] = 0.f;
      }
      float c1[4];
      {
        const float4 x = *reinterpret_cast<const float4*>(st_c1 + it * NG + h0);
        const float4 z = *reinterpret_cast<const float4*>(st_qz + it * NG + h0);
        c1[0] = x.x; c1[1] = x.y; c1[2] = x.z; c1[3] = x.w;
        add[0] += z.x; add[1] += z.y; add[2] += z.z; add[3] += z.w;
      }
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int lo = (int)v[4 * i + 1] * 256 + (int)v[4 * i];
        const int hi = (int)v[4 * i + 3] * 256 + (int)v[4 * i + 2];
        lg[i] = fmaf(fmaf((float)hi, 65536.f, (float)lo), c1[i], add[i]);
      }
      if (L_t < 128 && tq >= L_t) {
#pragma unroll
        for (int i = 0; i < 4; ++i) lg[i] = -INFINITY;
      }
    }
    // (ii) next block's K side (A_K and B_QK are free: QK(b) is complete)
    if (more) {
      k_side(it + 1);
      st_wait();
      fence_proxy_async();
      tc_fence_before();
      // QK(b + 1) as soon as every warp's A_K rows are in: the last warp waits and issues (warp
      // 0 issues PV / W), the others only arrive
      if (warp == NT / 32 - 1) {
        asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory");
        if (lane == 0) {
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ts(T + C_DS, T + C_AK + 8 * k, dqk + 32 * k, ID_QK, k > 0);
          mma_commit(mbS);
        }
        __syncwarp();
      } else {
        asm volatile("bar.arrive 2, %0;" ::"n"(NT) : "memory");
      }
      // all of the iteration's global loads go out here and in (iv): every load shares one
      // scoreboard, so metadata issued at the top of the loop made the next K-side read (the
      // first consumer) wait for loads just issued (measured 0.600 -> 0.659 ms, here 0.582)
      load_meta();
      if (it + 2 < nit) load_k();
    }
    // (iii) softmax of token tq: p' = 2^31 exp2(lg - m_ref), digits of p' and p' s_t 2^(Ev-31)
    // (lg[0] > -inf marks a valid token: head h0 < G always, NG = 8 only serves G > 4)
    float p8[4];
    uint32_t xw[4], xv[4];
    bool flag;
    auto probs = [&]() {
      // evs31 = +inf until the first V scale exponent is set: any valid token with s_t > 0 flags
      const float sE = vs_t * evs31;
      float dmax = (lg[0] > -INFINITY && sE >= 1.f) ? INFINITY : -INFINITY;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float d = lg[i] - (mref[i] - 31.f);
        dmax = fmaxf(dmax, d);
        p8[i] = ex2(d);
        xw[i] = __float2uint_rn(p8[i]);
        xv[i] = __float2uint_rn(p8[i] * sE);
      }
      flag = dmax > 31.f;
    };
    probs();
    {
      const bool any = __any_sync(0xffffffffu, flag);
      if (lane == 0) ri[(it & 1 ? R_FLAG1 : R_FLAG) + warp] = any;
    }
    // (iv) after PV / W of block b - 1: V planes -> A_V, one-hot and B rows of block b
    tc_fence_after();
    if (it > 0) mbar_wait(mbPV, (it - 1) & 1);
    tc_fence_after();
    {
      uint32_t ra[2 * VT], rb[2 * VT];
#pragma unroll
      for (int ti = 0; ti < VT; ++ti) {
        if (BITS == 2) {
          const uint32_t p0 = prmt(vw[ti].x, vw[ti].y, (wq & 1) ? 0x7531u : 0x6420u);
          ra[2 * ti] = p0 & 0x03030303u;
          ra[2 * ti + 1] = p0 & 0x0C0C0C0Cu;
          rb[2 * ti] = p0 & 0x30303030u;
          rb[2 * ti + 1] = p0 & 0xC0C0C0C0u;
        } else {
          const uint32_t p0 = prmt(vw[ti].x, vw[ti].y, 0x6420u), p1 = prmt(vw[ti].x, vw[ti].y, 0x7531u);
          ra[2 * ti] = p0 & 0x0F0F0F0Fu;
          ra[2 * ti + 1] = p0 & 0xF0F0F0F0u;
          rb[2 * ti] = p1 & 0x0F0F0F0Fu;
          rb[2 * ti + 1] = p1 & 0xF0F0F0F0u;
        }
      }
      const uint32_t cav = C_AV + 4 * vt0;
      if constexpr (VT == 8) {
        st16x128x8(T + lrow + cav, ra);
        st16x128x8(T + lrow + (16u << 16) + cav, rb);
      } else {
        st16x128x4(T + lrow + cav, ra);
        st16x128x4(T + lrow + (16u << 16) + cav, rb);
      }
    }
    if (more) load_v();
    if (hh == 0) {
      if (oh_off >= 0) onehot[oh_off] = 0;
      oh_off = (lg[0] > -INFINITY && vidx_t >= 0 && vidx_t < Pv) ? (vidx_t >> 7) * 16384 + (vidx_t & 127) * 16 + oh_base : -1;
      if (oh_off >= 0) onehot[oh_off] = 1;
    }
    auto write_rows = [&]() {
      *reinterpret_cast<uint4*>(bw + hh * 2048 + kposv * 16) = make_uint4(xw[0], xw[1], xw[2], xw[3]);
      *reinterpret_cast<uint4*>(bpv + hh * 2048 + kposv * 16) = make_uint4(xv[0], xv[1], xv[2], xv[3]);
    };
    write_rows();
    st_wait();
    fence_proxy_async();
    tc_fence_before();
    bar_sync1<NT>();
    const int* fl = ri + (it & 1 ? R_FLAG1 : R_FLAG);
    int anyf = 0;
#pragma unroll
    for (int w = 0; w < 4 * HH; ++w) anyf |= fl[w];
    if (anyf != 0) {
      // CTA-uniform slow path: new running max / V scale exponent; flush the TMEM sums
      tc_fence_after();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = __reduce_max_sync(0xffffffffu, fkey(lg[i]));
        if (lane == 0) ri[R_BMAX + wq * 8 + h0 + i] = k;
      }
      {
        const unsigned m = __reduce_max_sync(0xffffffffu, lg[0] > -INFINITY ? __float_as_uint(vs_t) : 0u);
        if (lane == 0 && hh == 0) ri[R_SVM + wq] = (int)m;
      }
      bar_sync1<NT>();
      float alpha[4], mnew[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int k = ri[R_BMAX + h0 + i];
#pragma unroll
        for (int w = 1; w < 4; ++w) k = max(k, ri[R_BMAX + w * 8 + h0 + i]);
        const float bm = funkey(k);
        mnew[i] = bm == -INFINITY ? mref[i] : fmaxf(mref[i], bm + TH);
        alpha[i] = mref[i] == -FLT_MAX ? 0.f : ex2(mref[i] - mnew[i]);
      }
      flush(alpha);
      unsigned svm = 0;
#pragma unroll
      for (int w = 0; w < 4; ++w) svm = max(svm, (unsigned)ri[R_SVM + w]);
      const float sv = __uint_as_float(svm);
      if (svm && sv * evs31 >= 1.f) {
        Ev = 30 - ceil_exp(sv);
        evs31 = ldexpf(1.f, Ev - 31);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) mref[i] = mnew[i];
      probs();
      write_rows();
      fence_proxy_async();
      tc_fence_before();
      bar_sync1<NT>();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      lsum[i] += p8[i];
      zsum[i] = fmaf(p8[i], vz_t, zsum[i]);
    }
    if (tid == 0) {
      tc_fence_after();
      const uint32_t acc0 = fresh ? 0u : 1u;
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_ts(T + C_DO, T + C_AV + 8 * k, dpv + 32 * k, ID_PV, k > 0 ? 1u : acc0);
      for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_ss(T + C_DW + N * mt, doh + 1024 * mt + 256 * k, dbw + 32 * k, ID_PV, k > 0 ? 1u : acc0);
      }
      mma_commit(mbPV);
    }
    fresh = false;
    next_meta();
  }

  // ---- chunk epilogue -------------------------------------------------------------------------
  if (nit > 0) {
    mbar_wait(mbPV, (nit - 1) & 1);
    tc_fence_after();
    float one[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) one[i] = 1.f;
    flush(one);
  }
  // l and z: token partials summed over the CTA (units of 2^-31)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float l = lsum[i], z = zsum[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
      z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    if (lane == 0) { rf[R_LS + wq * 8 + h0 + i] = l; rf[R_ZS + wq * 8 + h0 + i] = z; }
  }
  // pattern weights: thread (hh, tq) holds W of its heads for patterns tq and 128 + tq
  float* Wt = reinterpret_cast<float*>(onehot);  // [MT*128][NG], the one-hot is no longer read
  __syncthreads();
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    if (mt >= MT) break;
    *reinterpret_cast<float4*>(Wt + (mt * 128 + tq) * NG + h0) = make_float4(Wf[mt][0], Wf[mt][1], Wf[mt][2], Wf[mt][3]);
  }
  __syncthreads();
  // output of channel tq, heads h0 .. h0 + 3: one pass over the V pattern rows for all 4 heads
  float* out = a.part + (((int64_t)u * a.nchunk + chunk) * G) * (c.Dp + 2);
  float o4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float zt = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) zt += rf[R_ZS + w * 8 + h0 + i];
    o4[i] = fmaf(zt, 4.656612873077393e-10f, Of[i]);
  }
  if (tq < D) {
    const float* mv = c.vpat32 + (int64_t)u * c.Pcap * c.Dp + tq;
    for (int p = 0; p < Pv; ++p) {
      const float m = __ldg(mv + (int64_t)p * c.Dp);
      const float4 w4 = *reinterpret_cast<const float4*>(Wt + p * NG + h0);
      o4[0] = fmaf(w4.x, m, o4[0]); o4[1] = fmaf(w4.y, m, o4[1]);
      o4[2] = fmaf(w4.z, m, o4[2]); o4[3] = fmaf(w4.w, m, o4[3]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int h = h0 + i;
    if (h >= G) break;
    out[h * (c.Dp + 2) + tq] = o4[i];
    if (tq == 0) {
      float lt = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) lt += rf[R_LS + w * 8 + h];
      out[h * (c.Dp + 2) + c.Dp] = (nit > 0 && mref[i] != -FLT_MAX) ? mref[i] : -INFINITY;
      out[h * (c.Dp + 2) + c.Dp + 1] = lt * 4.656612873077393e-10f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<TCOLS>(T);
}

template <int BITS, int NG>
static cudaError_t launch_kt(const DevCache& c, const AttnArgs& a, int pkcap, int MT, cudaStream_t st) {
  const Smem L = carve(NG, MT, pkcap, a.bpc);
  const size_t smem = (size_t)L.total + 1024;
  cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<BITS, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  attn_tc_kernel<BITS, NG><<<dim3(a.nchunk, c.U), 32 * NG, smem, st>>>(c, a, pkcap, MT);
  return cudaGetLastError();
}

}  // namespace atc

// K3-TC entry: cudaErrorNotSupported outside its envelope (head_dim padding 128, 2/4-bit,
// <= 8 query heads per KV head, <= 256 patterns per side, <= 256 blocks per chunk) or when
// PKV_ATTN_TC=0; the caller then runs the CUDA-core K3.
cudaError_t launch_attn_tc(const DevCache& c, const AttnArgs& a, int Pk_max, int Pv_max, cudaStream_t st) {
  const char* env = getenv("PKV_ATTN_TC");
  if (env && env[0] == '0') return cudaErrorNotSupported;
  if (c.Dp != 128 || (c.bits != 2 && c.bits != 4) || a.G > 8 || c.ntile_blk > 8) return cudaErrorNotSupported;
  if (Pk_max > atc::MAXP || Pv_max > atc::MAXP || a.bpc > atc::MAX_BPC) return cudaErrorNotSupported;
  const int MT = Pv_max > 0 ? (Pv_max + 127) / 128 : 0;
  const int pkcap = (Pk_max + 3) & ~3;
  if (a.G <= 4) return c.bits == 2 ? atc::launch_kt<2, 4>(c, a, pkcap, MT, st) : atc::launch_kt<4, 4>(c, a, pkcap, MT, st);
  return c.bits == 2 ? atc::launch_kt<2, 8>(c, a, pkcap, MT, st) : atc::launch_kt<4, 8>(c, a, pkcap, MT, st);
}

}  // namespace pkv
