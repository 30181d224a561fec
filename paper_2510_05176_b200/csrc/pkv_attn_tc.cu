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
// One 128-thread CTA per (unit, chunk of <= 256 blocks); a thread is a token in the softmax
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

constexpr int THREADS = 128;
constexpr float TH = 2.f;          // on a rescale, m_ref = block max + TH (log2 units)
constexpr int MAX_BPC = 256;       // blocks per chunk: keeps the s32 D_O digits below 2^31
constexpr int MAXP = 256;          // patterns per side served (one-hot M tiles of 128)

__device__ __forceinline__ void bar_sync1() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st16x128x8(uint32_t ta, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
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
// scratch inside `red` (32-bit words)
constexpr int R_FLAG = 0;     // [4] per-warp slow-path votes
constexpr int R_BMAX = 4;     // [4][8] block max keys (also the prologue's max |q|)
constexpr int R_SVM = 36;     // [4] max V scale
constexpr int R_EQ = 40;      // [8] e_q per head
constexpr int R_LS = 48;      // [4][8] final l
constexpr int R_ZS = 80;      // [4][8] final z
constexpr int R_BAR = 112;    // 2 mbarriers (8-byte aligned)
constexpr int R_TMEM = 116;   // TMEM base

template <int BITS, int NG>
__global__ void __launch_bounds__(THREADS, NG == 4 ? 4 : 2) attn_tc_kernel(DevCache c, AttnArgs a, int pkcap, int MT) {
  constexpr int N = 4 * NG;                  // MMA N: heads x base-256 digits
  constexpr uint32_t C_AK = 0, C_AV = 32, C_DS = 64, C_DO = 64 + N, C_DW = 64 + 2 * N;
  constexpr uint32_t TCOLS = NG == 4 ? 128 : 256;
  constexpr int NWK = 16 * BITS / 8;         // K fragment words per lane per tile (4 or 8)
  constexpr int TB = 16 * 128 * BITS / 8;    // bytes per 16-token tile
  constexpr uint32_t ID_QK = idesc_i8(128, N, 0, 1, 0, 1);
  constexpr uint32_t ID_PV = idesc_i8(128, N, 0, 0, 0, 1);
  const int u = blockIdx.y, chunk = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
  for (int i = tid; i < NG * 128; i += THREADS) {
    const int h = i >> 7, ch = i & 127;
    sq[i] = (h < G && ch < D) ? a.q[((int64_t)u * G + h) * D + ch] : 0.f;
  }
  for (int i = tid; i < MT * 1024; i += THREADS) reinterpret_cast<uint4*>(onehot)[i] = make_uint4(0, 0, 0, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t T = *tslot;
  const uint32_t lrow = (uint32_t)(32 * warp) << 16;  // this warp's TMEM lane quarter
#pragma unroll
  for (int h = 0; h < NG; ++h) {
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(sq[h * 128 + tid])));
    if (lane == 0) ri[R_BMAX + warp * 8 + h] = (int)m;
  }
  __syncthreads();
  // channel role constants: B_QK row, q o 4^-m scaled so |x| < 2^29
  int kshift;
  const int kposc = kpos_k<BITS>(tid, kshift);
  float qf[NG];
#pragma unroll
  for (int h = 0; h < NG; ++h) {
    unsigned m = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) m = max(m, (unsigned)ri[R_BMAX + w * 8 + h]);
    const int eq = m ? ceil_exp(__uint_as_float(m)) : 0;
    if (tid == 0) ri[R_EQ + h] = eq;
    qf[h] = ldexpf(sq[h * 128 + tid], 29 - eq - kshift);
  }
  // q.M table (scale_log2 folded in)
  for (int p = tid; p < Pk; p += THREADS) {
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
  for (int i = tid; i < nit; i += THREADS) {
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
  // this unit's arenas from this thread's view; a block adds (32-bit) b * stride
  const uint32_t bbytes = (uint32_t)c.blk_bytes, gp = (uint32_t)c.GP, kps = 2u * (uint32_t)c.Dp;
  const uint8_t* klane = c.kcodes + ubase * c.blk_bytes + (2 * warp) * TB + lane * (4 * NWK);
  const uint8_t* vlane = c.vcodes + ubase * c.blk_bytes + lane * (8 * BITS) + (BITS == 2 ? 8 * (warp >> 1) : 8 * warp);
  const bool has_slot = tid < c.GP;
  const int16_t* kidx_u = c.kidx + ubase * c.GP + tid;
  const int16_t* vidx_u = c.vidx + ubase * c.GP + tid;
  const float2* vp_u = reinterpret_cast<const float2*>(c.vparam32) + ubase * c.GP + tid;
  const float* ks_u = c.kparam32 + ubase * 2 * c.Dp + tid;
  uint32_t kw[2][NWK];   // K fragment words of tiles 2w, 2w+1 (block b + 1)
  uint2 vw[8];           // V fragment words, this warp's channel quarter of the 8 tiles (block b)
  float s_nx = 0.f;      // K scale of channel tid (block b + 1)
  int kidx_t = RAW, vidx_t = RAW, kidx_n = RAW, vidx_n = RAW, L_t = 128, L_n = 128;
  float vs_t = 0.f, vz_t = 0.f, vs_n = 0.f, vz_n = 0.f;
  auto load_k = [&](int bb) {
    const uint8_t* p = klane + (uint32_t)bb * bbytes;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (ntile == 8 || 2 * warp + i < ntile) {
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
    s_nx = __ldg(ks_u + (uint32_t)bb * kps);
  };
  auto load_v = [&](int bb) {
    const uint8_t* p = vlane + (uint32_t)bb * bbytes;
    if (ntile == 8) {
#pragma unroll
      for (int ti = 0; ti < 8; ++ti) vw[ti] = __ldg(reinterpret_cast<const uint2*>(p + ti * TB));
    } else {
#pragma unroll
      for (int ti = 0; ti < 8; ++ti) vw[ti] = ti < ntile ? __ldg(reinterpret_cast<const uint2*>(p + ti * TB)) : make_uint2(0u, 0u);
    }
  };
  auto load_meta = [&](int bb) {  // token tid of block bb -> the *_n registers
    L_n = __ldg(c.blk_len + bb);
    if (has_slot) {
      const uint32_t o = (uint32_t)bb * gp;
      kidx_n = __ldg(kidx_u + o);
      vidx_n = __ldg(vidx_u + o);
      const float2 vp = __ldg(vp_u + o);
      vs_n = vp.x; vz_n = vp.y;
    } else {
      kidx_n = RAW; vidx_n = RAW; vs_n = 0.f; vz_n = 0.f;
    }
  };
  auto next_meta = [&]() { kidx_t = kidx_n; vidx_t = vidx_n; vs_t = vs_n; vz_t = vz_n; L_t = L_n; };
  // K planes of the loaded block -> A_K, B_QK row of channel tid (block local index i)
  auto k_side = [&](int i) {
    constexpr int NP = BITS == 2 ? 4 : 2;  // planes per word
#pragma unroll
    for (int t2 = 0; t2 < 2; ++t2) {
      uint32_t r[16];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {  // repeat rr: word pair (2 (rr / NP), +1), plane rr % NP
        const int wi = 2 * (rr / NP), m = rr % NP;
        const uint32_t mask = BITS == 2 ? (0x03030303u << (2 * m)) : (m ? 0xF0F0F0F0u : 0x0F0F0F0Fu);
        r[2 * rr] = kw[t2][wi] & mask;
        r[2 * rr + 1] = kw[t2][wi + 1] & mask;
      }
      st16x128x8(T + lrow + ((uint32_t)(16 * t2) << 16) + C_AK, r);
    }
    const float t = s_nx * st_si[i];
    uint32_t x[NG];
#pragma unroll
    for (int h = 0; h < NG; ++h) x[h] = ((uint32_t)__float2int_rn(qf[h] * t) + 0x80808080u) ^ 0x80808080u;
#pragma unroll
    for (int gp = 0; gp < NG / 4; ++gp)
      *reinterpret_cast<uint4*>(bqk + gp * 2048 + kposc * 16) = make_uint4(x[4 * gp], x[4 * gp + 1], x[4 * gp + 2], x[4 * gp + 3]);
  };

  float mref[NG], lsum[NG], zsum[NG], Of[NG], Wf[2][NG];
#pragma unroll
  for (int h = 0; h < NG; ++h) {
    mref[h] = -FLT_MAX; lsum[h] = 0.f; zsum[h] = 0.f; Of[h] = 0.f; Wf[0][h] = 0.f; Wf[1][h] = 0.f;
  }
  int Ev = 0;
  float evs31 = INFINITY;  // 2^(Ev - 31); +inf until the first V block sets Ev
  bool fresh = true;
  const int vsh = vshift<BITS>(tid);
  const int kposv = kpos_v(tid);
  int oh_off = -1;  // this token's one-hot byte (cleared after the block's W MMA)
  // descriptors (thread 0 issues every MMA)
  const uint64_t dqk = desc_none(bqk, 128, 2048), dpv = desc_none(bpv, 128, 2048), dbw = desc_none(bw, 128, 2048);
  const uint64_t doh = desc_none(onehot, 2048, 128);

  // flush the TMEM sums into fp32 registers (current Ev), then scale everything by alpha
  auto flush = [&](const float (&alpha)[NG]) {
    if (!fresh) {
      uint32_t v[32];
      if constexpr (N == 16) tmem_ld16(T + lrow + C_DO, v); else tmem_ld32(T + lrow + C_DO, v);
      tmem_ld_wait();
      const float so = ldexpf(1.f, -Ev - vsh);
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        float x = (float)(int)v[4 * h + 3];
        x = fmaf(x, 256.f, (float)(int)v[4 * h + 2]);
        x = fmaf(x, 256.f, (float)(int)v[4 * h + 1]);
        x = fmaf(x, 256.f, (float)(int)v[4 * h]);
        Of[h] = fmaf(x, so, Of[h]);
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        if (mt >= MT) break;
        if constexpr (N == 16) tmem_ld16(T + lrow + C_DW + N * mt, v); else tmem_ld32(T + lrow + C_DW + N * mt, v);
        tmem_ld_wait();
#pragma unroll
        for (int h = 0; h < NG; ++h) {
          float x = (float)(int)v[4 * h + 3];
          x = fmaf(x, 256.f, (float)(int)v[4 * h + 2]);
          x = fmaf(x, 256.f, (float)(int)v[4 * h + 1]);
          x = fmaf(x, 256.f, (float)(int)v[4 * h]);
          Wf[mt][h] = fmaf(x, 4.656612873077393e-10f, Wf[mt][h]);  // 2^-31
        }
      }
    }
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      Of[h] *= alpha[h]; lsum[h] *= alpha[h]; zsum[h] *= alpha[h];
      Wf[0][h] *= alpha[h]; Wf[1][h] *= alpha[h];
    }
    fresh = true;
  };

  __syncthreads();  // block statistics
  if (nit > 0) {
    load_k(b0);
    load_v(b0);
    load_meta(b0);
    next_meta();
    k_side(0);
    if (nit > 1) load_k(b0 + 1);
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
    const int b = b0 + it;
    const bool more = it + 1 < nit;
    if (more) load_meta(b + 1);
    // (i) scores of token tid
    float lg[NG];
    {
      mbar_wait(mbS, it & 1);
      tc_fence_after();
      uint32_t v[32];
      if constexpr (N == 16) tmem_ld16(T + lrow + C_DS, v); else tmem_ld32(T + lrow + C_DS, v);
      float add[NG];
      if (kidx_t >= 0 && kidx_t < Pk) {
#pragma unroll
        for (int gp = 0; gp < NG / 4; ++gp) {
          const float4 x = *reinterpret_cast<const float4*>(qm + kidx_t * NG + 4 * gp);
          add[4 * gp] = x.x; add[4 * gp + 1] = x.y; add[4 * gp + 2] = x.z; add[4 * gp + 3] = x.w;
        }
      } else {
#pragma unroll
        for (int h = 0; h < NG; ++h) add[h] = 0.f;
      }
      float c1[NG];
#pragma unroll
      for (int gp = 0; gp < NG / 4; ++gp) {
        const float4 x = *reinterpret_cast<const float4*>(st_c1 + it * NG + 4 * gp);
        const float4 z = *reinterpret_cast<const float4*>(st_qz + it * NG + 4 * gp);
        c1[4 * gp] = x.x; c1[4 * gp + 1] = x.y; c1[4 * gp + 2] = x.z; c1[4 * gp + 3] = x.w;
        add[4 * gp] += z.x; add[4 * gp + 1] += z.y; add[4 * gp + 2] += z.z; add[4 * gp + 3] += z.w;
      }
      tmem_ld_wait();
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        const int lo = (int)v[4 * h + 1] * 256 + (int)v[4 * h];
        const int hi = (int)v[4 * h + 3] * 256 + (int)v[4 * h + 2];
        lg[h] = fmaf(fmaf((float)hi, 65536.f, (float)lo), c1[h], add[h]);
      }
      if (L_t < 128 && tid >= L_t) {
#pragma unroll
        for (int h = 0; h < NG; ++h) lg[h] = -INFINITY;
      }
    }
    // (ii) next block's K side (A_K and B_QK are free: QK(b) is complete)
    if (more) {
      k_side(it + 1);
      st_wait();
      fence_proxy_async();
      tc_fence_before();
      // QK(b + 1) as soon as every warp's A_K rows are in: warp 0 waits, the others only arrive
      if (warp == 0) {
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (lane == 0) {
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ts(T + C_DS, T + C_AK + 8 * k, dqk + 32 * k, ID_QK, k > 0);
          mma_commit(mbS);
        }
        __syncwarp();
      } else {
        asm volatile("bar.arrive 2, 128;" ::: "memory");
      }
      if (it + 2 < nit) load_k(b + 2);
    }
    // (iii) softmax of token tid: p' = 2^31 exp2(lg - m_ref), digits of p' and p' s_t 2^(Ev-31)
    float p8[NG];
    uint32_t xw[NG], xv[NG];
    bool flag;
    auto probs = [&]() {
      // evs31 = +inf until the first V scale exponent is set: any valid token with s_t > 0 flags
      const float sE = vs_t * evs31;
      float dmax = (lg[0] > -INFINITY && sE >= 1.f) ? INFINITY : -INFINITY;
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        const float d = lg[h] - (mref[h] - 31.f);
        dmax = fmaxf(dmax, d);
        p8[h] = ex2(d);
        xw[h] = __float2uint_rn(p8[h]);
        xv[h] = __float2uint_rn(p8[h] * sE);
      }
      flag = dmax > 31.f;
    };
    probs();
    {
      const bool any = __any_sync(0xffffffffu, flag);
      if (lane == 0) ri[R_FLAG + warp] = any;
    }
    // (iv) after PV / W of block b - 1: V planes -> A_V, one-hot and B rows of block b
    tc_fence_after();
    if (it > 0) mbar_wait(mbPV, (it - 1) & 1);
    tc_fence_after();
    {
      uint32_t ra[16], rb[16];
#pragma unroll
      for (int ti = 0; ti < 8; ++ti) {
        if (BITS == 2) {
          const uint32_t p0 = prmt(vw[ti].x, vw[ti].y, (warp & 1) ? 0x7531u : 0x6420u);
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
      st16x128x8(T + lrow + C_AV, ra);
      st16x128x8(T + lrow + (16u << 16) + C_AV, rb);
    }
    if (more) load_v(b + 1);
    if (oh_off >= 0) onehot[oh_off] = 0;
    oh_off = (lg[0] > -INFINITY && vidx_t >= 0 && vidx_t < Pv) ? (vidx_t >> 7) * 16384 + (kposv >> 4) * 2048 + (vidx_t & 127) * 16 + (kposv & 15) : -1;
    if (oh_off >= 0) onehot[oh_off] = 1;
    auto write_rows = [&]() {
#pragma unroll
      for (int gp = 0; gp < NG / 4; ++gp) {
        *reinterpret_cast<uint4*>(bw + gp * 2048 + kposv * 16) = make_uint4(xw[4 * gp], xw[4 * gp + 1], xw[4 * gp + 2], xw[4 * gp + 3]);
        *reinterpret_cast<uint4*>(bpv + gp * 2048 + kposv * 16) = make_uint4(xv[4 * gp], xv[4 * gp + 1], xv[4 * gp + 2], xv[4 * gp + 3]);
      }
    };
    write_rows();
    st_wait();
    fence_proxy_async();
    tc_fence_before();
    bar_sync1();
    if ((ri[R_FLAG] | ri[R_FLAG + 1] | ri[R_FLAG + 2] | ri[R_FLAG + 3]) != 0) {
      // CTA-uniform slow path: new running max / V scale exponent; flush the TMEM sums
      tc_fence_after();
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        const int k = __reduce_max_sync(0xffffffffu, fkey(lg[h]));
        if (lane == 0) ri[R_BMAX + warp * 8 + h] = k;
      }
      {
        const unsigned m = __reduce_max_sync(0xffffffffu, lg[0] > -INFINITY ? __float_as_uint(vs_t) : 0u);
        if (lane == 0) ri[R_SVM + warp] = (int)m;
      }
      bar_sync1();
      float alpha[NG], mnew[NG];
#pragma unroll
      for (int h = 0; h < NG; ++h) {
        int k = ri[R_BMAX + h];
#pragma unroll
        for (int w = 1; w < 4; ++w) k = max(k, ri[R_BMAX + w * 8 + h]);
        const float bm = funkey(k);
        mnew[h] = bm == -INFINITY ? mref[h] : fmaxf(mref[h], bm + TH);
        alpha[h] = mref[h] == -FLT_MAX ? 0.f : ex2(mref[h] - mnew[h]);
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
      for (int h = 0; h < NG; ++h) mref[h] = mnew[h];
      probs();
      write_rows();
      fence_proxy_async();
      tc_fence_before();
      bar_sync1();
    }
#pragma unroll
    for (int h = 0; h < NG; ++h) {
      lsum[h] += p8[h];
      zsum[h] = fmaf(p8[h], vz_t, zsum[h]);
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
    float one[NG];
#pragma unroll
    for (int h = 0; h < NG; ++h) one[h] = 1.f;
    flush(one);
  }
  // l and z: token partials summed over the CTA (units of 2^-31)
#pragma unroll
  for (int h = 0; h < NG; ++h) {
    float l = lsum[h], z = zsum[h];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
      z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    if (lane == 0) { rf[R_LS + warp * 8 + h] = l; rf[R_ZS + warp * 8 + h] = z; }
  }
  // pattern weights: thread tid holds W for patterns tid and 128 + tid
  float* Wt = reinterpret_cast<float*>(onehot);  // [MT*128][NG], the one-hot is no longer read
  __syncthreads();
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    if (mt >= MT) break;
#pragma unroll
    for (int h = 0; h < NG; ++h) Wt[(mt * 128 + tid) * NG + h] = Wf[mt][h];
  }
  __syncthreads();
  float* out = a.part + (((int64_t)u * a.nchunk + chunk) * G) * (c.Dp + 2);
  for (int h = 0; h < G; ++h) {
    float lt = 0.f, zt = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) { lt += rf[R_LS + w * 8 + h]; zt += rf[R_ZS + w * 8 + h]; }
    float o = fmaf(zt, 4.656612873077393e-10f, Of[h]);
    if (tid < D) {
      const float* mv = c.vpat32 + (int64_t)u * c.Pcap * c.Dp + tid;
      for (int p = 0; p < Pv; ++p) o = fmaf(Wt[p * NG + h], __ldg(mv + (int64_t)p * c.Dp), o);
    }
    out[h * (c.Dp + 2) + tid] = o;
    if (tid == 0) {
      out[h * (c.Dp + 2) + c.Dp] = (nit > 0 && mref[h] != -FLT_MAX) ? mref[h] : -INFINITY;
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
  attn_tc_kernel<BITS, NG><<<dim3(a.nchunk, c.U), THREADS, smem, st>>>(c, a, pkcap, MT);
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
