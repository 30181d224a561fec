// K3 decode_attn: softmax(q K^T * scale) V over the PatternKV cache of every
// unit (new; the reference defines only the reconstruction it must equal,
// engine.py:255-303 + the exact window, SPEC.md:318 has no attention).
//
// K is never materialised: with k_t = s_b*code_t + z_b + M[idx_t] (per-channel
// block params s_b, z_b),
//   q.k_t = (q o s_b).code_t + q.z_b + (q.M)[idx_t]
// and with v_t = s_t*code_t + z_t + M'[idx_t] (per-token params),
//   sum_t p_t v_t = sum_t (p_t s_t) code_t + (sum_t p_t z_t) 1 + sum_p W_p M'_p,
// W_p = sum_{t: idx_t = p} p_t.  The code products run on tensor cores
// (mma.m16n8k16, fp32 accumulate) with A fragments dequantized in registers
// straight from one vector load of the fragment-ordered codes (LOP3 + HFMA2);
// q o s and p o s are split hi+lo into two fp16 columns so the fp16 operand
// rounding stays below 2^-22 relative.  Flash-decoding: CTA = chunk of blocks,
// warp = stream of whole 128-token blocks, lazy online-softmax rescale; a
// per-unit merge kernel adds the fp16 window exactly and combines chunks.
#include "pkv_common.cuh"

namespace pkv {

constexpr int ATT_WARPS = 4;
constexpr int ATT_THREADS = ATT_WARPS * 32;
constexpr int MAXG = 8;         // GQA group size served (query heads per KV head)
constexpr float RESCALE_TH = 8.f;  // lazy rescale threshold (log2 units)

__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float fast_exp2(float x) {  // MUFU.EX2 (2^-22 rel), exp2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t lop3_magic(uint32_t w, uint32_t mask) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "r"(mask), "r"(0x64006400u));  // (w & mask) | magic
  return r;
}
__device__ __forceinline__ uint32_t hfma2_u(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
// register transpose of an 8x8 b16 tile held in mma C/A-fragment order
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
  uint32_t r;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
  return (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
}

// Dequantize slot s of a code word into the half2 (1024 + 2^k c_lo, 1024 + 2^k c_hi),
// k = frag_slot_shift(s): one LOP3 (plus a shared byte shift for the upper slots).
// The constant 1024 and the per-channel 2^k are removed exactly outside the MMA
// (K: folded into B and a per-block bias; V: per-row correction of the output).
template <int BITS>
__device__ __forceinline__ uint32_t slot_raw(uint32_t w, int s) {
  constexpr int PER = 8 / BITS;  // slots in the low byte of each half
  const uint32_t ww = s >= PER ? (w >> 8) : w;
  const int ss = s >= PER ? s - PER : s;
  const uint32_t mask = ((1u << BITS) - 1) * 0x00010001u << (ss * BITS);
  return lop3_magic(ww, mask);
}

// exact code values (c_lo, c_hi): raw value * 2^-k - 1024 * 2^-k in one HFMA2
template <int BITS>
__device__ __forceinline__ uint32_t slot_exact(uint32_t w, int s) {
  constexpr int PER = 8 / BITS;
  const int k = (s % PER) * BITS;
  const float sc = 1.f / (float)(1 << k);
  const __half hs = __float2half_rn(sc), hb = __float2half_rn(-1024.f * sc);
  return hfma2_u(slot_raw<BITS>(w, s), pack_h2(hs, hs), pack_h2(hb, hb));
}

template <int BITS>
__device__ __forceinline__ void load_words(const uint8_t* tile, int lane, uint32_t* w, int WL) {
  constexpr int NW = 16 * BITS / 8;  // words per lane at Dp = 128
  if (WL == NW) {
    const uint4* p = reinterpret_cast<const uint4*>(tile) + lane * (NW / 4);
#pragma unroll
    for (int i = 0; i < NW / 4; ++i) {
      uint4 v = __ldg(p + i);
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  } else {  // head_dim < 128: fewer words per lane
    const uint32_t* p = reinterpret_cast<const uint32_t*>(tile) + lane * WL;
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = i < WL ? __ldg(p + i) : 0u;
  }
}

// per-lane private pattern-weight copies while they fit in 64 KB
__host__ __device__ inline bool attn_w_private(int Pv, int NT) {
  return (size_t)ATT_WARPS * 8 * (Pv > 1 ? Pv : 1) * 4 * NT * 4 <= 64 * 1024;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BITS>
__device__ __forceinline__ void load_stage_words(const unsigned char* p, uint32_t* w, int WL) {
  constexpr int NW = 16 * BITS / 8;  // words per lane at Dp = 128
  if (WL == NW) {
#pragma unroll
    for (int i = 0; i < NW / 4; ++i) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[i];
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = i < WL ? reinterpret_cast<const uint32_t*>(p)[i] : 0u;
  }
}

// A fragments of sub-tile j (4 half2 registers) from the lane's code words.
template <int BITS, int SIDE>
__device__ __forceinline__ void afrag(const uint32_t* w, int j, uint32_t* a) {
#pragma unroll
  for (int reg = 0; reg < 4; ++reg) {
    int word, slot;
    frag_word_slot(SIDE, 4 * j + reg, BITS, word, slot);
    // K: raw 1024 + 2^k c (bias and 2^k folded into B); V: exact c (the PV accumulator runs
    // over thousands of tiles; a folded 1024 bias would cost it ~10 bits)
    a[reg] = SIDE == 0 ? slot_raw<BITS>(w[word], slot) : slot_exact<BITS>(w[word], slot);
  }
}

template <int BITS, int NT, int KT>
__global__ void __launch_bounds__(ATT_THREADS, NT == 1 ? 4 : 2) attn_chunk_kernel(DevCache c, AttnArgs a) {
  const int u = blockIdx.y, chunk = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, qd = lane & 3;
  constexpr int Dp = 16 * KT;  // == c.Dp
  constexpr int WL = Dp * BITS / 64;
  const int D = c.D, G = a.G;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* sq = reinterpret_cast<float*>(smem_raw);                 // [MAXG][Dp]
  float* sqm = sq + MAXG * Dp;                                     // [Pk][MAXG]
  const int Pk = c.use_kp ? c.nk[u] : 0;
  const int Pv = c.use_vp ? c.nv[u] : 0;
  // pattern weights W_p = sum_{t: idx_t = p} p_t.  priv: one private copy per lane
  // ([warps][g][Pv][HN], plain read-modify-write, no atomics); else shared per warp
  // ([warps][Pv][MAXG]) with atomics.  Wc = the merged [Pv][MAXG] table.
  constexpr int HN = 4 * NT;
  const bool priv = attn_w_private(Pv, NT);
  const size_t wfl = priv ? (size_t)ATT_WARPS * 8 * max(Pv, 1) * HN : (size_t)ATT_WARPS * max(Pv, 1) * MAXG;
  float* sW = sqm + (size_t)max(Pk, 1) * MAXG;
  float* Wc = sW + wfl;                                             // [Pv][MAXG]
  __half* sP = reinterpret_cast<__half*>(Wc + (size_t)max(Pv, 1) * MAXG);  // [warps][16][16]
  float* sred = reinterpret_cast<float*>(sP + ATT_WARPS * 256);   // [warps][MAXG][4]

  // ---- per-unit setup: q, q.M table, zeroed pattern weights -----------------------
  for (int i = tid; i < MAXG * Dp; i += ATT_THREADS) {
    const int h = i / Dp, ch = i - h * Dp;
    sq[i] = (h < G && ch < D) ? a.q[((int64_t)u * G + h) * D + ch] : 0.f;
  }
  for (size_t i = tid; i < wfl; i += ATT_THREADS) sW[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < Pk * MAXG; i += ATT_THREADS) {
    const int p = i / MAXG, h = i - p * MAXG;
    float s = 0.f;
    if (h < G) {
      const float* m = c.kpat32 + ((int64_t)u * c.Pcap + p) * Dp;
      const float* qq = sq + h * Dp;
      for (int ch = 0; ch < D; ++ch) s = fmaf(qq[ch], m[ch], s);
    }
    sqm[i] = s;
  }
  __syncthreads();

  // ---- per-warp streaming state ----------------------------------------------------
  float oacc[8][NT][4];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) oacc[mt][nt][r] = 0.f;
  float mrun[NT], lsum[NT], zsum[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) { mrun[nt] = -INFINITY; lsum[nt] = 0.f; zsum[nt] = 0.f; }
  // this lane's W slot for (pattern p, head 4nt+qd)
  auto wslot = [&](int p, int nt) -> float* {
    return priv ? sW + (((size_t)warp * 8 + g) * max(Pv, 1) + p) * HN + 4 * nt + qd
                : sW + ((size_t)warp * max(Pv, 1) + p) * MAXG + 4 * nt + qd;
  };

  const int b0 = a.blk0 + chunk * a.bpc;
  const int b1 = min(a.blk0 + a.nb, b0 + a.bpc);
  // ---- register-prefetched tile stream: the lane's 16*BITS/8 code words per side come
  // straight from HBM (fragment order makes them one contiguous vector per lane) while the
  // previous tile computes; metadata: kidx / vidx / vparam of tokens g, g+8
  constexpr int NW = 16 * BITS / 8;
  constexpr int tbytes = 16 * Dp * BITS / 8;
  struct Tile {
    uint32_t kw[NW], vw[NW];
    int ki0, ki1, vi0, vi1;
    float2 vp0, vp1;
  };
  // per-block base: the block offset, and at 2 bits (where registers allow) the code pointers,
  // so the per-tile address work is a few adds
  struct BlkPtr {
    int64_t bo;
    const uint8_t* k;
    const uint8_t* v;
  };
  auto blk_ptr = [&](int bb) {
    BlkPtr p;
    p.bo = (int64_t)u * c.NBcap + bb;
    if constexpr (BITS == 2) {
      p.k = c.kcodes + p.bo * c.blk_bytes;
      p.v = c.vcodes + p.bo * c.blk_bytes;
    }
    return p;
  };
  auto load_tile = [&](const BlkPtr& bp, int ti, Tile& t) {
    const uint8_t* kb = BITS == 2 ? bp.k : c.kcodes + bp.bo * c.blk_bytes;
    const uint8_t* vb = BITS == 2 ? bp.v : c.vcodes + bp.bo * c.blk_bytes;
    load_words<BITS>(kb + ti * tbytes, lane, t.kw, WL);
    load_words<BITS>(vb + ti * tbytes, lane, t.vw, WL);
    const int64_t slot = bp.bo * c.GP + g + 16 * ti;
    t.ki0 = __ldg(c.kidx + slot); t.ki1 = __ldg(c.kidx + slot + 8);
    t.vi0 = __ldg(c.vidx + slot); t.vi1 = __ldg(c.vidx + slot + 8);
    t.vp0 = __ldg(reinterpret_cast<const float2*>(c.vparam32) + slot);
    t.vp1 = __ldg(reinterpret_cast<const float2*>(c.vparam32) + slot + 8);
  };
  // this lane's pattern-weight column base: W slot (p, head 4nt+qd) = wbase + p * wstride + 4nt
  float* const wbase = priv ? sW + ((size_t)warp * 8 + g) * max(Pv, 1) * HN + qd : sW + (size_t)warp * max(Pv, 1) * MAXG + qd;
  const int wstride = priv ? HN : MAXG;

  uint32_t bq[8][NT][2];
  float qz[NT], kbias[NT];
  auto block_setup = [&](int bb) {
    const float* kp = c.kparam32 + ((int64_t)u * c.NBcap + bb) * 2 * Dp;
    // B fragments of 64 * 2^-k(c) * (q o s_b) (hi/lo columns), q.z_b per head, and
    // the per-column bias 1024 * sum_c B[c][col] the magic-number A operand adds
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int col = 8 * nt + g, h = col >> 1, hl = col & 1;
      float zpart = 0.f, bpart = 0.f;
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
        if (kt < KT) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int ch = 16 * kt + 2 * qd + 8 * hh;
            constexpr int HS = 8 / BITS;
            const float fk = (float)(64 >> frag_slot_shift(2 * (kt % HS) + hh, BITS));  // 2^(6-k)
            const float2 s2 = __ldg(reinterpret_cast<const float2*>(kp + ch));
            const float2 z2 = __ldg(reinterpret_cast<const float2*>(kp + Dp + ch));
            const float q0 = sq[h * Dp + ch], q1 = sq[h * Dp + ch + 1];
            const float t0 = q0 * s2.x * fk, t1 = q1 * s2.y * fk;
            const __half2 hi = __floats2half2_rn(t0, t1);
            const float2 bk = __half22float2(hi);
            const __half2 lo = __floats2half2_rn(t0 - bk.x, t1 - bk.y);
            const __half2 e = hl ? lo : hi;
            const float2 ef = __half22float2(e);
            bpart += ef.x + ef.y;
            bq[kt][nt][hh] = *reinterpret_cast<const uint32_t*>(&e);
            zpart = fmaf(q0, z2.x, fmaf(q1, z2.y, zpart));
          }
        }
      }
      zpart += __shfl_xor_sync(0xffffffffu, zpart, 1);
      zpart += __shfl_xor_sync(0xffffffffu, zpart, 2);
      bpart += __shfl_xor_sync(0xffffffffu, bpart, 1);
      bpart += __shfl_xor_sync(0xffffffffu, bpart, 2);
      qz[nt] = __shfl_sync(0xffffffffu, zpart, 8 * qd);  // head 4nt+qd lives at g = 2qd
      kbias[nt] = 1024.f * (__shfl_sync(0xffffffffu, bpart, 8 * qd) + __shfl_sync(0xffffffffu, bpart, 8 * qd + 4));
    }
  };

  int b = b0 + warp, ti = 0;
  Tile ta, tb;
  BlkPtr bp{};  // current block of this warp
  int L = 0;
  if (b < b1) {
    bp = blk_ptr(b);
    L = __ldg(c.blk_len + b);
    load_tile(bp, 0, ta);
    block_setup(b);
  }
  // one tile of block b (state cur), prefetching the next tile of the warp into nxt
  auto step = [&](Tile& cur, Tile& nxt) {
    const int ntile = (L + 15) >> 4;
    int nti = ti + 1;
    const bool nextblk = nti >= ntile;
    if (nextblk) nti = 0;
    if (!nextblk) load_tile(bp, nti, nxt);  // prefetch while this tile computes
    else if (b + ATT_WARPS < b1) load_tile(blk_ptr(b + ATT_WARPS), 0, nxt);
    const int r0 = 16 * ti + g, r1 = r0 + 8;
    const bool ok0 = r0 < L, ok1 = r1 < L;
    const int vi0 = ok0 ? cur.vi0 : -1, vi1 = ok1 ? cur.vi1 : -1;
    const float2 vp0 = ok0 ? cur.vp0 : make_float2(0.f, 0.f);
    const float2 vp1 = ok1 ? cur.vp1 : make_float2(0.f, 0.f);

    // ---- S = K . (q o s): tokens on M, hi/lo head columns on N ----
    // two accumulator chains (even / odd k-tiles) halve the dependent-MMA latency
    float sacc[NT][4], sacc2[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) { sacc[nt][r] = 0.f; sacc2[nt][r] = 0.f; }
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      if (kt < KT) {
        uint32_t af[4];
        afrag<BITS, 0>(cur.kw, kt, af);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mma16816((kt & 1) ? sacc2[nt] : sacc[nt], af, bq[kt][nt][0], bq[kt][nt][1]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) sacc[nt][r] += sacc2[nt][r];
    // ---- online softmax (lazy rescale), P~ = p * s_t split hi/lo ----
    uint32_t pt[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int h = 4 * nt + qd;
      const float add0 = qz[nt] + (cur.ki0 >= 0 && ok0 ? sqm[cur.ki0 * MAXG + h] : 0.f);
      const float add1 = qz[nt] + (cur.ki1 >= 0 && ok1 ? sqm[cur.ki1 * MAXG + h] : 0.f);
      const float s0 = ok0 ? fmaf(sacc[nt][0] + sacc[nt][1] - kbias[nt], 0.015625f, add0) * a.scale_log2 : -INFINITY;
      const float s1 = ok1 ? fmaf(sacc[nt][2] + sacc[nt][3] - kbias[nt], 0.015625f, add1) * a.scale_log2 : -INFINITY;
      // lazy rescale: only when some lane's score passes the running max by the threshold
      if (__any_sync(0xffffffffu, fmaxf(s0, s1) > mrun[nt] + RESCALE_TH)) {
        float tmax = fmaxf(s0, s1);
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
        if (tmax > mrun[nt] + RESCALE_TH) {  // uniform over the 8 lanes of head 4nt+qd
          const float mnew = fmaxf(tmax, mrun[nt]);
          const float alpha = mrun[nt] == -INFINITY ? 0.f : fast_exp2(mrun[nt] - mnew);
          lsum[nt] *= alpha;
          zsum[nt] *= alpha;
#pragma unroll
          for (int mt = 0; mt < 8; ++mt)
#pragma unroll
            for (int r = 0; r < 4; ++r) oacc[mt][nt][r] *= alpha;
          if (priv) {
            for (int p = 0; p < Pv; ++p) wbase[p * wstride + 4 * nt] *= alpha;
          } else {
            for (int p = g; p < Pv; p += 8) wbase[p * wstride + 4 * nt] *= alpha;
          }
          mrun[nt] = mnew;
        }
      }
      const float p0 = fast_exp2(s0 - mrun[nt]), p1 = fast_exp2(s1 - mrun[nt]);
      lsum[nt] += p0 + p1;
      zsum[nt] = fmaf(p0, vp0.y, fmaf(p1, vp1.y, zsum[nt]));
      if (priv) {
        if (vi0 >= 0) wbase[vi0 * wstride + 4 * nt] += p0;
        if (vi1 >= 0) wbase[vi1 * wstride + 4 * nt] += p1;
      } else {
        __syncwarp();  // rescaled W visible before other lanes add into it
        if (vi0 >= 0 && p0 != 0.f) atomicAdd(&wbase[vi0 * wstride + 4 * nt], p0);
        if (vi1 >= 0 && p1 != 0.f) atomicAdd(&wbase[vi1 * wstride + 4 * nt], p1);
      }
      const float w0 = p0 * vp0.x, w1 = p1 * vp1.x;
      const __half2 wh = __floats2half2_rn(w0, w1);
      const float2 wb = __half22float2(wh);
      const __half2 wl = __floats2half2_rn(w0 - wb.x, w1 - wb.y);
      // P~ rows g / g+8 (cols 2qd, 2qd+1 = hi, lo of head 4nt+qd) are C-fragment
      // 8x8 b16 tiles; their transposes are exactly the PV B fragments (k = token, n = col)
      const __half2 rr0 = __halves2half2(__low2half(wh), __low2half(wl));
      const __half2 rr1 = __halves2half2(__high2half(wh), __high2half(wl));
      pt[nt][0] = movmatrix_t(*reinterpret_cast<const uint32_t*>(&rr0));
      pt[nt][1] = movmatrix_t(*reinterpret_cast<const uint32_t*>(&rr1));
    }
    // ---- O^T += V^T . P~ : channels on M ----
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      if (mt < KT) {
        uint32_t af[4];
        afrag<BITS, 1>(cur.vw, mt, af);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mma16816(oacc[mt][nt], af, pt[nt][0], pt[nt][1]);
      }
    }
    ti = nti;
    if (nextblk) {
      b += ATT_WARPS;
      if (b < b1) {
        bp = blk_ptr(b);
        L = __ldg(c.blk_len + b);
        block_setup(b);
      }
    }
  };
  while (b < b1) {
    step(ta, tb);
    ta = tb;
  }

  // ---- merge the warps of the CTA --------------------------------------------------
  // per-head running max m (same for the 8 lanes of a head), l and z partial per lane
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    float l = lsum[nt], z = zsum[nt];
    l += __shfl_xor_sync(0xffffffffu, l, 4); l += __shfl_xor_sync(0xffffffffu, l, 8); l += __shfl_xor_sync(0xffffffffu, l, 16);
    z += __shfl_xor_sync(0xffffffffu, z, 4); z += __shfl_xor_sync(0xffffffffu, z, 8); z += __shfl_xor_sync(0xffffffffu, z, 16);
    const int h = 4 * nt + qd;
    if (g == 0 && h < MAXG) {
      sred[(warp * MAXG + h) * 4 + 0] = mrun[nt];
      sred[(warp * MAXG + h) * 4 + 1] = l;
      sred[(warp * MAXG + h) * 4 + 2] = z;
    }
  }
  __syncthreads();
  // global max per head and each warp's factor
  float fac[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int h = min(4 * nt + qd, MAXG - 1);
    float M = -INFINITY;
    for (int w = 0; w < ATT_WARPS; ++w) M = fmaxf(M, sred[(w * MAXG + h) * 4]);
    fac[nt] = (mrun[nt] == -INFINITY) ? 0.f : exp2f(mrun[nt] - M);
  }
  // O reduction buffer reuses sq: [MAXG][Dp] (q no longer needed)
  __syncthreads();
  for (int i = tid; i < MAXG * Dp; i += ATT_THREADS) sq[i] = 0.f;
  __syncthreads();
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    if (mt < KT) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int h = 4 * nt + qd;
        if (h < MAXG) {
          atomicAdd(&sq[h * Dp + 16 * mt + g], (oacc[mt][nt][0] + oacc[mt][nt][1]) * fac[nt]);
          atomicAdd(&sq[h * Dp + 16 * mt + g + 8], (oacc[mt][nt][2] + oacc[mt][nt][3]) * fac[nt]);
        }
      }
    }
  }
  __syncthreads();
  // pattern weights merged over warps (and private lane copies): Wc[p][h] = sum_w fac_w(h) W_w[p][h]
  for (int i = tid; i < Pv * HN; i += ATT_THREADS) {
    const int p = i / HN, h = i - p * HN;
    float M = -INFINITY;
    for (int w = 0; w < ATT_WARPS; ++w) M = fmaxf(M, sred[(w * MAXG + h) * 4]);
    float acc = 0.f;
    for (int w = 0; w < ATT_WARPS; ++w) {
      const float mw = sred[(w * MAXG + h) * 4];
      if (mw == -INFINITY) continue;
      float sw = 0.f;
      if (priv) {
        for (int gg = 0; gg < 8; ++gg) sw += sW[(((size_t)w * 8 + gg) * Pv + p) * HN + h];
      } else {
        sw = sW[((size_t)w * Pv + p) * MAXG + h];
      }
      acc = fmaf(exp2f(mw - M), sw, acc);
    }
    Wc[p * MAXG + h] = acc;
  }
  __syncthreads();
  // final per-head sums and the pattern / zero-point terms, then write the partial
  float* out = a.part + (((int64_t)u * a.nchunk + chunk) * G) * (Dp + 2);
  for (int i = tid; i < G * Dp; i += ATT_THREADS) {
    const int h = i / Dp, ch = i - h * Dp;
    float M = -INFINITY, zt = 0.f;
    for (int w = 0; w < ATT_WARPS; ++w) M = fmaxf(M, sred[(w * MAXG + h) * 4]);
    for (int w = 0; w < ATT_WARPS; ++w) {
      const float mw = sred[(w * MAXG + h) * 4];
      if (mw != -INFINITY) zt += exp2f(mw - M) * sred[(w * MAXG + h) * 4 + 2];
    }
    float o = sq[i] + zt;
    if (ch < D) {
      for (int p = 0; p < Pv; ++p) o = fmaf(Wc[p * MAXG + h], c.vpat32[((int64_t)u * c.Pcap + p) * Dp + ch], o);
    }
    out[h * (Dp + 2) + ch] = o;
    if (ch == 0) {
      float l = 0.f;
      for (int w = 0; w < ATT_WARPS; ++w) {
        const float mw = sred[(w * MAXG + h) * 4];
        if (mw != -INFINITY) l += exp2f(mw - M) * sred[(w * MAXG + h) * 4 + 1];
      }
      out[h * (Dp + 2) + Dp] = M;
      out[h * (Dp + 2) + Dp + 1] = l;
    }
  }
}

// merge: exact fp32 attention over the window rows + combine chunk partials.
// grid U, block 32*G threads.  The window is shared by the unit's G query heads and every row is
// read from HBM once per unit: (1) thread per window row scores it against all G queries (the
// row's loads are all issued before the first FMA, so a row costs one HBM latency, not D), (2)
// warp h takes the max / exp2 / sum of head h's scores, (3) warp w accumulates p_r v_r for all G
// heads over rows r = w (mod G) with lanes over 4-channel vectors, 8 rows in flight, (4) warp h
// sums the G per-warp partials of head h in a fixed order (deterministic) and LSE-combines the
// chunk partials.  VEC needs D % 4 == 0 (4-element vector loads); otherwise scalar loads.
// (A warp per head walking the rows with a 5-shuffle reduction and an online rescale per row cost
// ~12% of a cfg2 decode step; a thread-per-row variant with scalar loads was no faster.)
template <typename T>
struct Vec4 { using raw = uint2; };
template <> struct Vec4<float> { using raw = uint4; };
template <> struct Vec4<double> { struct raw { uint4 a, b; }; };
template <typename T>
__device__ __forceinline__ typename Vec4<T>::raw ld4(const T* p) {
  return __ldg(reinterpret_cast<const typename Vec4<T>::raw*>(p));
}
template <>
__device__ __forceinline__ Vec4<double>::raw ld4<double>(const double* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  return {__ldg(q), __ldg(q + 1)};
}
__device__ __forceinline__ float4 cvt4(uint2 r, const __half*) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float4 cvt4(uint2 r, const __nv_bfloat16*) {
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float4 cvt4(uint4 r, const float*) {
  return make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z), __uint_as_float(r.w));
}
__device__ __forceinline__ float4 cvt4(Vec4<double>::raw r, const double*) {
  const double2 a = *reinterpret_cast<const double2*>(&r.a), b = *reinterpret_cast<const double2*>(&r.b);
  return make_float4((float)a.x, (float)a.y, (float)b.x, (float)b.y);
}
template <typename T>
__device__ __forceinline__ float to_f32(T x) { return (float)to_f64(x); }
template <>
__device__ __forceinline__ float to_f32<__half>(__half x) { return __half2float(x); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

constexpr int MERGE_WT = 1024;  // window rows scored per tile (online softmax across tiles)

template <typename T, bool VEC, int GC, bool TILED>
__global__ void attn_merge_kernel(DevCache c, AttnArgs a, int win_len, int win_slot0, float* out) {
  extern __shared__ float msm[];
  constexpr int GM = GC > 0 ? GC : MAXG;  // compile-time head count (GC = 0: a.G at run time)
  const int u = blockIdx.x, G = GC > 0 ? GC : a.G, NTH = 32 * G;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  // TILED: the window may exceed one score tile (else one tile: no rescale of the running sums)
  const int D = c.D, Dp = c.Dp, Wcap = c.Wcap, WT = TILED ? MERGE_WT : Wcap;
  float* qs = msm;                 // [G][D] queries
  float* sc = qs + G * D;          // [G][WT] scores, then probabilities, of one window tile
  float* rs = sc + G * WT;         // [G] per-head rescale of the running sums at this tile
  float* red = msm + ((G * D + G * WT + G + 3) & ~3);  // [G warps][G heads][D] partial outputs (VEC), 16-B aligned
  for (int i = tid; i < G * D; i += NTH) qs[i] = a.q[(int64_t)u * G * D + i];
  const T* wk = reinterpret_cast<const T*>(c.wk) + (int64_t)u * Wcap * D;
  const T* wv = reinterpret_cast<const T*>(c.wv) + (int64_t)u * Wcap * D;
  const int h = w;                 // phase (2) / (4): warp h = head h
  float m = -INFINITY, l = 0.f;    // head h's running max (log2 units) and sum
  float o[4] = {0.f, 0.f, 0.f, 0.f};
  float acc3[VEC ? GM : 1][4];     // VEC phase (3): this warp's rows, all heads
#pragma unroll
  for (int g = 0; g < (VEC ? GM : 1); ++g)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc3[g][j] = 0.f;
  auto tile = [&](int w0) {
    const int wn = min(WT, win_len - w0);
    __syncthreads();  // queries staged / the previous tile's probabilities consumed
    // (1) scores: thread per window row, all G heads
    for (int rr = tid; rr < wn; rr += NTH) {
      const int slot = win_slot0 + w0 + rr;  // ring slot: win_slot0 < Wcap and w0 + rr < Wcap
      const T* kr = wk + (int64_t)(slot >= Wcap ? slot - Wcap : slot) * D;
      float acc[GM];
#pragma unroll
      for (int g = 0; g < GM; ++g) acc[g] = 0.f;
      if constexpr (VEC) {
        constexpr int NB = sizeof(T) == 8 ? 4 : 16;  // 4-element vectors in flight per batch
        for (int d0 = 0; d0 < D; d0 += 4 * NB) {
          typename Vec4<T>::raw kv[NB];
#pragma unroll
          for (int j = 0; j < NB; ++j)
            if (d0 + 4 * j < D) kv[j] = ld4(kr + d0 + 4 * j);
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            if (d0 + 4 * j >= D) break;
            const float4 k4 = cvt4(kv[j], (const T*)nullptr);
#pragma unroll
            for (int g = 0; g < GM; ++g) {
              if (g >= G) break;
              const float4 q4 = *reinterpret_cast<const float4*>(qs + g * D + d0 + 4 * j);
              acc[g] = fmaf(q4.x, k4.x, fmaf(q4.y, k4.y, fmaf(q4.z, k4.z, fmaf(q4.w, k4.w, acc[g]))));
            }
          }
        }
      } else {
#pragma unroll 4
        for (int d = 0; d < D; ++d) {
          const float kv = to_f32(kr[d]);
#pragma unroll
          for (int g = 0; g < GM; ++g)
            if (g < G) acc[g] = fmaf(qs[g * D + d], kv, acc[g]);
        }
      }
#pragma unroll
      for (int g = 0; g < GM; ++g)
        if (g < G) sc[g * WT + rr] = acc[g] * a.scale_log2;
    }
    __syncthreads();
    // (2) warp h: tile max, running max, probabilities, running sum (log2 units)
    {
      float* sh = sc + h * WT;
      float mt = -INFINITY;
      for (int rr = lane; rr < wn; rr += 32) mt = fmaxf(mt, sh[rr]);
#pragma unroll
      for (int off = 16; off; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
      const float mn = fmaxf(m, mt);
      const float al = m == -INFINITY ? 0.f : exp2f(m - mn);
      float lt = 0.f;
      for (int rr = lane; rr < wn; rr += 32) {
        const float p = exp2f(sh[rr] - mn);
        sh[rr] = p;
        lt += p;
      }
      l = l * al + warp_sum_f(lt);
      m = mn;
      if (!TILED) {
      } else if (VEC) {
        if (lane == 0) rs[h] = al;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] *= al;
      }
    }
    if constexpr (VEC) {
      __syncthreads();
      // (3) warp w: rows r = w (mod G) of the tile, all heads, lane = channels 4*lane .. 4*lane+3
#pragma unroll
      for (int g = 0; g < GM; ++g) {
        if (g >= G || !TILED) break;
        const float al = rs[g];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc3[g][j] *= al;
      }
      const bool on = 4 * lane < D;
      constexpr int RB = 8;
      for (int r0 = w; r0 < wn; r0 += RB * G) {
        typename Vec4<T>::raw vv[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          const int rr = r0 + i * G;
          const int slot = win_slot0 + w0 + rr;
          if (on && rr < wn) vv[i] = ld4(wv + (int64_t)(slot >= Wcap ? slot - Wcap : slot) * D + 4 * lane);
        }
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          const int rr = r0 + i * G;
          if (rr >= wn) break;
          const float4 v4 = on ? cvt4(vv[i], (const T*)nullptr) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int g = 0; g < GM; ++g) {
            if (g >= G) break;
            const float p = sc[g * WT + rr];
            acc3[g][0] = fmaf(p, v4.x, acc3[g][0]);
            acc3[g][1] = fmaf(p, v4.y, acc3[g][1]);
            acc3[g][2] = fmaf(p, v4.z, acc3[g][2]);
            acc3[g][3] = fmaf(p, v4.w, acc3[g][3]);
          }
        }
      }
    } else {
      __syncwarp();
      // (3) o = sum_r p_r v_r for head h, lanes over channels
      const float* sh = sc + h * WT;
#pragma unroll 2
      for (int rr = 0; rr < wn; ++rr) {
        const int slot = win_slot0 + w0 + rr;
        const T* vr = wv + (int64_t)(slot >= Wcap ? slot - Wcap : slot) * D;
        const float p = sh[rr];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (lane + 32 * j < D) o[j] = fmaf(p, to_f32(vr[lane + 32 * j]), o[j]);
      }
    }
  };
  if constexpr (TILED) {
    for (int w0 = 0; w0 < win_len; w0 += WT) tile(w0);
  } else {  // one tile: the running sums are born in phase (3), not carried across a loop
    tile(0);
  }
  if constexpr (VEC) {
    const bool on = 4 * lane < D;
    if (on) {
#pragma unroll
      for (int g = 0; g < GM; ++g)
        if (g < G)
          *reinterpret_cast<float4*>(red + ((int64_t)w * G + g) * D + 4 * lane) =
              make_float4(acc3[g][0], acc3[g][1], acc3[g][2], acc3[g][3]);
    }
    __syncthreads();
    if (on)
      for (int ww = 0; ww < G; ++ww) {
        const float4 x = *reinterpret_cast<const float4*>(red + ((int64_t)ww * G + h) * D + 4 * lane);
        o[0] += x.x; o[1] += x.y; o[2] += x.z; o[3] += x.w;
      }
  }
  // channel of o[j]: VEC 4*lane + j, else lane + 32*j
  auto chan = [&](int j) { return VEC ? 4 * lane + j : lane + 32 * j; };
  // (4) combine with chunk partials (written by the chunk grid this launch depends on)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int ch = 0; ch < a.nchunk; ++ch) {
    const float* pp = a.part + (((int64_t)u * a.nchunk + ch) * G + h) * (Dp + 2);
    const float pm = pp[Dp], pl = pp[Dp + 1];
    if (pm == -INFINITY) continue;
    const float mn = fmaxf(m, pm);
    const float al = m == -INFINITY ? 0.f : exp2f(m - mn), be = exp2f(pm - mn);
    l = l * al + pl * be;
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = o[j] * al + (chan(j) < Dp ? pp[chan(j)] * be : 0.f);
    m = mn;
  }
  float* dst = out + ((int64_t)u * G + h) * D;
  if (a.ml) {  // partial (o, m, l) for a cross-rank LSE merge: m in natural-log units
#pragma unroll
    for (int j = 0; j < 4; ++j) if (chan(j) < D) dst[chan(j)] = o[j];
    if (lane == 0) {
      a.ml[((int64_t)u * G + h) * 2] = m * 0.6931471805599453f;
      a.ml[((int64_t)u * G + h) * 2 + 1] = l;
    }
    return;
  }
  const float inv = 1.f / l;
#pragma unroll
  for (int j = 0; j < 4; ++j) if (chan(j) < D) dst[chan(j)] = o[j] * inv;
}

template <typename T, bool VEC, int GC, bool TILED>
static cudaError_t launch_merge(const DevCache& c, const AttnArgs& a, int win_len, int win_slot0, float* out,
                                cudaStream_t st) {
  const size_t msmem =
      ((((size_t)a.G * c.D + (size_t)a.G * (TILED ? MERGE_WT : c.Wcap) + a.G + 3) & ~(size_t)3) +
       (VEC ? (size_t)a.G * a.G * c.D : 0)) * 4;
  if (msmem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(attn_merge_kernel<T, VEC, GC, TILED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)msmem);
    if (e != cudaSuccess) return e;
  }
  // programmatic dependent launch after a chunk grid: phases (1)-(3) read only the window and
  // the queries (written before the chunk grid started) and overlap the chunk grid's tail;
  // griddepcontrol.wait precedes the partials
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c.U);
  cfg.blockDim = dim3(32 * a.G);
  cfg.dynamicSmemBytes = msmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.nchunk > 0 ? 1 : 0;  // no chunk grid: the predecessor may be the window writer
  return cudaLaunchKernelEx(&cfg, attn_merge_kernel<T, VEC, GC, TILED>, c, a, win_len, win_slot0, out);
}

template <typename T, bool VEC>
static cudaError_t launch_merge_g(const DevCache& c, const AttnArgs& a, int win_len, int win_slot0, float* out,
                                  cudaStream_t st) {
  const bool tiled = c.Wcap > MERGE_WT;  // score tile of every window row fits smem otherwise
  switch (a.G) {
    case 4: return tiled ? launch_merge<T, VEC, 4, true>(c, a, win_len, win_slot0, out, st)
                         : launch_merge<T, VEC, 4, false>(c, a, win_len, win_slot0, out, st);
    case 8: return tiled ? launch_merge<T, VEC, 8, true>(c, a, win_len, win_slot0, out, st)
                         : launch_merge<T, VEC, 8, false>(c, a, win_len, win_slot0, out, st);
    default: return tiled ? launch_merge<T, VEC, 0, true>(c, a, win_len, win_slot0, out, st)
                          : launch_merge<T, VEC, 0, false>(c, a, win_len, win_slot0, out, st);
  }
}

size_t attn_smem_bytes(int Dp, int Pk, int Pv, int bits, int NT) {
  const size_t wfl = attn_w_private(Pv, NT) ? (size_t)ATT_WARPS * 8 * max(Pv, 1) * 4 * NT
                                             : (size_t)ATT_WARPS * max(Pv, 1) * MAXG;
  return (size_t)MAXG * Dp * 4 + (size_t)max(Pk, 1) * MAXG * 4 + wfl * 4 + (size_t)max(Pv, 1) * MAXG * 4 +
         ATT_WARPS * 256 * 2 + ATT_WARPS * MAXG * 4 * 4 + 16;
}

template <int BITS, int NT, int KT>
static cudaError_t launch_chunks_kt(const DevCache& c, const AttnArgs& a, size_t smem, cudaStream_t st) {
  const cudaError_t e = cudaFuncSetAttribute(attn_chunk_kernel<BITS, NT, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
  if (e != cudaSuccess) return e;
  attn_chunk_kernel<BITS, NT, KT><<<dim3(a.nchunk, c.U), ATT_THREADS, smem, st>>>(c, a);
  return cudaGetLastError();
}
template <int BITS, int NT>
static cudaError_t launch_chunks(const DevCache& c, const AttnArgs& a, size_t smem, cudaStream_t st) {
  switch (c.Dp / 16) {
    case 4: return launch_chunks_kt<BITS, NT, 4>(c, a, smem, st);
    default: return launch_chunks_kt<BITS, NT, 8>(c, a, smem, st);
  }
}

template <typename T>
cudaError_t launch_attn(const DevCache& c, const AttnArgs& a, int Pk_max, int Pv_max, int win_len, int win_slot0,
                        float* out, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  if (a.nb > 0) e = launch_attn_tc(c, a, Pk_max, Pv_max, st);  // K3-TC (pkv_attn_tc.cu)
  if (a.nb > 0 && e == cudaErrorNotSupported) {
    e = cudaSuccess;
    const int nt = a.G <= 4 ? 1 : 2;
    size_t smem = attn_smem_bytes(c.Dp, Pk_max, Pv_max, c.bits, nt);
    if (smem > 227 * 1024) return cudaErrorNotSupported;  // pkv_decode_attn reports the pattern-count limit
    if (c.bits == 2) e = nt == 1 ? launch_chunks<2, 1>(c, a, smem, st) : launch_chunks<2, 2>(c, a, smem, st);
    else if (c.bits == 4) e = nt == 1 ? launch_chunks<4, 1>(c, a, smem, st) : launch_chunks<4, 2>(c, a, smem, st);
    else e = nt == 1 ? launch_chunks<8, 1>(c, a, smem, st) : launch_chunks<8, 2>(c, a, smem, st);
    if (e != cudaSuccess) return e;
  }
  AttnArgs a2 = a;
  if (a.nb == 0) a2.nchunk = 0;
  return c.D % 4 == 0 ? launch_merge_g<T, true>(c, a2, win_len, win_slot0, out, st)
                      : launch_merge_g<T, false>(c, a2, win_len, win_slot0, out, st);
}
template cudaError_t launch_attn<__half>(const DevCache&, const AttnArgs&, int, int, int, int, float*, cudaStream_t);
template cudaError_t launch_attn<__nv_bfloat16>(const DevCache&, const AttnArgs&, int, int, int, int, float*, cudaStream_t);
template cudaError_t launch_attn<float>(const DevCache&, const AttnArgs&, int, int, int, int, float*, cudaStream_t);
template cudaError_t launch_attn<double>(const DevCache&, const AttnArgs&, int, int, int, int, float*, cudaStream_t);

}  // namespace pkv
