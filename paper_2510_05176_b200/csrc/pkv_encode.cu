// K1 encode_span: fused match -> gate -> residual -> quantize -> pack.
//
// One CTA per (span, unit).  Replaces, for one committed span of <= G tokens,
// the reference's _commit_span (engine.py:201-252): match_many
// (patterns.py:206-221), decide (gate.py:174-188), quantize_group and
// pack_codes (quant.py:70-146).  K groups run per channel over the span's
// tokens (engine.py:222); V groups per token over channels (engine.py:243).
//
// Exactness: the d_mm argmin is computed in fp32 (FADD + FMNMX3) with a
// rigorous error bound; a token whose best two fp32 distances are within the
// bound is re-matched over the whole table in IEEE fp64 (the reference's own
// arithmetic), so indices are bit-identical, ties to the lowest index.  Group
// extrema, scales and the gate ratio are fp64; codes use a guarded fp32
// quotient with an exact fp64 fallback.
#include "pkv_common.cuh"

namespace pkv {

constexpr int ENC_THREADS = 256;
#define INF32 __int_as_float(0x7f800000)
constexpr int NPROBE = 16;      // channels of the d_mm lower bound
constexpr int PRUNE_PMAX = 64;  // pruned matcher serves tables of <= 64 patterns
constexpr int PRUNE_MAXCAND = 6;
constexpr int PRUNE_WIDE_PMAX = 256;  // match_pruned_wide: probe table in the pattern staging rows
constexpr int MS_ROWS = 33;     // 32 staged patterns + one zero row (RAW payload)
constexpr float TWO_M22 = 2.384185791015625e-07f;  // 2^-22
constexpr float TWO_M21 = 4.76837158203125e-07f;   // 2^-21
constexpr float TWO_M20 = 9.5367431640625e-07f;    // 2^-20

struct EncSmem {
  int DS, Dm;
  float* xs;      // [GMAX][DS] span rows (fp32; exact for 16/32-bit inputs); codes overwrite
                  // byte 0 of each element slot after its last use (cslot)
  float* ms;      // [MS_ROWS][DS] pattern chunk + zero row
  float* xp;      // [GMAX][NPROBE] x at the probe channels
  float* xabs;    // [GMAX] max |x| per token
  float* best1; float* best2; int* bidx; int* fidx;  // [GMAX]
  double* qlo; double* qhi;  // [2][DMAX] (also exchange scratch)
  int* probe;     // [NPROBE]
  float* mpk;     // [NPROBE][PRUNE_PMAX] pattern values at the probe channels
};

__host__ __device__ inline size_t enc_smem_bytes(int D) {
  const int Dm = round_up(D, 4), DS = Dm + 4;
  size_t b = (size_t)(GMAX + MS_ROWS) * DS * 4 + (size_t)GMAX * NPROBE * 4 + 5 * GMAX * 4;
  b = (b + 15) / 16 * 16;
  b += 4 * DMAX * 8 + NPROBE * 4 + NPROBE * PRUNE_PMAX * 4;
  return b;
}

__device__ __forceinline__ uint8_t* cslot(const EncSmem& sm, int t, int c) {
  return reinterpret_cast<uint8_t*>(sm.xs + t * sm.DS + c);
}

// top-2 (value, lowest index) merge used by the warp reduction
__device__ __forceinline__ void top2_merge(float& a1, int& ai, float& a2, float b1, int bi, float b2) {
  if (b1 < a1 || (b1 == a1 && bi < ai)) {
    a2 = fminf(a1, b2);
    a1 = b1; ai = bi;
  } else {
    a2 = fminf(a2, b1);
  }
}

template <typename T>
__device__ __forceinline__ const T* span_row(const SpanSrc<T>& s, int u, int64_t off, int r, int D) {
  int64_t rr = s.row0 + off + r;
  if (rr >= s.ring) rr = rr < 2 * s.ring ? rr - s.ring : rr % s.ring;  // window ring wrap (rare, small)
  return s.base + (int64_t)u * s.unit_stride + rr * (int64_t)D;
}

template <typename T>
__device__ __forceinline__ double xval(const EncSmem& sm, const T* row, int r, int c) {
  if constexpr (exact_in_f32<T>::value) return (double)sm.xs[r * sm.DS + c];
  else return to_f64(row[c]);
}

// fp64 re-match of one vector over the whole table (patterns.py:217-221 exactly).
template <typename T>
__device__ int refine_match64(const EncSmem& sm, const T* row, int r, const double* p64, int P, int D, int lane) {
  double bestv = __longlong_as_double(0x7ff0000000000000LL);
  int besti = 0;
  for (int pb = 0; pb < P; pb += 32) {
    int p = pb + lane;
    double v = __longlong_as_double(0x7ff0000000000000LL);
    if (p < P) {
      double mx = -v, mn = v;
      const double* m = p64 + (int64_t)p * D;
      for (int c = 0; c < D; ++c) {
        double d = __dsub_rn(xval<T>(sm, row, r, c), m[c]);
        mx = fmax(mx, d);
        mn = fmin(mn, d);
      }
      v = __dsub_rn(mx, mn);
    }
    int pi = p;
    warp_argmin_d(v, pi);
    if (v < bestv) { bestv = v; besti = pi; }
  }
  return besti;
}

// ---- guarded fp32 quantizer (inputs exact in fp32) ------------------------------------
// t = (v32 - lo32)/scale + 1/2 with a per-group guard covering |v32 - v64| <= 2^-23 S
// (S bounds |x| + |m|) and the fp32 rounding of the quotient; a code whose fraction
// lands inside the guard is recomputed from the exact payload in IEEE fp64.
struct FastQ {
  QuantParamsDev qp;
  float lo32, guard;
};
__device__ __forceinline__ FastQ make_fastq(double lo, double hi, int qmax, float S) {
  FastQ f;
  f.qp = make_qparams(lo, hi, qmax);
  f.lo32 = (float)lo;
  if (f.qp.scale == 0.0) { f.guard = 0.f; return f; }
  const float span = (float)(hi - lo);
  const float g = TWO_M21 * (S + fabsf(f.lo32) + span) * f.qp.inv32 + TWO_M20 * (float)(qmax + 1);
  f.guard = fminf(g, 0.5f);
  return f;
}
// branch-free fast code; *bad set when the exact fp64 path must decide
__device__ __forceinline__ int code_fast(float v32, const FastQ& f, bool& bad) {
  const float t = __fmaf_rn(v32 - f.lo32, f.qp.inv32, 0.5f);
  const float fl = floorf(t);
  const float fr = t - fl;
  bad |= (fr <= f.guard) | (fr >= 1.f - f.guard);
  const int cde = (int)fl;
  return cde < 0 ? 0 : (cde > f.qp.qmax ? f.qp.qmax : cde);
}
__device__ __forceinline__ bool code_needs_exact(float v32, const FastQ& f) {
  const float t = __fmaf_rn(v32 - f.lo32, f.qp.inv32, 0.5f);
  const float fr = t - floorf(t);
  return (fr <= f.guard) | (fr >= 1.f - f.guard);
}
__device__ __forceinline__ int code_exact(double v64, const FastQ& f) {
  const double q = __dadd_rn(__ddiv_rn(__dsub_rn(v64, f.qp.lo), f.qp.scale), 0.5);
  const int cde = (int)floor(q);
  return cde < 0 ? 0 : (cde > f.qp.qmax ? f.qp.qmax : cde);
}

// pattern row of index idx for the fp32 residual (RAW -> the zero row)
struct PatRows {
  const float* ms;   // staged table (P <= 32) incl. zero row 32
  const float* p32;  // global table
  int DS, Dp, P;
  __device__ __forceinline__ const float* row(int idx) const {
    if (P <= 32) return ms + (idx >= 0 ? idx : 32) * DS;
    return idx >= 0 ? p32 + (int64_t)idx * Dp : ms + 32 * DS;
  }
};

// Stages C (per-token stats / gate / V quantization) and D (K per-channel
// quantization) for inputs exact in fp32 (fp16, bf16, fp32).  Group extrema are
// formed in fp64 only from the fp32 candidates within the error bound, so scale,
// zero, gate and codes equal the reference's fp64 arithmetic bit for bit.
template <typename T>
__device__ void encode_sides_fast(const DevCache& c, const EncSmem& sm, const SpanSrc<T>& src, int side, int u,
                                  int b, int64_t start, int64_t off, int L, int P, const float* p32,
                                  const double* p64, float pmax) {
  const int tid = threadIdx.x;
  const int D = c.D, Dp = c.Dp;
  unsigned* nex = c.stats ? &c.stats[1] : nullptr;
  const float INF = INF32;
  const double DINF = __longlong_as_double(0x7ff0000000000000LL);
  const PatRows pr{sm.ms, p32, sm.DS, Dp, P};

  // ---- C. per-token stats (V always, K when the K gate is on) ----
  // thread = (token t, channel half h), partner in tid ^ 128
  const bool per_token = (side == 1) || (c.use_kgate && P > 0);
  if (per_token) {
    const bool gate_on = side == 1 ? c.use_vgate : true;
    double* diag = side == 1 ? c.vdiag : c.kdiag;
    const int t = tid & (GMAX - 1), h = tid >> 7;
    const int HC = (D + 1) / 2;
    const int c0 = h ? HC : 0, c1 = h ? D : HC;
    float* xch = reinterpret_cast<float*>(sm.qlo);   // [2][GMAX][4] exchange
    double* dch = sm.qlo;                            // [2][GMAX][2]
    const bool act = t < L;
    const int idx = act ? sm.fidx[t] : RAW;
    const float* xr = sm.xs + t * sm.DS;
    const float* mr = pr.row(idx);
    float xmx = -INF, xmn = INF, rmx = -INF, rmn = INF;
    if (act) {
      for (int cc = c0; cc < c1; ++cc) {
        const float x = xr[cc];
        const float r = x - mr[cc];
        xmx = fmaxf(xmx, x); xmn = fminf(xmn, x);
        rmx = fmaxf(rmx, r); rmn = fminf(rmn, r);
      }
    }
    __syncthreads();
    xch[(h * GMAX + t) * 4 + 0] = xmx; xch[(h * GMAX + t) * 4 + 1] = xmn;
    xch[(h * GMAX + t) * 4 + 2] = rmx; xch[(h * GMAX + t) * 4 + 3] = rmn;
    __syncthreads();
    {
      const float* o = xch + ((h ^ 1) * GMAX + t) * 4;
      xmx = fmaxf(xmx, o[0]); xmn = fminf(xmn, o[1]); rmx = fmaxf(rmx, o[2]); rmn = fminf(rmn, o[3]);
    }
    const float S = act ? sm.xabs[t] + pmax : 0.f;
    const float tol2 = 2.f * TWO_M22 * S;
    const double* m = idx >= 0 ? p64 + (int64_t)idx * D : p64;
    double clo = DINF, chi = -DINF;
    if (act && idx >= 0) {
      const float lob = rmn + tol2, hib = rmx - tol2;
      for (int cc = c0; cc < c1; ++cc) {
        const float x = xr[cc];
        const float r = x - mr[cc];
        if (r <= lob || r >= hib) {
          const double r64 = __dsub_rn((double)x, m[cc]);
          if (r <= lob) clo = fmin(clo, r64);
          if (r >= hib) chi = fmax(chi, r64);
        }
      }
    }
    __syncthreads();
    dch[(h * GMAX + t) * 2 + 0] = clo;
    dch[(h * GMAX + t) * 2 + 1] = chi;
    __syncthreads();
    clo = fmin(clo, dch[((h ^ 1) * GMAX + t) * 2 + 0]);
    chi = fmax(chi, dch[((h ^ 1) * GMAX + t) * 2 + 1]);
    if (act) {
      bool flatten = false;
      if (idx >= 0) {
        const double raw = __dsub_rn((double)xmx, (double)xmn), flat = __dsub_rn(chi, clo);
        if (gate_on) flatten = raw > 0.0 && __ddiv_rn(flat, raw) <= c.thr;
        else flatten = true;
        if (h == 0 && c.keep_diag && diag) {
          const int64_t o = ((int64_t)u * c.Tcap + start + t) * 2;
          diag[o] = raw; diag[o + 1] = flat;
        }
      }
      const int fidx = flatten ? idx : RAW;
      if (side == 1) {
        const double lo = flatten ? clo : (double)xmn, hi = flatten ? chi : (double)xmx;
        const FastQ fq = make_fastq(lo, hi, c.qmax, flatten ? S : sm.xabs[t]);
        const float* mq = flatten ? mr : sm.ms + 32 * sm.DS;   // zero row for the raw payload
        if (fq.qp.scale == 0.0) {
          for (int cc = c0; cc < c1; ++cc) *cslot(sm, t, cc) = 0;
        } else {
          uint32_t bad0 = 0, bad1 = 0;  // guard-band hits, bit per channel of this half
          for (int cc = c0; cc < c1; ++cc) {
            bool bad = false;
            const int cd = code_fast(xr[cc] - mq[cc], fq, bad);
            if (cc - c0 < 32) bad0 |= (uint32_t)bad << (cc - c0); else bad1 |= (uint32_t)bad << (cc - c0 - 32);
            *cslot(sm, t, cc) = (uint8_t)cd;
          }
          if (bad0 | bad1) {  // rare: exact fp64 codes for fractions inside the guard band
            const T* row = span_row(src, u, off, t, D);
            while (bad0 | bad1) {
              int i;
              if (bad0) { i = __ffs(bad0) - 1; bad0 &= bad0 - 1; }
              else { i = 32 + __ffs(bad1) - 1; bad1 &= bad1 - 1; }
              const int cc = c0 + i;
              const float x = (float)to_f64(row[cc]);
              const double v64 = flatten ? __dsub_rn((double)x, m[cc]) : (double)x;
              *cslot(sm, t, cc) = (uint8_t)code_exact(v64, fq);
              if (nex) atomicAdd(nex, 1u);
            }
          }
        }
        if (h == 0) {
          const int64_t tok = (int64_t)u * c.Tcap + start + t;
          const int64_t slot = ((int64_t)u * c.NBcap + b) * c.GP + t;
          c.vparam64[2 * tok] = fq.qp.scale;
          c.vparam64[2 * tok + 1] = fq.qp.lo;
          c.vparam32[2 * slot] = (float)fq.qp.scale;
          c.vparam32[2 * slot + 1] = (float)fq.qp.lo;
          c.vidx[slot] = (int16_t)fidx;
        }
      }
      if (side == 0 && h == 0) sm.fidx[t] = fidx;  // K gate choice (read by stage D after its barrier)
    }
  }

  // ---- D. K: per-channel groups over the span's tokens; thread = (channel, token half) ----
  if (side == 0) {
    __syncthreads();
    // per-token pattern row: ms row (P <= 32, RAW -> zero row 32) or global row
    int* rowoff = sm.bidx;  // [GMAX], free after matching
    for (int t = tid; t < L; t += ENC_THREADS) {
      const int idx = sm.fidx[t];
      rowoff[t] = P <= 32 ? (idx >= 0 ? idx : 32) * sm.DS : idx;
    }
    __syncthreads();
    const int ch = tid & (DMAX - 1), half = tid >> 7;
    const int tb = half ? L / 2 : 0, te = half ? L : L / 2;
    float* f32buf = reinterpret_cast<float*>(sm.qlo);  // [3][2][DMAX] floats
    const bool small = P <= 32;
    auto mval = [&](int t) -> float {
      if (small) return sm.ms[rowoff[t] + ch];
      const int idx = rowoff[t];
      return idx >= 0 ? p32[(int64_t)idx * Dp + ch] : 0.f;
    };
    float mn = INF, mx = -INF, xab = 0.f;
    bool anyp = false;
    if (ch < D) {
      for (int t = tb; t < te; ++t) {
        const float x = sm.xs[t * sm.DS + ch];
        const float r = x - mval(t);
        mn = fminf(mn, r); mx = fmaxf(mx, r); xab = fmaxf(xab, fabsf(x));
        anyp |= sm.fidx[t] >= 0;
      }
    }
    f32buf[(0 * 2 + half) * DMAX + ch] = mn;
    f32buf[(1 * 2 + half) * DMAX + ch] = mx;
    f32buf[(2 * 2 + half) * DMAX + ch] = anyp ? xab + pmax : xab;
    __syncthreads();
    mn = fminf(f32buf[ch], f32buf[DMAX + ch]);
    mx = fmaxf(f32buf[2 * DMAX + ch], f32buf[3 * DMAX + ch]);
    const float S = fmaxf(f32buf[4 * DMAX + ch], f32buf[5 * DMAX + ch]);
    __syncthreads();
    const float tol2 = 2.f * TWO_M22 * S;
    double clo = DINF, chi = -DINF;
    if (ch < D) {
      const float lob = mn + tol2, hib = mx - tol2;
      for (int t = tb; t < te; ++t) {
        const float x = sm.xs[t * sm.DS + ch];
        const float r = x - mval(t);
        if (r <= lob || r >= hib) {
          const int idx = sm.fidx[t];
          const double r64 = idx >= 0 ? __dsub_rn((double)x, p64[(int64_t)idx * D + ch]) : (double)x;
          if (r <= lob) clo = fmin(clo, r64);
          if (r >= hib) chi = fmax(chi, r64);
        }
      }
    }
    sm.qlo[half * DMAX + ch] = clo;
    sm.qhi[half * DMAX + ch] = chi;
    __syncthreads();
    const double lo = fmin(sm.qlo[ch], sm.qlo[DMAX + ch]);
    const double hi = fmax(sm.qhi[ch], sm.qhi[DMAX + ch]);
    if (ch < D) {
      const FastQ fq = make_fastq(lo, hi, c.qmax, S);
      if (fq.qp.scale == 0.0) {
        for (int t = tb; t < te; ++t) *cslot(sm, t, ch) = 0;
      } else {
        uint32_t bad0 = 0, bad1 = 0;  // guard-band hits, bit per token of this half
        for (int t = tb; t < te; ++t) {
          const float x = sm.xs[t * sm.DS + ch];
          const float r = x - mval(t);
          bool bad = false;
          const int cd = code_fast(r, fq, bad);
          if (t - tb < 32) bad0 |= (uint32_t)bad << (t - tb); else bad1 |= (uint32_t)bad << (t - tb - 32);
          *cslot(sm, t, ch) = (uint8_t)cd;
        }
        while (bad0 | bad1) {  // rare: exact fp64 codes for fractions inside the guard band
          int i;
          if (bad0) { i = __ffs(bad0) - 1; bad0 &= bad0 - 1; }
          else { i = 32 + __ffs(bad1) - 1; bad1 &= bad1 - 1; }
          const int t = tb + i;
          const int idx = sm.fidx[t];
          const float x = (float)to_f64(span_row(src, u, off, t, D)[ch]);
          const double v64 = idx >= 0 ? __dsub_rn((double)x, p64[(int64_t)idx * D + ch]) : (double)x;
          *cslot(sm, t, ch) = (uint8_t)code_exact(v64, fq);
          if (nex) atomicAdd(nex, 1u);
        }
      }
      if (half == 0) {
        const int64_t o64 = ((int64_t)u * c.NBcap + b) * 2 * D;
        c.kparam64[o64 + ch] = fq.qp.scale;
        c.kparam64[o64 + D + ch] = fq.qp.lo;
      }
    }
    if (half == 0) {
      const int64_t o32 = ((int64_t)u * c.NBcap + b) * 2 * Dp;
      for (int cc = ch; cc < Dp; cc += DMAX) {
        float sc = 0.f, z = 0.f;
        if (cc < D) { sc = (float)__ddiv_rn(__dsub_rn(hi, lo), (double)c.qmax); z = (float)lo; }
        c.kparam32[o32 + cc] = sc;
        c.kparam32[o32 + Dp + cc] = z;
      }
    }
    for (int t = tid; t < L; t += ENC_THREADS) c.kidx[((int64_t)u * c.NBcap + b) * c.GP + t] = (int16_t)sm.fidx[t];
  }
}

// Full fp32 d_mm of token t against pattern p, warp-cooperative (lane = 4 channels).
__device__ __forceinline__ float coop_dmm(const EncSmem& sm, int t, int p, const float* p32, int Dp) {
  const int lane = threadIdx.x & 31;
  const int cc = 4 * lane;
  float mx = -INF32, mn = INF32;
  if (cc < sm.Dm) {
    const float4 x4 = *reinterpret_cast<const float4*>(sm.xs + t * sm.DS + cc);
    const float4 m4 = p < 32 ? *reinterpret_cast<const float4*>(sm.ms + p * sm.DS + cc)
                             : __ldg(reinterpret_cast<const float4*>(p32 + (int64_t)p * Dp + cc));
    const float r0 = x4.x - m4.x, r1 = x4.y - m4.y, r2 = x4.z - m4.z, r3 = x4.w - m4.w;
    mx = fmax3(fmaxf(r0, r1), r2, r3);
    mn = fmin3(fminf(r0, r1), r2, r3);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  return mx - mn;
}

// Exact nearest-pattern search with lower-bound pruning (P <= 64, inputs exact in
// fp32).  LB_p = range over NPROBE channels of (x - m_p) <= d32(x, m_p) exactly
// (the same fp32 residuals over a subset of channels), so a pattern with
// LB_p > d32(guess) + 2 tol is farther than the winner by more than the fp32
// error window and needs no full distance.  Survivors are evaluated in full; the
// top-2 ambiguity test and the fp64 re-match are those of the brute-force path.
template <typename T, bool TWO>
__device__ void match_pruned(const DevCache& c, const EncSmem& sm, const SpanSrc<T>& src, int u, int64_t off, int L,
                             int P, const float* p32, const double* p64, float pmax) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = c.D, Dp = c.Dp;
  for (int i = tid; i < NPROBE * PRUNE_PMAX; i += ENC_THREADS) {
    const int k = i / PRUNE_PMAX, p = i - k * PRUNE_PMAX;
    sm.mpk[i] = p < P ? p32[(int64_t)p * Dp + sm.probe[k]] : 0.f;
  }
  __syncthreads();
  float m0[NPROBE], m1[TWO ? NPROBE : 1];
#pragma unroll
  for (int k = 0; k < NPROBE; ++k) {
    m0[k] = sm.mpk[k * PRUNE_PMAX + lane];
    if constexpr (TWO) m1[k] = sm.mpk[k * PRUNE_PMAX + 32 + lane];
  }
  const bool v0 = lane < P, v1 = lane + 32 < P;
  for (int t0 = 16 * warp; t0 < 16 * warp + 16 && t0 < L; t0 += 4) {
    float a0[4], b0[4], a1[4], b1[4];  // max / min of the probe residuals
#pragma unroll
    for (int j = 0; j < 4; ++j) { a0[j] = -INF32; b0[j] = INF32; a1[j] = -INF32; b1[j] = INF32; }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4* xq = reinterpret_cast<const float4*>(sm.xp + (t0 + j) * NPROBE);
#pragma unroll
      for (int k4 = 0; k4 < NPROBE / 4; ++k4) {
        const float4 x4 = xq[k4];
        const float r0 = x4.x - m0[4 * k4], r1 = x4.y - m0[4 * k4 + 1];
        const float r2 = x4.z - m0[4 * k4 + 2], r3 = x4.w - m0[4 * k4 + 3];
        a0[j] = fmax3(a0[j], r0, r1); a0[j] = fmax3(a0[j], r2, r3);
        b0[j] = fmin3(b0[j], r0, r1); b0[j] = fmin3(b0[j], r2, r3);
        if constexpr (TWO) {
          const float s0 = x4.x - m1[4 * k4], s1 = x4.y - m1[4 * k4 + 1];
          const float s2 = x4.z - m1[4 * k4 + 2], s3 = x4.w - m1[4 * k4 + 3];
          a1[j] = fmax3(a1[j], s0, s1); a1[j] = fmax3(a1[j], s2, s3);
          b1[j] = fmin3(b1[j], s0, s1); b1[j] = fmin3(b1[j], s2, s3);
        }
      }
    }
#pragma unroll 1
    for (int j = 0; j < 4; ++j) {
      const int t = t0 + j;
      if (t >= L) break;
      const float lb0 = v0 ? a0[j] - b0[j] : INF32;
      const float lb1 = v1 ? a1[j] - b1[j] : INF32;
      // guess = lowest LB, lowest pattern index on ties
      float gv = fminf(lb0, lb1);
#pragma unroll
      for (int o = 16; o; o >>= 1) gv = fminf(gv, __shfl_xor_sync(0xffffffffu, gv, o));
      const unsigned e0 = __ballot_sync(0xffffffffu, lb0 == gv);
      const int gi = e0 ? __ffs(e0) - 1 : 32 + __ffs(__ballot_sync(0xffffffffu, lb1 == gv)) - 1;
      const float tol2 = 2.f * TWO_M20 * (sm.xabs[t] + pmax);
      float best = coop_dmm(sm, t, gi, p32, Dp);
      int bi = gi;
      float second = INF32;
      const float bound = best + tol2;
      unsigned c0 = __ballot_sync(0xffffffffu, lb0 <= bound);
      unsigned c1 = __ballot_sync(0xffffffffu, lb1 <= bound);
      if (gi < 32) c0 &= ~(1u << gi); else c1 &= ~(1u << (gi - 32));
      if (__popc(c0) + __popc(c1) > PRUNE_MAXCAND) {
        // poorly separated token: exhaustive search over the table (lane = pattern)
        float mx0 = -INF32, mn0 = INF32, mx1 = -INF32, mn1 = INF32;
        const float* xr = sm.xs + t * sm.DS;
        for (int cc = 0; cc < sm.Dm; cc += 4) {
          const float4 x4 = *reinterpret_cast<const float4*>(xr + cc);
          const float4 q0 = *reinterpret_cast<const float4*>(sm.ms + lane * sm.DS + cc);
          const float r0 = x4.x - q0.x, r1 = x4.y - q0.y, r2 = x4.z - q0.z, r3 = x4.w - q0.w;
          mx0 = fmax3(mx0, r0, r1); mx0 = fmax3(mx0, r2, r3);
          mn0 = fmin3(mn0, r0, r1); mn0 = fmin3(mn0, r2, r3);
          if (TWO && v1) {
            const float4 q1 = __ldg(reinterpret_cast<const float4*>(p32 + (int64_t)(lane + 32) * Dp + cc));
            const float s0 = x4.x - q1.x, s1 = x4.y - q1.y, s2 = x4.z - q1.z, s3 = x4.w - q1.w;
            mx1 = fmax3(mx1, s0, s1); mx1 = fmax3(mx1, s2, s3);
            mn1 = fmin3(mn1, s0, s1); mn1 = fmin3(mn1, s2, s3);
          }
        }
        const float va = v0 ? mx0 - mn0 : INF32, vb = v1 ? mx1 - mn1 : INF32;
        float w1 = va <= vb ? va : vb, w2 = va <= vb ? vb : va;
        int wi = va <= vb ? lane : lane + 32;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const float ob1 = __shfl_xor_sync(0xffffffffu, w1, o);
          const int obi = __shfl_xor_sync(0xffffffffu, wi, o);
          const float ob2 = __shfl_xor_sync(0xffffffffu, w2, o);
          top2_merge(w1, wi, w2, ob1, obi, ob2);
        }
        best = w1; bi = wi; second = w2;
      } else {
        while (c0 | c1) {
          int p;
          if (c0) { p = __ffs(c0) - 1; c0 &= c0 - 1; }
          else { p = 32 + __ffs(c1) - 1; c1 &= c1 - 1; }
          const float d = coop_dmm(sm, t, p, p32, Dp);
          if (d < best || (d == best && p < bi)) { second = best; best = d; bi = p; }
          else second = fminf(second, d);
        }
      }
      int idx = bi;
      if (second <= best + tol2) {
        idx = refine_match64<T>(sm, span_row(src, u, off, t, D), t, p64, P, D, lane);
        if (lane == 0 && c.stats) atomicAdd(&c.stats[0], 1u);
      }
      if (lane == 0) sm.fidx[t] = idx;
    }
  }
}

// The same pruned search for 64 < P <= 32 NC (NC = 4 or 8: decode flushes after many
// refreshes, e.g. cfg4's 156 patterns).  The probe table [NPROBE][32 NC] lives in the pattern
// staging rows of sm.ms (16 KB at NC = 8, rows 0..31; the zero row 32 is untouched), so full
// distances read pattern rows from the fp32 table in L2.  Lane l holds patterns l + 32 pc.
__device__ __forceinline__ float coop_dmm_g(const EncSmem& sm, int t, int p, const float* p32, int Dp) {
  const int lane = threadIdx.x & 31;
  const int cc = 4 * lane;
  float mx = -INF32, mn = INF32;
  if (cc < sm.Dm) {
    const float4 x4 = *reinterpret_cast<const float4*>(sm.xs + t * sm.DS + cc);
    const float4 m4 = __ldg(reinterpret_cast<const float4*>(p32 + (int64_t)p * Dp + cc));
    const float r0 = x4.x - m4.x, r1 = x4.y - m4.y, r2 = x4.z - m4.z, r3 = x4.w - m4.w;
    mx = fmax3(fmaxf(r0, r1), r2, r3);
    mn = fmin3(fminf(r0, r1), r2, r3);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  return mx - mn;
}
template <typename T, int NC>
__device__ void match_pruned_wide(const DevCache& c, const EncSmem& sm, const SpanSrc<T>& src, int u, int64_t off,
                                  int L, int P, const float* p32, const double* p64, float pmax) {
  constexpr int PM = 32 * NC;
  constexpr int TG = 2;  // tokens per probe-table pass (register budget of the inlined search)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = c.D, Dp = c.Dp;
  float* mpk = sm.ms;  // [NPROBE][PM]
  __syncthreads();     // every reader of the staged chunk-0 rows is done
  for (int i = tid; i < NPROBE * PM; i += ENC_THREADS) {
    const int k = i / PM, p = i - k * PM;
    mpk[i] = p < P ? p32[(int64_t)p * Dp + sm.probe[k]] : 0.f;
  }
  __syncthreads();
  for (int t0 = 16 * warp; t0 < 16 * warp + 16 && t0 < L; t0 += TG) {
    float lb[TG][NC];
#pragma unroll
    for (int pc = 0; pc < NC; ++pc) {
      float m[NPROBE];
#pragma unroll
      for (int k = 0; k < NPROBE; ++k) m[k] = mpk[k * PM + 32 * pc + lane];
      const bool valid = 32 * pc + lane < P;
#pragma unroll
      for (int j = 0; j < TG; ++j) {
        float a = -INF32, b = INF32;
        const float4* xq = reinterpret_cast<const float4*>(sm.xp + (t0 + j) * NPROBE);
#pragma unroll
        for (int k4 = 0; k4 < NPROBE / 4; ++k4) {
          const float4 x4 = xq[k4];
          const float r0 = x4.x - m[4 * k4], r1 = x4.y - m[4 * k4 + 1];
          const float r2 = x4.z - m[4 * k4 + 2], r3 = x4.w - m[4 * k4 + 3];
          a = fmax3(a, r0, r1); a = fmax3(a, r2, r3);
          b = fmin3(b, r0, r1); b = fmin3(b, r2, r3);
        }
        lb[j][pc] = valid ? a - b : INF32;
      }
    }
#pragma unroll 1
    for (int j = 0; j < TG; ++j) {
      const int t = t0 + j;
      if (t >= L) break;
      float lbj[NC];  // token j's bounds by selects (a dynamic index would put lb in local memory)
#pragma unroll
      for (int pc = 0; pc < NC; ++pc)
        lbj[pc] = j == 0 ? lb[0][pc] : (j == 1 ? lb[1][pc] : (j == 2 ? lb[TG > 2 ? 2 : 0][pc] : lb[TG > 3 ? 3 : 0][pc]));
      // guess = lowest LB, lowest pattern index on ties
      float gv = lbj[0];
#pragma unroll
      for (int pc = 1; pc < NC; ++pc) gv = fminf(gv, lbj[pc]);
#pragma unroll
      for (int o = 16; o; o >>= 1) gv = fminf(gv, __shfl_xor_sync(0xffffffffu, gv, o));
      int gi = -1;
#pragma unroll
      for (int pc = 0; pc < NC; ++pc) {
        const unsigned e = __ballot_sync(0xffffffffu, lbj[pc] == gv);
        if (gi < 0 && e) gi = 32 * pc + __ffs(e) - 1;
      }
      const float tol2 = 2.f * TWO_M20 * (sm.xabs[t] + pmax);
      float best = coop_dmm_g(sm, t, gi, p32, Dp);
      int bi = gi;
      float second = INF32;
      const float bound = best + tol2;
      unsigned cm[NC];
      int ncand = 0;
#pragma unroll
      for (int pc = 0; pc < NC; ++pc) {
        cm[pc] = __ballot_sync(0xffffffffu, lbj[pc] <= bound);
        if ((gi >> 5) == pc) cm[pc] &= ~(1u << (gi & 31));
        ncand += __popc(cm[pc]);
      }
      if (ncand > PRUNE_MAXCAND) {
        // poorly separated token: exhaustive search (lane = pattern, rows from L2)
        float w1 = INF32, w2 = INF32;
        int wi = 0x7fffffff;
        const float* xr = sm.xs + t * sm.DS;
#pragma unroll 1
        for (int pc = 0; pc < NC; ++pc) {
          const int pp = 32 * pc + lane;
          float mx = -INF32, mn = INF32;
          if (pp < P) {
            const float* mrow = p32 + (int64_t)pp * Dp;
            for (int cc = 0; cc < sm.Dm; cc += 4) {
              const float4 x4 = *reinterpret_cast<const float4*>(xr + cc);
              const float4 q = __ldg(reinterpret_cast<const float4*>(mrow + cc));
              const float r0 = x4.x - q.x, r1 = x4.y - q.y, r2 = x4.z - q.z, r3 = x4.w - q.w;
              mx = fmax3(mx, r0, r1); mx = fmax3(mx, r2, r3);
              mn = fmin3(mn, r0, r1); mn = fmin3(mn, r2, r3);
            }
          }
          const float v = pp < P ? mx - mn : INF32;
          top2_merge(w1, wi, w2, v, pp, INF32);  // lanes visit their patterns in increasing index
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const float ob1 = __shfl_xor_sync(0xffffffffu, w1, o);
          const int obi = __shfl_xor_sync(0xffffffffu, wi, o);
          const float ob2 = __shfl_xor_sync(0xffffffffu, w2, o);
          top2_merge(w1, wi, w2, ob1, obi, ob2);
        }
        best = w1; bi = wi; second = w2;
      } else {
#pragma unroll 1
        for (int pc = 0; pc < NC; ++pc) {
          while (cm[pc]) {
            const int p = 32 * pc + __ffs(cm[pc]) - 1;
            cm[pc] &= cm[pc] - 1;
            const float d = coop_dmm_g(sm, t, p, p32, Dp);
            if (d < best || (d == best && p < bi)) { second = best; best = d; bi = p; }
            else second = fminf(second, d);
          }
        }
      }
      int idx = bi;
      if (second <= best + tol2) {
        idx = refine_match64<T>(sm, span_row(src, u, off, t, D), t, p64, P, D, lane);
        if (lane == 0 && c.stats) atomicAdd(&c.stats[0], 1u);
      }
      if (lane == 0) sm.fidx[t] = idx;
    }
  }
}

// Exhaustive fp32 matching (lane = pattern, chunks of 32) for any table size.
template <typename T>
__device__ void match_brute(const DevCache& c, const EncSmem& sm, const SpanSrc<T>& src, int u, int64_t off, int L,
                            int P, const float* p32, const double* p64, float pmax) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = c.D, Dp = c.Dp;
  for (int pb = 0; pb < P; pb += 32) {
    const int pc = min(32, P - pb);
    if (pb > 0) {  // chunk 0 was staged with the zero row; later chunks overwrite rows 0..31
      __syncthreads();
      for (int i = tid; i < 32 * sm.Dm; i += ENC_THREADS) {
        const int p = i / sm.Dm, cc = i - p * sm.Dm;
        sm.ms[p * sm.DS + cc] = p < pc ? p32[(int64_t)(pb + p) * Dp + (cc < D ? cc : 0)] : 0.f;
      }
      __syncthreads();
    }
    const float* mrow = sm.ms + lane * sm.DS;
    for (int t0 = 16 * warp; t0 < 16 * warp + 16 && t0 < L; t0 += 4) {
      float mx[4], mn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) { mx[j] = -INF32; mn[j] = INF32; }
      for (int cc = 0; cc < sm.Dm; cc += 4) {
        const float4 m4 = *reinterpret_cast<const float4*>(mrow + cc);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 x4 = *reinterpret_cast<const float4*>(sm.xs + (t0 + j) * sm.DS + cc);
          const float r0 = x4.x - m4.x, r1 = x4.y - m4.y, r2 = x4.z - m4.z, r3 = x4.w - m4.w;
          mx[j] = fmax3(mx[j], r0, r1);
          mx[j] = fmax3(mx[j], r2, r3);
          mn[j] = fmin3(mn[j], r0, r1);
          mn[j] = fmin3(mn[j], r2, r3);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = t0 + j;
        float v1 = lane < pc ? mx[j] - mn[j] : INF32;
        int i1 = pb + lane;
        float v2 = INF32;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const float b1 = __shfl_xor_sync(0xffffffffu, v1, o);
          const int bi = __shfl_xor_sync(0xffffffffu, i1, o);
          const float b2 = __shfl_xor_sync(0xffffffffu, v2, o);
          top2_merge(v1, i1, v2, b1, bi, b2);
        }
        if (lane == 0 && t < L) {
          if (pb == 0) { sm.best1[t] = v1; sm.bidx[t] = i1; sm.best2[t] = v2; }
          else {
            float a1 = sm.best1[t], a2 = sm.best2[t]; int ai = sm.bidx[t];
            top2_merge(a1, ai, a2, v1, i1, v2);
            sm.best1[t] = a1; sm.bidx[t] = ai; sm.best2[t] = a2;
          }
        }
      }
    }
  }
  __syncthreads();
  for (int t = warp; t < L; t += ENC_THREADS / 32) {
    const float tol = TWO_M20 * (sm.xabs[t] + pmax);
    int idx = sm.bidx[t];
    if (sm.best2[t] <= sm.best1[t] + 2.f * tol) {
      idx = refine_match64<T>(sm, span_row(src, u, off, t, D), t, p64, P, D, lane);
      if (lane == 0 && c.stats) atomicAdd(&c.stats[0], 1u);
    }
    if (lane == 0) sm.fidx[t] = idx;
  }
}

template <typename T>
__global__ void __launch_bounds__(ENC_THREADS, 2)
encode_span_kernel(DevCache c, SpanSrc<T> srck, SpanSrc<T> srcv, int first_block, bool vec_rows) {
  const int u = blockIdx.y;
  const int b = first_block + blockIdx.x;
  const int64_t start = c.blk_start[b];
  const int L = c.blk_len[b];
  const int64_t off = start - c.blk_start[first_block];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = c.D, Dp = c.Dp;
  // prefill spans read caller rows (finiteness checked here); decode flushes read window rows
  // that window_put already checked
  const bool check_nf = srck.ring > (int64_t)1 << 40;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  EncSmem sm;
  sm.Dm = round_up(D, 4);
  sm.DS = sm.Dm + 4;
  sm.xs = reinterpret_cast<float*>(smem_raw);
  sm.ms = sm.xs + GMAX * sm.DS;
  sm.xp = sm.ms + MS_ROWS * sm.DS;
  sm.xabs = sm.xp + GMAX * NPROBE;
  sm.best1 = sm.xabs + GMAX;
  sm.best2 = sm.best1 + GMAX;
  sm.bidx = reinterpret_cast<int*>(sm.best2 + GMAX);
  sm.fidx = sm.bidx + GMAX;
  {
    size_t o = (size_t)(GMAX + MS_ROWS) * sm.DS * 4 + (size_t)GMAX * NPROBE * 4 + 5 * GMAX * 4;
    o = (o + 15) / 16 * 16;
    sm.qlo = reinterpret_cast<double*>(smem_raw + o);
    sm.qhi = sm.qlo + 2 * DMAX;
    sm.probe = reinterpret_cast<int*>(sm.qhi + 2 * DMAX);
    sm.mpk = reinterpret_cast<float*>(sm.probe + NPROBE);
  }

  for (int side = 0; side < 2; ++side) {
    const SpanSrc<T>& src = side == 0 ? srck : srcv;
    const bool usep = side == 0 ? c.use_kp : c.use_vp;
    const int P = usep ? (side == 0 ? c.nk[u] : c.nv[u]) : 0;
    const float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * Dp;
    const double* p64 = (side == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * D;
    const float pmax = P > 0 ? (side == 0 ? c.kpmax[u] : c.vpmax[u]) : 0.f;
    // wide tables: the probe table must fit the 32 staging rows (head_dim >= 124 at 256 patterns)
    const bool pruned = P > 0 && exact_in_f32<T>::value && c.prune &&
                        (P <= PRUNE_PMAX || (P <= PRUNE_WIDE_PMAX && NPROBE * (P > 128 ? 256 : 128) <= 32 * sm.DS));

    __syncthreads();  // previous side done with smem
    if (tid < NPROBE) sm.probe[tid] = c.probe[((int64_t)u * 2 + side) * 16 + tid];
    // patterns 0..31 (padded channels duplicate channel 0) and the zero row
    {
      const int np32 = min(P, 32), V4 = sm.Dm / 4;
      for (int i = tid; i < MS_ROWS * V4; i += ENC_THREADS) {
        const int p = i / V4, c4 = i - p * V4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p < np32) {
          v = __ldg(reinterpret_cast<const float4*>(p32 + (int64_t)p * Dp) + c4);  // Dp >= Dm, rows 16B aligned
          if (4 * c4 + 3 >= D) {  // padded tail channels duplicate channel 0
            const float m0 = p32[(int64_t)p * Dp];
            if (4 * c4 + 0 >= D) v.x = m0;
            if (4 * c4 + 1 >= D) v.y = m0;
            if (4 * c4 + 2 >= D) v.z = m0;
            if (4 * c4 + 3 >= D) v.w = m0;
          }
        }
        *reinterpret_cast<float4*>(sm.ms + p * sm.DS + 4 * c4) = v;
      }
    }
    __syncthreads();
    // ---- A. stage rows as fp32, |x|max per row, probe values ----------------------
    {
      constexpr int EPV = 16 / sizeof(T);  // elements per 16-byte vector
      const int VR = D / EPV;              // vectors per row
      if (vec_rows && VR <= 32 && (32 % VR) == 0) {
        // 32/VR rows per warp pass, 4 passes of loads in flight per lane
        const int RPI = 32 / VR;
        const int rl = lane / VR, vl = lane - rl * VR;
        const int stride = (ENC_THREADS / 32) * RPI;
        for (int r0 = warp * RPI; r0 < L; r0 += 4 * stride) {
          uint4 v[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = r0 + k * stride + rl;
            if (r < L) v[k] = __ldg(reinterpret_cast<const uint4*>(span_row(src, u, off, r, D)) + vl);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int r = r0 + k * stride + rl;
            float m = 0.f;
            if (r < L) {
              const T* e = reinterpret_cast<const T*>(&v[k]);
              float fv[EPV];
              unsigned nf = 0u;
#pragma unroll
              for (int q2 = 0; q2 < EPV; ++q2) {
                fv[q2] = (float)to_f64(e[q2]);
                m = fmaxf(m, fabsf(fv[q2]));
                if (check_nf && !is_finite_el(e[q2])) nf |= 1u << q2;
              }
              if (nf) atomicMin(c.bad, nf_key(u, side, start + r, vl * EPV + __ffs(nf) - 1));
              float* xr = sm.xs + r * sm.DS + vl * EPV;
              if constexpr (EPV % 4 == 0) {
#pragma unroll
                for (int q2 = 0; q2 < EPV; q2 += 4)
                  *reinterpret_cast<float4*>(xr + q2) = make_float4(fv[q2], fv[q2 + 1], fv[q2 + 2], fv[q2 + 3]);
              } else {
#pragma unroll
                for (int q2 = 0; q2 < EPV; ++q2) xr[q2] = fv[q2];
              }
            }
            for (int o = VR >> 1; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (vl == 0 && r < L) sm.xabs[r] = m;
          }
        }
      } else {
        for (int r = warp; r < L; r += ENC_THREADS / 32) {
          const T* row = span_row(src, u, off, r, D);
          float* xr = sm.xs + r * sm.DS;
          float m = 0.f;
          for (int ch = lane; ch < D; ch += 32) {
            const float f = (float)to_f64(row[ch]);
            xr[ch] = f;
            m = fmaxf(m, fabsf(f));
            if (check_nf && !is_finite_el(row[ch])) atomicMin(c.bad, nf_key(u, side, start + r, ch));
          }
          m = warp_max_f(m);
          if (lane == 0) sm.xabs[r] = m;
        }
      }
      __syncthreads();
      // padded channels duplicate channel 0; x at the probe channels
      if (sm.Dm > D)
        for (int i = tid; i < L * (sm.Dm - D); i += ENC_THREADS) {
          const int r = i / (sm.Dm - D), cc = D + i % (sm.Dm - D);
          sm.xs[r * sm.DS + cc] = sm.xs[r * sm.DS];
        }
      if (pruned)
        for (int i = tid; i < L * NPROBE; i += ENC_THREADS) {
          const int r = i / NPROBE, k = i % NPROBE;
          sm.xp[i] = sm.xs[r * sm.DS + sm.probe[k]];
        }
    }
    __syncthreads();

    // ---- B. nearest pattern -------------------------------------------------------
    if (pruned) {
      if (P > 128) match_pruned_wide<T, 8>(c, sm, src, u, off, L, P, p32, p64, pmax);
      else if (P > PRUNE_PMAX) match_pruned_wide<T, 4>(c, sm, src, u, off, L, P, p32, p64, pmax);
      else if (P > 32) match_pruned<T, true>(c, sm, src, u, off, L, P, p32, p64, pmax);
      else match_pruned<T, false>(c, sm, src, u, off, L, P, p32, p64, pmax);
    } else if (P > 0) {
      match_brute<T>(c, sm, src, u, off, L, P, p32, p64, pmax);
    } else {
      for (int t = tid; t < L; t += ENC_THREADS) sm.fidx[t] = RAW;
    }
    __syncthreads();

    // ---- C/D. residual extrema, gate, quantization ---------------------------------
    if constexpr (exact_in_f32<T>::value) {
      encode_sides_fast<T>(c, sm, src, side, u, b, start, off, L, P, p32, p64, pmax);
    } else {
    // ---- fp64-input path: residuals, ranges and codes in IEEE fp64 ---------
    const bool per_token = (side == 1) || (c.use_kgate && P > 0);
    if (per_token) {
      const bool gate_on = side == 1 ? c.use_vgate : true;
      double* diag = side == 1 ? c.vdiag : c.kdiag;
      for (int t = warp; t < L; t += ENC_THREADS / 32) {
        const T* row = span_row(src, u, off, t, D);
        const int idx = sm.fidx[t];
        const double* m = idx >= 0 ? p64 + (int64_t)idx * D : nullptr;
        double xmx = -1.0 / 0.0, xmn = 1.0 / 0.0, rmx = xmx, rmn = xmn;
        for (int cc = lane; cc < D; cc += 32) {
          double x = xval<T>(sm, row, t, cc);
          xmx = fmax(xmx, x); xmn = fmin(xmn, x);
          if (m) { double r = __dsub_rn(x, m[cc]); rmx = fmax(rmx, r); rmn = fmin(rmn, r); }
        }
        xmx = warp_max_d(xmx); xmn = warp_min_d(xmn);
        rmx = warp_max_d(rmx); rmn = warp_min_d(rmn);
        bool flatten = false;
        if (P > 0) {
          const double raw = __dsub_rn(xmx, xmn), flat = __dsub_rn(rmx, rmn);
          if (gate_on) flatten = raw > 0.0 && __ddiv_rn(flat, raw) <= c.thr;
          else flatten = true;
          if (lane == 0 && c.keep_diag && diag) {
            int64_t o = ((int64_t)u * c.Tcap + start + t) * 2;
            diag[o] = raw; diag[o + 1] = flat;
          }
        }
        const int fidx = flatten ? idx : RAW;
        if (side == 0) {  // K gate: only the index/payload choice; K quantizes per channel below
          __syncwarp();
          if (lane == 0) sm.fidx[t] = fidx;
          continue;
        }
        const double lo = flatten ? rmn : xmn, hi = flatten ? rmx : xmx;
        const QuantParamsDev qp = make_qparams(lo, hi, c.qmax);
        for (int cc = lane; cc < D; cc += 32) {
          double x = xval<T>(sm, row, t, cc);
          double v = flatten ? __dsub_rn(x, m[cc]) : x;
          *cslot(sm, t, cc) = (uint8_t)quant_code(v, qp, c.stats ? &c.stats[1] : nullptr);
        }
        if (lane == 0) {
          const int64_t tok = (int64_t)u * c.Tcap + start + t;
          c.vparam64[2 * tok] = qp.scale;
          c.vparam64[2 * tok + 1] = qp.lo;
          const int64_t slot = ((int64_t)u * c.NBcap + b) * c.GP + t;
          c.vparam32[2 * slot] = (float)qp.scale;
          c.vparam32[2 * slot + 1] = (float)qp.lo;
          c.vidx[slot] = (int16_t)fidx;
        }
      }
    }

    // ---- D. K: per-channel quantization over the span's tokens ---------------
    if (side == 0) {
      __syncthreads();
      const int ch = tid & (DMAX - 1), half = tid >> 7;
      const int tb = half ? L / 2 : 0, te = half ? L : L / 2;
      double lo = 1.0 / 0.0, hi = -1.0 / 0.0;
      if (ch < D) {
        for (int t = tb; t < te; ++t) {
          const int idx = sm.fidx[t];
          double x = xval<T>(sm, span_row(src, u, off, t, D), t, ch);
          double v = idx >= 0 ? __dsub_rn(x, p64[(int64_t)idx * D + ch]) : x;
          lo = fmin(lo, v); hi = fmax(hi, v);
        }
      }
      sm.qlo[half * DMAX + ch] = lo;
      sm.qhi[half * DMAX + ch] = hi;
      __syncthreads();
      if (ch < D) {
        lo = fmin(sm.qlo[ch], sm.qlo[DMAX + ch]);
        hi = fmax(sm.qhi[ch], sm.qhi[DMAX + ch]);
        const QuantParamsDev qp = make_qparams(lo, hi, c.qmax);
        for (int t = tb; t < te; ++t) {
          const int idx = sm.fidx[t];
          double x = xval<T>(sm, span_row(src, u, off, t, D), t, ch);
          double v = idx >= 0 ? __dsub_rn(x, p64[(int64_t)idx * D + ch]) : x;
          *cslot(sm, t, ch) = (uint8_t)quant_code(v, qp, c.stats ? &c.stats[1] : nullptr);
        }
        if (half == 0) {
          const int64_t o64 = ((int64_t)u * c.NBcap + b) * 2 * D;
          c.kparam64[o64 + ch] = qp.scale;
          c.kparam64[o64 + D + ch] = qp.lo;
        }
      }
      if (half == 0) {
        const int64_t o32 = ((int64_t)u * c.NBcap + b) * 2 * Dp;
        for (int cc = ch; cc < Dp; cc += DMAX) {
          float s = 0.f, z = 0.f;
          if (cc < D) { s = (float)__ddiv_rn(__dsub_rn(hi, lo), (double)c.qmax); z = (float)lo; }
          c.kparam32[o32 + cc] = s;
          c.kparam32[o32 + Dp + cc] = z;
        }
      }
      for (int t = tid; t < L; t += ENC_THREADS) c.kidx[((int64_t)u * c.NBcap + b) * c.GP + t] = (int16_t)sm.fidx[t];
      }
    }

    // ---- E. pack the codes into the mma-fragment layout ------------------------------
    // thread = (lane ln, word group); the words of one lane are contiguous in HBM
    __syncthreads();
    {
      const int WL = frag_words_per_lane(Dp, c.bits);
      const int S = 16 / c.bits;
      const int ln = tid & 31, grp = tid >> 5;
      const int g = ln >> 2, q = ln & 3;
      uint32_t* dst = reinterpret_cast<uint32_t*>((side == 0 ? c.kcodes : c.vcodes) +
                                                  ((int64_t)u * c.NBcap + b) * c.blk_bytes);
      auto code = [&](int t, int ch) -> uint32_t { return (t < L && ch < D) ? *cslot(sm, t, ch) : 0u; };
      for (int it = grp; it < c.ntile_blk * WL; it += ENC_THREADS / 32) {
        const int tile = it / WL, wl = it - tile * WL;
        uint32_t word = 0;
        for (int s2 = 0; s2 < S; ++s2) {
          const int R = frag_reg_of(side, wl, s2, c.bits);
          const int j = R >> 2, reg = R & 3;
          const int row = g + 8 * (reg & 1), col = 2 * q + 8 * (reg >> 1);
          const int shift = s2 * c.bits;
          if (side == 0) {
            const int t = tile * 16 + row, c0 = 16 * j + col;
            word |= code(t, c0) << shift;
            word |= code(t, c0 + 1) << (16 + shift);
          } else {
            const int ch = 16 * j + row, t0 = tile * 16 + col;
            word |= code(t0, ch) << shift;
            word |= code(t0 + 1, ch) << (16 + shift);
          }
        }
        dst[(tile * 32 + ln) * WL + wl] = word;
      }
    }
  }
}

template <typename T>
cudaError_t launch_encode(const DevCache& c, const SpanSrc<T>& k, const SpanSrc<T>& v, int first_block,
                          int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  const size_t smem = enc_smem_bytes(c.D);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(encode_span_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)enc_smem_bytes(DMAX));
    attr_set = true;
  }
  dim3 grid(nblocks, c.U);
  // 16-byte row loads need D * sizeof(T) % 16 == 0 and 16-byte aligned bases / unit strides
  const bool vec = (c.D * sizeof(T)) % 16 == 0 && ((uintptr_t)k.base % 16) == 0 && ((uintptr_t)v.base % 16) == 0 &&
                   (k.unit_stride * sizeof(T)) % 16 == 0 && (v.unit_stride * sizeof(T)) % 16 == 0;
  encode_span_kernel<T><<<grid, ENC_THREADS, smem, st>>>(c, k, v, first_block, vec);
  return cudaGetLastError();
}

template cudaError_t launch_encode<__half>(const DevCache&, const SpanSrc<__half>&, const SpanSrc<__half>&, int, int, cudaStream_t);
template cudaError_t launch_encode<__nv_bfloat16>(const DevCache&, const SpanSrc<__nv_bfloat16>&, const SpanSrc<__nv_bfloat16>&, int, int, cudaStream_t);
template cudaError_t launch_encode<float>(const DevCache&, const SpanSrc<float>&, const SpanSrc<float>&, int, int, cudaStream_t);
template cudaError_t launch_encode<double>(const DevCache&, const SpanSrc<double>&, const SpanSrc<double>&, int, int, cudaStream_t);

}  // namespace pkv
