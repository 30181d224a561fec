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
// arithmetic), so indices are bit-identical, ties to the lowest index.
// Residuals, ranges, scales and the gate ratio are fp64; codes use the
// guarded fp32 quotient of pkv_common.cuh.
#include "pkv_common.cuh"

namespace pkv {

constexpr int ENC_THREADS = 256;
#define INF32 __int_as_float(0x7f800000)

struct EncSmem {
  int DS, Dm;
  float* xs;      // [GMAX][DS] span rows (fp32; exact for 16/32-bit inputs)
  float* ms;      // [32][DS] pattern chunk
  uint8_t* codes; // [GMAX][Dp] code tile
  float* xabs;    // [GMAX]
  float* best1; float* best2; int* bidx; int* fidx;  // [GMAX]
  double* qlo; double* qhi;  // [2][DMAX]
};

__host__ __device__ inline size_t enc_smem_bytes(int D, int Dp) {
  int Dm = round_up(D, 4), DS = Dm + 4;
  size_t b = (size_t)(GMAX + 32) * DS * 4 + (size_t)GMAX * Dp + 4 * GMAX * 4 + 2 * GMAX * 4;
  b = (b + 15) / 16 * 16;
  b += 4 * DMAX * 8;
  return b;
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
  return s.base + (int64_t)u * s.unit_stride + ((s.row0 + off + r) % s.ring) * (int64_t)D;
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

template <typename T>
__global__ void __launch_bounds__(ENC_THREADS, 2)
encode_span_kernel(DevCache c, SpanSrc<T> srck, SpanSrc<T> srcv, int first_block) {
  const int u = blockIdx.y;
  const int b = first_block + blockIdx.x;
  const int64_t start = c.blk_start[b];
  const int L = c.blk_len[b];
  const int64_t off = start - c.blk_start[first_block];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int D = c.D, Dp = c.Dp;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  EncSmem sm;
  sm.Dm = round_up(D, 4);
  sm.DS = sm.Dm + 4;
  sm.xs = reinterpret_cast<float*>(smem_raw);
  sm.ms = sm.xs + GMAX * sm.DS;
  sm.codes = reinterpret_cast<uint8_t*>(sm.ms + 32 * sm.DS);
  sm.xabs = reinterpret_cast<float*>(sm.codes + GMAX * Dp);
  sm.best1 = sm.xabs + GMAX;
  sm.best2 = sm.best1 + GMAX;
  sm.bidx = reinterpret_cast<int*>(sm.best2 + GMAX);
  sm.fidx = sm.bidx + GMAX;
  {
    size_t o = (size_t)(GMAX + 32) * sm.DS * 4 + (size_t)GMAX * Dp + 6 * GMAX * 4;
    o = (o + 15) / 16 * 16;
    sm.qlo = reinterpret_cast<double*>(smem_raw + o);
    sm.qhi = sm.qlo + 2 * DMAX;
  }
  const int ntok = c.ntile_blk * 16;  // padded tokens in the block

  for (int side = 0; side < 2; ++side) {
    const SpanSrc<T>& src = side == 0 ? srck : srcv;
    const bool usep = side == 0 ? c.use_kp : c.use_vp;
    const int P = usep ? (side == 0 ? c.nk[u] : c.nv[u]) : 0;
    const float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * Dp;
    const double* p64 = (side == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * D;
    const float pmax = P > 0 ? (side == 0 ? c.kpmax[u] : c.vpmax[u]) : 0.f;

    __syncthreads();  // previous side done with smem
    // ---- A. stage rows as fp32, padded channels duplicate channel 0 ----------
    for (int i = tid; i < L * sm.Dm; i += ENC_THREADS) {
      int r = i / sm.Dm, cc = i - r * sm.Dm;
      const T* row = span_row(src, u, off, r, D);
      sm.xs[r * sm.DS + cc] = (float)to_f64(row[cc < D ? cc : 0]);
    }
    for (int i = tid; i < ntok * Dp; i += ENC_THREADS) {
      int r = i / Dp, cc = i - r * Dp;
      if (r >= L || cc >= D) sm.codes[i] = 0;
    }
    __syncthreads();
    for (int r = warp; r < L; r += ENC_THREADS / 32) {
      float m = 0.f;
      for (int cc = lane; cc < D; cc += 32) m = fmaxf(m, fabsf(sm.xs[r * sm.DS + cc]));
      m = warp_max_f(m);
      if (lane == 0) sm.xabs[r] = m;
    }

    // ---- B. fp32 min-max matching, lane = pattern ----------------------------
    if (P > 0) {
      for (int pb = 0; pb < P; pb += 32) {
        const int pc = min(32, P - pb);
        __syncthreads();
        for (int i = tid; i < 32 * sm.Dm; i += ENC_THREADS) {
          int p = i / sm.Dm, cc = i - p * sm.Dm;
          sm.ms[p * sm.DS + cc] = p < pc ? p32[(int64_t)(pb + p) * Dp + (cc < D ? cc : 0)] : 0.f;
        }
        __syncthreads();
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
              float r0 = x4.x - m4.x, r1 = x4.y - m4.y, r2 = x4.z - m4.z, r3 = x4.w - m4.w;
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
              float b1 = __shfl_xor_sync(0xffffffffu, v1, o);
              int bi = __shfl_xor_sync(0xffffffffu, i1, o);
              float b2 = __shfl_xor_sync(0xffffffffu, v2, o);
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
      // ambiguity test and fp64 refinement (rare)
      for (int t = warp; t < L; t += ENC_THREADS / 32) {
        const float tol = 9.5367431640625e-07f * (sm.xabs[t] + pmax);  // 2^-20 * S
        int idx = sm.bidx[t];
        if (sm.best2[t] <= sm.best1[t] + 2.f * tol) {
          idx = refine_match64<T>(sm, span_row(src, u, off, t, D), t, p64, P, D, lane);
          if (lane == 0 && c.stats) atomicAdd(&c.stats[0], 1u);
        }
        if (lane == 0) sm.fidx[t] = idx;
      }
    } else {
      for (int t = tid; t < L; t += ENC_THREADS) sm.fidx[t] = RAW;
    }
    __syncthreads();

    // ---- C. per-token residual stats, gate, and (V) per-token quantization ----
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
          sm.codes[t * Dp + cc] = (uint8_t)quant_code(v, qp, c.stats ? &c.stats[1] : nullptr);
        }
        if (lane == 0) {
          const int64_t tok = (int64_t)u * c.Tcap + start + t;
          c.vparam64[2 * tok] = qp.scale;
          c.vparam64[2 * tok + 1] = qp.lo;
          c.vparam32[2 * tok] = (float)qp.scale;
          c.vparam32[2 * tok + 1] = (float)qp.lo;
          c.vidx[tok] = (int16_t)fidx;
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
          sm.codes[t * Dp + ch] = (uint8_t)quant_code(v, qp, c.stats ? &c.stats[1] : nullptr);
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
      for (int t = tid; t < L; t += ENC_THREADS) c.kidx[(int64_t)u * c.Tcap + start + t] = (int16_t)sm.fidx[t];
    }

    // ---- E. pack the code tile into the mma-fragment layout -------------------
    __syncthreads();
    {
      const int WL = frag_words_per_lane(Dp, c.bits);
      const int S = 16 / c.bits;
      const int words = c.ntile_blk * 32 * WL;
      uint32_t* dst = reinterpret_cast<uint32_t*>((side == 0 ? c.kcodes : c.vcodes) +
                                                  ((int64_t)u * c.NBcap + b) * c.blk_bytes);
      for (int w = tid; w < words; w += ENC_THREADS) {
        const int tile = w / (32 * WL);
        const int rem = w - tile * 32 * WL;
        const int ln = rem / WL, wl = rem - ln * WL;
        uint32_t word = 0;
        for (int s = 0; s < S; ++s) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            FragPos p = frag_rc(ln, wl * S + s, e);
            int tok, ch;
            if (side == 0) { tok = tile * 16 + p.row; ch = 16 * p.j + p.col; }
            else { ch = 16 * p.j + p.row; tok = tile * 16 + p.col; }
            word |= (uint32_t)sm.codes[tok * Dp + ch] << ((e ? 16 : 0) + s * c.bits);
          }
        }
        dst[w] = word;
      }
    }
  }
}

template <typename T>
cudaError_t launch_encode(const DevCache& c, const SpanSrc<T>& k, const SpanSrc<T>& v, int first_block,
                          int nblocks, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
  size_t smem = enc_smem_bytes(c.D, c.Dp);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(encode_span_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)enc_smem_bytes(DMAX, DMAX));
    attr_set = true;
  }
  dim3 grid(nblocks, c.U);
  encode_span_kernel<T><<<grid, ENC_THREADS, smem, st>>>(c, k, v, first_block);
  return cudaGetLastError();
}

template cudaError_t launch_encode<__half>(const DevCache&, const SpanSrc<__half>&, const SpanSrc<__half>&, int, int, cudaStream_t);
template cudaError_t launch_encode<__nv_bfloat16>(const DevCache&, const SpanSrc<__nv_bfloat16>&, const SpanSrc<__nv_bfloat16>&, int, int, cudaStream_t);
template cudaError_t launch_encode<float>(const DevCache&, const SpanSrc<float>&, const SpanSrc<float>&, int, int, cudaStream_t);
template cudaError_t launch_encode<double>(const DevCache&, const SpanSrc<double>&, const SpanSrc<double>&, int, int, cudaStream_t);

}  // namespace pkv
