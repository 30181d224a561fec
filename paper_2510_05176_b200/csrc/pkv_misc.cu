// Small kernels around the hot path:
//   K4 pieces: window append + flush pattern refresh (engine.py:172-198,
//              midrange_center patterns.py:161-171, PatternSet.append :51-60)
//   K5 dequant: exact fp64 reconstruction (engine.py:255-303, quant.py:114-117)
//   export:     fragment layout -> reference packed layout (engine.py:222,243)
//   group API:  quantize_group / pack_codes / unpack_codes (quant.py:70-179),
//               match_many (patterns.py:206-221), validation (engine.py:132-139)
#include "pkv_common.cuh"

namespace pkv {

static inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---- non-finite scan: first flat index of a non-finite element --------------------
template <typename T>
__global__ void finite_kernel(const T* x, int64_t n, unsigned long long* first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = to_f64(x[i]);
    if (!isfinite(v)) atomicMin(first, (unsigned long long)i);
  }
}
template <typename T>
cudaError_t launch_finite(const T* x, int64_t n, unsigned long long* first, cudaStream_t st) {
  int blocks = (int)imin64((n + 255) / 256, 148 * 8);
  if (blocks < 1) blocks = 1;
  finite_kernel<T><<<blocks, 256, 0, st>>>(x, n, first);
  return cudaGetLastError();
}
template cudaError_t launch_finite<__half>(const __half*, int64_t, unsigned long long*, cudaStream_t);
template cudaError_t launch_finite<__nv_bfloat16>(const __nv_bfloat16*, int64_t, unsigned long long*, cudaStream_t);
template cudaError_t launch_finite<float>(const float*, int64_t, unsigned long long*, cudaStream_t);
template cudaError_t launch_finite<double>(const double*, int64_t, unsigned long long*, cudaStream_t);

// ---- window ring: copy rows [U][nrows][D] into ring slots (slot0 + r) % Wcap -------
// Row r is token token0 + r of its unit; non-finite elements are flagged in c.bad (the
// reference's finiteness checks, engine.py:136-138 / 180-181, fused into the copy).
template <typename T>
__global__ void window_put_kernel(DevCache c, const T* k, const T* v, int64_t src_unit_stride, int nrows, int slot0,
                                  int64_t token0) {
  const int u = blockIdx.y;
  const int64_t n = (int64_t)nrows * c.D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / c.D), ch = (int)(i - (int64_t)r * c.D);
    const int64_t dst = ((int64_t)u * c.Wcap + (slot0 + r) % c.Wcap) * c.D + ch;
    const int64_t src = (int64_t)u * src_unit_stride + i;
    const T kv = k[src], vv = v[src];
    reinterpret_cast<T*>(c.wk)[dst] = kv;
    reinterpret_cast<T*>(c.wv)[dst] = vv;
    if (!is_finite_el(kv)) atomicMin(c.bad, nf_key(u, 0, token0 + r, ch));
    if (!is_finite_el(vv)) atomicMin(c.bad, nf_key(u, 1, token0 + r, ch));
  }
}
template <typename T>
cudaError_t launch_window_put(const DevCache& c, const T* k, const T* v, int64_t sus, int nrows, int slot0, int64_t token0,
                              cudaStream_t st) {
  if (nrows <= 0) return cudaSuccess;
  int gx = (int)imin64(((int64_t)nrows * c.D + 255) / 256, 64);
  window_put_kernel<T><<<dim3(gx, c.U), 256, 0, st>>>(c, k, v, sus, nrows, slot0, token0);
  return cudaGetLastError();
}
template cudaError_t launch_window_put<__half>(const DevCache&, const __half*, const __half*, int64_t, int, int, int64_t, cudaStream_t);
template cudaError_t launch_window_put<__nv_bfloat16>(const DevCache&, const __nv_bfloat16*, const __nv_bfloat16*, int64_t, int, int, int64_t, cudaStream_t);
template cudaError_t launch_window_put<float>(const DevCache&, const float*, const float*, int64_t, int, int, int64_t, cudaStream_t);
template cudaError_t launch_window_put<double>(const DevCache&, const double*, const double*, int64_t, int, int, int64_t, cudaStream_t);

// ---- flush refresh: midrange of the oldest G ring rows appended as a pattern -------
// grid (U, 2 sides), block D threads.  0.5 * (min + max) in IEEE fp64.
template <typename T>
__global__ void refresh_kernel(DevCache c, int slot0, int G, int side_mask) {
  const int u = blockIdx.x, side = blockIdx.y, ch = threadIdx.x;
  if (!((side_mask >> side) & 1)) return;
  const T* w = reinterpret_cast<const T*>(side == 0 ? c.wk : c.wv) + (int64_t)u * c.Wcap * c.D;
  int* np_ = side == 0 ? c.nk : c.nv;
  const int p = np_[u];
  __shared__ float red[32];
  float a = 0.f;
  if (ch < c.D) {
    double mn = 1.0 / 0.0, mx = -1.0 / 0.0;
    for (int r = 0; r < G; ++r) {
      double x = to_f64(w[(int64_t)((slot0 + r) % c.Wcap) * c.D + ch]);
      mn = fmin(mn, x); mx = fmax(mx, x);
    }
    const double m = __dmul_rn(0.5, __dadd_rn(mn, mx));
    (side == 0 ? c.kpat64 : c.vpat64)[((int64_t)u * c.Pcap + p) * c.D + ch] = m;
    (side == 0 ? c.kpat32 : c.vpat32)[((int64_t)u * c.Pcap + p) * c.Dp + ch] = (float)m;
    a = fabsf((float)m) * (1.f + 1e-6f);
  }
  for (int cc = c.D + ch; cc < c.Dp; cc += blockDim.x)
    (side == 0 ? c.kpat32 : c.vpat32)[((int64_t)u * c.Pcap + p) * c.Dp + cc] = 0.f;
  a = warp_max_f(a);
  if ((ch & 31) == 0) red[ch >> 5] = a;
  __syncthreads();
  if (ch == 0) {
    float m = 0.f;
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) m = fmaxf(m, red[i]);
    float* pm = side == 0 ? c.kpmax : c.vpmax;
    pm[u] = fmaxf(pm[u], m);
    np_[u] = p + 1;
  }
}
template <typename T>
cudaError_t launch_refresh(const DevCache& c, int slot0, int G, int side_mask, cudaStream_t st) {
  int threads = round_up(c.D, 32);
  refresh_kernel<T><<<dim3(c.U, 2), threads, 0, st>>>(c, slot0, G, side_mask);
  return cudaGetLastError();
}
template cudaError_t launch_refresh<__half>(const DevCache&, int, int, int, cudaStream_t);
template cudaError_t launch_refresh<__nv_bfloat16>(const DevCache&, int, int, int, cudaStream_t);
template cudaError_t launch_refresh<float>(const DevCache&, int, int, int, cudaStream_t);
template cudaError_t launch_refresh<double>(const DevCache&, int, int, int, cudaStream_t);

// ---- probe channels of the pruned matcher: the 16 channels with the largest
// spread (max - min over the fp32 table) of each unit-side, ties to the lowest
// channel.  Recomputed whenever a table changes (mining, install, refresh).
__global__ void probe_kernel(DevCache c) {
  const int u = blockIdx.x, side = blockIdx.y, ch = threadIdx.x;
  const int P = side == 0 ? (c.use_kp ? c.nk[u] : 0) : (c.use_vp ? c.nv[u] : 0);
  const float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * c.Dp;
  __shared__ float spread[DMAX];
  if (ch < c.D) {
    float lo = 3.0e38f, hi = -3.0e38f;
    for (int p = 0; p < P; ++p) {
      const float v = p32[(int64_t)p * c.Dp + ch];
      lo = fminf(lo, v); hi = fmaxf(hi, v);
    }
    spread[ch] = P > 0 ? hi - lo : 0.f;
  }
  __syncthreads();
  int* out = c.probe + ((int64_t)u * 2 + side) * 16;
  const int np = c.D < 16 ? c.D : 16;
  if (ch < c.D) {
    const float sp = spread[ch];
    int rank = 0;
    for (int o = 0; o < c.D; ++o) rank += (spread[o] > sp) || (spread[o] == sp && o < ch);
    if (rank < np) out[rank] = ch;
  }
  __syncthreads();
  if (ch >= np && ch < 16) out[ch] = out[0];
}
cudaError_t launch_probes(const DevCache& c, cudaStream_t st) {
  probe_kernel<<<dim3(c.U, 2), DMAX, 0, st>>>(c);
  return cudaGetLastError();
}

// ---- pattern-table install (pkv_set_patterns / snapshot import): device [U][P][D] fp64
// -> the fp64 / fp32 arenas (rows past a unit's count zeroed), per-unit count and
// max |m| (x (1 + 1e-6), the bound the matchers use); no host round trip.
__global__ void install_patterns_kernel(DevCache c, int side, const double* pat, int P, const int* counts) {
  const int u = blockIdx.x;
  const int n = counts ? counts[u] : P;
  double* p64 = (side == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * c.D;
  float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * c.Dp;
  float m = 0.f;
  for (int64_t i = threadIdx.x; i < (int64_t)c.Pcap * c.Dp; i += blockDim.x) {
    const int p = (int)(i / c.Dp), ch = (int)(i % c.Dp);
    const bool in = p < n && ch < c.D;
    const double v = in ? pat[((int64_t)u * P + p) * c.D + ch] : 0.0;
    if (ch < c.D) p64[(int64_t)p * c.D + ch] = v;
    p32[i] = (float)v;
    if (in) m = fmaxf(m, fabsf((float)v) * (1.f + 1e-6f));
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    (side == 0 ? c.kpmax : c.vpmax)[u] = m;
    (side == 0 ? c.nk : c.nv)[u] = n;
  }
}
cudaError_t launch_install_patterns(const DevCache& c, int side, const double* pat, int P, const int* counts,
                                    cudaStream_t st) {
  install_patterns_kernel<<<c.U, 256, 0, st>>>(c, side, pat, P, counts);
  return cudaGetLastError();
}

// ---- fragment-layout addressing (inverse of frag_rc) -------------------------------
struct CodeLoc { int word; int shift; };
__device__ __forceinline__ CodeLoc frag_locate(int side, int row, int col16, int j, int bits, int WL) {
  // row/col16 are the A-fragment coordinates inside sub-tile j
  const int g = row & 7, hr = row >> 3, q = (col16 & 7) >> 1, hc = col16 >> 3, e = col16 & 1;
  const int reg = hr + 2 * hc, lane = 4 * g + q, R = 4 * j + reg;
  int word, slot;
  frag_word_slot(side, R, bits, word, slot);
  CodeLoc l;
  l.word = lane * WL + word;
  l.shift = (e ? 16 : 0) + slot * bits;
  return l;
}
__device__ __forceinline__ int read_code(const uint8_t* blk, int side, int tok, int ch, int Dp, int bits) {
  const int WL = frag_words_per_lane(Dp, bits);
  const int tile = tok >> 4;
  CodeLoc l = side == 0 ? frag_locate(0, tok & 15, ch & 15, ch >> 4, bits, WL)
                        : frag_locate(1, ch & 15, tok & 15, ch >> 4, bits, WL);
  const uint32_t w = reinterpret_cast<const uint32_t*>(blk + (size_t)tile * tile_bytes(Dp, bits))[l.word];
  return (w >> l.shift) & ((1 << bits) - 1);
}

// block index of committed token t (blocks are contiguous in token order)
__device__ __forceinline__ int find_block(const int64_t* start, int nb, int64_t t) {
  int lo = 0, hi = nb - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ---- K5 exact dequant of committed tokens [t0, t1) -> fp64 [U][n][D] ----------------
__global__ void dequant_kernel(DevCache c, int nb, int64_t t0, int64_t n, double* kout, double* vout) {
  const int u = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * c.D; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = t0 + i / c.D;
    const int ch = (int)(i % c.D);
    const int b = find_block(c.blk_start, nb, t);
    const int tb = (int)(t - c.blk_start[b]);
    const uint8_t* kb = c.kcodes + ((int64_t)u * c.NBcap + b) * c.blk_bytes;
    const uint8_t* vb = c.vcodes + ((int64_t)u * c.NBcap + b) * c.blk_bytes;
    // K: scale_c * code + zero_c (+ pattern)   engine.py:255-261
    const double* kp = c.kparam64 + ((int64_t)u * c.NBcap + b) * 2 * c.D;
    double kv = __dadd_rn(__dmul_rn(kp[ch], (double)read_code(kb, 0, tb, ch, c.Dp, c.bits)), kp[c.D + ch]);
    const int64_t slot = ((int64_t)u * c.NBcap + b) * c.GP + tb;
    const int ki = c.kidx[slot];
    if (ki >= 0) kv = __dadd_rn(kv, c.kpat64[((int64_t)u * c.Pcap + ki) * c.D + ch]);
    // V: scale_t * code + zero_t (+ pattern)   engine.py:264-268
    const double* vp = c.vparam64 + ((int64_t)u * c.Tcap + t) * 2;
    double vv = __dadd_rn(__dmul_rn(vp[0], (double)read_code(vb, 1, tb, ch, c.Dp, c.bits)), vp[1]);
    const int vi = c.vidx[slot];
    if (vi >= 0) vv = __dadd_rn(vv, c.vpat64[((int64_t)u * c.Pcap + vi) * c.D + ch]);
    kout[((int64_t)u * n + (i / c.D)) * c.D + ch] = kv;
    vout[((int64_t)u * n + (i / c.D)) * c.D + ch] = vv;
  }
}
cudaError_t launch_dequant(const DevCache& c, int nb, int64_t t0, int64_t n, double* k, double* v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int gx = (int)imin64((n * c.D + 255) / 256, 1024);
  dequant_kernel<<<dim3(gx, c.U), 256, 0, st>>>(c, nb, t0, n, k, v);
  return cudaGetLastError();
}

// ---- unpacked codes export: [U][n][D] uint8 for K and V (token-major) --------------
__global__ void codes_kernel(DevCache c, int nb, int64_t t0, int64_t n, uint8_t* kc, uint8_t* vc) {
  const int u = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * c.D; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = t0 + i / c.D;
    const int ch = (int)(i % c.D);
    const int b = find_block(c.blk_start, nb, t);
    const int tb = (int)(t - c.blk_start[b]);
    kc[(int64_t)u * n * c.D + i] = (uint8_t)read_code(c.kcodes + ((int64_t)u * c.NBcap + b) * c.blk_bytes, 0, tb, ch, c.Dp, c.bits);
    vc[(int64_t)u * n * c.D + i] = (uint8_t)read_code(c.vcodes + ((int64_t)u * c.NBcap + b) * c.blk_bytes, 1, tb, ch, c.Dp, c.bits);
  }
}
cudaError_t launch_codes(const DevCache& c, int nb, int64_t t0, int64_t n, uint8_t* k, uint8_t* v, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int gx = (int)imin64((n * c.D + 255) / 256, 1024);
  codes_kernel<<<dim3(gx, c.U), 256, 0, st>>>(c, nb, t0, n, k, v);
  return cudaGetLastError();
}

// ---- state import (resume from a PKVS snapshot, reference snapshot.py:148-220) ---------------
// Per committed token t of unit u (reference layout in, arena layout out): indices and V
// params into their block slots, fp64 params by token, gate records.
__global__ void import_tokens_kernel(DevCache c, int nb, int64_t C, const int32_t* kidx, const int32_t* vidx,
                                     const double* vparam, const double* kdiag, const double* vdiag) {
  const int u = blockIdx.y;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < C; t += (int64_t)gridDim.x * blockDim.x) {
    const int b = find_block(c.blk_start, nb, t);
    const int64_t slot = ((int64_t)u * c.NBcap + b) * c.GP + (t - c.blk_start[b]);
    const int64_t i = (int64_t)u * C + t;
    c.kidx[slot] = (int16_t)kidx[i];
    c.vidx[slot] = (int16_t)vidx[i];
    const int64_t tok = (int64_t)u * c.Tcap + t;
    c.vparam64[2 * tok] = vparam[2 * i];
    c.vparam64[2 * tok + 1] = vparam[2 * i + 1];
    c.vparam32[2 * slot] = (float)vparam[2 * i];
    c.vparam32[2 * slot + 1] = (float)vparam[2 * i + 1];
    if (c.keep_diag) {
      if (kdiag && c.kdiag) { c.kdiag[2 * tok] = kdiag[2 * i]; c.kdiag[2 * tok + 1] = kdiag[2 * i + 1]; }
      if (vdiag && c.vdiag) { c.vdiag[2 * tok] = vdiag[2 * i]; c.vdiag[2 * tok + 1] = vdiag[2 * i + 1]; }
    }
  }
}
// Per block: K params (fp64 and the fp32 attention copy, padded to Dp)
__global__ void import_kparams_kernel(DevCache c, int nb, const double* kparam) {
  const int u = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)nb * c.Dp;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / c.Dp), ch = (int)(i % c.Dp);
    const int64_t blk = (int64_t)u * c.NBcap + b;
    double sc = 0.0, z = 0.0;
    if (ch < c.D) {
      sc = kparam[(((int64_t)u * nb + b) * 2) * c.D + ch];
      z = kparam[(((int64_t)u * nb + b) * 2 + 1) * c.D + ch];
      c.kparam64[blk * 2 * c.D + ch] = sc;
      c.kparam64[blk * 2 * c.D + c.D + ch] = z;
    }
    c.kparam32[blk * 2 * c.Dp + ch] = (float)sc;
    c.kparam32[blk * 2 * c.Dp + c.Dp + ch] = (float)z;
  }
}
// Per (block, tile, lane, word): the mma-fragment code words from unpacked codes [U][C][D]
// (the same word assembly as stage E of encode_span_kernel)
__global__ void import_codes_kernel(DevCache c, int nb, int64_t C, const uint8_t* kcodes, const uint8_t* vcodes) {
  const int u = blockIdx.y;
  const int WL = frag_words_per_lane(c.Dp, c.bits), S = 16 / c.bits;
  const int64_t nw = (int64_t)nb * c.ntile_blk * 32 * WL;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * nw; i += (int64_t)gridDim.x * blockDim.x) {
    const int side = i >= nw;
    const int64_t k = side ? i - nw : i;
    const int wl = (int)(k % WL), ln = (int)((k / WL) % 32);
    const int tile = (int)((k / (WL * 32)) % c.ntile_blk), b = (int)(k / ((int64_t)WL * 32 * c.ntile_blk));
    const int g = ln >> 2, q = ln & 3;
    const int64_t s0 = c.blk_start[b];
    const int L = c.blk_len[b];
    const uint8_t* src = (side ? vcodes : kcodes) + (int64_t)u * C * c.D;
    auto code = [&](int t, int ch) -> uint32_t {
      return (t < L && ch < c.D && s0 + t < C) ? src[(s0 + t) * c.D + ch] : 0u;
    };
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
    uint8_t* dst = (side ? c.vcodes : c.kcodes) + ((int64_t)u * c.NBcap + b) * c.blk_bytes;
    reinterpret_cast<uint32_t*>(dst)[((int64_t)tile * 32 + ln) * WL + wl] = word;
  }
}
cudaError_t launch_import(const DevCache& c, int nb, int64_t C, const double* kparam, const int32_t* kidx,
                          const int32_t* vidx, const double* vparam, const uint8_t* kcodes, const uint8_t* vcodes,
                          const double* kdiag, const double* vdiag, cudaStream_t st) {
  if (nb <= 0 || C <= 0) return cudaSuccess;
  const int gx = (int)imin64((C + 255) / 256, 1024);
  import_tokens_kernel<<<dim3(gx, c.U), 256, 0, st>>>(c, nb, C, kidx, vidx, vparam, kdiag, vdiag);
  import_kparams_kernel<<<dim3((int)imin64(((int64_t)nb * c.Dp + 255) / 256, 1024), c.U), 256, 0, st>>>(c, nb, kparam);
  const int64_t nw = 2 * (int64_t)nb * c.ntile_blk * 32 * frag_words_per_lane(c.Dp, c.bits);
  import_codes_kernel<<<dim3((int)imin64((nw + 255) / 256, 4096), c.U), 256, 0, st>>>(c, nb, C, kcodes, vcodes);
  return cudaGetLastError();
}

// ---- group API ------------------------------------------------------------------------
// quantize_group over many groups: values fp64 concatenated, offsets[n+1].
// One warp per group (quant.py:70-111).
__global__ void quantize_groups_kernel(const double* vals, const int64_t* offs, int ngroups, int bits,
                                       double* scale, double* zero, uint8_t* codes) {
  const int lane = threadIdx.x & 31;
  const int gidx = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (gidx >= ngroups) return;
  const int64_t a = offs[gidx], b = offs[gidx + 1];
  double lo = 1.0 / 0.0, hi = -1.0 / 0.0;
  for (int64_t i = a + lane; i < b; i += 32) { lo = fmin(lo, vals[i]); hi = fmax(hi, vals[i]); }
  lo = warp_min_d(lo); hi = warp_max_d(hi);
  const QuantParamsDev qp = make_qparams(lo, hi, (1 << bits) - 1);
  for (int64_t i = a + lane; i < b; i += 32) codes[i] = (uint8_t)quant_code(vals[i], qp, nullptr);
  if (lane == 0) { scale[gidx] = qp.scale; zero[gidx] = qp.lo; }
}
cudaError_t launch_quantize_groups(const double* v, const int64_t* o, int n, int bits, double* s, double* z, uint8_t* c,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  quantize_groups_kernel<<<(n + 7) / 8, 256, 0, st>>>(v, o, n, bits, s, z, c);
  return cudaGetLastError();
}

// pack: out byte i = OR_k codes[i*per + k] << (k*bits)   (quant.py:120-146)
__global__ void pack_kernel(const uint8_t* codes, int64_t n, int bits, uint8_t* out) {
  const int per = 8 / bits;
  const int64_t nb = (n + per - 1) / per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned v = 0;
    for (int k = 0; k < per; ++k) {
      const int64_t j = i * per + k;
      if (j < n) v |= (unsigned)codes[j] << (k * bits);
    }
    out[i] = (uint8_t)v;
  }
}
__global__ void unpack_kernel(const uint8_t* in, int64_t n, int bits, uint8_t* codes) {
  const int per = 8 / bits;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    codes[j] = (in[j / per] >> ((j % per) * bits)) & ((1 << bits) - 1);
}
cudaError_t launch_pack(const uint8_t* c, int64_t n, int bits, uint8_t* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int g = (int)imin64((n + 1023) / 1024, 1024);
  pack_kernel<<<g, 256, 0, st>>>(c, n, bits, out);
  return cudaGetLastError();
}
cudaError_t launch_unpack(const uint8_t* in, int64_t n, int bits, uint8_t* c, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int g = (int)imin64((n + 255) / 256, 1024);
  unpack_kernel<<<g, 256, 0, st>>>(in, n, bits, c);
  return cudaGetLastError();
}

// match_many in IEEE fp64 (patterns.py:206-221): one warp per vector, lane = pattern.
__global__ void match_kernel(const double* x, int64_t n, const double* m, int P, int D, int64_t* idx, double* dist,
                             double* res) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= n) return;
  const double* xr = x + r * D;
  double bestv = 1.0 / 0.0;
  int besti = 0;
  for (int pb = 0; pb < P; pb += 32) {
    const int p = pb + lane;
    double v = 1.0 / 0.0;
    if (p < P) {
      double mx = -1.0 / 0.0, mn = 1.0 / 0.0;
      for (int c = 0; c < D; ++c) { double d = __dsub_rn(xr[c], m[(int64_t)p * D + c]); mx = fmax(mx, d); mn = fmin(mn, d); }
      v = __dsub_rn(mx, mn);
    }
    int pi = p;
    warp_argmin_d(v, pi);
    if (v < bestv) { bestv = v; besti = pi; }
  }
  if (lane == 0) { idx[r] = besti; dist[r] = bestv; }
  for (int c = lane; c < D; c += 32) res[r * D + c] = __dsub_rn(xr[c], m[(int64_t)besti * D + c]);
}
cudaError_t launch_match(const double* x, int64_t n, const double* m, int P, int D, int64_t* idx, double* dist, double* res,
                         cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  match_kernel<<<(int)((n + 7) / 8), 256, 0, st>>>(x, n, m, P, D, idx, dist, res);
  return cudaGetLastError();
}

// midrange over rows (patterns.py:161-171)
__global__ void midrange_kernel(const double* x, int64_t n, int D, double* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= D) return;
  double mn = 1.0 / 0.0, mx = -1.0 / 0.0;
  for (int64_t r = 0; r < n; ++r) { double v = x[r * D + c]; mn = fmin(mn, v); mx = fmax(mx, v); }
  out[c] = __dmul_rn(0.5, __dadd_rn(mn, mx));
}
cudaError_t launch_midrange(const double* x, int64_t n, int D, double* out, cudaStream_t st) {
  midrange_kernel<<<(D + 127) / 128, 128, 0, st>>>(x, n, D, out);
  return cudaGetLastError();
}

}  // namespace pkv

namespace pkv {

// ---- unit fork: copy every per-unit arena row of unit src[i] onto unit dst[i] ---------
// grid (n pairs, arenas); 16-byte vectors when the strides, bases and row size allow.
__global__ void fork_units_kernel(ForkArenas fa, const int* src, const int* dst) {
  const ForkArenas::Arena& ar = fa.a[blockIdx.y];
  if (!ar.src || !ar.dst || ar.bytes == 0) return;
  const int s = src[blockIdx.x], d = dst[blockIdx.x];
  const unsigned char* from = ar.src + (int64_t)s * ar.src_stride;
  unsigned char* to = ar.dst + (int64_t)d * ar.dst_stride;
  if (from == to) return;
  if (((ar.bytes | ar.src_stride | ar.dst_stride) & 15) == 0 && (((uintptr_t)ar.src | (uintptr_t)ar.dst) & 15) == 0) {
    const int64_t n = ar.bytes >> 4;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      reinterpret_cast<uint4*>(to)[i] = reinterpret_cast<const uint4*>(from)[i];
  } else {
    for (int64_t i = threadIdx.x; i < ar.bytes; i += blockDim.x) to[i] = from[i];
  }
}

cudaError_t launch_fork(const ForkArenas& fa, int n, const int* src, const int* dst, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fork_units_kernel<<<dim3(n, fa.n), 256, 0, st>>>(fa, src, dst);
  return cudaGetLastError();
}

}  // namespace pkv

namespace pkv {

// ---- single-group quantize+pack / unpack+dequantize (quant.py:70-179) -------------------
// One CTA: block min/max, the exact code rule of quant_code, the packed bytes straight out.
__global__ void qpack_kernel(const double* v, int64_t n, int bits, double* sz, uint8_t* packed) {
  __shared__ double rmin[32], rmax[32];
  double lo = 1.0 / 0.0, hi = -1.0 / 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) { lo = fmin(lo, v[i]); hi = fmax(hi, v[i]); }
  lo = warp_min_d(lo);
  hi = warp_max_d(hi);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) { rmin[warp] = lo; rmax[warp] = hi; }
  __syncthreads();
  lo = rmin[0]; hi = rmax[0];
  for (int w = 1; w < nw; ++w) { lo = fmin(lo, rmin[w]); hi = fmax(hi, rmax[w]); }
  const QuantParamsDev qp = make_qparams(lo, hi, (1 << bits) - 1);
  const int per = 8 / bits;
  const int64_t nb = (n + per - 1) / per;
  for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
    unsigned byte = 0;
    for (int k = 0; k < per; ++k) {
      const int64_t j = b * per + k;
      if (j < n) byte |= (unsigned)quant_code(v[j], qp, nullptr) << (k * bits);
    }
    packed[b] = (uint8_t)byte;
  }
  if (threadIdx.x == 0) { sz[0] = qp.scale; sz[1] = qp.lo; }
}
__global__ void dqunpack_kernel(const uint8_t* packed, int64_t n, int bits, double scale, double zero, double* out) {
  const int per = 8 / bits;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int code = (packed[j / per] >> ((j % per) * bits)) & ((1 << bits) - 1);
    out[j] = __dadd_rn(__dmul_rn(scale, (double)code), zero);
  }
}
cudaError_t launch_qpack(const double* v, int64_t n, int bits, double* sz, uint8_t* packed, cudaStream_t st) {
  qpack_kernel<<<1, 256, 0, st>>>(v, n, bits, sz, packed);
  return cudaGetLastError();
}
cudaError_t launch_dqunpack(const uint8_t* packed, int64_t n, int bits, double scale, double zero, double* out,
                            cudaStream_t st) {
  const int g = (int)imin64((n + 255) / 256, 1024);
  dqunpack_kernel<<<g, 256, 0, st>>>(packed, n, bits, scale, zero, out);
  return cudaGetLastError();
}

}  // namespace pkv
