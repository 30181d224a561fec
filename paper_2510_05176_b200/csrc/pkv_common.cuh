// PatternKV B200 codec -- shared device definitions.
//
// Data layout in HBM (per cache of U units = (batch, layer, kv-head)):
//   patterns   kpat64/vpat64 [U][Pcap][D] f64 (exact, reference semantics)
//              kpat32/vpat32 [U][Pcap][Dp] f32 (fast-filter copies, pad = 0)
//   K blocks   kcodes  [U][NBcap][blk_bytes]  mma-fragment order (see frag_pos)
//              kparam32[U][NBcap][2][Dp] f32 (scale, zero)  kparam64 [U][NBcap][2][D] f64
//              kidx    [U][NBcap][GP] int16 (RAW = -1), block-slot order (GP = 16*ntiles)
//   V tokens   vcodes  [U][NBcap][blk_bytes]  mma-fragment order (V^T operand)
//              vparam32[U][NBcap][GP][2] f32   vparam64 [U][Tcap][2] f64 (by token)
//              vidx    [U][NBcap][GP] int16   (per-token decode metadata in block slots,
//                                             so every tile's metadata is 16B aligned)
//   window     wk/wv   [U][Wcap][D] in the input dtype, ring of W+G rows
//
// A block is one K quantization group span (<= G <= 128 tokens), stored as
// ceil(G/16) tiles of 16 tokens.  Inside a tile each of the 32 lanes of the
// decode-attention warp finds its m16n8k16 A-fragments contiguous
// (16*Dp*bits/8/32 bytes per lane), so the attention kernel dequantizes
// straight from one coalesced vector load into registers.
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pkv {

constexpr int DMAX = 128;      // largest head_dim served by the kernels
constexpr int GMAX = 128;      // largest group_size (one span per CTA)
constexpr int16_t RAW = -1;    // engine.py:35 RAW_MARKER

enum DType { F16 = 1, F32 = 2, F64 = 3, BF16 = 4 };

__host__ __device__ inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ---- input element conversion ------------------------------------------------
template <typename T> __device__ __forceinline__ double to_f64(T x);
template <> __device__ __forceinline__ double to_f64<__half>(__half x) { return (double)__half2float(x); }
template <> __device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 x) { return (double)__bfloat162float(x); }
template <> __device__ __forceinline__ double to_f64<float>(float x) { return (double)x; }
template <> __device__ __forceinline__ double to_f64<double>(double x) { return x; }

// ---- non-finite inputs (engine.py:132-139, :180-181) ----------------------------------
template <typename T> __device__ __forceinline__ bool is_finite_el(T x);
template <> __device__ __forceinline__ bool is_finite_el<__half>(__half x) { return (__half_as_ushort(x) & 0x7c00u) != 0x7c00u; }
template <> __device__ __forceinline__ bool is_finite_el<__nv_bfloat16>(__nv_bfloat16 x) {
  return (__bfloat16_as_ushort(x) & 0x7f80u) != 0x7f80u;
}
template <> __device__ __forceinline__ bool is_finite_el<float>(float x) { return isfinite(x); }
template <> __device__ __forceinline__ bool is_finite_el<double>(double x) { return isfinite(x); }
// key of a non-finite input element: the smallest key is the reference's first DataError
// location -- lowest unit, K before V (engine.py:151-152 checks K first), then token, then dim
// (np.argwhere row-major order).  ~0 = none.
__device__ __forceinline__ unsigned long long nf_key(int u, int side, int64_t token, int dim) {
  return ((unsigned long long)u << 44) | ((unsigned long long)side << 43) | ((unsigned long long)token << 8) |
         (unsigned long long)(dim & 255);
}

template <typename T> struct exact_in_f32 { static constexpr bool value = true; };
template <> struct exact_in_f32<double> { static constexpr bool value = false; };

// ---- 3-input min/max (SASS FMNMX3 on sm_100a) ----------------------------------
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}

// ---- warp reductions -----------------------------------------------------------
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// argmin with lowest index on ties (np.argmin semantics)
__device__ __forceinline__ void warp_argmin_d(double& v, int& i) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
  }
}
// argmax with lowest index on ties (np.argmax semantics)
__device__ __forceinline__ void warp_argmax_d(double& v, long long& i) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
  }
}

// ---- exact quantizer code (quant.py:99-111) --------------------------------------
// code = clip(floor(fl(fl(v - lo) / scale) + 0.5), 0, qmax) in IEEE fp64.
// Fast path: fp32 quotient; when frac(t) is within `guard` of an integer the
// exact fp64 sequence decides.  |t32 - (q + 1/2)| <= 3*2^-24*(qmax+1/2), and
// guard = 2^-20*(qmax+1) leaves a >5x margin ("exact codes").
struct QuantParamsDev {
  double lo, scale;
  float inv32, guard;
  int qmax;
};
__device__ __forceinline__ QuantParamsDev make_qparams(double lo, double hi, int qmax) {
  QuantParamsDev p;
  p.lo = lo;
  p.scale = __ddiv_rn(__dsub_rn(hi, lo), (double)qmax);
  p.inv32 = p.scale == 0.0 ? 0.f : (float)__drcp_rn(p.scale);
  p.guard = (float)(qmax + 1) * 9.5367431640625e-07f;  // 2^-20 * (qmax + 1)
  p.qmax = qmax;
  return p;
}
__device__ __forceinline__ int quant_code(double v, const QuantParamsDev& p, unsigned* n_exact) {
  if (p.scale == 0.0) return 0;
  double diff = __dsub_rn(v, p.lo);
  float t = __fmaf_rn((float)diff, p.inv32, 0.5f);
  float fl = floorf(t);
  float fr = t - fl;
  int c;
  if (fr > p.guard && fr < 1.f - p.guard) {
    c = (int)fl;
  } else {
    double q = __dadd_rn(__ddiv_rn(diff, p.scale), 0.5);
    c = (int)floor(q);
    if (n_exact) atomicAdd(n_exact, 1u);
  }
  return c < 0 ? 0 : (c > p.qmax ? p.qmax : c);
}

// ---- fragment layout ---------------------------------------------------------------
// Within a 16-token tile, 32 lanes x (Dp*bits/64) 32-bit words.  Lane l holds the
// 4*KT mma.m16n8k16 A-fragment registers R = 4j + reg of its sub-tiles j (K: k-tiles
// over channels; V: m-tiles over channels), reg = hiRow + 2*hiCol, each register a
// half2 of elements (row, col) = (g + 8*hiRow, 2q + 8*hiCol + e), g = l/4, q = l%4.
//   K tile (A = K, M = tokens, K-dim = channels):  token = row, channel = 16j + col
//   V tile (A = V^T, M = channels, K-dim = tokens): channel = 16j + row, token = col
// Register R lives in word `word` at half2 slot `slot` (code bits at
// (e ? 16 : 0) + slot*bits).  The slot depends only on the operand's CHANNEL
// index (K: (j, hiCol); V: (j, hiRow)), so the power-of-two factor left by the
// LOP3 magic-number dequant (1024 + 2^k code) is constant per channel and folds
// into B (K) or the output rows (V) instead of costing an HFMA2 per element.
struct FragPos { int j, row, col; };  // sub-tile, row in [0,16), col in [0,16)
__device__ __forceinline__ FragPos frag_rc(int lane, int R, int e) {
  int reg = R & 3;
  FragPos p;
  p.j = R >> 2;
  p.row = (lane >> 2) + 8 * (reg & 1);
  p.col = 2 * (lane & 3) + 8 * (reg >> 1) + e;
  return p;
}
__host__ __device__ __forceinline__ void frag_word_slot(int side, int R, int bits, int& word, int& slot) {
  const int j = R >> 2, reg = R & 3, hiRow = reg & 1, hiCol = reg >> 1, HS = 8 / bits;
  const int inner = side == 0 ? hiCol : hiRow, outer = side == 0 ? hiRow : hiCol;
  word = outer + 2 * (j / HS);
  slot = 2 * (j % HS) + inner;
}
// inverse: (word, slot) -> register R
__host__ __device__ __forceinline__ int frag_reg_of(int side, int word, int slot, int bits) {
  const int HS = 8 / bits;
  const int j = (word >> 1) * HS + (slot >> 1);
  const int inner = slot & 1, outer = word & 1;
  const int hiRow = side == 0 ? outer : inner, hiCol = side == 0 ? inner : outer;
  return 4 * j + hiRow + 2 * hiCol;
}
// bit shift k of the dequantized value 1024 + 2^k * code for a slot
__host__ __device__ constexpr int frag_slot_shift(int slot, int bits) { return (slot % (8 / bits)) * bits; }
// words per lane per tile, bytes per tile
__host__ __device__ inline int frag_words_per_lane(int Dp, int bits) { return Dp * bits / 64; }
__host__ __device__ inline int tile_bytes(int Dp, int bits) { return 16 * Dp * bits / 8; }

// ---- device view of a cache -------------------------------------------------------
struct DevCache {
  int U, D, Dp, bits, qmax, G, W, Wcap, ntile_blk, blk_bytes, in_dtype;
  int GP;                          // token slots per block (16 * ntile_blk)
  int64_t Tcap, NBcap;
  int Pcap;
  int use_kp, use_vp, use_vgate, use_kgate, gen_new, keep_diag;
  int prune;                      // K1 lower-bound pruned matcher (exact; 0 = brute force)
  double thr;
  // patterns
  double* kpat64; double* vpat64;
  float* kpat32; float* vpat32;
  float* kpmax; float* vpmax;     // max |m| over each unit's table (filter tolerance)
  int* probe;                     // [U][2][16] probe channels of the pruned matcher
  int* nk; int* nv;               // per-unit pattern counts
  // blocks
  int64_t* blk_start; int* blk_len;  // [NBcap] (lockstep across units)
  uint8_t* kcodes; float* kparam32; double* kparam64; int16_t* kidx;
  uint8_t* vcodes; float* vparam32; double* vparam64; int16_t* vidx;
  double* kdiag; double* vdiag;   // [U][Tcap][2] raw/flat ranges (optional)
  // window ring
  void* wk; void* wv;
  // stats
  unsigned* stats;                // [0] fp64 refines, [1] exact-division fallbacks
  int* work;                      // [4] work-queue counters of the K1-TC encoder (reset per launch);
                                  // work[2] counts deferred K code fix-ups
  unsigned long long* fix;        // [fixcap] deferred K code fix-ups of K1-TC (see kfix_kernel)
  int fixcap;
  unsigned long long* bad;        // smallest nf_key of a non-finite input seen since the last prefill
};

// Source rows for an encode launch: row r of the span that starts `off` rows
// after the launch's first span lives at base + u*unit_stride + ((row0+off+r) % ring)*D
template <typename T>
struct SpanSrc {
  const T* base;
  int64_t unit_stride;
  int64_t row0;
  int64_t ring;
};

// ---- launch argument blocks shared between the C ABI and the kernels ---------------
template <typename E>
struct MineArgs {
  const E* x[2];              // K and V inputs, [U][T][D]
  int64_t unit_stride;        // elements between units
  int64_t T;
  const int64_t* first[2];    // device [U] first seed index per side
  int k;
  int side_mask;              // bit0 K, bit1 V
  double* near_;              // scratch [U][2][T]
  double* own;
  int* lab;
  int* lab2;
  int* list;
  double* hist;               // [U][2][25]
  int* niter;                 // [U][2]
  int* labels_out;            // optional [U][2][T]
  int64_t tstride;            // points per unit-side in the scratch arrays (>= T; 16-byte rows)
};

struct AttnArgs {
  const float* q;      // [U][G][D] fp32
  int G;               // query heads per unit
  float scale_log2;    // sm_scale * log2(e)
  int blk0;            // first committed block attended (sequence split: a rank's block range)
  int nb;              // committed blocks attended, [blk0, blk0 + nb)
  int nchunk, bpc;     // chunks per unit, blocks per chunk
  float* part;         // [U][nchunk][G][Dp + 2]  (o[Dp], m, l)
  float* ml;           // partial mode: [U][G][2] (m in natural-log units, l); out = unnormalised o
};

// per-unit arena rows copied by a unit fork: unit s of src -> unit d of dst,
// `bytes` from src + s*src_stride to dst + d*dst_stride (same or different caches)
struct ForkArenas {
  struct Arena { const unsigned char* src; unsigned char* dst; int64_t src_stride, dst_stride, bytes; };
  Arena a[24];
  int n;
};

// ---- launchers ------------------------------------------------------------------------
template <typename T> cudaError_t launch_encode(const DevCache&, const SpanSrc<T>&, const SpanSrc<T>&, int, int, cudaStream_t);
template <typename T> cudaError_t launch_mine(const DevCache&, const MineArgs<T>&, cudaStream_t);
template <typename T> cudaError_t launch_finite(const T*, int64_t, unsigned long long*, cudaStream_t);
template <typename T> cudaError_t launch_window_put(const DevCache&, const T*, const T*, int64_t, int, int, int64_t, cudaStream_t);
template <typename T> cudaError_t launch_refresh(const DevCache&, int, int, int, cudaStream_t);
template <typename T> cudaError_t launch_attn(const DevCache&, const AttnArgs&, int, int, int, int, float*, cudaStream_t);
cudaError_t launch_dequant(const DevCache&, int, int64_t, int64_t, double*, double*, cudaStream_t);
cudaError_t launch_fork(const ForkArenas&, int, const int*, const int*, cudaStream_t);
cudaError_t launch_codes(const DevCache&, int, int64_t, int64_t, uint8_t*, uint8_t*, cudaStream_t);
cudaError_t launch_quantize_groups(const double*, const int64_t*, int, int, double*, double*, uint8_t*, cudaStream_t);
cudaError_t launch_pack(const uint8_t*, int64_t, int, uint8_t*, cudaStream_t);
cudaError_t launch_qpack(const double*, int64_t, int, double*, uint8_t*, cudaStream_t);
cudaError_t launch_dqunpack(const uint8_t*, int64_t, int, double, double, double*, cudaStream_t);
cudaError_t launch_unpack(const uint8_t*, int64_t, int, uint8_t*, cudaStream_t);
cudaError_t launch_match(const double*, int64_t, const double*, int, int, int64_t*, double*, double*, cudaStream_t);
cudaError_t launch_midrange(const double*, int64_t, int, double*, cudaStream_t);
size_t mine_smem_bytes(int k, int D, bool tc);
cudaError_t launch_probes(const DevCache&, cudaStream_t);
cudaError_t launch_install_patterns(const DevCache&, int, const double*, int, const int*, cudaStream_t);
cudaError_t launch_import(const DevCache& c, int nb, int64_t C, const double* kparam, const int32_t* kidx,
                          const int32_t* vidx, const double* vparam, const uint8_t* kcodes, const uint8_t* vcodes,
                          const double* kdiag, const double* vdiag, cudaStream_t st);
// K3-TC decode attention on tcgen05 kind::i8 (pkv_attn_tc.cu); cudaErrorNotSupported outside its
// envelope (the caller then runs the CUDA-core K3)
cudaError_t launch_attn_tc(const DevCache& c, const AttnArgs& a, int Pk_max, int Pv_max, cudaStream_t st);
// K1-TC persistent fp16 prefill encoder (pkv_encode_tc.cu); cudaErrorNotSupported outside its envelope
cudaError_t launch_encode_tc(const DevCache& c, int max_p, const __half* k, const __half* v, int64_t rows,
                             int64_t unit_stride, int first_block, int nblocks, cudaStream_t st);

}  // namespace pkv
