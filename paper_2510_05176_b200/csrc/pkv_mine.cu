// K2 mine_kmeans (v1, CUDA-core fp64): batched Lloyd k-means, one CTA per
// (unit, side).  Restates lloyd_kmeans / _farthest_point_seeds / mine_patterns
// (patterns.py:72-158) for every unit of a cache at once:
//   * distinct-rows shortcut (patterns.py:95-101) detected during seeding: if
//     the farthest remaining point is at distance 0 after n <= k seeds, the
//     data has exactly n distinct rows; they are returned in lexicographic
//     order (np.unique(axis=0)) with history [0.0];
//   * farthest-point seeding from a host-supplied first index
//     (np.random.default_rng(seed).integers(T), patterns.py:103,135), argmax
//     ties to the lowest index (patterns.py:137-141);
//   * <= 25 Lloyd rounds with once-per-round empty-cluster repair
//     (patterns.py:112-118), centers = means (patterns.py:119-120) summed
//     sequentially in point order exactly like numpy's axis-0 reduction, and
//     the rel-tol 1e-6 stop (patterns.py:121-125).
// Squared distances: v1 path = fp64 FMA chains on CUDA cores; tensor-core path
// (fp16 inputs, d = 128, k <= 64) = the T x k x d product on tcgen05: TMA streams
// 128-point tiles of X (fp16, exact) into 128B-swizzled smem, one thread issues
// tcgen05.mma kind::f16 against the centers split hi+lo into two fp16 columns,
// accumulating in TMEM; four epilogue warps read the accumulator with tcgen05.ld
// and take the argmin of ||c||^2 - 2 x.c, re-deciding in fp64 any point whose two
// best candidates lie within the error bound.  The objective and the centroid
// means stay fp64 on CUDA cores (O(T d) per round).  The reference's einsum order
// is CPU specific, so mining is "parity-unpinned at ulp level".
#include "pkv_common.cuh"
#include "pkv_sm100.cuh"

#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace pkv {

constexpr int MINE_THREADS = 256;
constexpr int KMAX = 96;
constexpr int KCH = 16;  // centers per register chunk

struct MineSmem {
  double* cen;    // [k][CST] (CST = D + 1: conflict-free per-thread row reads)
  int CST;
  // tensor-core assignment (TC path only)
  unsigned char* sA;  // [2 stages][2 K-halves][128 rows x 128 B], 1024-aligned, 128B swizzle
  unsigned char* sB;  // [2 K-halves][NP rows x 128 B]
  float* cc;          // [NP/2] ||c_j||^2 (+inf for padding)
  uint64_t* bars;     // full[2], empty[2], tfull[2], tempty[2]
  uint32_t* tmem;     // TMEM base address
  int* cnt;       // [KMAX]
  int* off;       // [KMAX]
  int* wcnt;      // [16][KMAX]
  double* redv;   // [32]
  long long* redi;// [32]
  int* chosen;    // [KMAX]
  int* flags;     // [4]
};

__device__ __forceinline__ void block_argmax(double v, long long i, MineSmem& sm, double& ov, long long& oi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmax_d(v, i);
  if (lane == 0) { sm.redv[warp] = v; sm.redi[warp] = i; }
  __syncthreads();
  if (warp == 0) {
    v = lane < MINE_THREADS / 32 ? sm.redv[lane] : -1.0 / 0.0;
    i = lane < MINE_THREADS / 32 ? sm.redi[lane] : 0x7fffffffffffffffLL;
    warp_argmax_d(v, i);
    if (lane == 0) { sm.redv[0] = v; sm.redi[0] = i; }
  }
  __syncthreads();
  ov = sm.redv[0];
  oi = sm.redi[0];
  __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, MineSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sm.redv[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < MINE_THREADS / 32 ? sm.redv[lane] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sm.redv[0] = v;
  }
  __syncthreads();
  double r = sm.redv[0];
  __syncthreads();
  return r;
}

// squared distance of a point row to the staged fp64 seed row (fp64, same
// operands as the reference's x - x_seed); fp16 rows at d = 128 load as 16
// independent 16-byte vectors so the whole row is in flight at once
template <typename T>
__device__ __forceinline__ double sqdist_seed(const T* a, const double* b, int D) {
  if constexpr (std::is_same<T, __half>::value) {
    if (D == 128) {
      uint4 v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __ldg(reinterpret_cast<const uint4*>(a) + i);
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const __half* h = reinterpret_cast<const __half*>(&v[i]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double d = __dsub_rn((double)__half2float(h[e]), b[8 * i + e]);
          s = fma(d, d, s);
        }
      }
      return s;
    }
  }
  double s = 0.0;
  for (int c = 0; c < D; ++c) {
    const double d = __dsub_rn(to_f64(a[c]), b[c]);
    s = fma(d, d, s);
  }
  return s;
}

template <typename T>
__device__ __forceinline__ double sqdist_row(const T* a, const T* b, int D) {
  double s = 0.0;
  for (int c = 0; c < D; ++c) {
    double d = __dsub_rn(to_f64(a[c]), to_f64(b[c]));
    s = fma(d, d, s);
  }
  return s;
}

// assignment pass: labels/own from the current centers; returns sum of
// d2[t][lab_old[t]] when lab_old != nullptr (the objective of the previous round)
template <typename T>
__device__ double assign_pass(const T* X, int64_t Tn, int D, int k, MineSmem& sm, const int* lab_old,
                              int* lab_new, double* own, bool count) {
  if (count) {
    for (int j = threadIdx.x; j < k; j += MINE_THREADS) sm.cnt[j] = 0;
    __syncthreads();
  }
  double obj = 0.0;
  for (int64_t t = threadIdx.x; t < Tn; t += MINE_THREADS) {
    const T* xr = X + t * D;
    const int lo = lab_old ? lab_old[t] : -1;
    double best = 1.0 / 0.0;
    int bi = 0;
    for (int j0 = 0; j0 < k; j0 += KCH) {
      double acc[KCH];
#pragma unroll
      for (int j = 0; j < KCH; ++j) acc[j] = 0.0;
      for (int c = 0; c < D; ++c) {
        const double xv = to_f64(xr[c]);
#pragma unroll
        for (int j = 0; j < KCH; ++j) {
          if (j0 + j < k) {
            double d = __dsub_rn(xv, sm.cen[(j0 + j) * sm.CST + c]);
            acc[j] = fma(d, d, acc[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < KCH; ++j) {
        if (j0 + j < k) {
          if (acc[j] < best) { best = acc[j]; bi = j0 + j; }
          if (j0 + j == lo) obj += acc[j];
        }
      }
    }
    lab_new[t] = bi;
    own[t] = best;
    if (count) atomicAdd(&sm.cnt[bi], 1);
  }
  __syncthreads();
  return obj;
}

// ---------------------------------------------------------------------------------
// tensor-core assignment pass (fp16 points, d = 128, k <= 64)
// ---------------------------------------------------------------------------------
constexpr int TC_TILE = 128;
constexpr int TC_EPI_WARP0 = 4;  // warps 4..7: epilogue, TMEM lane quarter = warp % 4

__host__ __device__ inline int tc_np(int k) { return ((2 * k + 15) / 16) * 16; }

__device__ __forceinline__ unsigned char* tc_sa(const MineSmem& sm, int stage, int half) {
  return sm.sA + (stage * 2 + half) * (TC_TILE * 128);
}

// fp64 squared distance of smem point row r (swizzled fp16 tile) to center j
__device__ __forceinline__ double tc_d2_exact(const MineSmem& sm, int stage, int row, int j) {
  double acc = 0.0;
  const double* cj = sm.cen + j * sm.CST;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const unsigned char* base = tc_sa(sm, stage, half) + row * 128;
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      const uint4 v = *reinterpret_cast<const uint4*>(base + ((ch ^ (row & 7)) << 4));
      const __half* hv = reinterpret_cast<const __half*>(&v);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double d = __dsub_rn((double)__half2float(hv[e]), cj[half * 64 + ch * 8 + e]);
        acc = fma(d, d, acc);
      }
    }
  }
  return acc;
}

// One assignment pass over the T points of this unit-side.  Returns this thread's
// share of sum_t d2(x_t, c[lab_old[t]]) (fp64) when lab_old != nullptr.
__device__ double assign_tc(int64_t Tn, int k, MineSmem& sm, const int* lab_old, int* lab_new, bool count,
                            const CUtensorMap* map, int64_t row_base, uint32_t& gtile) {
  using namespace sm100;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NP = tc_np(k);
  const int NT = (int)((Tn + TC_TILE - 1) / TC_TILE);
  uint64_t* full = sm.bars;
  uint64_t* empty = sm.bars + 2;
  uint64_t* tfull = sm.bars + 4;
  uint64_t* tempty = sm.bars + 6;
  if (count)
    for (int j = tid; j < k; j += MINE_THREADS) sm.cnt[j] = 0;
  // B operand: row 2j = hi(c_j), row 2j+1 = lo(c_j) = fp16(c_j - hi), K-major, 128B swizzle
  for (int i = tid; i < NP * 16; i += MINE_THREADS) {
    const int row = i >> 4, half = (i >> 3) & 1, chunk = i & 7;
    const int j = row >> 1, part = row & 1;
    __half hv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      __half h = __float2half(0.f);
      if (j < k) {
        const double cv = sm.cen[j * sm.CST + half * 64 + chunk * 8 + e];
        const __half hi = __double2half(cv);
        h = part == 0 ? hi : __double2half(cv - (double)__half2float(hi));
      }
      hv[e] = h;
    }
    *reinterpret_cast<uint4*>(sm.sB + half * NP * 128 + row * 128 + ((chunk ^ (row & 7)) << 4)) =
        *reinterpret_cast<const uint4*>(hv);
  }
  for (int j = tid; j < NP / 2; j += MINE_THREADS) {
    double a = 0.0;
    if (j < k)
      for (int c = 0; c < 128; ++c) a = fma(sm.cen[j * sm.CST + c], sm.cen[j * sm.CST + c], a);
    sm.cc[j] = j < k ? (float)a : __int_as_float(0x7f800000);
  }
  fence_proxy_async();
  __syncthreads();
  float ccmax = 0.f;
  for (int j = 0; j < k; ++j) ccmax = fmaxf(ccmax, sm.cc[j]);
  const float cnorm = sqrtf(ccmax);
  double obj = 0.0;

  if (warp == 0) {
    if (lane == 0) {
      for (int m = 0; m < NT; ++m) {
        const uint32_t g = gtile + m, s = g & 1, ph = (g >> 1) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], 2 * TC_TILE * 128);
        const int r0 = (int)(row_base + (int64_t)m * TC_TILE);
        tma_load_2d(tc_sa(sm, s, 0), map, &full[s], 0, r0);
        tma_load_2d(tc_sa(sm, s, 1), map, &full[s], 64, r0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_f16_f32(TC_TILE, NP);
      const uint64_t db0 = smem_desc_k_sw128(sm.sB), db1 = smem_desc_k_sw128(sm.sB + NP * 128);
      for (int m = 0; m < NT; ++m) {
        const uint32_t g = gtile + m, s = g & 1, ph = (g >> 1) & 1;
        const uint32_t acc = g & 1, aph = (g >> 1) & 1;
        mbar_wait(&full[s], ph);
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint64_t da0 = smem_desc_k_sw128(tc_sa(sm, s, 0)), da1 = smem_desc_k_sw128(tc_sa(sm, s, 1));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 8 x K=16 over d = 128 (two 64-wide swizzle halves)
          const uint64_t da = (kk < 4 ? da0 : da1) + 2 * (kk & 3);  // +32 B per K step
          const uint64_t db = (kk < 4 ? db0 : db1) + 2 * (kk & 3);
          mma_f16_ss(*sm.tmem + acc * 128, da, db, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= TC_EPI_WARP0 && warp < TC_EPI_WARP0 + 4) {
    const int q = warp & 3, row = 32 * q + lane;
    for (int m = 0; m < NT; ++m) {
      const uint32_t g = gtile + m, s = g & 1, acc = g & 1, aph = (g >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int64_t t = (int64_t)m * TC_TILE + row;
      float vb = __int_as_float(0x7f800000), vs = vb;
      int bi = 0;
      for (int c0 = 0; c0 < NP; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(*sm.tmem + acc * 128 + c0 + ((uint32_t)(32 * q) << 16), v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int j = c0 / 2 + e;
          if (j < k) {  // columns past N (last 32-column load) are not centers
            const float dot = __uint_as_float(v[2 * e]) + __uint_as_float(v[2 * e + 1]);
            const float val = fmaf(-2.f, dot, sm.cc[j]);
            if (val < vb) { vs = vb; vb = val; bi = j; }
            else vs = fminf(vs, val);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (t < Tn) {
        // |x|^2 for the error bound; fp64 objective against the previous labels
        float xx = 0.f;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const unsigned char* base = tc_sa(sm, s, half) + row * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint4 w = *reinterpret_cast<const uint4*>(base + ((ch ^ (row & 7)) << 4));
            const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(h2[e]);
              xx = fmaf(f.x, f.x, fmaf(f.y, f.y, xx));
            }
          }
        }
        if (lab_old) obj += tc_d2_exact(sm, s, row, lab_old[t]);
        // |err(||c||^2 - 2 x.c)| <= 2^-16 |x||c| + 2^-21 (|c|^2 + |x|^2): B split (2^-22),
        // tensor-core fp32 accumulation over 8 K-steps, fp32 roundings (K2)
        const float tol = 1.52587890625e-05f * sqrtf(xx) * cnorm + 4.76837158203125e-07f * (ccmax + xx);
        if (vs - vb <= 2.f * tol) {  // near tie: decide in fp64 (reference arithmetic, lowest index)
          double best = __longlong_as_double(0x7ff0000000000000LL);
          for (int j = 0; j < k; ++j) {
            const double d = tc_d2_exact(sm, s, row, j);
            if (d < best) { best = d; bi = j; }
          }
        }
        lab_new[t] = bi;
        if (count) atomicAdd(&sm.cnt[bi], 1);
      }
      mbar_arrive(&empty[s]);
    }
  }
  gtile += NT;
  __syncthreads();
  return obj;
}

template <typename T, bool TC>
__global__ void __launch_bounds__(MINE_THREADS, 1)
kmeans_kernel(DevCache c, MineArgs<T> a, const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV) {
  const int u = blockIdx.x, side = blockIdx.y;
  if (!((a.side_mask >> side) & 1)) return;
  const int D = c.D, k = a.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t Tn = a.T;
  const T* X = a.x[side] + (int64_t)u * a.unit_stride;
  const int64_t so = ((int64_t)u * 2 + side) * a.tstride;
  double* near_ = a.near_ + so;
  double* own = a.own + so;
  int* lab = a.lab + so;
  int* lab2 = a.lab2 + so;
  int* list = a.list + so;
  double* hist = a.hist + ((int64_t)u * 2 + side) * 25;
  double* p64 = (side == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * D;
  float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * c.Dp;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  MineSmem sm;
  sm.CST = D + 1;
  unsigned char* sbase = smem_raw;
  if (TC) {
    // 1024-aligned swizzled operand tiles first
    const uintptr_t p = reinterpret_cast<uintptr_t>(smem_raw);
    sbase = reinterpret_cast<unsigned char*>((p + 1023) & ~(uintptr_t)1023);
    sm.sA = sbase;
    sm.sB = sm.sA + 4 * TC_TILE * 128;
    sbase = sm.sB + 2 * tc_np(k) * 128;
  }
  sm.cen = reinterpret_cast<double*>(sbase);
  sm.redv = sm.cen + (size_t)k * sm.CST;
  sm.redi = reinterpret_cast<long long*>(sm.redv + 32);
  sm.cnt = reinterpret_cast<int*>(sm.redi + 32);
  sm.off = sm.cnt + KMAX;
  sm.wcnt = sm.off + KMAX;
  sm.chosen = sm.wcnt + 16 * KMAX;
  sm.flags = sm.chosen + KMAX;
  uint32_t gtile = 0;
  const CUtensorMap* tmap = side == 0 ? &tmK : &tmV;
  if (TC) {
    sm.bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uintptr_t>(sm.flags + 4 + 1) & ~(uintptr_t)7);
    sm.tmem = reinterpret_cast<uint32_t*>(sm.bars + 8);
    sm.cc = reinterpret_cast<float*>(sm.tmem + 4);
    if (tid == 0) {
      for (int i = 0; i < 2; ++i) {
        sm100::mbar_init(&sm.bars[i], 1);                       // full: producer arrive + tx
        sm100::mbar_init(&sm.bars[2 + i], 128);                 // empty: epilogue threads
        sm100::mbar_init(&sm.bars[4 + i], 1);                   // tmem full: MMA commit
        sm100::mbar_init(&sm.bars[6 + i], 128);                 // tmem empty: epilogue threads
      }
      sm100::fence_mbar_init();
      sm100::tma_prefetch(tmap);
    }
    if (warp == 1) sm100::tmem_alloc<256>(sm.tmem);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
  }

  // ---- seeding (patterns.py:134-142) with distinct-rows detection --------------
  const int64_t first = a.first[side][u];
  if (tid == 0) sm.chosen[0] = (int)first;
  double vmax; long long imax;
  {
    double bv = -1.0 / 0.0; long long bi = 0x7fffffffffffffffLL;
    for (int c2 = tid; c2 < D; c2 += MINE_THREADS) sm.cen[c2] = to_f64(X[first * D + c2]);  // seed row (cen is free here)
    __syncthreads();
    for (int64_t t = tid; t < Tn; t += MINE_THREADS) {
      double d = sqdist_seed(X + t * D, sm.cen, D);
      near_[t] = d;
      if (d > bv) { bv = d; bi = t; }
    }
    block_argmax(bv, bi, sm, vmax, imax);
  }
  int n = 1;
  bool shortcut = false;
  while (true) {
    if (vmax == 0.0) { shortcut = true; break; }
    if (n == k) break;
    if (tid == 0) sm.chosen[n] = (int)imax;
    ++n;
    for (int c2 = tid; c2 < D; c2 += MINE_THREADS) sm.cen[c2] = to_f64(X[imax * D + c2]);
    __syncthreads();
    double bv = -1.0 / 0.0; long long bi = 0x7fffffffffffffffLL;
    for (int64_t t = tid; t < Tn; t += MINE_THREADS) {
      double d = fmin(near_[t], sqdist_seed(X + t * D, sm.cen, D));
      near_[t] = d;
      if (d > bv) { bv = d; bi = t; }
    }
    block_argmax(bv, bi, sm, vmax, imax);
  }
  __syncthreads();

  int iters = 0;
  if (shortcut) {
    // np.unique(axis=0): the n distinct rows in lexicographic order
    for (int i = tid; i < n; i += MINE_THREADS) {
      const T* ri = X + (int64_t)sm.chosen[i] * D;
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const T* rj = X + (int64_t)sm.chosen[j] * D;
        for (int cc = 0; cc < D; ++cc) {
          double x1 = to_f64(rj[cc]), x2 = to_f64(ri[cc]);
          if (x1 < x2) { ++rank; break; }
          if (x1 > x2) break;
        }
      }
      for (int cc = 0; cc < D; ++cc) sm.cen[rank * sm.CST + cc] = to_f64(ri[cc]);
    }
    __syncthreads();
    assign_pass(X, Tn, D, n, sm, nullptr, lab, own, false);
    if (tid == 0) hist[0] = 0.0;
    iters = 1;
  } else {
    for (int i = tid; i < k * D; i += MINE_THREADS) {
      int j = i / D, cc = i - j * D;
      sm.cen[j * sm.CST + cc] = to_f64(X[(int64_t)sm.chosen[j] * D + cc]);
    }
    __syncthreads();
    if (TC) assign_tc(Tn, k, sm, nullptr, lab, true, tmap, (int64_t)u * Tn, gtile);
    else assign_pass(X, Tn, D, k, sm, nullptr, lab, own, true);
    bool own_valid = !TC;  // the TC pass computes labels only; own d2 is rebuilt on demand
    double prev = 1.0 / 0.0;
    for (int it = 0; it < 25; ++it) {
      // ---- empty-cluster repair (patterns.py:112-118) ----------------------------
      if (tid == 0) {
        int ne = 0;
        for (int j = 0; j < k; ++j) if (sm.cnt[j] == 0) sm.off[ne++] = j;
        sm.flags[0] = ne;
      }
      __syncthreads();
      const int ne = sm.flags[0];
      if (ne > 0 && !own_valid) {  // rare: exact fp64 d2 to the assigned centers
        for (int64_t t = tid; t < Tn; t += MINE_THREADS) {
          const T* xr = X + t * D;
          const double* cj = sm.cen + lab[t] * sm.CST;
          double acc = 0.0;
          for (int cc = 0; cc < D; ++cc) { const double d = __dsub_rn(to_f64(xr[cc]), cj[cc]); acc = fma(d, d, acc); }
          own[t] = acc;
        }
        __syncthreads();
      }
      for (int ei = 0; ei < ne; ++ei) {
        const int e = sm.off[ei];
        double bv = -1.0 / 0.0; long long bi = 0x7fffffffffffffffLL;
        for (int64_t t = tid; t < Tn; t += MINE_THREADS) {
          double v = sm.cnt[lab[t]] > 1 ? own[t] : -1.0;
          if (v > bv) { bv = v; bi = t; }
        }
        double fv; long long far_;
        block_argmax(bv, bi, sm, fv, far_);
        if (tid == 0) {
          sm.cnt[lab[far_]] -= 1;
          sm.cnt[e] += 1;
          lab[far_] = e;
          own[far_] = 0.0;
        }
        __syncthreads();
      }
      // ---- centers = sequential fp64 means (numpy axis-0 reduction order) -------
      // Points stream in index order, one thread per channel: every (cluster, channel) chain
      // receives its members' values in point order, exactly the additions of a per-cluster
      // walk; the running sum of the current label run stays in a register, and a chain's
      // first member is assigned (numpy starts the reduction from the first row, so a lone
      // -0.0 stays -0.0).  Coalesced row loads, no member lists.
      for (int c0 = 0; c0 < D; c0 += MINE_THREADS) {
        const int c = c0 + tid;
        const bool act = c < D;  // warp-uniform for D % 32 == 0; inactive lanes still shuffle
        uint32_t started[(KMAX + 31) / 32];
#pragma unroll
        for (int w = 0; w < (KMAX + 31) / 32; ++w) started[w] = 0u;
        int curj = -1;
        double racc = 0.0;
        // 16-point blocks: lane e holds the label of point tb + e (one coalesced load); the
        // next block's labels and values load while this block's additions run
        constexpr int PB = 16;
        int myl = lane < PB && lane < Tn ? lab[lane] : -1;
        T xv[PB];
#pragma unroll
        for (int e = 0; e < PB; ++e) xv[e] = (act && e < Tn) ? X[(int64_t)e * D + c] : T(0);
        for (int64_t tb = 0; tb < Tn; tb += PB) {
          const int64_t tn = tb + PB;
          const int nl = (lane < PB && tn + lane < Tn) ? lab[tn + lane] : -1;
          T nx[PB];
#pragma unroll
          for (int e = 0; e < PB; ++e) nx[e] = (act && tn + e < Tn) ? X[(tn + e) * D + c] : T(0);
#pragma unroll
          for (int e = 0; e < PB; ++e) {
            const int jt = __shfl_sync(0xffffffffu, myl, e);
            if (jt < 0) break;  // past Tn (uniform)
            const double x = to_f64(xv[e]);
            if (jt == curj) {
              racc = __dadd_rn(racc, x);
            } else {
              if (curj >= 0 && act) sm.cen[curj * sm.CST + c] = racc;
              const uint32_t bit = 1u << (jt & 31);
              racc = ((started[jt >> 5] & bit) && act) ? __dadd_rn(sm.cen[jt * sm.CST + c], x) : x;
              started[jt >> 5] |= bit;
              curj = jt;
            }
          }
          myl = nl;
#pragma unroll
          for (int e = 0; e < PB; ++e) xv[e] = nx[e];
        }
        if (act) {
          if (curj >= 0) sm.cen[curj * sm.CST + c] = racc;
          for (int jj = 0; jj < k; ++jj)
            if ((started[jj >> 5] >> (jj & 31)) & 1)
              sm.cen[jj * sm.CST + c] = __ddiv_rn(sm.cen[jj * sm.CST + c], (double)sm.cnt[jj]);
        }
      }
      __syncthreads();
      // The objective of this round (patterns.py:121) against the new means: any order
      // (compared at 1e-12); thread = (channel, quarter of the points), four partial sums.
      double part = 0.0;
      {
        constexpr int NQ = MINE_THREADS / 64;  // >= 1
        for (int w0 = tid; w0 < D * NQ; w0 += MINE_THREADS) {
          const int c = w0 % D, qq = w0 / D;
          const int64_t t0 = Tn * qq / NQ, t1 = Tn * (qq + 1) / NQ;
          double p4[4] = {0.0, 0.0, 0.0, 0.0};
          int64_t t = t0;
          for (; t + 4 <= t1; t += 4) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const double d = __dsub_rn(to_f64(X[(t + e) * D + c]), sm.cen[lab[t + e] * sm.CST + c]);
              p4[e] = fma(d, d, p4[e]);
            }
          }
          for (; t < t1; ++t) {
            const double d = __dsub_rn(to_f64(X[t * D + c]), sm.cen[lab[t] * sm.CST + c]);
            p4[0] = fma(d, d, p4[0]);
          }
          part += (p4[0] + p4[1]) + (p4[2] + p4[3]);
        }
      }
      __syncthreads();
      const double obj = block_sum(part, sm);
      if (tid == 0) hist[it] = obj;
      iters = it + 1;
      if (obj == 0.0 || (isfinite(prev) && prev - obj < 1e-6 * prev)) break;
      prev = obj;
      if (it + 1 == 25) break;  // keep the labels the final centers were built from
      // ---- next assignment --------------------------------------------------------------
      if (TC) {
        assign_tc(Tn, k, sm, nullptr, lab2, true, tmap, (int64_t)u * Tn, gtile);
        own_valid = false;
      } else {
        assign_pass(X, Tn, D, k, sm, nullptr, lab2, near_, true);
        own_valid = true;
        double* to = own; own = near_; near_ = to;
      }
      int* tl = lab; lab = lab2; lab2 = tl;
    }
    n = k;
  }
  // ---- write the pattern tables ---------------------------------------------------
  float amax = 0.f;
  for (int i = tid; i < n * D; i += MINE_THREADS) {
    const int j = i / D, cc = i - j * D;
    const double v = sm.cen[j * sm.CST + cc];
    p64[(int64_t)j * D + cc] = v;
    p32[(int64_t)j * c.Dp + cc] = (float)v;
    amax = fmaxf(amax, fabsf((float)v) * (1.f + 1e-6f));
  }
  for (int i = tid; i < n * (c.Dp - D); i += MINE_THREADS) {
    const int j = i / (c.Dp - D), cc = D + i % (c.Dp - D);
    p32[(int64_t)j * c.Dp + cc] = 0.f;
  }
  amax = warp_max_f(amax);
  if (lane == 0) sm.redv[warp] = amax;
  __syncthreads();
  if (tid == 0) {
    float m = 0.f;
    for (int w = 0; w < MINE_THREADS / 32; ++w) m = fmaxf(m, (float)sm.redv[w]);
    (side == 0 ? c.kpmax : c.vpmax)[u] = m;
    (side == 0 ? c.nk : c.nv)[u] = n;
    a.niter[u * 2 + side] = iters;
  }
  if (a.labels_out) {
    const int* fin = lab;
    for (int64_t t = tid; t < Tn; t += MINE_THREADS) a.labels_out[so + t] = fin[t];
  }
  if (TC) {
    __syncthreads();
    if (warp == 1) sm100::tmem_free<256>(*sm.tmem);
  }
}

// =================================================================================
// K2 v2: streamed k-means (fp16 points, d = 128, k <= 48), one CTA per unit-side.
// Every pass over the points is one TMA stream of 128-point tiles through a 3-stage
// smem ring, consumed by 4 row warps (thread per point) and 4 channel warps (thread
// per channel), so a Lloyd round costs ONE pass instead of three:
//   * labels of round r on tcgen05 (distance GEMM vs the centers split hi + lo, TMEM
//     accumulator, fp64 re-decision of near ties) -- as in the v1 kernel;
//   * the centroid sums of round r by the channel warps from the same tile;
//   * the objective (patterns.py:121: the new means against the labels that built them)
//     needs no pass: sum_t ||x_t||^2 (first seeding pass) minus per-cluster terms of the
//     exact sums, in double-double (sk_objective).
// The sums are exact in fp64 whenever T * max|x| < 2^29: fp16 values are multiples of
// 2^-24, so every partial sum of at most T of them is a multiple of 2^-24 below 2^53 *
// 2^-24 and every fp64 addition is exact -- the result is independent of the order and
// equals numpy's sequential axis-0 sum bit for bit (accumulators start at -0.0, so an
// all -0.0 column keeps its sign as numpy's first-row start does).  Otherwise (and after
// an empty-cluster repair) the sums are recomputed in numpy's point order (v1 code).
// Farthest-point seeding streams the same ring: fp64 distances to the newest seed from
// the smem tile, running minima in HBM, block argmax (lowest index on ties).
// The stop rule (patterns.py:123) is applied right after each round's means, as in the
// reference; a round whose sums are not the exact ones (repair, huge values) takes one
// objective pass (fp64 distances from the smem tile).
// =================================================================================
constexpr int SK_THREADS = 384;   // warp 0 TMA, 1 MMA, 2-3 idle, 4-7 rows, 8-11 channels
constexpr int SK_NS = 4;          // smem ring stages (even: split seeding gives each consumer group its own stages)
constexpr int SK_ROW0 = 4, SK_CH0 = 8;
constexpr int SK_KMAX = 32;

struct SkSmem {
  unsigned char* sA;   // [NS][2 halves][128 rows x 128 B] swizzled fp16 tiles
  unsigned char* sB;   // [2 halves][NP rows x 128 B]
  double* cen;         // [k][129]
  double* acc;         // [k][128] centroid sums
  double* seed;        // [128] newest seed row (fp64)
  float* seed32;       // [128] the same row in fp32 (exact: fp16 values)
  double* sNear;       // [NS][128] running seeding minima of the tile's points (bulk-loaded)
  int* sLab;           // [NS][128] previous labels of the tile's points (bulk-loaded)
  int* labs;           // [NS][128] labels of the tile's rows (row -> channel warps)
  float* cc;           // [NP/2]
  int* cnt;            // [k]
  int* off;            // [k]
  int* flags;          // [8]
  double* redv;        // [16]
  long long* redi;     // [16]
  uint64_t* bars;      // full[NS], empty[NS], lready[NS], tfull[2], tempty[2]
  uint32_t* tmem;
};
__host__ __device__ inline size_t sk_smem_bytes(int k) {
  const int NP = ((2 * k + 15) / 16) * 16;
  return 1024 + (size_t)SK_NS * 2 * 16384 + 2 * (size_t)NP * 128 + (size_t)k * 129 * 8 + (size_t)k * 128 * 8 + 128 * 12 +
         SK_NS * 128 * 12 +
         SK_NS * 128 * 4 + (size_t)NP / 2 * 4 + 2 * (size_t)k * 4 + 8 * 4 + 16 * 8 + 16 * 8 + (3 * SK_NS + 4) * 8 + 16 + 64 +
         14 * 16;  // 16-byte carve alignment
}
__device__ __forceinline__ unsigned char* sk_tile(const SkSmem& s, int stage, int half) {
  return s.sA + (stage * 2 + half) * 16384;
}
using sm100::smem_u32;
// explicit shared-space loads on 32-bit addresses (no generic->shared conversions in the
// hot loops); volatile keeps them ordered against the mbarrier waits
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ double ldsd(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float ldsf(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void stsd(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ unsigned short lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double h2d_bits(unsigned short h) {  // one F2F.F64.F16
  double r;
  asm("cvt.f64.f16 %0, %1;" : "=d"(r) : "h"(h));
  return r;
}
__device__ __forceinline__ double h2d(__half h) { return h2d_bits(__half_as_ushort(h)); }
// shared address of 16-byte chunk q (channels 8q .. 8q+7) of row `row` of a swizzled tile
__device__ __forceinline__ uint32_t sk_chunk(uint32_t tile_s, int row, int q) {
  return tile_s + (q >> 3) * 16384 + row * 128 + ((((q & 7) ^ (row & 7))) << 4);
}
// fp64 squared distance of tile row `row` to a fp64 row at cj_s, channel order, one fma
// chain (the v1 arithmetic)
__device__ __forceinline__ double sk_d2(uint32_t tile_s, int row, uint32_t cj_s) {
  double a0 = 0.0;
#pragma unroll 2
  for (int q = 0; q < 16; ++q) {
    const uint4 v = lds128(sk_chunk(tile_s, row, q));
    const __half* h = reinterpret_cast<const __half*>(&v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double d = __dsub_rn(h2d(h[e]), ldsd(cj_s + 8 * (8 * q + e)));
      a0 = fma(d, d, a0);
    }
  }
  return a0;
}
// the same distance with four independent accumulators (a 32-deep instead of a 128-deep
// dependency chain: seeding minima, the objective, near-tie candidates); |x|max on request
template <bool XMAX>
__device__ __forceinline__ double sk_d2x4(uint32_t tile_s, int row, uint32_t cj_s, float* xmax) {
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  float xm = 0.f;
#pragma unroll 4
  for (int q = 0; q < 16; ++q) {
    const uint4 v = lds128(sk_chunk(tile_s, row, q));
    const __half* h = reinterpret_cast<const __half*>(&v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (XMAX) xm = fmaxf(xm, fabsf(__half2float(h[e])));
      const double d = __dsub_rn(h2d(h[e]), ldsd(cj_s + 8 * (8 * q + e)));
      a[e & 3] = fma(d, d, a[e & 3]);
    }
  }
  if (XMAX) *xmax = fmaxf(*xmax, xm);
  return (a[0] + a[1]) + (a[2] + a[3]);
}
// fp32 squared distance of tile row `row` to the fp32 seed row, four partial sums:
// |d2_32 - d2| <= 2^-18 d2 (x and the seed are fp16 values, exact in fp32; one rounding
// per difference, <= 34 roundings per partial-sum chain), so d2_32 (1 - 2^-16) is a
// lower bound of the exact distance
__device__ __forceinline__ float sk_d2_f32(uint32_t tile_s, int row, uint32_t s32_s) {
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
  for (int q = 0; q < 16; ++q) {
    const uint4 v = lds128(sk_chunk(tile_s, row, q));
    const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
    const uint4 sa = lds128(s32_s + 32 * q), sb = lds128(s32_s + 32 * q + 16);
    const float sv[8] = {__uint_as_float(sa.x), __uint_as_float(sa.y), __uint_as_float(sa.z), __uint_as_float(sa.w),
                         __uint_as_float(sb.x), __uint_as_float(sb.y), __uint_as_float(sb.z), __uint_as_float(sb.w)};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // x - s straight from the packed fp16 (one FHADD each: exact conversion, one rounding)
      float d0, d1;
      asm("sub.rn.f32.f16 %0, %1, %2;" : "=f"(d0) : "h"((unsigned short)(vw[e] & 0xffffu)), "f"(sv[2 * e]));
      asm("sub.rn.f32.f16 %0, %1, %2;" : "=f"(d1) : "h"((unsigned short)(vw[e] >> 16)), "f"(sv[2 * e + 1]));
      a[e] = fmaf(d0, d0, a[e]);
      a[e] = fmaf(d1, d1, a[e]);
    }
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}

// ---- double-double arithmetic (error-free transforms) for the objective identity --------
struct DD { double h, l; };
__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
  return DD{s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ DD two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return DD{p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.h, b.h);
  const double e = __dadd_rn(s.l, __dadd_rn(a.l, b.l));
  const double h = __dadd_rn(s.h, e);
  return DD{h, __dsub_rn(e, __dsub_rn(h, s.h))};
}
// sum_c x_c^2 of tile row `row` in double-double (every x_c^2 of an fp16 value is exact in
// fp64, so the pair carries the row's squared norm to ~2^-104 relative)
__device__ __forceinline__ void sk_x2_row(uint32_t tile_s, int row, DD& acc) {
#pragma unroll 2
  for (int q = 0; q < 16; ++q) {
    const uint4 v = lds128(sk_chunk(tile_s, row, q));
    const __half* h = reinterpret_cast<const __half*>(&v);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const double x = h2d(h[e]);
      const DD t = two_sum(acc.h, __dmul_rn(x, x));
      acc.h = t.h;
      acc.l = __dadd_rn(acc.l, t.l);
    }
  }
}

struct SkCounters { uint32_t gt, gm, gl; };  // tiles streamed, MMA tiles, label hand-offs

enum { SK_SEED = 1, SK_ASSIGN = 2, SK_OBJ = 4, SK_SUMS = 8, SK_FIRST = 16, SK_SPLIT = 32 };

// Block reductions over the 8 consumer warps (rows 4-7 carry the values; others pass identity)
__device__ __forceinline__ double sk_block_sum(double v, const SkSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sm.redv[warp] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < SK_THREADS / 32; ++w) r += sm.redv[w];
  __syncthreads();
  return r;
}
__device__ __forceinline__ void sk_block_argmax(double v, long long i, const SkSmem& sm, double& ov, long long& oi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmax_d(v, i);
  if (lane == 0) { sm.redv[warp] = v; sm.redi[warp] = i; }
  __syncthreads();
  ov = -1.0 / 0.0;
  oi = 0x7fffffffffffffffLL;
  for (int w = 0; w < SK_THREADS / 32; ++w) {
    const double v2 = sm.redv[w];
    const long long i2 = sm.redi[w];
    if (v2 > ov || (v2 == ov && i2 < oi)) { ov = v2; oi = i2; }
  }
  __syncthreads();
}

// Double-double block sum (every thread contributes; all threads get the result)
__device__ __forceinline__ DD sk_block_sum_dd(DD v, const SkSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const DD w{__shfl_xor_sync(0xffffffffu, v.h, o), __shfl_xor_sync(0xffffffffu, v.l, o)};
    v = dd_add(v, w);
  }
  double* lo = reinterpret_cast<double*>(sm.redi);
  if (lane == 0) { sm.redv[warp] = v.h; lo[warp] = v.l; }
  __syncthreads();
  DD r{0.0, 0.0};
  for (int w = 0; w < SK_THREADS / 32; ++w) r = dd_add(r, DD{sm.redv[w], lo[w]});
  __syncthreads();
  return r;
}
// Objective of the labels the current centers were built from (patterns.py:121,
// sum_t ||x_t - c_l(t)||^2) without a pass over the points:
//   sum_t ||x_t - c_l(t)||^2 = sum_t ||x_t||^2 - sum_j sum_c (2 c_jc S_jc - n_j c_jc^2)
// with S_jc the cluster sums, exact in fp64 on the streamed path (kernel header), X2 =
// sum_t ||x_t||^2 from the first seeding pass and every product split exactly (two_prod),
// all in double-double: the only roundings are ~2^-104 of the terms, so the value is the
// exact objective to ~2^-102 X2 / obj relative before the final rounding (the reference's
// own einsum + pairwise sum rounds at ~1e-15).  Valid only when S holds the exact sums.
__device__ double sk_objective(const SkSmem& sm, int k, DD X2) {
  DD acc{0.0, 0.0};
  for (int i = threadIdx.x; i < k * 128; i += SK_THREADS) {
    const int j = i >> 7, cc = i & 127;
    const double cv = sm.cen[j * 129 + cc], S = sm.acc[i], n = (double)sm.cnt[j];
    const DD p = two_prod(cv, S);                 // c S
    const DD q = two_prod(cv, cv);                // c^2
    const DD r = two_prod(n, q.h);                // n c^2 (hi part)
    acc = dd_add(acc, DD{2.0 * p.h, 2.0 * p.l});  // x 2 is exact
    acc = dd_add(acc, DD{-r.h, -__fma_rn(n, q.l, r.l)});
  }
  const DD T = sk_block_sum_dd(acc, sm);
  const DD d = two_sum(X2.h, -T.h);
  return __dadd_rn(d.h, __dadd_rn(d.l, __dsub_rn(X2.l, T.l)));
}

// Split seeding: the row warps take the even tiles and the channel warps the odd ones.
// With an even stage count each group owns its stages, so no group ever skips a phase of
// a stage's mbarrier (a skipped phase would make the parity test ambiguous).
// Seeding update of one tile row: running minimum of the fp64 squared distances to the
// chosen seeds (exact fp64 only where the newest seed can lower it), argmax tracking.
__device__ __forceinline__ void sk_seed_row(const SkSmem& sm, uint32_t tile_s, int s, int row, int64_t t, int mode,
                                            double* near_, double& bv, long long& bi_out, float& xmax, DD& x2) {
  const uint32_t seed_s = smem_u32(sm.seed);
  double nv;
  if (mode & SK_FIRST) {
    nv = sk_d2x4<true>(tile_s, row, seed_s, &xmax);
    near_[t] = nv;
    sk_x2_row(tile_s, row, x2);
  } else {
    nv = sm.sNear[s * 128 + row];
    const float lb = sk_d2_f32(tile_s, row, smem_u32(sm.seed32)) * 0.9999847412109375f;  // (1 - 2^-16)
    if ((double)lb < nv) {
      const double d = sk_d2x4<false>(tile_s, row, seed_s, nullptr);
      if (d < nv) { nv = d; near_[t] = nv; }
    }
  }
  if (nv > bv) { bv = nv; bi_out = t; }
}

// One streamed pass.  Returns, on row threads, this thread's share of the objective
// (SK_OBJ) and its running argmax of the seeding minima (SK_SEED via bv/bi) and |x|max.
__device__ void sk_pass(int mode, int64_t Tn, int k, const SkSmem& sm, const CUtensorMap* map, int64_t row_base,
                        SkCounters& ctr, double* near_, const int* lab_old, int* lab_new, double& obj, double& bv,
                        long long& bi_out, float& xmax, DD& x2) {
  using namespace sm100;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = (int)((Tn + 127) / 128);
  const int NP = ((2 * k + 15) / 16) * 16;
  uint64_t* full = sm.bars;
  uint64_t* empty = sm.bars + SK_NS;
  uint64_t* lready = sm.bars + 2 * SK_NS;
  uint64_t* tfull = sm.bars + 3 * SK_NS;
  uint64_t* tempty = sm.bars + 3 * SK_NS + 2;
  const bool assign = mode & SK_ASSIGN, sums = mode & SK_SUMS;
  if (assign) {
    for (int j = tid; j < k; j += SK_THREADS) sm.cnt[j] = 0;
    // B operand: row 2j = hi(c_j), row 2j+1 = lo(c_j) = fp16(c_j - hi), K-major, 128B swizzle
    for (int i = tid; i < NP * 16; i += SK_THREADS) {
      const int row = i >> 4, half = (i >> 3) & 1, chunk = i & 7;
      const int j = row >> 1, part = row & 1;
      __half hv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        __half h = __float2half(0.f);
        if (j < k) {
          const double cv = sm.cen[j * 129 + half * 64 + chunk * 8 + e];
          const __half hi = __double2half(cv);
          h = part == 0 ? hi : __double2half(cv - (double)__half2float(hi));
        }
        hv[e] = h;
      }
      *reinterpret_cast<uint4*>(sm.sB + half * NP * 128 + row * 128 + ((chunk ^ (row & 7)) << 4)) =
          *reinterpret_cast<const uint4*>(hv);
    }
    for (int j = tid; j < NP / 2; j += SK_THREADS) {
      double a = 0.0;
      if (j < k)
        for (int c = 0; c < 128; ++c) a = fma(sm.cen[j * 129 + c], sm.cen[j * 129 + c], a);
      sm.cc[j] = j < k ? (float)a : __int_as_float(0x7f800000);
    }
  }
  if (sums)
    for (int i = tid; i < k * 128; i += SK_THREADS) sm.acc[i] = -0.0;
  fence_proxy_async();
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      const bool ld_near = (mode & SK_SEED) && !(mode & SK_FIRST), ld_lab = mode & SK_OBJ;
      for (int m = 0; m < NT; ++m) {
        const uint32_t g = ctr.gt + m, s = g % SK_NS, ph = (g / SK_NS) & 1;
        const int rows = (int)min((int64_t)128, Tn - (int64_t)m * 128);
        const uint32_t nb_near = ld_near ? (uint32_t)((rows * 8 + 15) & ~15) : 0u;
        const uint32_t nb_lab = ld_lab ? (uint32_t)((rows * 4 + 15) & ~15) : 0u;
        mbar_wait_sleep(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], 2 * 16384 + nb_near + nb_lab);
        const int r0 = (int)(row_base + (int64_t)m * 128);
        tma_load_2d(sk_tile(sm, s, 0), map, &full[s], 0, r0);
        tma_load_2d(sk_tile(sm, s, 1), map, &full[s], 64, r0);
        // per-point state rides with the tile (no global load on the consumers' path)
        if (nb_near) bulk_load(sm.sNear + s * 128, near_ + (int64_t)m * 128, nb_near, &full[s]);
        if (nb_lab) bulk_load(sm.sLab + s * 128, lab_old + (int64_t)m * 128, nb_lab, &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (assign && lane == 0) {
      const uint32_t idesc = idesc_f16_f32(128, NP);
      const uint64_t db0 = smem_desc_k_sw128(sm.sB), db1 = smem_desc_k_sw128(sm.sB + NP * 128);
      for (int m = 0; m < NT; ++m) {
        const uint32_t g = ctr.gt + m, s = g % SK_NS, ph = (g / SK_NS) & 1;
        const uint32_t gm = ctr.gm + m, acc = gm & 1, aph = (gm >> 1) & 1;
        mbar_wait_sleep(&full[s], ph);
        mbar_wait_sleep(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint64_t da0 = smem_desc_k_sw128(sk_tile(sm, s, 0)), da1 = smem_desc_k_sw128(sk_tile(sm, s, 1));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t da = (kk < 4 ? da0 : da1) + 2 * (kk & 3);
          const uint64_t db = (kk < 4 ? db0 : db1) + 2 * (kk & 3);
          mma_f16_ss(*sm.tmem + acc * 128, da, db, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= SK_ROW0 && warp < SK_ROW0 + 4) {
    const int q = warp & 3, row = 32 * q + lane;
    float ccmax = 0.f;
    if (assign)
      for (int j = 0; j < k; ++j) ccmax = fmaxf(ccmax, sm.cc[j]);
    const float cnorm = sqrtf(ccmax);
    const uint32_t cc_s = smem_u32(sm.cc);
    const bool seedp = mode & SK_SEED, split = seedp && (mode & SK_SPLIT);
    for (int m = 0; m < NT; m += split ? 2 : 1) {  // split seeding: even tiles (channel warps: odd)
      const uint32_t g = ctr.gt + m, s = g % SK_NS, ph = (g / SK_NS) & 1;
      const int64_t t = (int64_t)m * 128 + row;
      const bool live = t < Tn;
      const unsigned char* tile = sk_tile(sm, s, 0);
      const uint32_t tile_s = smem_u32(tile);
      int bi = 0;
      float vb = __int_as_float(0x7f800000), vs = vb;
      mbar_wait_sleep(&full[s], ph);
      if (assign) {
        const uint32_t gm = ctr.gm + m, acc = gm & 1, aph = (gm >> 1) & 1;
        const uint32_t tbase = *sm.tmem + acc * 128 + ((uint32_t)(32 * q) << 16);
        // |x|^2 for the error bound (the tile has landed: the MMA consumed it)
        float xq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint4 w = lds128(sk_chunk(tile_s, row, 8 * half + ch));
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // x^2 + acc straight from fp16 (FHFMA, no conversion)
              asm("fma.rn.f32.f16 %0, %1, %1, %0;" : "+f"(xq[e]) : "h"((unsigned short)(ww[e] >> 16)));
              asm("fma.rn.f32.f16 %0, %1, %1, %0;" : "+f"(xq[e]) : "h"((unsigned short)(ww[e] & 0xffffu)));
            }
          }
        }
        const float xx = (xq[0] + xq[1]) + (xq[2] + xq[3]);
        // same error bound as the v1 tensor-core pass (K2)
        const float tol = 1.52587890625e-05f * sqrtf(xx) * cnorm + 4.76837158203125e-07f * (ccmax + xx);
        mbar_wait_sleep(&tfull[acc], aph);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < NP; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(tbase + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = c0 / 2 + e;
            if (j < k) {
              const float dot = __uint_as_float(v[2 * e]) + __uint_as_float(v[2 * e + 1]);
              const float val = fmaf(-2.f, dot, ldsf(cc_s + 4 * j));
              if (val < vb) { vs = vb; vb = val; bi = j; }
              else vs = fminf(vs, val);
            }
          }
        }
        // near tie: fp64 over the candidates inside the error window only (every other center
        // is provably farther), lowest index among equal fp64 distances
        const bool tie = live && vs - vb <= 2.f * tol;
        if (__any_sync(0xffffffffu, tie)) {
          const float lim = vb + 2.f * tol;
          double best = __longlong_as_double(0x7ff0000000000000LL);
          int bj = bi;
#pragma unroll 1
          for (int c0 = 0; c0 < NP; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tbase + c0, v);  // warp-collective reload
            tmem_ld_wait();
            uint32_t cand = 0u;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int j = c0 / 2 + e;
              if (j < k && fmaf(-2.f, __uint_as_float(v[2 * e]) + __uint_as_float(v[2 * e + 1]), ldsf(cc_s + 4 * j)) <= lim)
                cand |= 1u << e;
            }
            if (!tie) cand = 0u;
            while (cand) {
              const int j = c0 / 2 + __ffs(cand) - 1;
              cand &= cand - 1;
              const double d = sk_d2x4<false>(tile_s, row, smem_u32(sm.cen + j * 129), nullptr);
              if (d < best) { best = d; bj = j; }
            }
          }
          bi = bj;
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      }
      if (live) {
        if (seedp) sk_seed_row(sm, tile_s, s, row, t, mode, near_, bv, bi_out, xmax, x2);
        if (assign) {
          lab_new[t] = bi;
          atomicAdd(&sm.cnt[bi], 1);
        }
        if (mode & SK_OBJ) obj += sk_d2x4<false>(tile_s, row, smem_u32(sm.cen + sm.sLab[s * 128 + row] * 129), nullptr);
      }

      if (sums) {  // label hand-off slot/barrier follow their own counter (gl), not the tile stage
        const uint32_t ls = (ctr.gl + m) % SK_NS;
        sm.labs[ls * 128 + row] = live ? bi : -1;
        mbar_arrive(&lready[ls]);
      }
      if (split) mbar_arrive_cnt(&empty[s], 2);  // this group alone consumed the tile
      else mbar_arrive(&empty[s]);
    }
  } else if (warp >= SK_CH0 && warp < SK_CH0 + 4) {
    const int c = tid - 32 * SK_CH0;  // channel
    const int hoff = (c >> 6) * 16384 + ((c & 7) << 1), cb = (c & 63) >> 3;
    for (int m = 0; m < NT; ++m) {
      const uint32_t g = ctr.gt + m, s = g % SK_NS, ph = (g / SK_NS) & 1;
      if (sums) {
        const uint32_t gl = ctr.gl + m, ls = gl % SK_NS, lph = (gl / SK_NS) & 1;
        mbar_wait_sleep(&lready[ls], lph);
        const uint32_t tile_s = smem_u32(sk_tile(sm, s, 0)) + hoff;
        const uint32_t lb_s = smem_u32(sm.labs + ls * 128);
        const uint32_t acc_s = smem_u32(sm.acc + c);
        // rows in blocks of 8: labels and values load up front; the current label's run is
        // summed in two interleaved registers (exact sums: any order) and flushed on a change
        int curj = -1;
        double run0 = -0.0, run1 = -0.0;
        for (int r0 = 0; r0 < 128; r0 += 8) {
          const uint4 la = lds128(lb_s + 4 * r0);
          const uint4 lb4 = lds128(lb_s + 4 * r0 + 16);
          const int js[8] = {(int)la.x, (int)la.y, (int)la.z, (int)la.w, (int)lb4.x, (int)lb4.y, (int)lb4.z, (int)lb4.w};
          double xs[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int r = r0 + e;
            xs[e] = h2d_bits(lds16(tile_s + r * 128 + ((cb ^ (r & 7)) << 4)));
          }
          bool same = curj >= 0;
#pragma unroll
          for (int e = 0; e < 8; ++e) same &= js[e] == curj;
          if (same) {  // the whole block continues the current run (uniform over the warp)
            run0 = __dadd_rn(run0, __dadd_rn(__dadd_rn(xs[0], xs[1]), __dadd_rn(xs[2], xs[3])));
            run1 = __dadd_rn(run1, __dadd_rn(__dadd_rn(xs[4], xs[5]), __dadd_rn(xs[6], xs[7])));
            continue;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = js[e];
            if (j < 0) continue;  // past Tn
            if (j != curj) {
              if (curj >= 0) stsd(acc_s + curj * 1024, __dadd_rn(ldsd(acc_s + curj * 1024), __dadd_rn(run0, run1)));
              curj = j;
              run0 = xs[e];
              run1 = -0.0;
            } else if (e & 1) {
              run1 = __dadd_rn(run1, xs[e]);
            } else {
              run0 = __dadd_rn(run0, xs[e]);
            }
          }
        }
        if (curj >= 0) stsd(acc_s + curj * 1024, __dadd_rn(ldsd(acc_s + curj * 1024), __dadd_rn(run0, run1)));
      } else if ((mode & SK_SEED) && (mode & SK_SPLIT)) {  // seeding: the odd tiles (row warps: even)
        if (m & 1) {
          mbar_wait_sleep(&full[s], ph);
          const int64_t t = (int64_t)m * 128 + c;
          if (t < Tn) sk_seed_row(sm, smem_u32(sk_tile(sm, s, 0)), s, c, t, mode, near_, bv, bi_out, xmax, x2);
          mbar_arrive_cnt(&empty[s], 2);
        }
        continue;
      } else {
        mbar_wait_sleep(&full[s], ph);
      }
      mbar_arrive(&empty[s]);
    }
  }
  ctr.gt += NT;
  if (assign) ctr.gm += NT;
  if (sums) ctr.gl += NT;
  fence_proxy_async_global();  // near_/labels written here are bulk-read (async proxy) next pass
  __syncthreads();
}

// centroid sums in numpy's point order straight from HBM (v1 order; any data)
__device__ void sk_seq_sums(const __half* X, int64_t Tn, int k, const int* lab, const SkSmem& sm) {
  const int tid = threadIdx.x;
  if (tid < 128) {
    const int c = tid;
    for (int j = 0; j < k; ++j) sm.acc[j * 128 + c] = 0.0;
    uint64_t started = 0ull;  // k <= 48
    int curj = -1;
    double racc = 0.0;
    for (int64_t t = 0; t < Tn; ++t) {
      const int jt = lab[t];
      const double x = (double)__half2float(X[t * 128 + c]);
      if (jt == curj) {
        racc = __dadd_rn(racc, x);
      } else {
        if (curj >= 0) sm.acc[curj * 128 + c] = racc;
        racc = ((started >> jt) & 1ull) ? __dadd_rn(sm.acc[jt * 128 + c], x) : x;
        started |= 1ull << jt;
        curj = jt;
      }
    }
    if (curj >= 0) sm.acc[curj * 128 + c] = racc;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(SK_THREADS, 1)
kmeans_stream_kernel(DevCache c, MineArgs<__half> a, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, int side0, int nsides) {
  using namespace sm100;
  // K sides first (they run ~25 rounds, V ~2): longest-first over the waves
  const int side = side0 + (int)blockIdx.x / c.U, u = (int)blockIdx.x % c.U;
  (void)nsides;
  const int k = a.k, tid = threadIdx.x, warp = tid >> 5;
  const int64_t Tn = a.T;
  const __half* X = a.x[side] + (int64_t)u * a.unit_stride;
  const int64_t so = ((int64_t)u * 2 + side) * a.tstride;
  double* near_ = a.near_ + so;
  double* own = a.own + so;
  int* lab = a.lab + so;
  double* hist = a.hist + ((int64_t)u * 2 + side) * 25;
  double* p64 = (side == 0 ? c.kpat64 : c.vpat64) + (int64_t)u * c.Pcap * 128;
  float* p32 = (side == 0 ? c.kpat32 : c.vpat32) + (int64_t)u * c.Pcap * c.Dp;
  const CUtensorMap* map = side == 0 ? &tmK : &tmV;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  SkSmem sm;
  {
    const int NP = ((2 * k + 15) / 16) * 16;
    // 1024-aligned base as pointer arithmetic on the shared array (keeps the address space
    // visible to the compiler: plain LDS/STS, and the SK_SMEM assumptions hold)
    unsigned char* p = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    auto carve = [&](size_t bytes) { unsigned char* q = p; p += (bytes + 15) & ~(size_t)15; return q; };
    sm.sA = carve(SK_NS * 2 * 16384);
    sm.sB = carve(2 * NP * 128);
    sm.cen = reinterpret_cast<double*>(carve((size_t)k * 129 * 8));
    sm.acc = reinterpret_cast<double*>(carve((size_t)k * 128 * 8));
    sm.seed = reinterpret_cast<double*>(carve(128 * 8));
    sm.seed32 = reinterpret_cast<float*>(carve(128 * 4));
    sm.sNear = reinterpret_cast<double*>(carve(SK_NS * 128 * 8));
    sm.sLab = reinterpret_cast<int*>(carve(SK_NS * 128 * 4));
    sm.redv = reinterpret_cast<double*>(carve(16 * 8));
    sm.redi = reinterpret_cast<long long*>(carve(16 * 8));
    sm.bars = reinterpret_cast<uint64_t*>(carve((3 * SK_NS + 4) * 8));
    sm.labs = reinterpret_cast<int*>(carve(SK_NS * 128 * 4));
    sm.cc = reinterpret_cast<float*>(carve(NP / 2 * 4));
    sm.cnt = reinterpret_cast<int*>(carve(k * 4));
    sm.off = reinterpret_cast<int*>(carve(k * 4));
    sm.flags = reinterpret_cast<int*>(carve(8 * 4));
    sm.tmem = reinterpret_cast<uint32_t*>(p);
  }
  if (tid == 0) {
    for (int i = 0; i < SK_NS; ++i) {
      mbar_init(&sm.bars[i], 1);                 // full: producer arrive + tx
      mbar_init(&sm.bars[SK_NS + i], 256);       // empty: row + channel threads
      mbar_init(&sm.bars[2 * SK_NS + i], 128);   // lready: row threads
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.bars[3 * SK_NS + i], 1);     // tmem full: MMA commit
      mbar_init(&sm.bars[3 * SK_NS + 2 + i], 128);  // tmem empty: row threads
    }
    fence_mbar_init();
    tma_prefetch(map);
  }
  if (warp == 1) tmem_alloc<256>(sm.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  SkCounters ctr{0u, 0u, 0u};
  const int64_t row_base = (int64_t)u * Tn;
  double objp = 0.0, bv = -1.0 / 0.0;
  long long bi = 0x7fffffffffffffffLL;
  float xmax = 0.f;
  DD x2sum{0.0, 0.0};  // this thread's share of sum_t ||x_t||^2 (first seeding pass)

  // ---- seeding (patterns.py:134-142) with distinct-rows detection -------------------
  const int64_t first = a.first[side][u];
  int* chosen = sm.off;  // seed indices (k)
  if (tid == 0) chosen[0] = (int)first;
  for (int c2 = tid; c2 < 128; c2 += SK_THREADS) {
    sm.seed32[c2] = __half2float(X[first * 128 + c2]);
    sm.seed[c2] = (double)sm.seed32[c2];
  }
  __syncthreads();
  const int split = (a.side_mask & 4) ? 0 : SK_SPLIT;  // bit 2: debugging switch (one consumer group)
  sk_pass(SK_SEED | SK_FIRST | split, Tn, k, sm, map, row_base, ctr, near_, nullptr, nullptr, objp, bv, bi, xmax, x2sum);
  const DD X2 = sk_block_sum_dd(x2sum, sm);
  double vmax;
  long long imax;
  sk_block_argmax(bv, bi, sm, vmax, imax);
  // exact-sum condition: T * max|x| < 2^29 (see the header)
  {
    float xm = warp_max_f(xmax);
    if ((tid & 31) == 0) sm.redv[warp] = xm;
    __syncthreads();
    float m = 0.f;
    for (int w = 0; w < SK_THREADS / 32; ++w) m = fmaxf(m, (float)sm.redv[w]);
    __syncthreads();
    xmax = m;
  }
  const bool exact_sums = (double)xmax * (double)Tn < 536870912.0;
  int n = 1;
  bool shortcut = false;
  while (true) {
    if (vmax == 0.0) { shortcut = true; break; }
    if (n == k) break;
    if (tid == 0) chosen[n] = (int)imax;
    ++n;
    for (int c2 = tid; c2 < 128; c2 += SK_THREADS) {
      sm.seed32[c2] = __half2float(X[imax * 128 + c2]);
      sm.seed[c2] = (double)sm.seed32[c2];
    }
    __syncthreads();
    bv = -1.0 / 0.0;
    bi = 0x7fffffffffffffffLL;
    sk_pass(SK_SEED | split, Tn, k, sm, map, row_base, ctr, near_, nullptr, nullptr, objp, bv, bi, xmax, x2sum);
    sk_block_argmax(bv, bi, sm, vmax, imax);
  }

  int iters = 0;
  int* fin = lab;
  if (shortcut) {
    // np.unique(axis=0): the n distinct rows in lexicographic order, labels = nearest
    for (int i = tid; i < n; i += SK_THREADS) {
      const __half* ri = X + (int64_t)chosen[i] * 128;
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const __half* rj = X + (int64_t)chosen[j] * 128;
        for (int cc = 0; cc < 128; ++cc) {
          const float x1 = __half2float(rj[cc]), x2 = __half2float(ri[cc]);
          if (x1 < x2) { ++rank; break; }
          if (x1 > x2) break;
        }
      }
      for (int cc = 0; cc < 128; ++cc) sm.cen[rank * 129 + cc] = (double)__half2float(ri[cc]);
    }
    __syncthreads();
    for (int64_t t = tid; t < Tn; t += SK_THREADS) {
      double best = 1.0 / 0.0;
      int b = 0;
      for (int j = 0; j < n; ++j) {
        double s2 = 0.0;
        for (int cc = 0; cc < 128; ++cc) {
          const double d = __dsub_rn((double)__half2float(X[t * 128 + cc]), sm.cen[j * 129 + cc]);
          s2 = fma(d, d, s2);
        }
        if (s2 < best) { best = s2; b = j; }
      }
      lab[t] = b;
    }
    if (tid == 0) hist[0] = 0.0;
    iters = 1;
  } else {
    for (int i = tid; i < k * 128; i += SK_THREADS) {
      const int j = i >> 7, cc = i & 127;
      sm.cen[j * 129 + cc] = (double)__half2float(X[(int64_t)chosen[j] * 128 + cc]);
    }
    __syncthreads();
    int* lcur = lab;  // labels of the newest assignment (the centers are built from them)
    double prev = 1.0 / 0.0;
    for (int r = 0; r < 25; ++r) {  // KMEANS_MAX_ITERS rounds (patterns.py:107-124)
      sk_pass(SK_ASSIGN | (exact_sums ? SK_SUMS : 0), Tn, k, sm, map, row_base, ctr, nullptr, nullptr, lcur, objp, bv,
              bi, xmax, x2sum);
      // ---- empty-cluster repair of the new labels (patterns.py:112-118) -----------------
      if (tid == 0) {
        int ne = 0;
        for (int j = 0; j < k; ++j) if (sm.cnt[j] == 0) sm.flags[1 + ne++] = j;
        sm.flags[0] = ne;
      }
      __syncthreads();
      const int ne = sm.flags[0];
      bool seq = !exact_sums;
      if (ne > 0) {
        seq = true;
        for (int64_t t = tid; t < Tn; t += SK_THREADS) {  // exact d2 to the assigned centers
          const double* cj = sm.cen + lcur[t] * 129;
          double s2 = 0.0;
          for (int cc = 0; cc < 128; ++cc) {
            const double d = __dsub_rn((double)__half2float(X[t * 128 + cc]), cj[cc]);
            s2 = fma(d, d, s2);
          }
          own[t] = s2;
        }
        __syncthreads();
        for (int ei = 0; ei < ne; ++ei) {
          const int e = sm.flags[1 + ei];
          double b2 = -1.0 / 0.0;
          long long i2 = 0x7fffffffffffffffLL;
          for (int64_t t = tid; t < Tn; t += SK_THREADS) {
            const double v = sm.cnt[lcur[t]] > 1 ? own[t] : -1.0;
            if (v > b2) { b2 = v; i2 = t; }
          }
          double fv;
          long long far_;
          sk_block_argmax(b2, i2, sm, fv, far_);
          if (tid == 0) {
            sm.cnt[lcur[far_]] -= 1;
            sm.cnt[e] += 1;
            lcur[far_] = e;
            own[far_] = 0.0;
            sm100::fence_proxy_async_global();  // lcur is bulk-read (async proxy) by the next pass
          }
          __syncthreads();
        }
      }
      if (seq) sk_seq_sums(X, Tn, k, lcur, sm);
      // ---- centers = means (patterns.py:119-120) ---------------------------------------
      for (int i = tid; i < k * 128; i += SK_THREADS) {
        const int j = i >> 7, cc = i & 127;
        sm.cen[j * 129 + cc] = __ddiv_rn(sm.acc[i], (double)sm.cnt[j]);
      }
      __syncthreads();
      // ---- objective and stop rule (patterns.py:121-124) ---------------------------------
      // exact sums: the double-double identity, no pass; otherwise (repair, huge values) an
      // objective pass over the points (fp64 distance to the assigned center)
      double obj;
      if (!seq) {
        obj = sk_objective(sm, k, X2);
      } else {
        objp = 0.0;
        sk_pass(SK_OBJ, Tn, k, sm, map, row_base, ctr, nullptr, lcur, nullptr, objp, bv, bi, xmax, x2sum);
        obj = sk_block_sum(objp, sm);
      }
      if (tid == 0) hist[r] = obj;
      iters = r + 1;
      if (obj == 0.0 || (isfinite(prev) && prev - obj < 1e-6 * prev)) break;
      prev = obj;
    }
    fin = lcur;
    n = k;
  }
  // ---- write the pattern tables -------------------------------------------------------
  float amax = 0.f;
  for (int i = tid; i < n * 128; i += SK_THREADS) {
    const int j = i >> 7, cc = i & 127;
    const double v = sm.cen[j * 129 + cc];
    p64[(int64_t)j * 128 + cc] = v;
    p32[(int64_t)j * c.Dp + cc] = (float)v;
    amax = fmaxf(amax, fabsf((float)v) * (1.f + 1e-6f));
  }
  for (int i = tid; i < n * (c.Dp - 128); i += SK_THREADS) {
    const int j = i / (c.Dp - 128), cc = 128 + i % (c.Dp - 128);
    p32[(int64_t)j * c.Dp + cc] = 0.f;
  }
  amax = warp_max_f(amax);
  if ((tid & 31) == 0) sm.redv[warp] = amax;
  __syncthreads();
  if (tid == 0) {
    float m = 0.f;
    for (int w = 0; w < SK_THREADS / 32; ++w) m = fmaxf(m, (float)sm.redv[w]);
    (side == 0 ? c.kpmax : c.vpmax)[u] = m;
    (side == 0 ? c.nk : c.nv)[u] = n;
    a.niter[u * 2 + side] = iters;
  }
  if (a.labels_out)
    for (int64_t t = tid; t < Tn; t += SK_THREADS) a.labels_out[so + t] = fin[t];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_free<256>(*sm.tmem);
}

size_t mine_smem_bytes(int k, int D, bool tc) {
  size_t b = (size_t)k * (D + 1) * 8 + 32 * 8 + 32 * 8 + (size_t)(KMAX * 3 + 16 * KMAX + 4 + 2) * 4;
  if (tc) b += 1024 + 4 * TC_TILE * 128 + 2 * (size_t)tc_np(k) * 128 + 8 * 8 + 16 + (size_t)tc_np(k) / 2 * 4 + 64;
  return b;
}

// TMA descriptor of a [rows][128] fp16 matrix, 64 x 128 boxes, 128-byte swizzle
static bool make_tmap(CUtensorMap* map, const void* base, uint64_t rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return false;
    fn = reinterpret_cast<EncodeFn>(p);
  }
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t strides[1] = {128 * 2};
  const cuuint32_t box[2] = {64, TC_TILE};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T>
cudaError_t launch_mine(const DevCache& c, const MineArgs<T>& a, cudaStream_t st) {
  CUtensorMap tk, tv;
  memset(&tk, 0, sizeof tk);
  memset(&tv, 0, sizeof tv);
  bool tc = false;
  if constexpr (std::is_same<T, __half>::value) {
    const char* env = getenv("PKV_MINE_CUDA_CORES");
    tc = c.D == 128 && a.k <= 64 && a.unit_stride == a.T * 128 && !(env && env[0] == '1') &&
         make_tmap(&tk, a.x[0], (uint64_t)c.U * a.T) && make_tmap(&tv, a.x[1], (uint64_t)c.U * a.T);
  }
  const size_t smem = mine_smem_bytes(a.k, c.D, tc);
  if constexpr (std::is_same<T, __half>::value) {
    const char* v1 = getenv("PKV_MINE_V1");
    if (tc && a.k <= SK_KMAX && !(v1 && v1[0] == '1') && sk_smem_bytes(a.k) <= 227 * 1024) {
      const int s0 = (a.side_mask & 1) ? 0 : 1, ns = (a.side_mask & 1) + ((a.side_mask >> 1) & 1);
      const char* ns1 = getenv("PKV_MINE_NOSPLIT");
      MineArgs<__half> a2 = a;
      if (ns1 && ns1[0] == '1') a2.side_mask |= 4;
      const size_t sb = sk_smem_bytes(a.k);
      const cudaError_t e = cudaFuncSetAttribute(kmeans_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
      if (e != cudaSuccess) return e;
      kmeans_stream_kernel<<<c.U * ns, SK_THREADS, sb, st>>>(c, a2, tk, tv, s0, ns);
      return cudaGetLastError();
    }
    if (tc) {
      cudaFuncSetAttribute(kmeans_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kmeans_kernel<T, true><<<dim3(c.U, 2), MINE_THREADS, smem, st>>>(c, a, tk, tv);
      return cudaGetLastError();
    }
  }
  {
    cudaFuncSetAttribute(kmeans_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kmeans_kernel<T, false><<<dim3(c.U, 2), MINE_THREADS, smem, st>>>(c, a, tk, tv);
  }
  return cudaGetLastError();
}

template cudaError_t launch_mine<__half>(const DevCache&, const MineArgs<__half>&, cudaStream_t);
template cudaError_t launch_mine<__nv_bfloat16>(const DevCache&, const MineArgs<__nv_bfloat16>&, cudaStream_t);
template cudaError_t launch_mine<float>(const DevCache&, const MineArgs<float>&, cudaStream_t);
template cudaError_t launch_mine<double>(const DevCache&, const MineArgs<double>&, cudaStream_t);

}  // namespace pkv
