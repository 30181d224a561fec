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
// Squared distances are fp64 FMA chains (the reference's einsum order is CPU
// specific; mining is "parity-unpinned at ulp level").
#include "pkv_common.cuh"

namespace pkv {

constexpr int MINE_THREADS = 512;
constexpr int KMAX = 96;
constexpr int KCH = 16;  // centers per register chunk

struct MineSmem {
  double* cen;    // [k][D]
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
            double d = __dsub_rn(xv, sm.cen[(j0 + j) * D + c]);
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

template <typename T>
__global__ void __launch_bounds__(MINE_THREADS, 1) kmeans_kernel(DevCache c, MineArgs<T> a) {
  const int u = blockIdx.x, side = blockIdx.y;
  if (!((a.side_mask >> side) & 1)) return;
  const int D = c.D, k = a.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t Tn = a.T;
  const T* X = a.x[side] + (int64_t)u * a.unit_stride;
  const int64_t so = ((int64_t)u * 2 + side) * Tn;
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
  sm.cen = reinterpret_cast<double*>(smem_raw);
  sm.redv = sm.cen + (size_t)k * D;
  sm.redi = reinterpret_cast<long long*>(sm.redv + 32);
  sm.cnt = reinterpret_cast<int*>(sm.redi + 32);
  sm.off = sm.cnt + KMAX;
  sm.wcnt = sm.off + KMAX;
  sm.chosen = sm.wcnt + 16 * KMAX;
  sm.flags = sm.chosen + KMAX;

  // ---- seeding (patterns.py:134-142) with distinct-rows detection --------------
  const int64_t first = a.first[side][u];
  if (tid == 0) sm.chosen[0] = (int)first;
  double vmax; long long imax;
  {
    double bv = -1.0 / 0.0; long long bi = 0x7fffffffffffffffLL;
    const T* xf = X + first * D;
    for (int64_t t = tid; t < Tn; t += MINE_THREADS) {
      double d = sqdist_row(X + t * D, xf, D);
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
    const T* xn = X + imax * D;
    double bv = -1.0 / 0.0; long long bi = 0x7fffffffffffffffLL;
    for (int64_t t = tid; t < Tn; t += MINE_THREADS) {
      double d = fmin(near_[t], sqdist_row(X + t * D, xn, D));
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
      for (int cc = 0; cc < D; ++cc) sm.cen[rank * D + cc] = to_f64(ri[cc]);
    }
    __syncthreads();
    assign_pass(X, Tn, D, n, sm, nullptr, lab, own, false);
    if (tid == 0) hist[0] = 0.0;
    iters = 1;
  } else {
    for (int i = tid; i < k * D; i += MINE_THREADS) {
      int j = i / D, cc = i - j * D;
      sm.cen[i] = to_f64(X[(int64_t)sm.chosen[j] * D + cc]);
    }
    __syncthreads();
    assign_pass(X, Tn, D, k, sm, nullptr, lab, own, true);
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
      // ---- stable per-cluster point lists (index order) ------------------------
      if (tid == 0) {
        int s = 0;
        for (int j = 0; j < k; ++j) { sm.off[j] = s; s += sm.cnt[j]; }
      }
      __syncthreads();
      for (int64_t base = 0; base < Tn; base += MINE_THREADS) {
        const int64_t t = base + tid;
        const int l = t < Tn ? lab[t] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, l);
        const int rank_w = __popc(peers & ((1u << lane) - 1));
        for (int i = tid; i < 16 * k; i += MINE_THREADS) sm.wcnt[i] = 0;
        __syncthreads();
        if (l >= 0 && rank_w == 0) sm.wcnt[warp * k + l] = __popc(peers);
        __syncthreads();
        if (l >= 0) {
          int pre = 0;
          for (int w = 0; w < warp; ++w) pre += sm.wcnt[w * k + l];
          list[sm.off[l] + pre + rank_w] = (int)t;
        }
        __syncthreads();
        for (int j = tid; j < k; j += MINE_THREADS) {
          int tot = 0;
          for (int w = 0; w < 16; ++w) tot += sm.wcnt[w * k + j];
          sm.off[j] += tot;
        }
        __syncthreads();
      }
      if (tid == 0) {
        int s = 0;
        for (int j = 0; j < k; ++j) { sm.off[j] = s; s += sm.cnt[j]; }
      }
      __syncthreads();
      // ---- centers = sequential fp64 means (numpy axis-0 reduction order) -------
      for (int i = tid; i < k * D; i += MINE_THREADS) {
        const int j = i / D, cc = i - j * D;
        const int n_j = sm.cnt[j];
        const int* lj = list + sm.off[j];
        double s = to_f64(X[(int64_t)lj[0] * D + cc]);
        for (int q = 1; q < n_j; ++q) s = __dadd_rn(s, to_f64(X[(int64_t)lj[q] * D + cc]));
        sm.cen[i] = __ddiv_rn(s, (double)n_j);
      }
      __syncthreads();
      // ---- objective of this round fused with the next assignment ----------------
      double part = assign_pass(X, Tn, D, k, sm, lab, lab2, near_, true);
      const double obj = block_sum(part, sm);
      if (tid == 0) hist[it] = obj;
      iters = it + 1;
      if (obj == 0.0 || (isfinite(prev) && prev - obj < 1e-6 * prev)) break;
      prev = obj;
      if (it + 1 == 25) break;  // keep the labels the final centers were built from
      int* tl = lab; lab = lab2; lab2 = tl;
      double* to = own; own = near_; near_ = to;
    }
    n = k;
  }
  // ---- write the pattern tables ---------------------------------------------------
  float amax = 0.f;
  for (int i = tid; i < n * D; i += MINE_THREADS) {
    const int j = i / D, cc = i - j * D;
    const double v = sm.cen[i];
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
}

size_t mine_smem_bytes(int k, int D) {
  return (size_t)k * D * 8 + 32 * 8 + 32 * 8 + (size_t)(KMAX * 3 + 16 * KMAX + 4) * 4;
}

template <typename T>
cudaError_t launch_mine(const DevCache& c, const MineArgs<T>& a, cudaStream_t st) {
  size_t smem = mine_smem_bytes(a.k, c.D);
  cudaFuncSetAttribute(kmeans_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kmeans_kernel<T><<<dim3(c.U, 2), MINE_THREADS, smem, st>>>(c, a);
  return cudaGetLastError();
}

template cudaError_t launch_mine<__half>(const DevCache&, const MineArgs<__half>&, cudaStream_t);
template cudaError_t launch_mine<__nv_bfloat16>(const DevCache&, const MineArgs<__nv_bfloat16>&, cudaStream_t);
template cudaError_t launch_mine<float>(const DevCache&, const MineArgs<float>&, cudaStream_t);
template cudaError_t launch_mine<double>(const DevCache&, const MineArgs<double>&, cudaStream_t);

}  // namespace pkv
