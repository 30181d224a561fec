// C ABI of the B200 PatternKV codec (include/pkv.h): cache arenas, lockstep
// lifecycle (prefill / append-and-refresh / decode attention / dequant) and
// the group-level API.  Host logic mirrors engine.py:142-198 (geometry,
// flush trigger, window retention) and gate.py:23-106 (threshold).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/pkv.h"
#include "pkv_common.cuh"


using namespace pkv;

// ---------------------------------------------------------------------------------
// errors (errors.py:9-14 taxonomy)
// ---------------------------------------------------------------------------------
static thread_local std::string g_err;
static thread_local int64_t g_err_idx = -1;

static int fail(int code, int64_t idx, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  g_err_idx = idx;
  return code;
}
#define CU(x)                                                                                  \
  do {                                                                                         \
    cudaError_t _e = (x);                                                                      \
    if (_e != cudaSuccess) return fail(PKV_CUDA, -1, "%s: %s", #x, cudaGetErrorString(_e));   \
  } while (0)

extern "C" int pkv_version(void) { return 1; }
extern "C" const char* pkv_last_error(int64_t* index) {
  if (index) *index = g_err_idx;
  return g_err.c_str();
}

// ---------------------------------------------------------------------------------
// gate constants (gate.py:23-106), host double arithmetic in the reference order
// ---------------------------------------------------------------------------------
static double horner(const double* c, int n, double r) {
  double acc = c[n - 1];
  for (int i = n - 2; i >= 0; --i) acc = acc * r + c[i];
  return acc;
}
static const double kA[8] = {3.3871328727963666080e0, 1.3314166789178437745e2, 1.9715909503065514427e3, 1.3731693765509461125e4,
                             4.5921953931549871457e4, 6.7265770927008700853e4, 3.3430575583588128105e4, 2.5090809287301226727e3};
static const double kB[8] = {1.0, 4.2313330701600911252e1, 6.8718700749205790830e2, 5.3941960214247511077e3,
                             2.1213794301586595867e4, 3.9307895800092710610e4, 2.8729085735721942674e4, 5.2264952788528545610e3};
static const double kC[8] = {1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0, 3.64784832476320460504e0,
                             1.27045825245236838258e0, 2.41780725177450611770e-1, 2.27238449892691845833e-2, 7.74545014278341407640e-4};
static const double kD[8] = {1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
                             1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4, 1.05075007164441684324e-9};
static const double kE[8] = {6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0, 2.96560571828504891230e-1,
                             2.65321895265761230930e-2, 1.24266094738807843860e-3, 2.71155556874348757815e-5, 2.01033439929228813265e-7};
static const double kF[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
                             7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7, 2.04426310338993978564e-15};

extern "C" int pkv_z_quantile(double alpha, double* out) {
  if (!(alpha > 0.0 && alpha <= 0.5)) return fail(PKV_USAGE, -1, "alpha must lie in (0, 0.5], got %g", alpha);
  const double q = alpha - 0.5;
  double z;
  if (std::fabs(q) <= 0.425) {
    const double r = 0.180625 - q * q;
    z = q * horner(kA, 8, r) / horner(kB, 8, r);
  } else {
    double r = q < 0 ? alpha : 1.0 - alpha;
    r = std::sqrt(-std::log(r));
    if (r <= 5.0) { r -= 1.6; z = horner(kC, 8, r) / horner(kD, 8, r); }
    else { r -= 5.0; z = horner(kE, 8, r) / horner(kF, 8, r); }
    if (q < 0) z = -z;
  }
  *out = -z;
  return PKV_OK;
}

extern "C" int pkv_threshold(int32_t head_dim, double alpha, double* out) {
  if (head_dim < 1) return fail(PKV_USAGE, -1, "head_dim must be >= 1, got %d", head_dim);
  double z;
  int rc = pkv_z_quantile(alpha, &z);
  if (rc) return rc;
  if (z <= 0.0) { *out = 1.0; return PKV_OK; }
  const double c = 2.0 * z / std::sqrt(5.0 * head_dim);
  if (c >= 1.0)
    return fail(PKV_USAGE, -1, "no contraction ratio reaches significance for head_dim=%d, alpha=%g", head_dim, alpha);
  double lo = 0.0, hi = 1.0;
  while (hi - lo > 1e-12) {
    const double mid = 0.5 * (lo + hi);
    if ((1.0 - mid * mid) - c * std::sqrt(1.0 + std::pow(mid, 4)) >= 0.0) lo = mid;
    else hi = mid;
  }
  *out = 0.5 * (lo + hi);
  return PKV_OK;
}

extern "C" int pkv_config_validate(const pkv_config* c) {
  if (!c) return fail(PKV_USAGE, -1, "null config");
  if (c->bits != 2 && c->bits != 4 && c->bits != 8)
    return fail(PKV_USAGE, -1, "unsupported bit width %d; expected one of (2, 4, 8)", c->bits);
  if (c->pattern_count < 1) return fail(PKV_USAGE, -1, "pattern_count must be >= 1, got %d", c->pattern_count);
  if (c->group_size < 1) return fail(PKV_USAGE, -1, "group_size must be >= 1, got %d", c->group_size);
  if (c->residual_window < c->group_size)
    return fail(PKV_USAGE, -1, "residual_window (%d) must be >= group_size (%d) so flushes always fill whole groups",
                c->residual_window, c->group_size);
  if (!(c->alpha > 0.0 && c->alpha <= 0.5)) return fail(PKV_USAGE, -1, "alpha must lie in (0, 0.5], got %g", c->alpha);
  return PKV_OK;
}

// ---------------------------------------------------------------------------------
// cache
// ---------------------------------------------------------------------------------
struct pkv_cache {
  pkv_config cfg;
  int U, D, Dp, dtype, esize, flags;
  DevCache dev;
  int64_t token_count = 0, committed = 0;
  int win_len = 0, win_slot0 = 0, nb = 0;
  int nb_prefill = 0;          // blocks laid out by prefill; later blocks are decode flushes of G
  int64_t decode_base = 0;     // committed count after prefill
  std::vector<int64_t> blk_start;
  std::vector<int> blk_len;
  int pk_bound = 0, pv_bound = 0;  // upper bounds of per-unit pattern counts
  float* part = nullptr;
  size_t part_bytes = 0;
  unsigned* stats = nullptr;
  unsigned long long* scratch_flag = nullptr;
  int64_t uploaded_nbcap = -1, uploaded_base = -1;   // last block table sent to the device
  std::vector<int64_t> uploaded_start;
  bool blocks_stale = false;   // reset dropped the prefill geometry; re-upload before the next flush
  unsigned char* mine_scratch = nullptr;   // k-means scratch (pkv_cache_reserve_mining), else per call
  size_t mine_scratch_bytes = 0;
  // fused non-finite detection: the kernels atomicMin dev.bad; every prefill / append copies it
  // into pinned host memory behind an event, so the host reads it without a stream sync
  unsigned long long* bad_host = nullptr;
  cudaEvent_t bad_ev = nullptr;
  int64_t prefill_tokens = 0;  // tokens of the last prefill (keys below are prefill rows)
};

// k-means scratch for U units x 2 sides x T points: near, own (f64), lab, lab2, list (i32),
// labels out (i32), history [U][2][25] f64, niter [U][2] i32, first [U][2] i64
static size_t mine_scratch_need(int U, int64_t T) {
  const size_t n2 = (size_t)U * 2 * T;
  return n2 * 8 * 2 + n2 * 4 * 4 + (size_t)U * 2 * 25 * 8 + (size_t)U * 2 * 4 + (size_t)U * 2 * 8 + 9 * 256;  // + carve alignment
}

static int esize_of(int dtype) {
  switch (dtype) {
    case PKV_F16: case PKV_BF16: return 2;
    case PKV_F32: return 4;
    case PKV_F64: return 8;
    default: return 0;
  }
}

template <typename P>
static cudaError_t dalloc(P** p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc((void**)p, bytes);
  if (e != cudaSuccess) return e;
  return cudaMemset(*p, 0, bytes);
}

// grow [U][old][row] -> [U][new][row]
template <typename P>
static cudaError_t regrow(P** p, int U, int64_t old_rows, int64_t new_rows, size_t row_bytes, cudaStream_t st) {
  P* np_ = nullptr;
  cudaError_t e = dalloc(&np_, (size_t)U * new_rows * row_bytes);
  if (e != cudaSuccess) return e;
  if (*p && old_rows > 0) {
    e = cudaMemcpy2DAsync(np_, new_rows * row_bytes, *p, old_rows * row_bytes, old_rows * row_bytes, U,
                          cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    cudaStreamSynchronize(st);
  }
  if (*p) cudaFree(*p);
  *p = np_;
  return cudaSuccess;
}

static int64_t nb_cap_for(int64_t Tcap, int G) { return (Tcap + G - 1) / G + 2; }

// block table for every future decode flush is precomputed on the device, so a
// flush needs no host->device traffic (CUDA-graph friendly)
static int upload_blocks(pkv_cache* c, cudaStream_t st) {
  const int G = c->cfg.group_size;
  if (c->uploaded_nbcap == c->dev.NBcap && c->uploaded_start == c->blk_start && c->uploaded_base == c->decode_base)
    return PKV_OK;
  std::vector<int64_t> s(c->dev.NBcap);
  std::vector<int> l(c->dev.NBcap);
  for (int64_t b = 0; b < c->dev.NBcap; ++b) {
    if (b < (int64_t)c->blk_start.size()) { s[b] = c->blk_start[b]; l[b] = c->blk_len[b]; }
    else { s[b] = c->decode_base + (b - c->nb_prefill) * (int64_t)G; l[b] = G; }
  }
  CU(cudaMemcpyAsync(c->dev.blk_start, s.data(), s.size() * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(c->dev.blk_len, l.data(), l.size() * 4, cudaMemcpyHostToDevice, st));
  CU(cudaStreamSynchronize(st));
  c->uploaded_nbcap = c->dev.NBcap;
  c->uploaded_start = c->blk_start;
  c->uploaded_base = c->decode_base;
  return PKV_OK;
}

// publish the device non-finite flag to pinned host memory (stream ordered, no sync)
static int publish_bad(pkv_cache* c, cudaStream_t st) {
  CU(cudaMemcpyAsync(c->bad_host, c->dev.bad, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaEventRecord(c->bad_ev, st));
  return PKV_OK;
}

// PKV_DATA with the reference's message when a finished prefill / append saw a non-finite
// input; wait = block until the last published flag is on the host
static int check_bad(pkv_cache* c, int wait, int64_t* where) {
  if (wait) CU(cudaEventSynchronize(c->bad_ev));
  else if (cudaEventQuery(c->bad_ev) != cudaSuccess) { (void)cudaGetLastError(); return PKV_OK; }
  const unsigned long long key = *(volatile unsigned long long*)c->bad_host;
  if (key == ~0ull) return PKV_OK;
  const int u = (int)(key >> 44), side = (int)((key >> 43) & 1), dim = (int)(key & 255);
  const int64_t tok = (int64_t)((key >> 8) & ((1ull << 35) - 1));
  if (where) { where[0] = u; where[1] = side; where[2] = tok; where[3] = dim; }
  if (tok < c->prefill_tokens)  // engine.py:138
    return fail(PKV_DATA, tok, "non-finite prefill %s element at token %lld, dim %d (unit %d)", side ? "V" : "K",
                (long long)tok, dim, u);
  return fail(PKV_DATA, tok, "non-finite decode vector at token %lld (unit %d)", (long long)tok, u);  // engine.py:181
}

static int reserve(pkv_cache* c, int64_t Tcap, int Pcap, cudaStream_t st) {
  DevCache& d = c->dev;
  const int U = c->U, D = c->D, Dp = c->Dp;
  if (Pcap > 32767) return fail(PKV_USAGE, -1, "pattern table would exceed 32767 entries (16-bit indices)");
  if (Pcap > d.Pcap) {
    int64_t o = d.Pcap;
    CU(regrow(&d.kpat64, U, o, Pcap, (size_t)D * 8, st));
    CU(regrow(&d.vpat64, U, o, Pcap, (size_t)D * 8, st));
    CU(regrow(&d.kpat32, U, o, Pcap, (size_t)Dp * 4, st));
    CU(regrow(&d.vpat32, U, o, Pcap, (size_t)Dp * 4, st));
    d.Pcap = Pcap;
  }
  if (Tcap > d.Tcap) {
    const int64_t oT = d.Tcap, oNB = d.NBcap;
    const int64_t nNB = nb_cap_for(Tcap, d.G);
    CU(regrow(&d.vparam64, U, oT, Tcap, 16, st));
    if (d.keep_diag) {
      CU(regrow(&d.kdiag, U, oT, Tcap, 16, st));
      CU(regrow(&d.vdiag, U, oT, Tcap, 16, st));
    }
    CU(regrow(&d.kcodes, U, oNB, nNB, (size_t)d.blk_bytes, st));
    CU(regrow(&d.vcodes, U, oNB, nNB, (size_t)d.blk_bytes, st));
    CU(regrow(&d.kparam32, U, oNB, nNB, (size_t)2 * Dp * 4, st));
    CU(regrow(&d.kparam64, U, oNB, nNB, (size_t)2 * D * 8, st));
    CU(regrow(&d.kidx, U, oNB, nNB, (size_t)d.GP * 2, st));
    CU(regrow(&d.vidx, U, oNB, nNB, (size_t)d.GP * 2, st));
    CU(regrow(&d.vparam32, U, oNB, nNB, (size_t)d.GP * 8, st));
    CU(regrow(&d.blk_start, 1, oNB, nNB, 8, st));
    CU(regrow(&d.blk_len, 1, oNB, nNB, 4, st));
    d.Tcap = Tcap;
    d.NBcap = nNB;
    int rc = upload_blocks(c, st);
    if (rc) return rc;
  }
  return PKV_OK;
}

extern "C" int pkv_cache_create(const pkv_config* cfg, int32_t n_units, int32_t head_dim, int32_t in_dtype,
                                int64_t max_tokens, int32_t max_patterns, int32_t flags, pkv_cache** out) {
  int rc = pkv_config_validate(cfg);
  if (rc) return rc;
  if (n_units < 1) return fail(PKV_USAGE, -1, "n_units must be >= 1, got %d", n_units);
  if (head_dim < 1 || head_dim > DMAX)
    return fail(PKV_USAGE, -1, "head_dim must lie in [1, %d] on the B200 path, got %d", DMAX, head_dim);
  if (cfg->group_size > GMAX)
    return fail(PKV_USAGE, -1, "group_size must be <= %d on the B200 path, got %d", GMAX, cfg->group_size);
  if (cfg->pattern_count > 96)
    return fail(PKV_USAGE, -1, "pattern_count must be <= 96 on the B200 path, got %d", cfg->pattern_count);
  if (!esize_of(in_dtype)) return fail(PKV_USAGE, -1, "unknown dtype code %d", in_dtype);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(PKV_USAGE, -1, "no CUDA device: the PatternKV B200 codec has no CPU fallback");
  double thr = 1.0;
  rc = pkv_threshold(head_dim, cfg->alpha, &thr);
  if (rc && (cfg->use_v_gate || cfg->use_k_gate)) return rc;

  pkv_cache* c = new pkv_cache();
  c->cfg = *cfg;
  c->U = n_units;
  c->D = head_dim;
  c->Dp = round_up(head_dim, 64);  // whole k-tile groups of the fragment layout at every bit width
  c->dtype = in_dtype;
  c->esize = esize_of(in_dtype);
  c->flags = flags;
  DevCache& d = c->dev;
  std::memset(&d, 0, sizeof d);
  d.U = n_units; d.D = head_dim; d.Dp = c->Dp; d.bits = cfg->bits; d.qmax = (1 << cfg->bits) - 1;
  d.G = cfg->group_size; d.W = cfg->residual_window; d.Wcap = cfg->residual_window + cfg->group_size;
  d.ntile_blk = (cfg->group_size + 15) / 16;
  d.GP = 16 * d.ntile_blk;
  d.blk_bytes = d.ntile_blk * tile_bytes(c->Dp, cfg->bits);
  d.in_dtype = in_dtype;
  d.use_kp = cfg->use_k_patterns; d.use_vp = cfg->use_v_patterns; d.use_vgate = cfg->use_v_gate;
  d.use_kgate = cfg->use_k_gate; d.gen_new = cfg->generate_new_patterns;
  d.keep_diag = (flags & PKV_FLAG_DECISIONS) ? 1 : 0;
  d.prune = (flags & PKV_FLAG_BRUTE_FORCE) ? 0 : 1;
  d.thr = thr;
  cudaStream_t st = 0;
  auto bail = [&](int code) { pkv_cache_destroy(c); return code; };
  if (dalloc(&d.kpmax, (size_t)n_units * 4) || dalloc(&d.vpmax, (size_t)n_units * 4) ||
      dalloc(&d.nk, (size_t)n_units * 4) || dalloc(&d.nv, (size_t)n_units * 4) ||
      dalloc(&d.probe, (size_t)n_units * 2 * 16 * 4) ||
      dalloc(&d.wk, (size_t)n_units * d.Wcap * head_dim * c->esize) ||
      dalloc(&d.wv, (size_t)n_units * d.Wcap * head_dim * c->esize) || dalloc(&c->scratch_flag, 8) ||
      dalloc(&d.work, 16) || dalloc(&d.bad, 8))
    return bail(fail(PKV_CUDA, -1, "cudaMalloc failed: %s", cudaGetErrorString(cudaGetLastError())));
  if (cudaMemset(d.bad, 0xff, 8) != cudaSuccess || cudaHostAlloc((void**)&c->bad_host, 8, cudaHostAllocDefault) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->bad_ev, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(PKV_CUDA, -1, "non-finite flag allocation failed: %s", cudaGetErrorString(cudaGetLastError())));
  *c->bad_host = ~0ull;
  if (flags & PKV_FLAG_STATS) {
    if (dalloc(&c->stats, 16)) return bail(fail(PKV_CUDA, -1, "cudaMalloc failed"));
    d.stats = c->stats;
  }
  rc = reserve(c, std::max<int64_t>(max_tokens, 1), std::max(max_patterns, cfg->pattern_count + 8), st);
  if (rc) return bail(rc);
  {  // decode-attention chunk partials, sized once for the largest chunking attn_impl picks
    // (U * nchunk <= 16 * SMs + U) and 8 query heads, so decode steps never allocate
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    c->part_bytes = (size_t)(16 * std::max(nsm, 1) + n_units) * 8 * (c->Dp + 2) * 4;
    if (cudaMalloc((void**)&c->part, c->part_bytes) != cudaSuccess)
      return bail(fail(PKV_CUDA, -1, "cudaMalloc of %zu attention partial bytes failed", c->part_bytes));
  }
  *out = c;
  return PKV_OK;
}

extern "C" int pkv_cache_destroy(pkv_cache* c) {
  if (!c) return PKV_OK;
  DevCache& d = c->dev;
  void* ptrs[] = {d.kpat64, d.vpat64, d.kpat32, d.vpat32, d.kpmax, d.vpmax, d.nk, d.nv, d.probe, d.blk_start, d.blk_len,
                  d.kcodes, d.kparam32, d.kparam64, d.kidx, d.vcodes, d.vparam32, d.vparam64, d.vidx, d.kdiag,
                  d.vdiag, d.wk, d.wv, c->stats, c->part, c->scratch_flag, d.work, c->mine_scratch, d.fix};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (d.bad) cudaFree(d.bad);
  if (c->bad_host) cudaFreeHost(c->bad_host);
  if (c->bad_ev) cudaEventDestroy(c->bad_ev);
  delete c;
  return PKV_OK;
}

extern "C" int pkv_cache_info_get(pkv_cache* c, pkv_cache_info* o) {
  if (!c || !o) return fail(PKV_USAGE, -1, "null argument");
  o->n_units = c->U; o->head_dim = c->D; o->head_dim_padded = c->Dp; o->in_dtype = c->dtype;
  o->token_count = c->token_count; o->committed_count = c->committed;
  o->window_len = c->win_len; o->window_slot0 = c->win_slot0; o->n_blocks = c->nb;
  o->pattern_capacity = c->dev.Pcap; o->token_capacity = c->dev.Tcap; o->block_bytes = c->dev.blk_bytes;
  o->n_refined = 0; o->n_exact_div = 0;
  if (c->stats) {
    unsigned s[4];
    CU(cudaMemcpy(s, c->stats, 16, cudaMemcpyDeviceToHost));
    o->n_refined = s[0]; o->n_exact_div = s[1];
  }
  return PKV_OK;
}

extern "C" int pkv_cache_reserve_mining(pkv_cache* c, int64_t max_tokens, void* stream) {
  if (!c) return fail(PKV_USAGE, -1, "null cache");
  if (max_tokens < 1) return fail(PKV_USAGE, -1, "max_tokens must be >= 1");
  const size_t need = mine_scratch_need(c->U, (max_tokens + 3) / 4 * 4);
  if (need <= c->mine_scratch_bytes) return PKV_OK;
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  if (c->mine_scratch) cudaFree(c->mine_scratch);
  c->mine_scratch = nullptr;
  c->mine_scratch_bytes = 0;
  CU(cudaMalloc((void**)&c->mine_scratch, need));
  c->mine_scratch_bytes = need;
  return PKV_OK;
}

extern "C" int pkv_cache_reserve(pkv_cache* c, int64_t max_tokens, int32_t max_patterns, void* stream) {
  if (!c) return fail(PKV_USAGE, -1, "null cache");
  return reserve(c, std::max(max_tokens, c->dev.Tcap), std::max<int>(max_patterns, c->dev.Pcap), (cudaStream_t)stream);
}

extern "C" int pkv_cache_reset(pkv_cache* c, int32_t keep_patterns, void* stream) {
  if (!c) return fail(PKV_USAGE, -1, "null cache");
  cudaStream_t st = (cudaStream_t)stream;
  c->token_count = 0;
  c->committed = 0;
  c->win_len = 0;
  c->win_slot0 = 0;
  c->nb = 0;
  // the next flush (without a prefill) starts a fresh block table at token 0
  c->blk_start.clear();
  c->blk_len.clear();
  c->nb_prefill = 0;
  c->decode_base = 0;
  c->blocks_stale = true;
  c->prefill_tokens = 0;
  CU(cudaMemsetAsync(c->dev.bad, 0xff, 8, st));
  {
    const int rc = publish_bad(c, st);
    if (rc) return rc;
  }
  if (!keep_patterns) {
    CU(cudaMemsetAsync(c->dev.nk, 0, (size_t)c->U * 4, st));
    CU(cudaMemsetAsync(c->dev.nv, 0, (size_t)c->U * 4, st));
    CU(cudaMemsetAsync(c->dev.kpmax, 0, (size_t)c->U * 4, st));
    CU(cudaMemsetAsync(c->dev.vpmax, 0, (size_t)c->U * 4, st));
    c->pk_bound = c->pv_bound = 0;
    CU(launch_probes(c->dev, st));
  }
  return PKV_OK;
}

extern "C" int pkv_cache_buffer(pkv_cache* c, const char* name, void** ptr, int64_t* bytes) {
  if (!c || !name || !ptr) return fail(PKV_USAGE, -1, "null argument");
  DevCache& d = c->dev;
  const int64_t U = c->U, T = d.Tcap, NB = d.NBcap, P = d.Pcap, D = c->D;
  struct { const char* n; void* p; int64_t b; } tab[] = {
      {"kpat64", d.kpat64, U * P * D * 8}, {"vpat64", d.vpat64, U * P * D * 8},
      {"kparam64", d.kparam64, U * NB * 2 * D * 8}, {"vparam64", d.vparam64, U * T * 16},
      {"kidx", d.kidx, U * NB * d.GP * 2}, {"vidx", d.vidx, U * NB * d.GP * 2},
      {"kdiag", d.kdiag, d.keep_diag ? U * T * 16 : 0}, {"vdiag", d.vdiag, d.keep_diag ? U * T * 16 : 0},
      {"wk", d.wk, U * d.Wcap * D * c->esize}, {"wv", d.wv, U * d.Wcap * D * c->esize},
      {"nk", d.nk, U * 4}, {"nv", d.nv, U * 4}, {"blk_start", d.blk_start, NB * 8}, {"blk_len", d.blk_len, NB * 4},
      {"kcodes", d.kcodes, U * NB * d.blk_bytes}, {"vcodes", d.vcodes, U * NB * d.blk_bytes},
      {"kparam32", d.kparam32, U * NB * 2 * d.Dp * 4}, {"vparam32", d.vparam32, U * NB * d.GP * 8},
      {"kpat32", d.kpat32, U * P * d.Dp * 4}, {"vpat32", d.vpat32, U * P * d.Dp * 4},
      {"stats", c->stats, c->stats ? 16 : 0},
  };
  for (auto& e : tab) {
    if (std::strcmp(e.n, name) == 0) {
      *ptr = e.p;
      if (bytes) *bytes = e.b;
      return PKV_OK;
    }
  }
  return fail(PKV_USAGE, -1, "unknown buffer name '%s'", name);
}

extern "C" int pkv_cache_read(pkv_cache* c, const char* name, int64_t offset, int64_t n, void* dst, void* stream) {
  void* p = nullptr;
  int64_t bytes = 0;
  int rc = pkv_cache_buffer(c, name, &p, &bytes);
  if (rc) return rc;
  if (offset < 0 || n < 0 || offset + n > bytes)
    return fail(PKV_USAGE, offset, "read [%lld, %lld) outside arena '%s' of %lld bytes", (long long)offset,
                (long long)(offset + n), name, (long long)bytes);
  if (n) CU(cudaMemcpyAsync(dst, (const char*)p + offset, n, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return PKV_OK;
}

// ---------------------------------------------------------------------------------
// finiteness (engine.py:132-139)
// ---------------------------------------------------------------------------------
extern "C" int pkv_check_finite(const void* x, int32_t dtype, int64_t n, int64_t* first_bad, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* flag = nullptr;
  CU(cudaMallocAsync((void**)&flag, 8, st));
  CU(cudaMemsetAsync(flag, 0xff, 8, st));
  cudaError_t e;
  switch (dtype) {
    case PKV_F16: e = launch_finite((const __half*)x, n, flag, st); break;
    case PKV_BF16: e = launch_finite((const __nv_bfloat16*)x, n, flag, st); break;
    case PKV_F32: e = launch_finite((const float*)x, n, flag, st); break;
    case PKV_F64: e = launch_finite((const double*)x, n, flag, st); break;
    default: cudaFreeAsync(flag, st); return fail(PKV_USAGE, -1, "unknown dtype code %d", dtype);
  }
  CU(e);
  unsigned long long h = ~0ull;
  CU(cudaMemcpyAsync(&h, flag, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaFreeAsync(flag, st));
  CU(cudaStreamSynchronize(st));
  *first_bad = h == ~0ull ? -1 : (int64_t)h;
  return PKV_OK;
}

// ---------------------------------------------------------------------------------
// dtype dispatch helper
// ---------------------------------------------------------------------------------
template <typename F>
static cudaError_t dispatch(int dtype, F&& f) {
  switch (dtype) {
    case PKV_F16: return f((__half*)nullptr);
    case PKV_BF16: return f((__nv_bfloat16*)nullptr);
    case PKV_F32: return f((float*)nullptr);
    default: return f((double*)nullptr);
  }
}

// ---------------------------------------------------------------------------------
// mining (patterns.py:145-158 per unit)
// ---------------------------------------------------------------------------------
static int mine_impl(pkv_cache* c, int side_mask, const void* xk, const void* xv, int64_t T, const int64_t* fk,
                     const int64_t* fv, double* hist_host, int32_t* niter_host, int32_t* labels_dev, cudaStream_t st) {
  const int U = c->U, k = c->cfg.pattern_count;
  if (T < 1) return fail(PKV_USAGE, -1, "pattern mining expects a non-empty 2-D array of row vectors");
  for (int s = 0; s < 2; ++s) {
    const int64_t* f = s == 0 ? fk : fv;
    if (!((side_mask >> s) & 1)) continue;
    for (int u = 0; u < U; ++u)
      if (f[u] < 0 || f[u] >= T) return fail(PKV_USAGE, f[u], "first seed index %lld outside [0, %lld)", (long long)f[u], (long long)T);
  }
  int rc = reserve(c, c->dev.Tcap, std::max(c->dev.Pcap, k + 8), st);
  if (rc) return rc;
  const int64_t Tp = (T + 3) / 4 * 4;  // scratch stride: 16-byte aligned rows per unit-side
  const size_t n2 = (size_t)U * 2 * Tp;
  double *near_ = nullptr, *own = nullptr, *hist = nullptr;
  int *lab = nullptr, *lab2 = nullptr, *list = nullptr, *niter = nullptr;
  int64_t* first = nullptr;
  int* lab_out = nullptr;
  const size_t need = mine_scratch_need(U, Tp);
  const bool own_scratch = c->mine_scratch_bytes >= need;
  unsigned char* base = c->mine_scratch;
  if (!own_scratch) CU(cudaMallocAsync((void**)&base, need, st));
  {
    size_t off = 0;
    auto carve = [&](size_t bytes) { unsigned char* p = base + off; off += (bytes + 255) & ~(size_t)255; return p; };
    near_ = (double*)carve(n2 * 8); own = (double*)carve(n2 * 8);
    lab = (int*)carve(n2 * 4); lab2 = (int*)carve(n2 * 4); list = (int*)carve(n2 * 4);
    if (labels_dev) lab_out = (int*)carve(n2 * 4); else carve(n2 * 4);
    hist = (double*)carve((size_t)U * 2 * 25 * 8); niter = (int*)carve((size_t)U * 2 * 4);
    first = (int64_t*)carve((size_t)U * 2 * 8);
  }
  std::vector<int64_t> fh((size_t)U * 2, 0);
  for (int u = 0; u < U; ++u) {
    if (side_mask & 1) fh[u] = fk[u];
    if (side_mask & 2) fh[U + u] = fv[u];
  }
  CU(cudaMemcpyAsync(first, fh.data(), fh.size() * 8, cudaMemcpyHostToDevice, st));
  cudaError_t e = dispatch(c->dtype, [&](auto* tp) {
    using T_ = std::remove_pointer_t<decltype(tp)>;
    MineArgs<T_> a;
    a.x[0] = (const T_*)xk; a.x[1] = (const T_*)xv;
    a.unit_stride = T * c->D; a.T = T;
    a.first[0] = first; a.first[1] = first + U;
    a.k = k; a.side_mask = side_mask;
    a.near_ = near_; a.own = own; a.lab = lab; a.lab2 = lab2; a.list = list;
    a.hist = hist; a.niter = niter; a.labels_out = lab_out; a.tstride = Tp;
    return launch_mine<T_>(c->dev, a, st);
  });
  CU(e);
  if (labels_dev) {  // [U][2][T] -> the mined side's [U][T]
    const int s = (side_mask & 1) ? 0 : 1;
    CU(cudaMemcpy2DAsync(labels_dev, (size_t)T * 4, lab_out + (size_t)s * Tp, (size_t)2 * Tp * 4, (size_t)T * 4, U,
                         cudaMemcpyDeviceToDevice, st));
  }
  if (hist_host || niter_host) {
    std::vector<double> hh((size_t)U * 2 * 25);
    std::vector<int> nh((size_t)U * 2);
    CU(cudaMemcpyAsync(hh.data(), hist, hh.size() * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(nh.data(), niter, nh.size() * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const int s = (side_mask & 1) ? 0 : 1;
    for (int u = 0; u < U; ++u) {
      if (hist_host) std::memcpy(hist_host + (size_t)u * 25, hh.data() + ((size_t)u * 2 + s) * 25, 25 * 8);
      if (niter_host) niter_host[u] = nh[(size_t)u * 2 + s];
    }
  }
  if (!own_scratch) CU(cudaFreeAsync(base, st));
  if (side_mask & 1) c->pk_bound = k;
  if (side_mask & 2) c->pv_bound = k;
  CU(launch_probes(c->dev, st));
  return PKV_OK;
}

extern "C" int pkv_mine(pkv_cache* c, int32_t side, const void* x, int64_t T, const int64_t* first_idx, double* history,
                        int32_t* niter, int32_t* labels, void* stream) {
  if (!c || !x || !first_idx) return fail(PKV_USAGE, -1, "null argument");
  if (side != 0 && side != 1) return fail(PKV_USAGE, -1, "side must be 0 (K) or 1 (V)");
  return mine_impl(c, 1 << side, x, x, T, first_idx, first_idx, history, niter, labels, (cudaStream_t)stream);
}

// pattern tables with per-unit counts (device [U][P][D] fp64, host counts [U] <= P): installed by
// a kernel on the stream (no host round trip of the table)
static int load_patterns(pkv_cache* c, int side, const double* pat, int P, const int32_t* counts, cudaStream_t st) {
  int bound = P;
  int* dcounts = nullptr;
  if (counts) {
    bound = 0;
    for (int u = 0; u < c->U; ++u) bound = std::max(bound, (int)counts[u]);
    CU(cudaMallocAsync((void**)&dcounts, (size_t)c->U * 4, st));
    CU(cudaMemcpyAsync(dcounts, counts, (size_t)c->U * 4, cudaMemcpyHostToDevice, st));
  }
  CU(launch_install_patterns(c->dev, side, pat, P, dcounts, st));
  CU(launch_probes(c->dev, st));
  if (dcounts) CU(cudaFreeAsync(dcounts, st));
  if (side == 0) c->pk_bound = bound; else c->pv_bound = bound;
  return PKV_OK;
}

extern "C" int pkv_cache_import(pkv_cache* c, int64_t token_count, int32_t nb, const int64_t* blk_start,
                                const int32_t* blk_len, int32_t nb_prefill, int32_t win_len, int32_t Pk, int32_t Pv,
                                const int32_t* nk, const int32_t* nv, const double* kpat, const double* vpat,
                                const double* kparam, const int32_t* kidx, const int32_t* vidx, const double* vparam,
                                const uint8_t* kcodes, const uint8_t* vcodes, const void* wk, const void* wv,
                                const double* kdiag, const double* vdiag, void* stream) {
  if (!c) return fail(PKV_USAGE, -1, "null cache");
  const pkv_config& cfg = c->cfg;
  const int G = cfg.group_size, W = cfg.residual_window;
  if (nb < 0 || nb_prefill < 0 || nb_prefill > nb || win_len < 0 || Pk < 0 || Pv < 0 || token_count < 0)
    return fail(PKV_USAGE, -1, "invalid import geometry");
  if (nb > 0 && (!blk_start || !blk_len || !kparam || !kidx || !vidx || !vparam || !kcodes || !vcodes))
    return fail(PKV_USAGE, -1, "null argument");
  int64_t C = 0;
  for (int b = 0; b < nb; ++b) {
    if (blk_len[b] < 1 || blk_len[b] > G || blk_start[b] != C)
      return fail(PKV_DATA, b, "block %d: start %lld / length %d do not continue the committed tokens", b,
                  (long long)blk_start[b], blk_len[b]);
    if (b >= nb_prefill && blk_len[b] != G) return fail(PKV_DATA, b, "decode block %d has length %d != G", b, blk_len[b]);
    C += blk_len[b];
  }
  if (C + win_len != token_count)
    return fail(PKV_DATA, -1, "committed %lld + window %d != token count %lld", (long long)C, win_len,
                (long long)token_count);
  if (win_len > W + G - 1) return fail(PKV_DATA, -1, "window of %d rows exceeds W + G - 1 = %d", win_len, W + G - 1);
  cudaStream_t st = (cudaStream_t)stream;
  int rc = pkv_cache_reset(c, 0, stream);
  if (rc) return rc;
  rc = reserve(c, std::max<int64_t>(c->dev.Tcap, token_count + 4 * G), std::max(c->dev.Pcap, std::max(Pk, Pv) + 8), st);
  if (rc) return rc;
  while ((int64_t)nb + 2 > c->dev.NBcap) {
    rc = reserve(c, c->dev.Tcap * 2, c->dev.Pcap, st);
    if (rc) return rc;
  }
  if (Pk > 0 && cfg.use_k_patterns) { rc = load_patterns(c, 0, kpat, Pk, nk, st); if (rc) return rc; }
  if (Pv > 0 && cfg.use_v_patterns) { rc = load_patterns(c, 1, vpat, Pv, nv, st); if (rc) return rc; }
  DevCache& d = c->dev;
  c->blk_start.assign(blk_start, blk_start + nb);
  c->blk_len.assign(blk_len, blk_len + nb);
  c->nb = nb;
  c->nb_prefill = nb_prefill;
  c->decode_base = nb_prefill > 0 ? blk_start[nb_prefill - 1] + blk_len[nb_prefill - 1] : 0;
  rc = upload_blocks(c, st);
  if (rc) return rc;
  c->blocks_stale = false;
  CU(launch_import(d, nb, C, kparam, kidx, vidx, vparam, kcodes, vcodes, kdiag, vdiag, st));
  if (win_len > 0) {
    const size_t row = (size_t)c->D * c->esize;
    CU(cudaMemcpy2DAsync(d.wk, (size_t)d.Wcap * row, wk, (size_t)win_len * row, (size_t)win_len * row, c->U,
                         cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpy2DAsync(d.wv, (size_t)d.Wcap * row, wv, (size_t)win_len * row, (size_t)win_len * row, c->U,
                         cudaMemcpyDeviceToDevice, st));
  }
  CU(cudaStreamSynchronize(st));
  c->win_slot0 = 0;
  c->win_len = win_len;
  c->token_count = token_count;
  c->committed = C;
  return PKV_OK;
}

extern "C" int pkv_set_patterns(pkv_cache* c, int32_t side, const double* pat, int32_t P, void* stream) {
  if (!c) return fail(PKV_USAGE, -1, "null cache");
  if (P < 0) return fail(PKV_USAGE, -1, "negative pattern count");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reserve(c, c->dev.Tcap, std::max(c->dev.Pcap, P + 8), st);
  if (rc) return rc;
  return load_patterns(c, side, pat, P, nullptr, st);
}

// ---------------------------------------------------------------------------------
// prefill (engine.py:142-169)
// ---------------------------------------------------------------------------------
extern "C" int pkv_prefill(pkv_cache* c, const void* k, const void* v, int64_t T, const int64_t* first_k,
                           const int64_t* first_v, void* stream) {
  if (!c || !k || !v) return fail(PKV_USAGE, -1, "null argument");
  if (T < 1) return fail(PKV_USAGE, -1, "prefill K must be a non-empty (tokens, dim) matrix");
  if (c->token_count != 0) return fail(PKV_USAGE, -1, "prefill on a cache that already holds %lld tokens", (long long)c->token_count);
  cudaStream_t st = (cudaStream_t)stream;
  const pkv_config& cfg = c->cfg;
  const int W = cfg.residual_window, G = cfg.group_size;
  const int64_t commit_n = T - std::min<int64_t>(T, W);
  int rc = reserve(c, std::max<int64_t>(c->dev.Tcap, T + 4 * G), c->dev.Pcap, st);
  if (rc) return rc;
  CU(cudaMemsetAsync(c->dev.bad, 0xff, 8, st));  // a prefill starts a new stream of inputs
  c->prefill_tokens = T;
  // mining (engine.py:156-159)
  int mask = 0;
  if (cfg.use_k_patterns && first_k) mask |= 1;
  if (cfg.use_v_patterns && first_v) mask |= 2;
  if (mask) {
    rc = mine_impl(c, mask, k, v, T, first_k, first_v, nullptr, nullptr, nullptr, st);
    if (rc) return rc;
  }
  // block geometry (engine.py:161-165): spans of G from 0, short tail allowed
  c->blk_start.clear();
  c->blk_len.clear();
  for (int64_t s = 0; s < commit_n; s += G) {
    c->blk_start.push_back(s);
    c->blk_len.push_back((int)std::min<int64_t>(G, commit_n - s));
  }
  c->nb = c->nb_prefill = (int)c->blk_start.size();
  c->decode_base = commit_n;
  rc = upload_blocks(c, st);
  if (rc) return rc;
  c->blocks_stale = false;
  cudaError_t e = dispatch(c->dtype, [&](auto* tp) {
    using T_ = std::remove_pointer_t<decltype(tp)>;
    SpanSrc<T_> sk{(const T_*)k, T * c->D, 0, INT64_MAX / 4};
    SpanSrc<T_> sv{(const T_*)v, T * c->D, 0, INT64_MAX / 4};
    cudaError_t e1 = cudaErrorNotSupported;
    if constexpr (std::is_same<T_, __half>::value) {
      // deferred code fix-up list (~0.25 pairs per token-unit at cfg2: 64 per block leaves 4x
      // headroom); an overflow is fixed in line
      int64_t want = std::min<int64_t>(std::max<int64_t>((int64_t)c->U * c->nb * 64, 1 << 16), 1 << 27);
      const char* fcap = getenv("PKV_FIX_CAP");  // tests: a tiny list exercises the in-line fix
      if (fcap) want = std::max<int64_t>(atoll(fcap), 1);
      if (c->dev.fixcap < want || (fcap && c->dev.fixcap != want)) {
        if (c->dev.fix) cudaFree(c->dev.fix);
        c->dev.fix = nullptr;
        c->dev.fixcap = 0;
        if (cudaMalloc((void**)&c->dev.fix, (size_t)want * 8) == cudaSuccess) c->dev.fixcap = (int)want;
        else (void)cudaGetLastError();
      }
      e1 = launch_encode_tc(c->dev, std::max(c->pk_bound, c->pv_bound), (const __half*)k, (const __half*)v, T,
                            T * c->D, 0, c->nb, st);
    }
    if (e1 == cudaErrorNotSupported) {
      (void)cudaGetLastError();
      e1 = launch_encode<T_>(c->dev, sk, sv, 0, c->nb, st);
    }
    if (e1 != cudaSuccess) return e1;
    // window = newest min(T, W) rows (engine.py:166-167)
    const size_t off = (size_t)commit_n * c->D;
    return launch_window_put<T_>(c->dev, (const T_*)k + off, (const T_*)v + off, T * c->D, (int)(T - commit_n), 0,
                                 commit_n, st);
  });
  CU(e);
  c->win_slot0 = 0;
  c->win_len = (int)(T - commit_n);
  c->token_count = T;
  c->committed = commit_n;
  return publish_bad(c, st);
}

// ---------------------------------------------------------------------------------
// append-and-refresh (engine.py:172-198)
// ---------------------------------------------------------------------------------
extern "C" int pkv_append(pkv_cache* c, const void* k, const void* v, void* stream) {
  if (!c || !k || !v) return fail(PKV_USAGE, -1, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const pkv_config& cfg = c->cfg;
  const int W = cfg.residual_window, G = cfg.group_size;
  DevCache& d = c->dev;
  {  // a cache whose earlier input was non-finite refuses further appends (reset / prefill clears it)
    int rc = check_bad(c, 0, nullptr);
    if (rc) return rc;
  }
  if (c->blocks_stale) {
    int rc = upload_blocks(c, st);
    if (rc) return rc;
    c->blocks_stale = false;
  }
  const int slot = (c->win_slot0 + c->win_len) % d.Wcap;
  cudaError_t e = dispatch(c->dtype, [&](auto* tp) {
    using T_ = std::remove_pointer_t<decltype(tp)>;
    return launch_window_put<T_>(d, (const T_*)k, (const T_*)v, c->D, 1, slot, c->token_count, st);
  });
  CU(e);
  c->win_len += 1;
  c->token_count += 1;
  if (c->win_len == W + G) {
    // capacity for one more block and one more pattern per side
    const bool grow_p = cfg.generate_new_patterns;
    int need_p = std::max(c->pk_bound, c->pv_bound) + (grow_p ? 1 : 0);
    if (c->committed + G > d.Tcap || c->nb + 1 > d.NBcap - 1 || need_p > d.Pcap) {
      int rc = reserve(c, std::max<int64_t>(d.Tcap * 2, c->committed + 2 * G),
                       need_p > d.Pcap ? std::max(2 * d.Pcap, need_p) : d.Pcap, st);
      if (rc) return rc;
    }
    if (grow_p) {
      int mask = (cfg.use_k_patterns ? 1 : 0) | (cfg.use_v_patterns ? 2 : 0);
      if (mask) {
        e = dispatch(c->dtype, [&](auto* tp) {
          using T_ = std::remove_pointer_t<decltype(tp)>;
          return launch_refresh<T_>(d, c->win_slot0, G, mask, st);
        });
        CU(e);
        if (mask & 1) c->pk_bound += 1;
        if (mask & 2) c->pv_bound += 1;
        CU(launch_probes(d, st));
      }
    }
    // commit the oldest G rows against the refreshed tables (engine.py:195)
    e = dispatch(c->dtype, [&](auto* tp) {
      using T_ = std::remove_pointer_t<decltype(tp)>;
      SpanSrc<T_> sk{(const T_*)d.wk, (int64_t)d.Wcap * c->D, c->win_slot0, d.Wcap};
      SpanSrc<T_> sv{(const T_*)d.wv, (int64_t)d.Wcap * c->D, c->win_slot0, d.Wcap};
      return launch_encode<T_>(d, sk, sv, c->nb, 1, st);
    });
    CU(e);
    c->blk_start.push_back(c->committed);
    c->blk_len.push_back(G);
    c->nb += 1;
    c->committed += G;
    c->win_slot0 = (c->win_slot0 + G) % d.Wcap;
    c->win_len -= G;
  }
  return publish_bad(c, st);
}

extern "C" int pkv_cache_check(pkv_cache* c, int32_t wait, int64_t* where) {
  if (!c) return fail(PKV_USAGE, -1, "null cache");
  return check_bad(c, wait, where);
}

// ---------------------------------------------------------------------------------
// decode attention
// ---------------------------------------------------------------------------------
static int attn_impl(pkv_cache* c, const float* q, int32_t gqa, float sm_scale, int32_t blk0, int32_t blk1,
                     int32_t with_window, float* out, float* ml, cudaStream_t st) {
  if (!c || !q || !out) return fail(PKV_USAGE, -1, "null argument");
  if (gqa < 1 || gqa > 8) return fail(PKV_USAGE, -1, "query heads per KV head must lie in [1, 8], got %d", gqa);
  if (c->token_count == 0) return fail(PKV_USAGE, -1, "attention over an empty cache");
  if (blk0 < 0 || blk1 > c->nb || blk0 > blk1)
    return fail(PKV_USAGE, blk0, "block range [%d, %d) outside the %d committed blocks", blk0, blk1, c->nb);
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  AttnArgs a;
  a.q = q; a.G = gqa; a.scale_log2 = sm_scale * 1.4426950408889634f;
  a.blk0 = blk0; a.nb = blk1 - blk0; a.ml = ml;
  // enough CTAs for ~4 waves (K3-TC: 4 CTAs/SM at GQA <= 4, 2 CTAs of two head halves above),
  // >= 4 blocks per chunk (one per warp)
  static const char* tenv = getenv("PKV_ATTN_CTAS_PER_SM");  // tuning: CTAs per SM the chunking aims at
  const int target = (tenv ? std::max(1, atoi(tenv)) : (gqa <= 4 ? 16 : 8)) * num_sms;
  int nchunk = std::max(1, std::min((target + c->U - 1) / c->U, (a.nb + 3) / 4));
  nchunk = std::max(nchunk, (a.nb + 255) / 256);  // K3-TC: <= 256 blocks per chunk (s32 digit sums)
  a.bpc = std::max(1, (a.nb + nchunk - 1) / nchunk);
  a.nchunk = std::max(1, (a.nb + a.bpc - 1) / a.bpc);
  const size_t need = (size_t)c->U * a.nchunk * gqa * (c->Dp + 2) * 4;
  if (need > c->part_bytes) {
    if (c->part) { CU(cudaStreamSynchronize(st)); cudaFree(c->part); c->part = nullptr; c->part_bytes = 0; }
    CU(cudaMalloc((void**)&c->part, need));
    c->part_bytes = need;
  }
  a.part = c->part;
  const int pk = c->cfg.use_k_patterns ? c->pk_bound : 0, pv = c->cfg.use_v_patterns ? c->pv_bound : 0;
  const int wl = with_window ? c->win_len : 0;
  cudaError_t e = dispatch(c->dtype, [&](auto* tp) {
    using T_ = std::remove_pointer_t<decltype(tp)>;
    return launch_attn<T_>(c->dev, a, pk, pv, wl, c->win_slot0, out, st);
  });
  if (e == cudaErrorNotSupported)
    return fail(PKV_USAGE, -1, "decode attention holds the q.M table and pattern weights in shared memory: %d K / %d V "
                "patterns exceed its 227 KB (about 1100 patterns per side)", pk, pv);
  CU(e);
  return PKV_OK;
}

extern "C" int pkv_decode_attn(pkv_cache* c, const float* q, int32_t gqa, float sm_scale, float* out, void* stream) {
  if (!c) return fail(PKV_USAGE, -1, "null cache");
  return attn_impl(c, q, gqa, sm_scale, 0, c->nb, 1, out, nullptr, (cudaStream_t)stream);
}

extern "C" int pkv_decode_attn_partial(pkv_cache* c, const float* q, int32_t gqa, float sm_scale, int32_t blk0,
                                       int32_t blk1, int32_t with_window, float* o, float* ml, void* stream) {
  if (!c || !ml) return fail(PKV_USAGE, -1, "null argument");
  return attn_impl(c, q, gqa, sm_scale, blk0, blk1, with_window, o, ml, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------------
// unit fork (parallel sampling from one prompt: a unit's whole state copied)
// ---------------------------------------------------------------------------------
// arena rows of every unit of `src` to the matching units of `dst` (dst capacities >= src's)
static ForkArenas fork_arenas(const pkv_cache* src, const pkv_cache* dst) {
  const DevCache& a = src->dev;
  const DevCache& b = dst->dev;
  const int64_t D = src->D, Dp = src->Dp;
  ForkArenas fa;
  std::memset(&fa, 0, sizeof fa);
  auto add = [&](const void* ps, void* pd, int64_t ss, int64_t ds, int64_t bytes) {
    fa.a[fa.n++] = ForkArenas::Arena{(const unsigned char*)ps, (unsigned char*)pd, ss, ds, (ps && pd) ? bytes : 0};
  };
  add(a.kpat64, b.kpat64, a.Pcap * D * 8, b.Pcap * D * 8, a.Pcap * D * 8);
  add(a.vpat64, b.vpat64, a.Pcap * D * 8, b.Pcap * D * 8, a.Pcap * D * 8);
  add(a.kpat32, b.kpat32, a.Pcap * Dp * 4, b.Pcap * Dp * 4, a.Pcap * Dp * 4);
  add(a.vpat32, b.vpat32, a.Pcap * Dp * 4, b.Pcap * Dp * 4, a.Pcap * Dp * 4);
  add(a.kpmax, b.kpmax, 4, 4, 4); add(a.vpmax, b.vpmax, 4, 4, 4);
  add(a.nk, b.nk, 4, 4, 4); add(a.nv, b.nv, 4, 4, 4);
  add(a.probe, b.probe, 128, 128, 128);
  const int64_t bb = a.blk_bytes;
  add(a.kcodes, b.kcodes, a.NBcap * bb, b.NBcap * bb, a.NBcap * bb);
  add(a.vcodes, b.vcodes, a.NBcap * bb, b.NBcap * bb, a.NBcap * bb);
  add(a.kparam32, b.kparam32, a.NBcap * 2 * Dp * 4, b.NBcap * 2 * Dp * 4, a.NBcap * 2 * Dp * 4);
  add(a.kparam64, b.kparam64, a.NBcap * 2 * D * 8, b.NBcap * 2 * D * 8, a.NBcap * 2 * D * 8);
  add(a.kidx, b.kidx, a.NBcap * a.GP * 2, b.NBcap * b.GP * 2, a.NBcap * a.GP * 2);
  add(a.vidx, b.vidx, a.NBcap * a.GP * 2, b.NBcap * b.GP * 2, a.NBcap * a.GP * 2);
  add(a.vparam32, b.vparam32, a.NBcap * a.GP * 8, b.NBcap * b.GP * 8, a.NBcap * a.GP * 8);
  add(a.vparam64, b.vparam64, a.Tcap * 16, b.Tcap * 16, a.Tcap * 16);
  if (a.keep_diag && b.keep_diag) {
    add(a.kdiag, b.kdiag, a.Tcap * 16, b.Tcap * 16, a.Tcap * 16);
    add(a.vdiag, b.vdiag, a.Tcap * 16, b.Tcap * 16, a.Tcap * 16);
  }
  const int64_t wrow = (int64_t)a.Wcap * D * src->esize;
  add(a.wk, b.wk, wrow, wrow, wrow);
  add(a.wv, b.wv, wrow, wrow, wrow);
  return fa;
}

static int run_fork(const ForkArenas& fa, const std::vector<int>& hs, const std::vector<int>& hd, cudaStream_t st) {
  const int n = (int)hs.size();
  if (n == 0) return PKV_OK;
  int* dev_pairs = nullptr;
  CU(cudaMallocAsync((void**)&dev_pairs, (size_t)2 * n * 4, st));
  std::vector<int> pairs(hs);
  pairs.insert(pairs.end(), hd.begin(), hd.end());
  CU(cudaMemcpyAsync(dev_pairs, pairs.data(), (size_t)2 * n * 4, cudaMemcpyHostToDevice, st));
  CU(launch_fork(fa, n, dev_pairs, dev_pairs + n, st));
  CU(cudaFreeAsync(dev_pairs, st));
  return PKV_OK;
}

extern "C" int pkv_cache_fork(pkv_cache* c, const int32_t* src_units, const int32_t* dst_units, int32_t n,
                              void* stream) {
  if (!c || (n > 0 && (!src_units || !dst_units))) return fail(PKV_USAGE, -1, "null argument");
  if (n < 0) return fail(PKV_USAGE, -1, "negative unit count");
  std::vector<int> hs(n), hd(n), seen(c->U, 0);
  for (int i = 0; i < n; ++i) {
    if (src_units[i] < 0 || src_units[i] >= c->U || dst_units[i] < 0 || dst_units[i] >= c->U)
      return fail(PKV_USAGE, i, "fork pair %d (%d -> %d) outside the %d units", i, src_units[i], dst_units[i], c->U);
    if (seen[dst_units[i]]++) return fail(PKV_USAGE, i, "unit %d is a fork destination twice", dst_units[i]);
    hs[i] = src_units[i];
    hd[i] = dst_units[i];
  }
  for (int i = 0; i < n; ++i)
    if (seen[hs[i]] && hs[i] != hd[i])
      return fail(PKV_USAGE, i, "unit %d is both a fork source and a destination", hs[i]);
  return run_fork(fork_arenas(c, c), hs, hd, (cudaStream_t)stream);
}

extern "C" int pkv_cache_fork_from(pkv_cache* dst, const pkv_cache* src, const int32_t* src_units, void* stream) {
  if (!dst || !src || !src_units) return fail(PKV_USAGE, -1, "null argument");
  if (dst == src) return fail(PKV_USAGE, -1, "fork_from needs two caches (use pkv_cache_fork within one)");
  const pkv_config &a = src->cfg, &b = dst->cfg;
  if (src->D != dst->D || src->dtype != dst->dtype || a.bits != b.bits || a.group_size != b.group_size ||
      a.residual_window != b.residual_window || a.use_k_patterns != b.use_k_patterns ||
      a.use_v_patterns != b.use_v_patterns || a.generate_new_patterns != b.generate_new_patterns ||
      a.use_v_gate != b.use_v_gate || a.use_k_gate != b.use_k_gate || a.alpha != b.alpha)
    return fail(PKV_USAGE, -1, "fork_from: caches differ in head_dim, dtype or config");
  std::vector<int> hs(dst->U), hd(dst->U);
  for (int i = 0; i < dst->U; ++i) {
    if (src_units[i] < 0 || src_units[i] >= src->U)
      return fail(PKV_USAGE, i, "source unit %d of destination unit %d outside the %d units", src_units[i], i, src->U);
    hs[i] = src_units[i];
    hd[i] = i;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = reserve(dst, std::max(dst->dev.Tcap, src->dev.Tcap), std::max(dst->dev.Pcap, src->dev.Pcap), st);
  if (rc) return rc;
  // the destination takes the source's lockstep geometry
  dst->token_count = src->token_count; dst->committed = src->committed;
  dst->win_len = src->win_len; dst->win_slot0 = src->win_slot0; dst->nb = src->nb;
  dst->nb_prefill = src->nb_prefill; dst->decode_base = src->decode_base;
  dst->blk_start = src->blk_start; dst->blk_len = src->blk_len;
  dst->pk_bound = src->pk_bound; dst->pv_bound = src->pv_bound;
  dst->prefill_tokens = src->prefill_tokens;
  rc = upload_blocks(dst, st);
  if (rc) return rc;
  dst->blocks_stale = false;
  return run_fork(fork_arenas(src, dst), hs, hd, st);
}

// ---------------------------------------------------------------------------------
// reconstruction / export
// ---------------------------------------------------------------------------------
extern "C" int pkv_dequant(pkv_cache* c, int64_t t0, int64_t t1, double* k_out, double* v_out, void* stream) {
  if (!c || ((!k_out || !v_out) && t1 > t0)) return fail(PKV_USAGE, -1, "null argument");
  if (t0 < 0 || t1 > c->committed || t0 > t1)
    return fail(PKV_USAGE, t0, "token range [%lld, %lld) outside committed [0, %lld)", (long long)t0, (long long)t1,
                (long long)c->committed);
  CU(launch_dequant(c->dev, c->nb, t0, t1 - t0, k_out, v_out, (cudaStream_t)stream));
  return PKV_OK;
}

extern "C" int pkv_export_codes(pkv_cache* c, int64_t t0, int64_t t1, uint8_t* kc, uint8_t* vc, void* stream) {
  if (!c || ((!kc || !vc) && t1 > t0)) return fail(PKV_USAGE, -1, "null argument");
  if (t0 < 0 || t1 > c->committed || t0 > t1) return fail(PKV_USAGE, t0, "token range outside committed tokens");
  CU(launch_codes(c->dev, c->nb, t0, t1 - t0, kc, vc, (cudaStream_t)stream));
  return PKV_OK;
}

// ---------------------------------------------------------------------------------
// group-level API
// ---------------------------------------------------------------------------------
extern "C" int pkv_quantize_groups(const double* values, const int64_t* offsets, int32_t n, int32_t bits, double* scale,
                                   double* zero, uint8_t* codes, void* stream) {
  if (bits != 2 && bits != 4 && bits != 8)
    return fail(PKV_USAGE, -1, "unsupported bit width %d; expected one of (2, 4, 8)", bits);
  CU(launch_quantize_groups(values, offsets, n, bits, scale, zero, codes, (cudaStream_t)stream));
  return PKV_OK;
}
// single-group host API: a per-thread pinned staging buffer + device buffer + stream, one
// H2D, one kernel, one D2H per call (the reference's per-group functions are called in loops)
struct GroupCtx {
  cudaStream_t st = nullptr;
  unsigned char* host = nullptr;
  unsigned char* dev = nullptr;
  size_t cap = 0;
  ~GroupCtx() {
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    if (st) cudaStreamDestroy(st);
  }
};
static thread_local GroupCtx g_group;
static int group_ctx(size_t bytes) {
  GroupCtx& g = g_group;
  if (!g.st) CU(cudaStreamCreateWithFlags(&g.st, cudaStreamNonBlocking));
  if (bytes > g.cap) {
    if (g.host) cudaFreeHost(g.host);
    if (g.dev) cudaFree(g.dev);
    g.host = nullptr; g.dev = nullptr; g.cap = 0;
    const size_t cap = std::max<size_t>(bytes, 64 * 1024);
    CU(cudaHostAlloc((void**)&g.host, cap, cudaHostAllocDefault));
    CU(cudaMalloc((void**)&g.dev, cap));
    g.cap = cap;
  }
  return PKV_OK;
}

extern "C" int pkv_quantize_group_host(const double* values, int64_t n, int32_t bits, double* scale, double* zero,
                                       uint8_t* packed) {
  if (bits != 2 && bits != 4 && bits != 8)
    return fail(PKV_USAGE, -1, "unsupported bit width %d; expected one of (2, 4, 8)", bits);
  if (n < 1) return fail(PKV_USAGE, -1, "cannot quantize an empty group");
  if (!values || !scale || !zero || !packed) return fail(PKV_USAGE, -1, "null argument");
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(values[i])) return fail(PKV_DATA, i, "non-finite value at index %lld: %g", (long long)i, values[i]);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(PKV_USAGE, -1, "no CUDA device: the PatternKV B200 codec has no CPU fallback");
  const size_t nb = (size_t)(n * bits + 7) / 8, vb = (size_t)n * 8, ob = 16 + ((nb + 15) & ~(size_t)15);
  int rc = group_ctx(vb + ob);
  if (rc) return rc;
  GroupCtx& g = g_group;
  std::memcpy(g.host, values, vb);
  CU(cudaMemcpyAsync(g.dev, g.host, vb, cudaMemcpyHostToDevice, g.st));
  CU(launch_qpack((const double*)g.dev, n, bits, (double*)(g.dev + vb), g.dev + vb + 16, g.st));
  CU(cudaMemcpyAsync(g.host + vb, g.dev + vb, 16 + nb, cudaMemcpyDeviceToHost, g.st));
  CU(cudaStreamSynchronize(g.st));
  std::memcpy(scale, g.host + vb, 8);
  std::memcpy(zero, g.host + vb + 8, 8);
  std::memcpy(packed, g.host + vb + 16, nb);
  return PKV_OK;
}

extern "C" int pkv_dequantize_group_host(const uint8_t* packed, int64_t n, int32_t bits, double scale, double zero,
                                         double* out) {
  if (bits != 2 && bits != 4 && bits != 8)
    return fail(PKV_USAGE, -1, "unsupported bit width %d; expected one of (2, 4, 8)", bits);
  if (n < 0 || (n > 0 && (!packed || !out))) return fail(PKV_USAGE, -1, "null argument");
  if (n == 0) return PKV_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(PKV_USAGE, -1, "no CUDA device: the PatternKV B200 codec has no CPU fallback");
  const size_t nb = (size_t)(n * bits + 7) / 8, pb = (nb + 15) & ~(size_t)15, ob = (size_t)n * 8;
  int rc = group_ctx(pb + ob);
  if (rc) return rc;
  GroupCtx& g = g_group;
  std::memcpy(g.host, packed, nb);
  CU(cudaMemcpyAsync(g.dev, g.host, nb, cudaMemcpyHostToDevice, g.st));
  CU(launch_dqunpack(g.dev, n, bits, scale, zero, (double*)(g.dev + pb), g.st));
  CU(cudaMemcpyAsync(g.host + pb, g.dev + pb, ob, cudaMemcpyDeviceToHost, g.st));
  CU(cudaStreamSynchronize(g.st));
  std::memcpy(out, g.host + pb, ob);
  return PKV_OK;
}

extern "C" int pkv_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint8_t* out, void* stream) {
  if (bits != 2 && bits != 4 && bits != 8)
    return fail(PKV_USAGE, -1, "unsupported bit width %d; expected one of (2, 4, 8)", bits);
  CU(launch_pack(codes, n, bits, out, (cudaStream_t)stream));
  return PKV_OK;
}
extern "C" int pkv_unpack_codes(const uint8_t* packed, int64_t n, int32_t bits, uint8_t* codes, void* stream) {
  if (bits != 2 && bits != 4 && bits != 8)
    return fail(PKV_USAGE, -1, "unsupported bit width %d; expected one of (2, 4, 8)", bits);
  CU(launch_unpack(packed, n, bits, codes, (cudaStream_t)stream));
  return PKV_OK;
}
extern "C" int pkv_match(const double* x, int64_t n, const double* pat, int32_t P, int32_t D, int64_t* idx, double* dist,
                         double* residual, void* stream) {
  if (P < 1) return fail(PKV_USAGE, -1, "cannot match against an empty pattern set");
  CU(launch_match(x, n, pat, P, D, idx, dist, residual, (cudaStream_t)stream));
  return PKV_OK;
}
extern "C" int pkv_midrange(const double* x, int64_t n, int32_t D, double* out, void* stream) {
  if (n < 1) return fail(PKV_USAGE, -1, "window must be a non-empty 2-D array of row vectors");
  CU(launch_midrange(x, n, D, out, (cudaStream_t)stream));
  return PKV_OK;
}

extern "C" int pkv_kmeans(const double* x, int64_t T, int32_t D, int32_t k, int64_t first_idx, double* centers,
                          int32_t* labels, double* history, int32_t* n_hist, int32_t* n_centers, void* stream) {
  if (T < 1) return fail(PKV_USAGE, -1, "k-means expects a non-empty 2-D array of row vectors");
  if (k < 1) return fail(PKV_USAGE, -1, "cluster count must be >= 1, got %d", k);
  if (k > 96) return fail(PKV_USAGE, -1, "cluster count must be <= 96 on the B200 path, got %d", k);
  if (D < 1 || D > 1024) return fail(PKV_USAGE, -1, "vector dimension must lie in [1, 1024], got %d", D);
  if (first_idx < 0 || first_idx >= T) return fail(PKV_USAGE, first_idx, "first seed index outside the point set");
  cudaStream_t st = (cudaStream_t)stream;
  DevCache d;
  std::memset(&d, 0, sizeof d);
  d.U = 1; d.D = D; d.Dp = round_up(D, 32); d.Pcap = k;
  d.kpat64 = centers;
  CU(cudaMallocAsync((void**)&d.kpat32, (size_t)k * d.Dp * 4, st));
  CU(cudaMallocAsync((void**)&d.kpmax, 4, st));
  CU(cudaMallocAsync((void**)&d.nk, 4, st));
  const size_t n2 = (size_t)2 * T;
  MineArgs<double> a;
  a.x[0] = x; a.x[1] = x; a.unit_stride = T * D; a.T = T;
  int64_t* first = nullptr;
  CU(cudaMallocAsync((void**)&first, 16, st));
  int64_t fh[2] = {first_idx, first_idx};
  CU(cudaMemcpyAsync(first, fh, 16, cudaMemcpyHostToDevice, st));
  a.first[0] = first; a.first[1] = first;
  a.k = k; a.side_mask = 1;
  CU(cudaMallocAsync((void**)&a.near_, n2 * 8, st));
  CU(cudaMallocAsync((void**)&a.own, n2 * 8, st));
  CU(cudaMallocAsync((void**)&a.lab, n2 * 4, st));
  CU(cudaMallocAsync((void**)&a.lab2, n2 * 4, st));
  CU(cudaMallocAsync((void**)&a.list, n2 * 4, st));
  CU(cudaMallocAsync((void**)&a.hist, 2 * 25 * 8, st));
  CU(cudaMallocAsync((void**)&a.niter, 8, st));
  a.labels_out = labels;
  a.tstride = T;
  CU(launch_mine<double>(d, a, st));
  int nc = 0, ni = 0;
  CU(cudaMemcpyAsync(&nc, d.nk, 4, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(&ni, a.niter, 4, cudaMemcpyDeviceToHost, st));
  if (history) CU(cudaMemcpyAsync(history, a.hist, 25 * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (void* p : {(void*)d.kpat32, (void*)d.kpmax, (void*)d.nk, (void*)first, (void*)a.near_, (void*)a.own, (void*)a.lab,
                  (void*)a.lab2, (void*)a.list, (void*)a.hist, (void*)a.niter})
    CU(cudaFreeAsync(p, st));
  if (n_hist) *n_hist = ni;
  if (n_centers) *n_centers = nc;
  return PKV_OK;
}
