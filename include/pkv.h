/*
 * pkv.h -- C ABI of the B200-native PatternKV codec (libpkv_b200.so).
 *
 * The reference (patternkv, pure Python/numpy) has no FFI; its drop-in
 * surface is the Python module API re-exported by pkg/src/patternkv/__init__.py:10-94.
 * Each entry point below names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/patternkv/).  Plain C types
 * only: device pointers are `void*`/typed pointers to CUDA global memory,
 * streams are `cudaStream_t` passed as `void*`.
 *
 * Status codes follow the reference error taxonomy (errors.py:9-14):
 *   PKV_OK 0, PKV_USAGE 1 (UsageError, CLI exit 1), PKV_DATA 2 (DataError,
 *   CLI exit 2), PKV_CUDA 3 (device/runtime failure; no reference analogue).
 * pkv_last_error() returns the thread-local message of the last failure and
 * the element index it refers to (-1 if none).
 *
 * Ownership: the library owns every cache arena; callers own the buffers they
 * pass.  One writer stream per cache (the reference's single-writer
 * HeadCacheState); reads are stream ordered.  Units (batch x
 * layer x kv-head) are independent and advance in lockstep (same token count).
 */
#ifndef PKV_H_
#define PKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PKV_OK 0
#define PKV_USAGE 1
#define PKV_DATA 2
#define PKV_CUDA 3

/* element types of caller tensors */
#define PKV_F16 1
#define PKV_F32 2
#define PKV_F64 3
#define PKV_BF16 4

/* cache flags */
#define PKV_FLAG_DECISIONS 1 /* keep per-token gate ranges (GateDecision records) */
#define PKV_FLAG_STATS 2     /* count fp64 refinements / exact-division fallbacks */
#define PKV_FLAG_BRUTE_FORCE 4 /* exhaustive d_mm matching (disable lower-bound pruning) */

/* EngineConfig, field for field (engine.py:38-83) */
typedef struct pkv_config {
  int32_t bits;              /* 2, 4 or 8 (quant.py:18 SUPPORTED_BITS) */
  int32_t pattern_count;     /* |M| mined per side at prefill */
  int32_t group_size;        /* G, K per-channel group length; <= 128 on the GPU */
  int32_t residual_window;   /* W >= G, exact window */
  double alpha;              /* gate level in (0, 0.5] */
  int32_t use_k_patterns;
  int32_t use_v_patterns;
  int32_t generate_new_patterns;
  int32_t use_v_gate;
  int32_t use_k_gate;
  int64_t seed;              /* K mining seed; V uses seed + 1 (engine.py:157-159) */
} pkv_config;

typedef struct pkv_cache pkv_cache;

typedef struct pkv_cache_info {
  int32_t n_units, head_dim, head_dim_padded, in_dtype;
  int64_t token_count;      /* HeadCacheState.token_count (engine.py:116) */
  int64_t committed_count;  /* engine.py:121-123 */
  int32_t window_len;       /* len(window_k) */
  int32_t window_slot0;     /* ring slot of the oldest window row */
  int32_t n_blocks;         /* len(k_blocks) */
  int32_t pattern_capacity;
  int64_t token_capacity;
  int32_t block_bytes;      /* packed bytes per K (or V) block, fragment layout */
  uint32_t n_refined;       /* fp64 re-matches (PKV_FLAG_STATS) */
  uint32_t n_exact_div;     /* exact-division quantizer fallbacks (PKV_FLAG_STATS) */
} pkv_cache_info;

int pkv_version(void);
const char* pkv_last_error(int64_t* index);

/* gate.py:23-71 z_quantile and gate.py:74-106 contraction_threshold (host) */
int pkv_z_quantile(double alpha, double* out);
int pkv_threshold(int32_t head_dim, double alpha, double* out);
/* engine.py:62-75 EngineConfig.__post_init__ */
int pkv_config_validate(const pkv_config* cfg);

/* HeadCacheState(config, head_dim) x n_units (engine.py:104-119); max_tokens and
 * max_patterns are initial capacities (the cache grows on demand). */
int pkv_cache_create(const pkv_config* cfg, int32_t n_units, int32_t head_dim, int32_t in_dtype,
                     int64_t max_tokens, int32_t max_patterns, int32_t flags, pkv_cache** out);
int pkv_cache_destroy(pkv_cache* c);
int pkv_cache_info_get(pkv_cache* c, pkv_cache_info* out);
int pkv_cache_reserve(pkv_cache* c, int64_t max_tokens, int32_t max_patterns, void* stream);
/* preallocate the k-means scratch for prefills/mining of up to max_tokens tokens, so
 * pkv_mine / pkv_prefill allocate nothing (otherwise they allocate it per call). */
int pkv_cache_reserve_mining(pkv_cache* c, int64_t max_tokens, void* stream);
/* drop every committed/window token (token_count = 0) but keep the pattern
 * tables when keep_patterns != 0, so the next pkv_prefill with NULL seed
 * indices re-encodes against the same tables (re-prefill of a slot). */
int pkv_cache_reset(pkv_cache* c, int32_t keep_patterns, void* stream);

/* Fused finiteness checks (engine.py:132-139 / :180-181): the kernels that read caller
 * K/V (K1-TC's tensor-core scores, K1's staging, the window copy) record the first
 * non-finite element (lowest unit, K before V, token, dim) in the cache; pkv_prefill /
 * pkv_append publish it to pinned host memory without synchronising.  pkv_cache_check
 * returns PKV_DATA with the reference's message ("non-finite prefill K element at token
 * t, dim j" / "non-finite decode vector at token t", plus the unit) once the flagged work
 * has run -- wait != 0 blocks until the last prefill/append has; where (optional) [4] =
 * unit, side, token, dim.  pkv_append refuses a flagged cache; pkv_cache_reset and
 * pkv_prefill clear the flag.  A flagged cache's contents are unspecified. */
int pkv_cache_check(pkv_cache* c, int32_t wait, int64_t* where);

/* standalone finiteness scan: *first_bad = flat index of the first non-finite element
 * or -1.  Synchronous on `stream`. */
int pkv_check_finite(const void* x, int32_t dtype, int64_t n, int64_t* first_bad, void* stream);

/* mine_patterns (patterns.py:145-158) for every unit of one side (0 = K, 1 = V).
 * x: device [U][T][D] of the cache dtype; first_idx: host [U] = first seed index
 * np.random.default_rng(seed).integers(T) (patterns.py:103,135).  history/niter
 * (optional, host) receive the objective history [U][25] and its length [U];
 * labels (optional, device int32 [U][T]) the final assignment (lloyd_kmeans's
 * second return value, patterns.py:84-85). */
int pkv_mine(pkv_cache* c, int32_t side, const void* x, int64_t T, const int64_t* first_idx,
             double* history, int32_t* niter, int32_t* labels, void* stream);
/* install pattern tables (device [U][P][D] fp64) for one side */
int pkv_set_patterns(pkv_cache* c, int32_t side, const double* pat, int32_t P, void* stream);

/* prefill (engine.py:142-169): mine K (first_k) and V (first_v) unless the
 * pointer is NULL (tables kept), commit T - min(T, W) tokens in spans of G,
 * keep the newest min(T, W) rows as the exact window.  k, v: device [U][T][D]. */
int pkv_prefill(pkv_cache* c, const void* k, const void* v, int64_t T, const int64_t* first_k,
                const int64_t* first_v, void* stream);

/* append_decode_token (engine.py:172-198) for all units: k, v device [U][D]. */
int pkv_append(pkv_cache* c, const void* k, const void* v, void* stream);

/* decode attention (new; semantics = softmax over committed_matrices +
 * window, engine.py:296-303): q device fp32 [U][gqa][D], out device fp32
 * [U][gqa][D]. */
int pkv_decode_attn(pkv_cache* c, const float* q, int32_t gqa, float sm_scale, float* out, void* stream);

/* Partial decode attention for a sequence split across ranks (new; SURVEY 8e,
 * cfg3 at 8 GPUs): attention over committed blocks [blk0, blk1) plus the exact
 * window when with_window != 0, returned unnormalised: o device fp32 [U][gqa][D]
 * = sum_t e^(s_t - m) v_t, ml device fp32 [U][gqa][2] = (m, l = sum_t e^(s_t - m)),
 * s_t = sm_scale q.k_t (natural-log units; m = -inf, l = 0 for an empty range).
 * Ranks exchange (o, m, l) once and LSE-merge (dist.gather_and_merge_partials). */
int pkv_decode_attn_partial(pkv_cache* c, const float* q, int32_t gqa, float sm_scale, int32_t blk0, int32_t blk1,
                            int32_t with_window, float* o, float* ml, void* stream);

/* Fork units (new; parallel sampling from one prompt, BASELINE configs[3]): unit
 * dst_units[i] becomes a copy of unit src_units[i] -- pattern tables, committed
 * codes/params/indices, gate records and window (all units share the token count
 * and block geometry, so a copy is a whole state).  The reference equivalent is
 * copy.deepcopy of a HeadCacheState (engine.py:104-129).  Host arrays [n]. */
int pkv_cache_fork(pkv_cache* c, const int32_t* src_units, const int32_t* dst_units, int32_t n, void* stream);
/* Fork across caches: every unit i of dst becomes a copy of unit src_units[i] of src
 * (host array [dst units]); dst takes src's token count and block geometry (e.g. a
 * one-prompt cache of L x H units -> a cache of S samples x L x H units). */
int pkv_cache_fork_from(pkv_cache* dst, const pkv_cache* src, const int32_t* src_units, void* stream);

/* committed_matrices / reconstruct_token (engine.py:271-303), exact fp64:
 * committed tokens [t0, t1) -> device [U][t1-t0][D] each. */
int pkv_dequant(pkv_cache* c, int64_t t0, int64_t t1, double* k_out, double* v_out, void* stream);

/* unpacked integer codes of committed tokens [t0, t1): device uint8 [U][n][D]
 * (token-major) for K and V; pack with pkv_pack_codes for the reference bytes. */
int pkv_export_codes(pkv_cache* c, int64_t t0, int64_t t1, uint8_t* k_codes, uint8_t* v_codes, void* stream);

/* Resume: install a committed state (reference snapshot.py:148-220 load_snapshot ->
 * engine HeadCacheState) into the cache, replacing its contents.  All units share the
 * token count and block geometry (lockstep).  Host: blk_start/blk_len [nb] (the
 * first nb_prefill blocks are prefill spans, the rest decode flushes of G), nk/nv
 * [U] pattern counts, npk/npv [U] how many of them came from prefill mining.
 * Device: kpat/vpat fp64 [U][Pk|Pv][D]; kparam fp64 [U][nb][2][D] (scale, zero);
 * kidx/vidx int32 [U][C] (RAW = -1); vparam fp64 [U][C][2]; kcodes/vcodes uint8
 * [U][C][D] unpacked; wk/wv [U][win][D] in the cache dtype; kdiag/vdiag fp64
 * [U][C][2] (raw, flat) or NULL.  C = sum(blk_len). */
int pkv_cache_import(pkv_cache* c, int64_t token_count, int32_t nb, const int64_t* blk_start, const int32_t* blk_len,
                     int32_t nb_prefill, int32_t win_len, int32_t Pk, int32_t Pv, const int32_t* nk,
                     const int32_t* nv, const double* kpat, const double* vpat, const double* kparam,
                     const int32_t* kidx, const int32_t* vidx, const double* vparam, const uint8_t* kcodes,
                     const uint8_t* vcodes, const void* wk, const void* wv, const double* kdiag,
                     const double* vdiag, void* stream);

/* Raw device arena pointers of the cache (read-only views for export / PKVS
 * snapshots): name in {"kpat64","vpat64","kparam64","vparam64","kidx","vidx",
 * "kdiag","vdiag","wk","wv","nk","nv","blk_start","blk_len","kcodes","vcodes"}. */
int pkv_cache_buffer(pkv_cache* c, const char* name, void** ptr, int64_t* bytes);
/* stream-ordered copy of bytes [offset, offset + n) of a named arena into a
 * caller device buffer (export path for the reference-shaped state). */
int pkv_cache_read(pkv_cache* c, const char* name, int64_t offset, int64_t n, void* dst, void* stream);

/* quantize_group over n groups (quant.py:70-111): values fp64 concatenated with
 * offsets[n+1] (device), outputs scale/zero [n] and unpacked codes. */
int pkv_quantize_groups(const double* values, const int64_t* offsets, int32_t n, int32_t bits, double* scale,
                        double* zero, uint8_t* codes, void* stream);
/* quantize_group (quant.py:70-111) + pack_codes (quant.py:120-146) of ONE group of n
 * host values: host outputs scale, zero and ceil(n*bits/8) packed bytes (the reference's
 * byte layout).  Non-finite value -> PKV_DATA with its index.  Synchronous. */
int pkv_quantize_group_host(const double* values, int64_t n, int32_t bits, double* scale, double* zero,
                            uint8_t* packed);
/* dequantize_group (quant.py:114-117): scale * code + zero in IEEE fp64 for n codes packed
 * in host memory -> host out[n].  Synchronous. */
int pkv_dequantize_group_host(const uint8_t* packed, int64_t n, int32_t bits, double scale, double zero, double* out);
/* pack_codes / unpack_codes (quant.py:120-179) on device buffers */
int pkv_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint8_t* out, void* stream);
int pkv_unpack_codes(const uint8_t* packed, int64_t n, int32_t bits, uint8_t* codes, void* stream);
/* match_many (patterns.py:206-221): x [n][D], patterns [P][D] fp64 device */
int pkv_match(const double* x, int64_t n, const double* pat, int32_t P, int32_t D, int64_t* idx, double* dist,
              double* residual, void* stream);
/* midrange_center (patterns.py:161-171) */
int pkv_midrange(const double* x, int64_t n, int32_t D, double* out, void* stream);
/* lloyd_kmeans (patterns.py:72-126) on one point set: x device fp64 [T][D];
 * outputs centers [k][D] fp64 (device), labels [T] int32 (device), history
 * (host, 25) and counts; *n_centers = min(k, distinct rows). */
int pkv_kmeans(const double* x, int64_t T, int32_t D, int32_t k, int64_t first_idx, double* centers,
               int32_t* labels, double* history, int32_t* n_hist, int32_t* n_centers, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PKV_H_ */
