"""Instrumented copy of pkv_encode_tc.cu timing the phases of token_stage (clock64, lane 0 of
every warp, summed per side in device memory; the last CTA to finish prints the per-item
averages) into _ab/enc_tc_tok.so:
    python tools/tok_phase_probe.py && PKV_LIB=$PWD/_ab/enc_tc_tok.so python tools/enc_stats.py 64"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "paper_2510_05176_b200/csrc/pkv_encode_tc.cu")).read()
s = "#include <cstdio>\n" + s


def sub(old, new):
    global s
    assert old in s, old[:70]
    s = s.replace(old, new, 1)


sub("namespace fe {\n", "namespace fe {\n__device__ unsigned long long g_tok[2][8];\n__device__ unsigned g_done;\n")
sub("  warp_converged();\n  const int g = lane >> 2, q = lane & 3;\n  const int tt_ = 32 * w + lane;  // this thread's token in stages A/C\n",
    "  warp_converged();\n  const int g = lane >> 2, q = lane & 3;\n  const int tt_ = 32 * w + lane;  // this thread's token in stages A/C\n"
    "  unsigned long long tp_ = clock64();\n"
    "  auto mk_ = [&](int i) { const unsigned long long t = clock64(); if (lane == 0) atomicAdd(&g_tok[SIDE][i], t - tp_); tp_ = t; };\n")
sub("  // ---- B. keyed residual extrema against the guess, per 16-token tile -----------------\n",
    "  mk_(0);\n  // ---- B. keyed residual extrema against the guess, per 16-token tile -----------------\n")
sub("  // ---- C. prune every other pattern by an exact lower bound (thread per token) --------\n",
    "  mk_(1);\n  // ---- C. prune every other pattern by an exact lower bound (thread per token) --------\n")
sub("  // ---- D. survivors: full fp32 distance, top-2 with error bounds, fp64 re-match ---------\n",
    "  mk_(2);\n  // ---- D. survivors: full fp32 distance, top-2 with error bounds, fp64 re-match ---------\n")
# end of token_stage: the final __syncwarp() before the closing brace of token_stage
i = s.index("__device__ __noinline__ void token_stage(")
j = s.index("\n}\n", i)
body = s[i:j]
k = body.rindex("  __syncwarp();")
body = body[:k] + "  mk_(3);\n  if (lane == 0) atomicAdd(&g_tok[SIDE][7], 1ull);\n" + body[k:]
s = s[:i] + body + s[j:]
sub("  if (warp == 0) tmem_free<256>(tmem);\n}",
    "  if (warp == 0) tmem_free<256>(tmem);\n"
    "  if (tid == 0 && A.c.stats) {\n"
    "    __threadfence();\n"
    "    if (atomicAdd(&g_done, 1u) == gridDim.x - 1) {\n"
    "      for (int sd = 0; sd < 2; ++sd) {\n"
    "        const double n = (double)g_tok[sd][7];\n"
    "        printf(\"TOK side %d warp-items %.0f | guess %.0f btile %.0f prune %.0f survivors %.0f (cycles per warp-item)\\n\", sd, n,\n"
    "               g_tok[sd][0] / n, g_tok[sd][1] / n, g_tok[sd][2] / n, g_tok[sd][3] / n);\n"
    "        for (int i = 0; i < 8; ++i) g_tok[sd][i] = 0;\n"
    "      }\n"
    "      g_done = 0;\n"
    "    }\n"
    "  }\n}")
open(os.path.join(ROOT, "_ab/enc_tc_tok.cu"), "w").write(s)
print(subprocess.run(["bash", os.path.join(ROOT, "tools/ab_build.sh"), "enc_tc_tok", "pkv_encode_tc", "_ab/enc_tc_tok.cu"],
                     cwd=ROOT, capture_output=True, text=True).stdout.strip().splitlines()[-1])
