"""Instrumented copy of pkv_mine.cu timing the roles of a Lloyd (assign + sums) pass of
kmeans_stream_kernel per tile: row warps (wait for the tile, wait for the MMA, the epilogue
work), channel warps (wait for the labels, the sums).  Lane 0 of warps 4 and 8 of every CTA
add clock64 deltas into device memory per side; the last CTA prints per-tile averages.
    python tools/mine_phase_probe.py && PKV_LIB=$PWD/_ab/mine_t.so U=256 python tools/mine_bench.py"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "paper_2510_05176_b200/csrc/pkv_mine.cu")).read()
s = "#include <cstdio>\n" + s


def sub(old, new):
    global s
    assert old in s, old[:70]
    s = s.replace(old, new, 1)


sub("constexpr int SK_THREADS = 384;", "__device__ unsigned long long g_mp[2][8];\n__device__ unsigned g_mdone;\nconstexpr int SK_THREADS = 384;")
# row warps
sub("      mbar_wait_sleep(&full[s], ph);\n      if (assign) {\n",
    "      unsigned long long r0_ = clock64();\n      mbar_wait_sleep(&full[s], ph);\n      unsigned long long r1_ = clock64(), r2_ = r1_, r3_ = r1_;\n      if (assign) {\n")
sub("        mbar_wait_sleep(&tfull[acc], aph);\n        tc_fence_after();\n",
    "        r2_ = clock64();\n        mbar_wait_sleep(&tfull[acc], aph);\n        tc_fence_after();\n        r3_ = clock64();\n")
sub("      if (split) mbar_arrive_cnt(&empty[s], 2);  // this group alone consumed the tile\n",
    "      if (sums && lane == 0 && (warp & 3) == 0) {\n"
    "        const int sd_ = blockIdx.x >= gridDim.x / 2;\n"
    "        const unsigned long long r4_ = clock64();\n"
    "        atomicAdd(&g_mp[sd_][0], r1_ - r0_); atomicAdd(&g_mp[sd_][1], r3_ - r2_);\n"
    "        atomicAdd(&g_mp[sd_][2], (r2_ - r1_) + (r4_ - r3_)); atomicAdd(&g_mp[sd_][5], 1ull);\n"
    "      }\n"
    "      if (split) mbar_arrive_cnt(&empty[s], 2);  // this group alone consumed the tile\n")
# near-tie fp64 re-decision (row warps): cycles and entries
sub("        if (__any_sync(0xffffffffu, tie)) {\n",
    "        const unsigned long long t0_ = clock64();\n        const bool anyt_ = __any_sync(0xffffffffu, tie);\n"
    "        if (anyt_) {\n")
sub("          bi = bj;\n        }\n",
    "          bi = bj;\n        }\n"
    "        if (lane == 0 && (warp & 3) == 0) {\n"
    "          const int sd_ = blockIdx.x >= gridDim.x / 2;\n"
    "          atomicAdd(&g_mp[sd_][6], clock64() - t0_); atomicAdd(&g_mp[sd_][7], anyt_ ? 1ull : 0ull);\n"
    "        }\n")
# channel warps
sub("        mbar_wait_sleep(&lready[ls], lph);\n",
    "        unsigned long long c0_ = clock64();\n        mbar_wait_sleep(&lready[ls], lph);\n        unsigned long long c1_ = clock64();\n")
sub("        if (curj >= 0) stsd(acc_s + curj * 1024, __dadd_rn(ldsd(acc_s + curj * 1024), __dadd_rn(run0, run1)));\n      } else if ((mode & SK_SEED) && (mode & SK_SPLIT)) {",
    "        if (curj >= 0) stsd(acc_s + curj * 1024, __dadd_rn(ldsd(acc_s + curj * 1024), __dadd_rn(run0, run1)));\n"
    "        if (lane == 0 && c < 32) {\n"
    "          const int sd_ = blockIdx.x >= gridDim.x / 2;\n"
    "          atomicAdd(&g_mp[sd_][3], c1_ - c0_); atomicAdd(&g_mp[sd_][4], clock64() - c1_);\n"
    "        }\n"
    "      } else if ((mode & SK_SEED) && (mode & SK_SPLIT)) {")
sub("  if (warp == 1) tmem_free<256>(*sm.tmem);\n}",
    "  if (warp == 1) tmem_free<256>(*sm.tmem);\n"
    "  if (tid == 0) {\n    __threadfence();\n"
    "    if (atomicAdd(&g_mdone, 1u) == gridDim.x - 1) {\n"
    "      for (int sd = 0; sd < 2; ++sd) {\n        const double n = (double)g_mp[sd][5];\n"
    "        if (n > 0) printf(\"MINE half %d tiles %.0f | row wait-tile %.0f wait-mma %.0f work %.0f | ch wait-labels %.0f sums %.0f | ties %.0f cyc, %.3f of tiles (cycles/tile)\\n\",\n"
    "               sd, n, g_mp[sd][0] / n, g_mp[sd][1] / n, g_mp[sd][2] / n, g_mp[sd][3] / n, g_mp[sd][4] / n, g_mp[sd][6] / n, g_mp[sd][7] / n);\n"
    "        for (int i = 0; i < 8; ++i) g_mp[sd][i] = 0;\n      }\n      g_mdone = 0;\n    }\n  }\n}")
open(os.path.join(ROOT, "_ab/mine_t.cu"), "w").write(s)
print(subprocess.run(["bash", os.path.join(ROOT, "tools/ab_build.sh"), "mine_t", "pkv_mine", "_ab/mine_t.cu"],
                     cwd=ROOT, capture_output=True, text=True).stdout.strip().splitlines()[-1])
