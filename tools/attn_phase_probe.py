"""Instrumented copy of pkv_attn_tc.cu timing the phases of one block iteration of K3-TC
(clock64 per warp, summed per warp in registers, one atomic per phase per warp at the end)
into _ab/attn_t.so; printed by the last CTA to finish:
    python tools/attn_phase_probe.py && PKV_LIB=$PWD/_ab/attn_t.so python tools/attn_time.py --units 512"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "paper_2510_05176_b200/csrc/pkv_attn_tc.cu")).read()
s = "#include <cstdio>\n" + s


def sub(old, new):
    global s
    assert old in s, old[:70]
    s = s.replace(old, new, 1)


sub("namespace atc {\n", "namespace atc {\n__device__ unsigned long long g_ph[2][10];\n__device__ unsigned g_dn[2];\n")
sub("  // ---- block loop: QK(b) was issued by the previous iteration --------------------------------\n",
    "  unsigned long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tp_ = clock64(), nb_ = 0;\n"
    "  auto mk_ = [&](int i) { const unsigned long long t = clock64(); ph_[i] += t - tp_; tp_ = t; };\n"
    "  // ---- block loop: QK(b) was issued by the previous iteration --------------------------------\n")
sub("    // (ii) next block's K side (A_K and B_QK are free: QK(b) is complete)\n",
    "    mk_(0);\n    ++nb_;\n    // (ii) next block's K side (A_K and B_QK are free: QK(b) is complete)\n")
sub("    // (iii) softmax of token tq: p' = 2^31 exp2(lg - m_ref), digits of p' and p' s_t 2^(Ev-31)\n",
    "    mk_(1);\n    // (iii) softmax of token tq: p' = 2^31 exp2(lg - m_ref), digits of p' and p' s_t 2^(Ev-31)\n")
sub("    // (iv) after PV / W of block b - 1: V planes -> A_V, one-hot and B rows of block b\n",
    "    mk_(2);\n    // (iv) after PV / W of block b - 1: V planes -> A_V, one-hot and B rows of block b\n")
sub("    auto write_rows = [&]() {\n", "    mk_(3);\n    auto write_rows = [&]() {\n")
sub("    if (anyf != 0) {\n", "    mk_(4);\n    if (anyf != 0) {\n")
sub("#pragma unroll\n    for (int i = 0; i < 4; ++i) {\n      lsum[i] += p8[i];", "    mk_(5);\n#pragma unroll\n    for (int i = 0; i < 4; ++i) {\n      lsum[i] += p8[i];")
sub("    fresh = false;\n    next_meta();\n  }\n", "    fresh = false;\n    next_meta();\n    mk_(6);\n  }\n")
sub("  if (warp == 0) tmem_free<TCOLS>(T);\n",
    "  if (warp == 0) tmem_free<TCOLS>(T);\n"
    "  {\n    const int bi_ = BITS == 2 ? 0 : 1;\n"
    "    if (lane == 0) { for (int i = 0; i < 7; ++i) atomicAdd(&g_ph[bi_][i], ph_[i]); atomicAdd(&g_ph[bi_][9], nb_); }\n"
    "    __syncthreads();\n"
    "    if (tid == 0) {\n      __threadfence();\n"
    "      if (atomicAdd(&g_dn[bi_], 1u) == gridDim.x * gridDim.y - 1) {\n"
    "        const double n = (double)g_ph[bi_][9];\n"
    "        printf(\"ATT bits %d NG %d warp-blocks %.0f | scores %.0f kside+qk %.0f softmax %.0f vplanes %.0f rows+bar %.0f slow %.0f mma+meta %.0f\\n\",\n"
    "               BITS, NG, n, g_ph[bi_][0] / n, g_ph[bi_][1] / n, g_ph[bi_][2] / n, g_ph[bi_][3] / n, g_ph[bi_][4] / n, g_ph[bi_][5] / n, g_ph[bi_][6] / n);\n"
    "        for (int i = 0; i < 10; ++i) g_ph[bi_][i] = 0;\n        g_dn[bi_] = 0;\n      }\n    }\n  }\n")
os.makedirs(os.path.join(ROOT, "_ab"), exist_ok=True)
open(os.path.join(ROOT, "_ab/attn_t.cu"), "w").write(s)
print(subprocess.run(["bash", os.path.join(ROOT, "tools/ab_build.sh"), "attn_t", "pkv_attn_tc", "_ab/attn_t.cu"],
                     cwd=ROOT, capture_output=True, text=True).stdout.strip().splitlines()[-1])
