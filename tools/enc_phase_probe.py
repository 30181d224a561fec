"""Build an instrumented copy of pkv_encode_tc.cu (clock64 per phase of each item, printed for a
few CTAs when the cache counts statistics) into _ab/enc_tc_t.so:
    python tools/enc_phase_probe.py && PKV_LIB=$PWD/_ab/enc_tc_t.so python tools/enc_stats.py 64
Phases per item and warp: TMA wait, token stage, barrier 1, K channel pass, barrier 2, scalar
pass, barrier 3, fix-ups/codes + release, next-item barrier (+ 2-bit code stores), metadata and
chunk barriers."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
s = open(os.path.join(ROOT, "paper_2510_05176_b200/csrc/pkv_encode_tc.cu")).read()
s = "#include <cstdio>\n" + s


def sub(old, new):
    global s
    assert old in s, old[:60]
    s = s.replace(old, new, 1)


sub("  int pending = -1;  // item whose TMA this subgroup already issued\n",
    "  int pending = -1;  // item whose TMA this subgroup already issued\n"
    "  unsigned long long ph_[12] = {0,0,0,0,0,0,0,0,0,0,0,0};\n"
    "  unsigned long long tprev_ = clock64(), nitems_ = 0;\n"
    "  auto mark_ = [&](int i) { const unsigned long long t = clock64(); ph_[i] += t - tprev_; tprev_ = t; };\n")
sub("      mbar_wait(xfull, ph);\n", "      mark_(9);\n      mbar_wait(xfull, ph);\n      mark_(0);\n")
sub("    if (u != staged) {\n      stage_patterns(A, SIDE, u, sb, gtid);\n      bar_side();\n      staged = u;\n    }\n",
    "    mark_(10);\n    if (u != staged) {\n      stage_patterns(A, SIDE, u, sb, gtid);\n      bar_side();\n      staged = u;\n    }\n    mark_(11);\n")
sub("      token_stage<SIDE>(sc, pt, X, M, mmab, ph, tcol, w, lane, P, pmx, p64, stats, u, start, L, c.bad);\n",
    "      token_stage<SIDE>(sc, pt, X, M, mmab, ph, tcol, w, lane, P, pmx, p64, stats, u, start, L, c.bad);\n"
    "      mark_(1);\n      ++nitems_;\n")
sub("        bar_sub(sgi);  // every token's final pattern index\n",
    "        bar_sub(sgi);  // every token's final pattern index\n        mark_(2);\n")
sub("        bar_sub(sgi);  // per-channel statistics of all 128 channels\n",
    "        mark_(3);\n        bar_sub(sgi);  // per-channel statistics of all 128 channels\n        mark_(4);\n")
sub("        bar_sub(sgi);  // per-channel fp64 params in HBM\n",
    "        mark_(5);\n        bar_sub(sgi);  // per-channel fp64 params in HBM\n        mark_(6);\n")
sub("        v_scalar<BITS>(A, X, M, pt, sc, st, L, start, u, blk, p64, stats);\n",
    "        v_scalar<BITS>(A, X, M, pt, sc, st, L, start, u, blk, p64, stats);\n        mark_(5);\n")
sub("      // release the x tile; the last warp out takes", "      mark_(7);\n      // release the x tile; the last warp out takes")
sub("          dst[ci] = make_uint4(wv[0], wv[1], wv[2], wv[3]);\n        }\n      }\n",
    "          dst[ci] = make_uint4(wv[0], wv[1], wv[2], wv[3]);\n        }\n      }\n      mark_(8);\n")
sub("      *cnext = (int)j0 + 4;\n    }\n    bar_side();\n  }\n}\n",
    "      *cnext = (int)j0 + 4;\n    }\n    bar_side();\n  }\n  mark_(9);\n"
    "  if (c.stats && blockIdx.x < 3 && lane == 0 && sgi < 2)\n"
    "    printf(\"ENC side %d cta %d warp %d items %llu | tma %.0f tok %.0f bar1 %.0f kpass %.0f bar2 %.0f scal %.0f "
    "bar3 %.0f fix/codes %.0f next+store %.0f meta %.0f chunkbar %.0f stage %.0f\\n\", SIDE, blockIdx.x, warp, nitems_,\n"
    "           ph_[0] / (double)nitems_, ph_[1] / (double)nitems_, ph_[2] / (double)nitems_, ph_[3] / (double)nitems_,\n"
    "           ph_[4] / (double)nitems_, ph_[5] / (double)nitems_, ph_[6] / (double)nitems_, ph_[7] / (double)nitems_,\n"
    "           ph_[8] / (double)nitems_, ph_[9] / (double)nitems_, ph_[10] / (double)nitems_, ph_[11] / (double)nitems_);\n}\n")
os.makedirs(os.path.join(ROOT, "_ab"), exist_ok=True)
open(os.path.join(ROOT, "_ab/enc_tc_t.cu"), "w").write(s)
print(subprocess.run(["bash", os.path.join(ROOT, "tools/ab_build.sh"), "enc_tc_t", "pkv_encode_tc", "_ab/enc_tc_t.cu"],
                     cwd=ROOT, capture_output=True, text=True).stdout.strip().splitlines()[-1])
