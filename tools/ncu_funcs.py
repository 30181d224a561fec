"""Per-function breakdown of an ncu source page (SASS): instructions executed and stall
samples attributed to each device function of the kernel, using the symbol offsets of the
kernel's cubin (nm -n on a cubin compiled from the same source).

    python tools/ncu_funcs.py <report.ncu-rep> <kernel.cubin> <kernel-symbol-substring>
"""
import csv
import subprocess
import sys


def main(rep, cubin, ksub):
    rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                          capture_output=True, text=True).stdout.splitlines()))
    h = rows[1]
    ia, ie, ist = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ino, iba = h.index("stall_no_inst"), h.index("stall_barrier")
    data = [(int(r[ia], 16), float(r[ie] or 0), float(r[ist] or 0), float(r[ino] or 0), float(r[iba] or 0))
            for r in rows[2:] if len(r) > iba]
    base = data[0][0]
    syms = []
    for line in subprocess.run(["nm", "-n", cubin], capture_output=True, text=True).stdout.splitlines():
        p = line.split()
        if len(p) == 3 and ksub in p[2]:
            name = p[2].split("$")[-1] if "$" in p[2] else "<kernel body>"
            syms.append((int(p[0], 16), name))
    syms.sort()
    agg = {}
    for a, e, s, no, ba in data:
        off = a - base
        name = "<kernel body>"
        for so, sn in syms:
            if off >= so:
                name = sn
        agg.setdefault(name, [0, 0, 0, 0, 0])
        agg[name][0] += e
        agg[name][1] += s
        agg[name][2] += 1
        agg[name][3] += no
        agg[name][4] += ba
    te = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print("  inst%  stall%  no_inst%  barrier%   sass  function")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{v[0] / te * 100:6.2f}% {v[1] / ts * 100:6.2f}%  {v[3] / ts * 100:7.2f}%  {v[4] / ts * 100:7.2f}% "
              f"{v[2]:6d}  {k[:70]}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
