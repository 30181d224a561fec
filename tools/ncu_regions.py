"""Instruction share of source-line ranges of one file in an ncu report.

    python tools/ncu_regions.py <rep> <file.cu> name:a-b [name:a-b ...]
"""
import csv
import subprocess
import sys

rep, target = sys.argv[1], sys.argv[2]
regions = []
for spec in sys.argv[3:]:
    name, rng = spec.rsplit(":", 1)
    a, b = map(int, rng.split("-"))
    regions.append((name, a, b))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
per_line, fname, hdr = {}, None, None
for line in out:
    r = next(csv.reader([line]))
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit() and len(r) > 7:
        try:
            ex = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        per_line[(fname, int(r[0]))] = per_line.get((fname, int(r[0])), 0) + ex
tot = sum(per_line.values()) or 1
print(f"total {tot:.3e}")
for name, a, b in regions:
    v = sum(e for (f, ln), e in per_line.items() if f == target and a <= ln <= b)
    print(f"{v / tot * 100:6.2f}%  {name} ({target}:{a}-{b})")
other = tot - sum(e for (f, ln), e in per_line.items() if f == target)
print(f"{other / tot * 100:6.2f}%  other files (inlined headers)")
