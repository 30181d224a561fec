"""Per-CUDA-source-line instruction counts and stall samples from an ncu report."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
rows = []
fname = None
hdr = None
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
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        rows.append((ex, st, fname, int(r[0]), r[1].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
tst = sum(x[1] for x in rows) or 1
print(f"total instr {tot:.3e}")
for ex, st, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{ex / tot * 100:5.1f}% inst {st / tst * 100:5.1f}% stall  {f}:{ln}  {src}")
