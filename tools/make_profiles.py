"""Write the committed evidence under profiles/ from ncu reports in gpurun_out/.

    python tools/make_profiles.py <round-tag>

For each full capture (prof_*_full.ncu-rep / prof_kmeans.ncu-rep) writes a text
summary (SOL metrics, DRAM traffic, tensor-pipe activity, instruction mix, hot
source lines) and a traffic.json consumed by bench.py for roofline.traffic; the
launch list (launches.csv) is summarised per kernel (share of the step).
"""

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, os.path.join(ROOT, "tools"))

import ncu_summary  # noqa: E402


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def lines(rep, top=30):
    return run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, str(top)])


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:90]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["kernel | launches | mean ms | share of all kernel time"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k} | {len(v)} | {sum(v) / len(v) / 1e6:.3f} | {sum(v) / tot * 100:.1f}%")
    return "\n".join(out)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "round1"
    os.makedirs(PROF, exist_ok=True)
    traffic = {}
    instr = {}
    kmeans_util = None
    # token-units (units x committed tokens) of the captured launches (tools/gpu_profiles.sh MED config)
    units = int(os.environ.get("PROF_UNITS", 2 * 32 * 8)) * int(os.environ.get("PROF_COMMITTED", 32768 - 128))
    # only reports from this capture: within an hour of the newest one (older reports left in
    # gpurun_out/ by earlier captures would describe superseded kernels)
    pre = os.environ.get("PROF_PREFIX", "")  # e.g. "r2_" for tools/gpu_r2.sh captures
    reps = {n: os.path.join(OUT, pre + n + ".ncu-rep")
            for n in ("prof_encode_full", "prof_attn_full", "prof_kmeans", "prof_encode", "prof_attn", "prof_merge")}
    newest = max((os.path.getmtime(r) for r in reps.values() if os.path.exists(r)), default=0.0)
    for name, rep in reps.items():
        if not os.path.exists(rep) or os.path.getmtime(rep) < newest - 3600:
            continue
        txt = "\n".join(ncu_summary.details(rep))
        raw = ncu_summary.raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum",
                                    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                                    "gpu__time_duration.sum", "launch__grid_size", "smsp__inst_executed.sum"])
        txt += "\n" + "\n".join(f"{k:60s} {v[0]} {v[1]}" for k, v in raw.items())
        txt += "\n\n" + "\n".join(ncu_summary.sass(rep, nwin=0))
        txt += "\n\nhot source lines (share of executed instructions / of stall samples):\n" + lines(rep)
        with open(os.path.join(PROF, f"{tag}_{name}.txt"), "w") as f:
            f.write(f"# ncu --set full capture: {name}.ncu-rep ({tag})\n\n" + txt)
        if "kmeans" in name:  # K2 utilisation for the bench line's `mining.ncu`
            import re

            def grab(label):
                m = re.search(r"^" + re.escape(label) + r"\s+([0-9.,]+)", txt, re.M)
                return float(m.group(1).replace(",", "")) if m else None
            kmeans_util = {"dram_throughput_pct": grab("DRAM Throughput"), "l2_hit_pct": grab("L2 Hit Rate"),
                           "issue_slots_busy_pct": grab("Issue Slots Busy"),
                           "tensor_pipe_pct": grab("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                           "grid": grab("Grid Size"),
                           "source": f"ncu --set full, {name}.ncu-rep ({tag}): one full K2 launch "
                                     "(32 units x 2 sides = 64 CTAs, so device-wide % understate a full grid)"}
        if "dram__bytes_read.sum" in raw and "kmeans" not in name and "merge" not in name:
            def to_bytes(v):
                val, unit = float(v[0].replace(",", "")), v[1]
                return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
            traffic[name.replace("prof_", "").replace("_full", "")] = (
                to_bytes(raw["dram__bytes_read.sum"]) + to_bytes(raw["dram__bytes_write.sum"])) / units
            if "smsp__inst_executed.sum" in raw:
                instr[name.replace("prof_", "").replace("_full", "")] = (
                    float(raw["smsp__inst_executed.sum"][0].replace(",", "")) / units)
    if traffic:
        with open(os.path.join(PROF, "traffic.json"), "w") as f:
            json.dump({"source": f"ncu --set full dram__bytes_read.sum + dram__bytes_write.sum ({tag}), "
                                 f"per token-unit of the captured launch ({units} token-units)",
                       "bytes_per_token_unit": traffic,
                       "warp_instr_per_token_unit": instr,
                       "kmeans": kmeans_util}, f, indent=1)
    lp = os.path.join(OUT, pre + "launches.csv")
    if os.path.exists(lp):
        with open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w") as f:
            f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 "
                    "python bench.py --steps 2 --warmup 3 --no-four-bit --no-cpu\n"
                    "# cold-cache, serialised launches: compare shares, not absolutes\n\n")
            f.write(launch_summary(lp) + "\n")
        import shutil
        shutil.copy(lp, os.path.join(PROF, f"{tag}_launches.csv"))
    print("wrote", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main()
