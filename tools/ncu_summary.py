"""Summarise an ncu report: key SOL metrics, instruction mix and hot SASS windows."""
import collections
import csv
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def details(rep):
    r = list(csv.reader(run([rep, "--page", "details", "--csv"]).splitlines()))
    h = r[0]
    keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
            "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Occupancy", "Grid Size",
            "Dynamic Shared Memory Per Block", "Eligible Warps Per Scheduler", "L2 Hit Rate", "Executed Instructions",
            "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "Compute (SM) Throughput")
    out = []
    for row in r[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in keep:
            out.append(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    return out


def raw(rep, names):
    r = list(csv.reader(run([rep, "--page", "raw", "--csv"]).splitlines()))
    h, units, vals = r[0], r[1], r[2]
    return {n: (vals[h.index(n)], units[h.index(n)]) for n in names if n in h}


def sass(rep, top=22, win=40, nwin=4):
    rows = list(csv.reader(run([rep, "--page", "source", "--csv", "--print-source", "sass"]).splitlines()))
    h = rows[1]
    data = rows[2:]
    isrc, iex, ist = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ex = [float(r[iex] or 0) if len(r) > iex else 0 for r in data]
    tot = sum(ex)
    ops, st = collections.Counter(), collections.Counter()
    for r, e in zip(data, ex):
        t = r[isrc].split() if len(r) > isrc else []
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += e
        st[op] += float(r[ist] or 0) if len(r) > ist else 0
    stt = sum(st.values()) or 1
    out = [f"total warp instructions {tot:.3e}"]
    out += [f"  {o:10s} {v / tot * 100:6.2f}%  stall {st[o] / stt * 100:5.1f}%" for o, v in ops.most_common(top)]
    blocks = sorted(((sum(ex[i:i + win]) / tot * 100, i) for i in range(0, len(ex), win)), reverse=True)
    for s, i in blocks[:nwin]:
        out.append(f"--- window at {i}: {s:.1f}% of instructions")
        out += ["     " + data[j][isrc][:72] for j in range(i, min(i + win, len(data)), 4)]
    return out


if __name__ == "__main__":
    rep = sys.argv[1]
    print("\n".join(details(rep)))
    for k, v in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                          "smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]).items():
        print(f"{k:40s} {v[0]} {v[1]}")
    print("\n".join(sass(rep, nwin=int(sys.argv[2]) if len(sys.argv) > 2 else 3)))
