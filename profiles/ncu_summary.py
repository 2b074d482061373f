"""Summarise an ncu report (raw metrics + per-opcode instruction mix + top
stalls) -- used to produce the profiles/*.txt files committed per round."""
import collections
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
        "launch__occupancy_limit_registers",
        # tensor pipes (the DMMA Gram): matched by suffix, ncu prefixes them with a section name
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def run(rep, points=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    out = []
    for r in rows[2:]:
        name = r[rows[0].index("Kernel Name")]
        out.append(f"kernel: {name}")
        for w in WANT:
            hits = [i for i, h in enumerate(rows[0]) if h == w or h.endswith("." + w)]
            if hits:
                i = hits[0]
                out.append(f"  {w} = {r[i]} {rows[1][i]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        hdr = srows[1]
        ie, sc, st = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        c = collections.Counter()
        tot = 0
        stalls = []
        for r in srows[2:]:
            if not r[ie].isdigit():
                continue
            t = r[sc].split()
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            c[op] += int(r[ie])
            tot += int(r[ie])
            stalls.append((int(r[st]) if r[st].isdigit() else 0, r[sc].strip()))
        out.append(f"  warp instructions executed: {tot}")
        if points:
            out.append(f"  lane instructions per point: {tot * 32 / points:.1f}")
            out.append("  mix per point: " + ", ".join(f"{k} {v * 32 / points:.1f}" for k, v in c.most_common(20)))
        out.append("  top stall sites:")
        for s, line in sorted(stalls, reverse=True)[:8]:
            out.append(f"    {s:7d}  {line}")
    return "\n".join(out)


if __name__ == "__main__":
    print(run(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None))
