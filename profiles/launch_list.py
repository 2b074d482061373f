"""ncu --csv launch list (gpu__time_duration.sum, dram bytes) -> the
per-launch table committed under profiles/ and the mean DRAM traffic per
headline launch used for bench.py's roofline.traffic."""
import collections
import csv
import json
import sys

ALG_BYTES = 32 * 167284151  # one variant launch of the headline step

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, ii, mi, vi = hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
k = collections.OrderedDict()
for r in rows[1:]:
    d = k.setdefault(r[ii], {"kernel": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
print("# ncu launch list of `python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-fit`")
print("# (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none)")
print("# cold-cache, serialised launches; compare shares, not absolutes")
print("id,kernel,duration_us,dram_read_GB,dram_write_GB,algorithmic_GB,dram_GBps")
tr = []
for i, d in k.items():
    name = d["kernel"]
    if not name.startswith("kcg_"):
        continue
    us = d["gpu__time_duration.sum"] / 1e3 if d["gpu__time_duration.sum"] > 1e5 else d["gpu__time_duration.sum"]
    rd, wr = d["dram__bytes_read.sum"] / 1e9, d["dram__bytes_write.sum"] / 1e9
    alg = ALG_BYTES / 1e9 if name.endswith("_tma") else 0.0
    print(f"{i},{name},{us:.1f},{rd:.3f},{wr:.3f},{alg:.3f},{(rd + wr) / us * 1e6:.0f}")
    if name.endswith("_tma"):
        tr.append((rd + wr) * 1e9)
if len(sys.argv) > 2 and tr:
    json.dump({"kernel": "kcg_eval_<variant>_tma", "traffic_bytes_per_launch": sum(tr) / len(tr),
               "source": f"profiles/r01_launches_eval.csv (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                         f"mean over the {len(tr)} launches)"}, open(sys.argv[2], "w"), indent=1)
