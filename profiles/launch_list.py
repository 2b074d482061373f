"""ncu --csv launch list (gpu__time_duration.sum, dram bytes) -> the
per-launch table committed under profiles/ and the mean DRAM traffic per
headline launch used for bench.py's roofline.traffic."""
import collections
import csv
import json
import sys

SIZES = 167284151  # sizes of the headline lattice (551^3)
ALG = {"multi": 72 * SIZES,   # kcg_multi_v6_tma: 24 B bindings read once + 6 x 8 B predictions per size
       "eval": 32 * SIZES}    # one per-variant kcg_eval_<k>_tma launch: 24 B in + 8 B out per point

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
ki, ii, mi, vi = hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
k = collections.OrderedDict()
for r in rows[1:]:
    d = k.setdefault(r[ii], {"kernel": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
print("# ncu launch list of `python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-fit --no-configs`")
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
    alg = (ALG["multi"] if name.startswith("kcg_multi") and name.endswith(("_tma", "_tmab"))
           else ALG["eval"] if name.startswith("kcg_eval") and name.endswith("_tma") else 0.0) / 1e9
    print(f"{i},{name},{us:.1f},{rd:.3f},{wr:.3f},{alg:.3f},{(rd + wr) / us * 1e6:.0f}")
    if name.startswith("kcg_multi") and name.endswith(("_tma", "_tmab")):
        tr.append((rd + wr) * 1e9)
if len(sys.argv) > 3 and tr:
    json.dump({"kernel": "kcg_multi_v6_tmab", "traffic_bytes_per_launch": sum(tr) / len(tr),
               "sizes_per_launch": SIZES, "algorithmic_bytes_per_launch": ALG["multi"],
               "source": f"{sys.argv[2]} (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                         f"mean over the {len(tr)} headline launches)"}, open(sys.argv[3], "w"), indent=1)
