"""DRAM bytes per step of the headline's pass kernels from an ncu launch-list CSV of the bench
command (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum), written
to profiles/pass_kernel_traffic.json for bench.py's roofline.traffic.

  python tools/traffic_from_launches.py profiles/TAG_launches_qaoa20_b256.csv TAG
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, tag = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ci = {h: i for i, h in enumerate(hdr)}
launches = []          # [(id, name, {metric: value})]
for r in rows[start + 1:]:
    key = (r[ci["ID"]], r[ci["Kernel Name"]])
    if not launches or launches[-1][0] != key[0]:
        launches.append((key[0], key[1], {}))
    launches[-1][2][r[ci["Metric Name"]]] = float(r[ci["Metric Value"]].replace(",", ""))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# steps start at qf_f_p0; the last complete step before the trailing launches is taken
starts = [i for i, l in enumerate(launches) if l[1] == "qf_f_p0"]
a, b = starts[-2], starts[-1]
step = launches[a:b]
passes = [l for l in step if l[1].startswith("qf_f_p") or l[1].startswith("qf_a_p") or l[1] == "qf_turn"]
byt = sum(l[2].get("dram__bytes_read.sum", 0) + l[2].get("dram__bytes_write.sum", 0) for l in passes)
t_pass = sum(l[2]["gpu__time_duration.sum"] for l in passes)
t_all = sum(l[2]["gpu__time_duration.sum"] for l in step)
out = {"bytes_per_step": byt,
       "source": f"{os.path.relpath(path, ROOT)}: dram__bytes_read.sum + dram__bytes_write.sum of one timed bench "
                 f"step's pass launches ({', '.join(l[1] for l in passes)}), capture {tag}",
       "algorithmic_bytes_per_step": 42949672960,
       "pass_kernel_share_of_step_launch_time": t_pass / t_all,
       "launches_per_step": len(step),
       "launch_names": [l[1] for l in step]}
json.dump(out, open(os.path.join(ROOT, "profiles", "pass_kernel_traffic.json"), "w"), indent=1)
print(json.dumps(out)[:600])
