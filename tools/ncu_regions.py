"""Split an ncu source-page CSV (SASS view) of one pass kernel at its BAR.SYNC barriers and
print, per region, the warp-stall samples (total and by reason) and the opcode mix, so the
load / gate / exchange / store phases of a tile can be compared.

  ncu -i X.ncu-rep --page source --csv --kernel-name regex:qf_a_p2 --print-source sass > k.csv
  python tools/ncu_regions.py k.csv
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ci = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
regions = [[]]
for r in data:
    regions[-1].append(r)
    if "BAR.SYNC" in r[ci["Source"]] or "BAR.RED" in r[ci["Source"]]:
        regions.append([])
tot_all = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"total samples {tot_all}, instructions {len(data)}")
for k, reg in enumerate(regions):
    if not reg:
        continue
    s = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in reg)
    st = collections.Counter()
    for r in reg:
        for h in reasons:
            st[h[6:]] += int(r[ci[h]] or 0)
    ops = collections.Counter(re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ci["Source"]]).group(2) for r in reg)
    print(f"region {k}: {len(reg)} instr, {100 * s / tot_all:.1f}% samples | "
          + " ".join(f"{a}={100 * b / max(s, 1):.0f}%" for a, b in st.most_common(5) if b)
          + " | " + " ".join(f"{a}:{b}" for a, b in ops.most_common(6)))
