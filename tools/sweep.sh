#!/bin/bash
# Geometry / occupancy sweep of the plan-specialised kernels on the headline workload.
# usage: tools/sweep.sh TAG "ENV1" "ENV2" ...   (each ENV is a space-separated VAR=VAL list)
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
i=0
for cfg in "$@"; do
  i=$((i+1))
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $OUT/c$i.json 2> $OUT/c$i.err
  python - "$cfg" $OUT/c$i.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[1]:45s} value={d['value']:.0f} frac={r['frac']:.3f} passes={d['config']['fwd_passes']}+{d['config']['adj_passes']} ms={r['pass_ms']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
