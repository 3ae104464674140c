#!/bin/bash
# Quick GPU check: build, parity suite (optionally filtered), bench line.
# usage: tools/gpu_quick.sh TAG [pytest -k expr]
set -u
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
if [ -n "${2:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$2" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
else
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
python - $OUT/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d["roofline"]
print("value",round(d["value"]),"e2e",round(d["e2e"]["value"]),"frac",round(r["frac"],3),"ms",round(d["ms_per_step"],3))
print("pass_ms",r["pass_ms"]); print("pass_gbs",r["pass_gbs"])
PY
