#!/bin/bash
# A/B pass times on the headline for env variants given as arguments (each "VAR=x VAR2=y").
OUT=gpurun_out/${AB_TAG:-ab}
mkdir -p $OUT
for v in "$@"; do
  env $v timeout 600 python tools/pass_times.py ${AB_CFG:-cfg2} --reps 5 > "$OUT/pt_$(echo $v | tr ' =,' '__-').json" 2>&1
done
for f in $OUT/pt_*.json; do echo "$f: $(tail -1 $f | cut -c40-220)"; done
if [ -n "${AB_TESTS:-}" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$AB_TESTS" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log; fi
