#!/bin/bash
# A/B of tools/configs_bench.py lines for env variants: CFG_AB="cfg1 cfg3" tools/cfg_ab.sh "VAR=x" "VAR=y" ...
OUT=gpurun_out/${AB_TAG:-cab}
mkdir -p $OUT
for v in "$@"; do
  f="$OUT/cb_$(echo $v | tr ' =,' '__-').jsonl"
  env $v timeout 900 python tools/configs_bench.py ${CFG_AB:-cfg1} --no-cpu > "$f" 2>&1
  echo "== $v"; cut -c1-150 "$f" | grep config
done
