#!/bin/bash
# Per-pass times of the QAOA 20q headline under timing-only kernel variants (jit.EXP_MODE).
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
for v in "" noload nocompute memonly; do
  QF_EXP=$v timeout 600 python tools/pass_times.py cfg2 --reps 5 > $OUT/pt_${v:-base}.json 2>&1
done
tail -n 2 $OUT/pt_*.json
