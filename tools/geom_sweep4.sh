#!/bin/bash
OUT=gpurun_out/${1:-geom4}
mkdir -p $OUT
run() { env "$@" timeout 600 python tools/pass_times.py cfg2 --reps 5 > $OUT/pt_$(echo "$@" | tr ' =,' '__-').json 2>&1; }
run QF_X=0
run QF_GRAD_CHAINS=4
run QF_GRAD_CHAINS=8
run QF_FUSED_GRAD=1
run QF_FUSED_GRAD=1 QF_GRAD_CHAINS=4
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=1
for f in $OUT/pt_*.json; do echo "$f: $(tail -1 $f | cut -c60-200)"; done
