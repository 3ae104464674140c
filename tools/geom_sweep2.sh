#!/bin/bash
OUT=gpurun_out/${1:-geom2}
mkdir -p $OUT
run() { env "$@" timeout 600 python tools/pass_times.py cfg2 --reps 5 > $OUT/pt_$(echo "$@" | tr ' =,' '__-').json 2>&1; }
run QF_GEOM_ADJ=12,4
run QF_GEOM_ADJ=12,4 QF_TB_MODE=cs
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=3
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=3 QF_TB_MODE=cs
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=2
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=3 QF_EXP=nodiag
for f in $OUT/pt_*.json; do echo "$f: $(tail -1 $f | cut -c1-200)"; done
