#!/bin/bash
OUT=gpurun_out/${1:-qcnn}
mkdir -p $OUT
run() { env "$@" timeout 900 python tools/pass_times.py cfg3 --reps 3 > $OUT/pt_$(echo "$@" | tr ' =,' '__-').json 2>&1; }
run QF_X=0
run QF_MINB_ADJ=1
run QF_GEOM_ADJ=12,3
run QF_GEOM_ADJ=12,3 QF_MINB_ADJ=1
run QF_MINB_FWD=2
run QF_GEOM_FWD=11,4
for f in $OUT/pt_*.json; do echo "$f: $(tail -1 $f | cut -c1-330)"; done
