#!/bin/bash
# Adjoint tile-geometry sweep on the headline (per-pass times; results must still be exact).
OUT=gpurun_out/${1:-geom}
mkdir -p $OUT
run() { env "$@" timeout 600 python tools/pass_times.py cfg2 --reps 5 > $OUT/pt_$(echo "$@" | tr ' =,' '__-').json 2>&1; }
run QF_GEOM_ADJ=12,4
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=3
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=2
run QF_GEOM_ADJ=13,5 QF_MINB_ADJ=1
run QF_GEOM_ADJ=12,4 QF_MINB_ADJ=3
for f in $OUT/pt_*.json; do echo "$f: $(tail -1 $f | cut -c1-300)"; done
