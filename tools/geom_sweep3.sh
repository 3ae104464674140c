#!/bin/bash
OUT=gpurun_out/${1:-geom3}
mkdir -p $OUT
run() { env "$@" timeout 600 python tools/pass_times.py cfg2 --reps 5 > $OUT/pt_$(echo "$@" | tr ' =,' '__-').json 2>&1; }
run QF_GEOM_ADJ=12,4
run QF_GEOM_ADJ=12,4 QF_LANE_ORDER=0
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=2
run QF_GEOM_ADJ=12,5 QF_MINB_ADJ=3
for f in $OUT/pt_*.json; do echo "$f: $(tail -1 $f | cut -c1-200)"; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_config_parity.py -q -x -k "not cfg4" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
