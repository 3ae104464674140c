#!/bin/bash
# ncu --set full of the middle adjoint pass (qf_a_p2) of the headline for the given env (B=32).
OUT=gpurun_out/${1:-ncuadj}; shift
mkdir -p $OUT
env "$@" QF_B=64 timeout 900 ncu --set full --clock-control none --import-source on -k regex:qf_a_p2 -c 1 \
  -o $OUT/adj_$(echo "$@" | tr ' =,' '__-') python tools/prof_qaoa.py > $OUT/ncu_$(echo "$@" | tr ' =,' '__-').log 2>&1
